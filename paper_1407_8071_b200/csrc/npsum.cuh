// numpy float64 summation order (shared by the reference-order resampler
// and the likelihood epilogues).
#pragma once

#include <stdint.h>

namespace pf {

// numpy's float64 sum is a fixed pairwise recursion (8 accumulators on
// blocks of <= 128, halves rounded down to a multiple of 8) and cumsum is
// strictly sequential.  Replicating both orders, plus IEEE division for
// w = e/total, makes the CDF bit-identical to the reference's whenever the
// exp() values agree, so ancestors are bit-exact even at N = 2^26 (the
// blocked parallel scan leaves O(10^2) rounding ties there).  Used in oracle
// (tape) mode for parity; the production path keeps the parallel scan.
static __device__ double np_pairwise_block(const double *a, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r = __dadd_rn(r, a[i]);
    return r;
  }
  double r0 = a[0], r1 = a[1], r2 = a[2], r3 = a[3], r4 = a[4], r5 = a[5], r6 = a[6], r7 = a[7];
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8) {
    r0 = __dadd_rn(r0, a[i]);
    r1 = __dadd_rn(r1, a[i + 1]);
    r2 = __dadd_rn(r2, a[i + 2]);
    r3 = __dadd_rn(r3, a[i + 3]);
    r4 = __dadd_rn(r4, a[i + 4]);
    r5 = __dadd_rn(r5, a[i + 5]);
    r6 = __dadd_rn(r6, a[i + 6]);
    r7 = __dadd_rn(r7, a[i + 7]);
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r0, r1), __dadd_rn(r2, r3)),
                         __dadd_rn(__dadd_rn(r4, r5), __dadd_rn(r6, r7)));
  for (; i < n; ++i) res = __dadd_rn(res, a[i]);
  return res;
}

// numpy's pairwise recursion  pw(a, n) = n <= 128 ? block(a, n)
//   : pw(a, n2) + pw(a + n2, n - n2),  n2 = n/2 - (n/2) % 8,
// evaluated iteratively (explicit stack, no device recursion).  Leaves are
// either summed here from `a` or, if leaf_sums != nullptr, taken in order
// from precomputed leaf sums.
static __device__ __noinline__ double np_pairwise_iter(const double *a, int64_t n_total, const double *leaf_sums) {
  int64_t st_lo[48], st_n[48];
  double st_left[48];
  int st_state[48];
  int sp = 0;
  st_lo[0] = 0;
  st_n[0] = n_total;
  st_state[0] = 0;
  sp = 1;
  double ret = 0.0;
  int64_t leaf = 0;
  while (sp > 0) {
    const int top = sp - 1;
    const int64_t n = st_n[top];
    if (n <= 128) {
      ret = leaf_sums ? leaf_sums[leaf++] : np_pairwise_block(a + st_lo[top], n);
      --sp;
      continue;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    if (st_state[top] == 0) {
      st_state[top] = 1;
      st_lo[sp] = st_lo[top];
      st_n[sp] = n2;
      st_state[sp] = 0;
      ++sp;
    } else if (st_state[top] == 1) {
      st_left[top] = ret;
      st_state[top] = 2;
      st_lo[sp] = st_lo[top] + n2;
      st_n[sp] = n - n2;
      st_state[sp] = 0;
      ++sp;
    } else {
      ret = __dadd_rn(st_left[top], ret);
      --sp;
    }
  }
  return ret;
}


// numpy's sum of n <= 128 contiguous doubles on one warp: lanes 0..7 run the
// 8 strided accumulators, then ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the
// remainder in order (pairwise_sum, numpy/_core/src/umath/loops_utils.h).
// Larger n falls back to the serial recursion on lane 0.  All 32 lanes must
// call; the result is valid on lane 0.
static __device__ __forceinline__ double np_pairwise_warp(const double *a, int n, int lane) {
  if (n > 128) return lane == 0 ? np_pairwise_iter(a, n, nullptr) : 0.0;
  if (n < 8) {
    double r = 0.0;
    if (lane == 0)
      for (int i = 0; i < n; ++i) r = __dadd_rn(r, a[i]);
    return r;
  }
  const int nblk = n - (n % 8);
  double acc = 0.0;
  if (lane < 8) {
    acc = a[lane];
    for (int i = lane + 8; i < nblk; i += 8) acc = __dadd_rn(acc, a[i]);
  }
  const double s01 = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, 1));
  const double s0123 = __dadd_rn(s01, __shfl_down_sync(0xffffffffu, s01, 2));
  double res = __dadd_rn(s0123, __shfl_down_sync(0xffffffffu, s0123, 4));
  if (lane == 0)
    for (int i = nblk; i < n; ++i) res = __dadd_rn(res, a[i]);
  return res;
}

// The order of the reference's observation sums, -0.5/var * np.sum(resid *
// resid, axis=1) over x[:, :K][:, obs_idx] (fhn.py:199-207): fancy indexing
// on the second axis yields a column-major (n, n_obs) array, so for n >= 2
// rows numpy reduces axis 1 as the OUTER loop - a strictly sequential sum per
// row - while a single row (n == 1) is contiguous and summed pairwise.
// All 32 lanes must call; the result is valid on lane 0.
static __device__ __forceinline__ double np_rows_sum(const double *a, int n, bool sequential,
                                                     int lane) {
  if (!sequential) return np_pairwise_warp(a, n, lane);
  double r = 0.0;
  if (lane == 0) {
    r = a[0];
    for (int i = 1; i < n; ++i) r = __dadd_rn(r, a[i]);
  }
  return r;
}

}  // namespace pf
