// Per-filter logsumexp normalisation + multinomial resampling (segmented).
//
// Reference (paths under parpf/):
//   normalize_log_weights   core.py:116-138   max, exp(lw-m), sum, w=e/total,
//                                             log_mean_raw = m + log(total) - log(N)
//   multinomial_resample_*  resampling.py:29-43  cum = cumsum(w) (fp64)
//   _sorted_uniforms        resampling.py:21-26  c = cumsum(Exp(1) x (N+1)); u = c[:N]/c[N]
//   resample_indices        accel.py:175-203     smallest k: cum[k] >= u, clamp N-1
//   bf_step collapse        filters.py:105-109   all -inf -> uniform, lnc unchanged
//
// Two paths, same arithmetic:
//  * bank path (N <= kBankMaxN): one CTA per filter, the filter's cum and u
//    resident in shared memory; one launch does everything.
//  * wide path (larger N, e.g. M=1 x N=2^26): tile kernels over HBM with a
//    per-filter tile-offset pass (max -> sum -> tile scan offsets -> cum ->
//    merge), workspace from pf_resample_workspace_bytes().
// Everything is fp64 (the reference upcasts: core.py:126, resampling.py:11);
// fp32 CDFs lose ~94% of ancestors at N=2^26 (SURVEY §7 hard part 1).
#include <cstring>
#include <cstdlib>
#include "block_ops.cuh"
#include "common.cuh"
#include "npsum.cuh"
#include "philox.cuh"

#include <type_traits>

namespace pf {

constexpr int kBankMaxN = 8192;

// Production fp32 log weights: exp(x) = 2^(x log2 e) on the MUFU
// (ex2.approx.ftz; relative error <= ~2^-21 + |x| 2^-24, below the input's own
// fp32 rounding of |lw| 2^-24); exp(-inf) = 0.
__device__ __forceinline__ float exp_fast(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x * 1.4426950408889634f));
  return y;
}
constexpr int kBankThreads = 256;
constexpr int kTile = 2048;          // wide path elements per tile
constexpr int kTileThreads = 256;

template <typename TW>
__device__ __forceinline__ double load_lw(const TW *p) {
  return static_cast<double>(*p);
}

// Production-mode exponential spacing E_j = -ln(U_j), one 32-bit Philox
// word per draw (4 draws per Philox block), MUFU log2: ~2^-22 relative
// accuracy, far below Monte Carlo noise; the order statistics are then formed
// by an fp64 scan exactly as in resampling.py:24-26.
__device__ __forceinline__ double spacing_exp_fast_word(uint32_t a) {
  const float u = fmaf(static_cast<float>(a), 2.3283064365386963e-10f, 1.1641532182693481e-10f);
  return static_cast<double>(-0.6931471805599453f * lg2_approx(u));
}
__device__ __forceinline__ double spacing_exp_fast(Key2 key, uint32_t t, int64_t j) {
  const uint4 r = philox10(make_uint4(static_cast<uint32_t>(j >> 2), t,
                                      static_cast<uint32_t>(j >> 34), kPurposeResample),
                           key);
  const uint32_t w = (j & 3) == 0 ? r.x : (j & 3) == 1 ? r.y : (j & 3) == 2 ? r.z : r.w;
  return spacing_exp_fast_word(w);
}

// Exclusive block scan of one fp64 value per thread; returns the exclusive
// prefix and writes the block total to *total.  scratch >= 33 doubles.
__device__ __forceinline__ double block_exclusive_scan(double v, double *scratch, double *total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  double x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x = __dadd_rn(x, y);
  }
  if (lane == 31) scratch[warp] = x;
  __syncthreads();
  // every warp scans the warp totals itself (no divergent single-warp
  // section, one barrier fewer); same association order
  double wv = lane < nw ? scratch[lane] : 0.0;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, wv, o);
    if (lane >= o) wv = __dadd_rn(wv, y);
  }
  const double woff = __shfl_sync(0xffffffffu, wv, warp > 0 ? warp - 1 : 0);
  *total = __shfl_sync(0xffffffffu, wv, nw - 1);
  const double prev = __shfl_up_sync(0xffffffffu, x, 1);
  const double excl = lane > 0 ? prev : 0.0;  // sum of lower lanes in this warp
  __syncthreads();
  return warp > 0 ? __dadd_rn(woff, excl) : excl;
}

// Exclusive block scan of a pair of fp64 values per thread (two independent
// scans in one pass: one barrier pair instead of two).  scratch >= 33.
__device__ __forceinline__ double2 block_exclusive_scan2(double2 v, double2 *scratch,
                                                         double2 *total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  double x = v.x, y = v.y;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double a = __shfl_up_sync(0xffffffffu, x, o);
    const double b = __shfl_up_sync(0xffffffffu, y, o);
    if (lane >= o) {
      x = __dadd_rn(x, a);
      y = __dadd_rn(y, b);
    }
  }
  if (lane == 31) scratch[warp] = make_double2(x, y);
  __syncthreads();
  double2 wv = lane < nw ? scratch[lane] : make_double2(0.0, 0.0);
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double a = __shfl_up_sync(0xffffffffu, wv.x, o);
    const double b = __shfl_up_sync(0xffffffffu, wv.y, o);
    if (lane >= o) {
      wv.x = __dadd_rn(wv.x, a);
      wv.y = __dadd_rn(wv.y, b);
    }
  }
  const int src = warp > 0 ? warp - 1 : 0;
  const double wox = __shfl_sync(0xffffffffu, wv.x, src);
  const double woy = __shfl_sync(0xffffffffu, wv.y, src);
  total->x = __shfl_sync(0xffffffffu, wv.x, nw - 1);
  total->y = __shfl_sync(0xffffffffu, wv.y, nw - 1);
  const double px = __shfl_up_sync(0xffffffffu, x, 1);
  const double py = __shfl_up_sync(0xffffffffu, y, 1);
  const double ex = lane > 0 ? px : 0.0, ey = lane > 0 ? py : 0.0;
  __syncthreads();
  return warp > 0 ? make_double2(__dadd_rn(wox, ex), __dadd_rn(woy, ey)) : make_double2(ex, ey);
}

// ---- bank path: one CTA per filter --------------------------------------
// Thread t owns the IPT consecutive particles [t*IPT, t*IPT+IPT): weights,
// CDF and sorted uniforms live in registers, per-thread sums are combined
// with one block scan; the CDF and the uniforms go to shared memory in a
// "thread-major" layout (element i at (i % IPT) * THREADS + i / IPT, so the
// per-thread stores are conflict-free) for the merge path.
// GATHER fuses the ancestor gather of a fp32 planar state (cfg1).

// Forward search from k for the first index >= k with c(i) >= x (n if none):
// a short linear probe, then galloping + binary search.  Keeps the merge
// O(log gap) per uniform when the CDF has long flat runs (weights that
// underflow below the CDF's ulp, e.g. sigma = 10 log weights).
template <typename I, typename F>
__device__ __forceinline__ I advance_to(F c, I k, I n, double x) {
  // common case: the next uniform lands within a few CDF entries
  int probe = 0;
  while (k < n && c(k) < x) {
    ++k;
    if (++probe == 8) break;
  }
  if (probe < 8 || k >= n || !(c(k) < x)) return k;
  I lo = k, step = 1;  // invariant: c(lo - 1) < x
  while (lo + step - 1 < n && c(lo + step - 1) < x) {
    lo += step;
    step <<= 1;
  }
  I hi = lo + step - 1 < n ? lo + step - 1 : n;  // c(hi) >= x or hi == n
  while (lo < hi) {
    const I mid = (lo + hi) >> 1;
    if (c(mid) < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// Fused posterior mean of the resampled set (filters.py:188) for planar
// states (Lorenz, HMM, linear-Gaussian; dim <= 8): the resampler already
// holds every particle's ancestor, so it sums x[d][anc] and writes the
// estimate - no separate pass over the particles.  Fixed order: per thread
// in particle order, warps by shuffle tree, warps in index order.
struct EstFuse {
  const void *x;  // planes x[d*mn + row] of the propagated particles (NULL: off)
  int dim;
  int64_t mn;
  double *est;  // filter f's row at est + f*stride
  int64_t stride;
  double *lnc_tr;    // optional: this step's lnc trace row (lnc_tr[f] = lnc[f] after)
  uint8_t *coll_tr;  // optional: this step's collapse trace row
};
constexpr int kEstMaxDim = 8;

template <int THREADS>
__device__ __forceinline__ void est_block_write(double (&acc)[kEstMaxDim], int dim,
                                                double *s_red, double *dst, double invN) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int d = 0; d < kEstMaxDim; ++d) {
    if (d >= dim) continue;
    double v = acc[d];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, o));
    if (lane == 0) s_red[warp * kEstMaxDim + d] = v;
  }
  __syncthreads();
  if (threadIdx.x < dim) {
    double sum = s_red[threadIdx.x];
    for (int w = 1; w < THREADS / 32; ++w) sum = __dadd_rn(sum, s_red[w * kEstMaxDim + threadIdx.x]);
    dst[threadIdx.x] = __dmul_rn(sum, invN);
  }
}

// The exponential spacing of element i is word (i & 3) of Philox block
// (i >> 2, t, 0, kPurposeResample) (spacing_exp_fast).  wd[h] = the word of
// element i + h for h < min(IPT, 4); i % IPT == 0, so for IPT < 4 the run
// lies inside one block but need not start at its first word.
template <int IPT>
__device__ __forceinline__ void spacing_words(Key2 key, uint32_t t, int i, uint32_t *wd) {
  const uint4 r = philox10(make_uint4(static_cast<uint32_t>(i >> 2), t, 0u, kPurposeResample), key);
  if constexpr (IPT >= 4) {
    wd[0] = r.x;
    wd[1] = r.y;
    wd[2] = r.z;
    wd[3] = r.w;
  } else if constexpr (IPT == 2) {
    const bool upper = (i & 2) != 0;
    wd[0] = upper ? r.z : r.x;
    wd[1] = upper ? r.w : r.y;
  } else {
    static_assert(IPT == 1, "IPT must be 1, 2 or a multiple of 4");
    const int w = i & 3;
    wd[0] = w == 0 ? r.x : w == 1 ? r.y : w == 2 ? r.z : r.w;
  }
}

template <typename TW, int MODE, int THREADS, int IPT, bool GATHER>
__global__ void __launch_bounds__(THREADS, THREADS == 128 ? 8 : 1) resample_bank_kernel(
    const TW *__restrict__ logw, int32_t N, const double *__restrict__ u_tape,
    const uint32_t *__restrict__ keys, uint32_t t, int32_t *__restrict__ anc,
    double *__restrict__ lnc, uint8_t *__restrict__ collapsed, uint32_t *__restrict__ status,
    const float *__restrict__ gx_in, float *__restrict__ gx_out, int gdims, int64_t gMN,
    EstFuse ef) {
  extern __shared__ double s_cum[];  // THREADS * IPT slots, thread-major
  __shared__ double scratch[33];
  __shared__ double2 scratch2[33];
  __shared__ double s_red[(THREADS / 32) * kEstMaxDim];
  const TW *ex = static_cast<const TW *>(ef.x);
  const double invN = 1.0 / static_cast<double>(N);
  const int tid = threadIdx.x;
  const int64_t f = blockIdx.x;
  const int64_t base = f * N;
  const int i0 = tid * IPT;

  // Production draws on fp32 log-weights (kFastExp) stay in fp32 through
  // the max, expf and the thread's running sum (the input's own rounding,
  // |lw| * 2^-24 relative, already exceeds these errors); the total, CDF and
  // uniforms are fp64.  Tape mode and fp64 inputs are fp64 throughout.
  constexpr bool kFastExp = MODE == 0 && std::is_same<TW, float>::value;
  // 1. load + max (NaN detection: np.max propagates NaN, core.py:132)
  double lw[IPT];
  float lf[IPT];
  double u[IPT];
  double erun64 = 0.0;  // the thread's exponential-spacing run (production draws)
  double mx = -INFINITY;
  int nan = 0;
  // VEC: whole runs in range and 16-byte aligned -> vector loads/stores
  // (fully coalesced: consecutive lanes own consecutive runs)
  const bool vec = (IPT % 4 == 0) && (N % IPT == 0) && sizeof(TW) == 4 && ((base & 3) == 0);
  double m;
  if constexpr (kFastExp) {
    if (vec && i0 < N) {
#pragma unroll
      for (int q = 0; q < IPT; q += 4) {
        const float4 v = __ldg(reinterpret_cast<const float4 *>(logw + base + i0 + q));
        lf[q] = v.x;
        lf[q + 1] = v.y;
        lf[q + 2] = v.z;
        lf[q + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int q = 0; q < IPT; ++q) lf[q] = i0 + q < N ? __ldg(logw + base + i0 + q) : -INFINITY;
    }
    // the thread's exponential spacings (independent of the weights) while
    // the log-weight loads are in flight
    {
      const Key2 key = load_key(keys, f);
#pragma unroll
      for (int q = 0; q < IPT; q += 4) {
        uint32_t wd[4];
        spacing_words<IPT>(key, t, i0 + q, wd);
#pragma unroll
        for (int h = 0; h < 4 && q + h < IPT; ++h) {
          const double e = i0 + q + h < N ? spacing_exp_fast_word(wd[h]) : 0.0;
          erun64 = __dadd_rn(erun64, e);
          u[q + h] = erun64;
        }
      }
    }
    float mf = -INFINITY;
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
      nan |= isnan(lf[q]);
      mf = fmaxf(mf, lf[q]);
    }
    nan = __syncthreads_or(nan);
    m = static_cast<double>(block_max_f(mf, reinterpret_cast<float *>(scratch)));
  } else {
  if (vec && i0 < N) {
#pragma unroll
    for (int q = 0; q < IPT; q += 4) {
      const float4 v = __ldg(reinterpret_cast<const float4 *>(logw + base + i0 + q));
      lw[q] = v.x;
      lw[q + 1] = v.y;
      lw[q + 2] = v.z;
      lw[q + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
      const int i = i0 + q;
      lw[q] = i < N ? static_cast<double>(__ldg(logw + base + i)) : -INFINITY;
    }
  }
  // production draws: this thread's exponential spacings are independent of
  // the weights - generated here, while the log-weight loads are in flight
  if constexpr (MODE == 0) {
    const Key2 key = load_key(keys, f);
#pragma unroll
    for (int q = 0; q < IPT; q += 4) {
      uint32_t wd[4];
      spacing_words<IPT>(key, t, i0 + q, wd);
#pragma unroll
      for (int h = 0; h < 4 && q + h < IPT; ++h) {
        const double e = i0 + q + h < N ? spacing_exp_fast_word(wd[h]) : 0.0;
        erun64 = __dadd_rn(erun64, e);
        u[q + h] = erun64;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < IPT; ++q) {
    if (i0 + q >= N) lw[q] = -INFINITY;
    nan |= isnan(lw[q]);
    mx = fmax(mx, lw[q]);
  }
  nan = __syncthreads_or(nan);
  m = block_max(mx, scratch);
  }
  if (nan || m == -INFINITY) {
    // NaN -> ValueError on the host; total underflow -> collapse: identity
    // ancestors, lnc unchanged (filters.py:105-109)
    double acc[kEstMaxDim] = {};
    for (int i = tid; i < N; i += blockDim.x) {
      anc[base + i] = static_cast<int32_t>(base + i);
      if (GATHER)
        for (int d = 0; d < gdims; ++d) gx_out[d * gMN + base + i] = gx_in[d * gMN + base + i];
      if (ex) {
#pragma unroll
        for (int d = 0; d < kEstMaxDim; ++d)
          if (d < ef.dim) acc[d] = __dadd_rn(acc[d], static_cast<double>(ex[d * ef.mn + base + i]));
      }
    }
    if (ex) est_block_write<THREADS>(acc, ef.dim, s_red, ef.est + f * ef.stride, invN);
    if (tid == 0) {
      collapsed[f] = nan ? 0 : 1;
      if (nan) atomicOr(status + f, PF_ST_NAN_WEIGHT);
      if (ef.lnc_tr) ef.lnc_tr[f] = lnc[f];
      if (ef.coll_tr) ef.coll_tr[f] = nan ? 0 : 1;
    }
    return;
  }

  // 2. e = exp(lw - m) and the total (core.py:134-135)
  // 3. w = e / total (IEEE division, core.py:136; production fp32 inputs:
  // reciprocal multiply), CDF = offset + local run
  double total, run = 0.0;
  if constexpr (kFastExp) {
    // production fp32: the thread's unnormalised weight runs and its
    // unnormalised exponential spacings (resampling.py:21-26) are scanned
    // together (one block scan of pairs); CDF = (offset + run) / total,
    // uniforms = (offset + run) / c[N]
    const float mf = static_cast<float>(m);
    float pf = 0.f;  // running sum of the thread's exp(lw - m)
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
      pf += exp_fast(lf[q] - mf);  // padding: exp(-inf) = 0
      lw[q] = static_cast<double>(pf);
    }
    const Key2 key = load_key(keys, f);
    double2 tot2;
    const double2 off2 =
        block_exclusive_scan2(make_double2(static_cast<double>(pf), erun64), scratch2, &tot2);
    total = tot2.x;
    const double inv_total = 1.0 / total;
#pragma unroll
    for (int q = 0; q < IPT; ++q)
      if (i0 + q < N) s_cum[q * THREADS + tid] = __dadd_rn(off2.x, lw[q]) * inv_total;
    const double cN = __dadd_rn(tot2.y, spacing_exp_fast(key, t, N));  // c[N]
    const double inv = 1.0 / cN;  // production draws: reciprocal multiply
#pragma unroll
    for (int q = 0; q < IPT; ++q) u[q] = i0 + q < N ? __dadd_rn(off2.y, u[q]) * inv : 2.0;
  } else {
    double part = 0.0;
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
      lw[q] = i0 + q < N ? exp(__dsub_rn(lw[q], m)) : 0.0;
      part = __dadd_rn(part, lw[q]);
    }
    total = block_sum(part, scratch);
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
      run = __dadd_rn(run, __ddiv_rn(lw[q], total));
      lw[q] = run;  // local inclusive prefix
    }
    // 4. this thread's sorted uniforms (resampling.py:21-26); production: the
    // CDF runs and the spacing runs in one block scan of pairs (each
    // component in block_exclusive_scan's association)
    double off;
    if constexpr (MODE == 1) {
      double wtot;
      off = block_exclusive_scan(run, scratch, &wtot);
#pragma unroll
      for (int q = 0; q < IPT; ++q) u[q] = i0 + q < N ? __ldg(u_tape + base + i0 + q) : 2.0;
    } else {
      double2 tot2;
      const double2 off2 = block_exclusive_scan2(make_double2(run, erun64), scratch2, &tot2);
      off = off2.x;
      const double cN = __dadd_rn(tot2.y, spacing_exp_fast(load_key(keys, f), t, N));  // c[N]
      const double inv = 1.0 / cN;  // production draws: reciprocal multiply
#pragma unroll
      for (int q = 0; q < IPT; ++q) u[q] = i0 + q < N ? __dadd_rn(off2.y, u[q]) * inv : 2.0;
    }
#pragma unroll
    for (int q = 0; q < IPT; ++q)
      if (i0 + q < N) s_cum[q * THREADS + tid] = __dadd_rn(off, lw[q]);
  }
  __syncthreads();  // s_cum complete

  // 5. merge: searchsorted(cum, u, 'left') clamped to N-1 (accel.py:175-197)
  // as a merge path over (cum, u): thread t merges the 2*IPT outputs on its
  // diagonal [2*IPT*t, 2*IPT*(t+1)), taking cum[a] before u[b] iff
  // cum[a] < u[b]; when u[b] is taken, a = #{cum < u[b]} is its ancestor.
  // Every thread does one diagonal binary search and exactly 2*IPT merge
  // steps, whatever the weight profile (flat CDF runs included).
  double *s_u = s_cum + THREADS * IPT;
  int32_t *s_anc = reinterpret_cast<int32_t *>(s_u + THREADS * IPT);
#pragma unroll
  for (int q = 0; q < IPT; ++q)
    if (i0 + q < N) s_u[q * THREADS + tid] = u[q];
  __syncthreads();
  {
    auto slot = [](unsigned i) { return (i & (IPT - 1)) * THREADS + i / IPT; };
    const int d0 = min(tid * 2 * IPT, 2 * N), d1 = min(d0 + 2 * IPT, 2 * N);
    const uint32_t sc = static_cast<uint32_t>(__cvta_generic_to_shared(s_cum));
    const uint32_t su = sc + 8u * static_cast<uint32_t>(THREADS * IPT);
    int lo = max(0, d0 - N), hi = min(d0, N);
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      double cm, um;
      asm volatile("ld.shared.f64 %0, [%1];" : "=d"(cm) : "r"(sc + 8u * slot(mid)));
      asm volatile("ld.shared.f64 %0, [%1];" : "=d"(um) : "r"(su + 8u * slot(d0 - 1 - mid)));
      if (cm < um)
        lo = mid + 1;
      else
        hi = mid;
    }
    int a = lo, b = d0 - lo;
    double ca = a < N ? s_cum[slot(a)] : INFINITY;
    double ub = b < N ? s_u[slot(b)] : INFINITY;
    // branch-free steps (no warp divergence): one predicated store and one
    // shared load of the next element of whichever sequence advanced, both
    // sequences addressed from one 32-bit shared base (s_u = s_cum +
    // THREADS*IPT; explicit ld/st.shared keep ptxas from re-deriving the
    // shared window address every step)
    const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(s_anc));
    auto step = [&]() {
      const bool ta = b >= N || ca < ub;
      const uint32_t av = static_cast<uint32_t>(base + (a < N - 1 ? a : N - 1));
      asm volatile(
          "{\n .reg .pred p;\n setp.eq.u32 p, %2, 0;\n @p st.shared.u32 [%0], %1;\n}\n" ::"r"(
              sa + 4u * slot(b)),
          "r"(av), "r"(static_cast<uint32_t>(ta))
          : "memory");
      a += ta;
      b += !ta;
      const int i = ta ? a : b;
      const uint32_t idx = slot(i) + (ta ? 0u : static_cast<uint32_t>(THREADS * IPT));
      double nv;
      asm volatile("ld.shared.f64 %0, [%1];" : "=d"(nv) : "r"(sc + 8u * idx));
      nv = i < N ? nv : INFINITY;
      ca = ta ? nv : ca;
      ub = ta ? ub : nv;
    };
    if (d1 - d0 == 2 * IPT) {  // every diagonal but the ones past 2N
#pragma unroll
      for (int st = 0; st < 2 * IPT; ++st) step();
    } else {
      for (int st = d0; st < d1; ++st) step();
    }
  }
  __syncthreads();
  if (i0 < N) {
    int32_t av[IPT];
#pragma unroll
    for (int q = 0; q < IPT; ++q) av[q] = i0 + q < N ? s_anc[q * THREADS + tid] : 0;
    if (vec) {
#pragma unroll
      for (int q = 0; q < IPT; q += 4)
        *reinterpret_cast<int4 *>(anc + base + i0 + q) =
            make_int4(av[q], av[q + 1], av[q + 2], av[q + 3]);
      if (GATHER && gdims == 3) {
        // 3-float state (cfg1): all 3*IPT gathered loads in flight first
        float g[3][IPT];
#pragma unroll
        for (int d = 0; d < 3; ++d)
#pragma unroll
          for (int q = 0; q < IPT; ++q) g[d][q] = __ldg(gx_in + d * gMN + av[q]);
#pragma unroll
        for (int d = 0; d < 3; ++d)
#pragma unroll
          for (int q = 0; q < IPT; q += 4)
            *reinterpret_cast<float4 *>(gx_out + d * gMN + base + i0 + q) =
                make_float4(g[d][q], g[d][q + 1], g[d][q + 2], g[d][q + 3]);
      } else if (GATHER) {
        for (int d = 0; d < gdims; ++d) {
          const float *src = gx_in + d * gMN;
          float *dst = gx_out + d * gMN + base + i0;
#pragma unroll
          for (int q = 0; q < IPT; q += 4)
            *reinterpret_cast<float4 *>(dst + q) =
                make_float4(__ldg(src + av[q]), __ldg(src + av[q + 1]), __ldg(src + av[q + 2]),
                            __ldg(src + av[q + 3]));
        }
      }
    } else {
#pragma unroll
      for (int q = 0; q < IPT; ++q) {
        if (i0 + q < N) {
          anc[base + i0 + q] = av[q];
          if (GATHER)
            for (int d = 0; d < gdims; ++d)
              gx_out[d * gMN + base + i0 + q] = __ldg(gx_in + d * gMN + av[q]);
        }
      }
    }
  }
  if (ex) {
    double acc[kEstMaxDim] = {};
#pragma unroll
    for (int q = 0; q < IPT; ++q)
      if (i0 + q < N) {
        const int64_t row = s_anc[q * THREADS + tid];
#pragma unroll
        for (int d = 0; d < kEstMaxDim; ++d)
          if (d < ef.dim) acc[d] = __dadd_rn(acc[d], static_cast<double>(ex[d * ef.mn + row]));
      }
    est_block_write<THREADS>(acc, ef.dim, s_red, ef.est + f * ef.stride, invN);
  }
  if (tid == 0) {
    collapsed[f] = 0;
    // log_mean_raw = (m + log(total)) - log(N); lnc += log_mean_raw
    const double lmr = __dsub_rn(__dadd_rn(m, log(total)), log(static_cast<double>(N)));
    const double l = __dadd_rn(lnc[f], lmr);
    lnc[f] = l;
    if (ef.lnc_tr) ef.lnc_tr[f] = l;
    if (ef.coll_tr) ef.coll_tr[f] = 0;
  }
}

// ---- wide path ----------------------------------------------------------
struct WideWs {
  double *tmax, *tsum, *twsum, *tesum, *twoff, *teoff;  // per tile
  double *m, *total, *cN;                               // per filter
  int *flag;                                            // per filter: 0 ok, 1 collapse, 2 nan
  double *cum;                                          // M*N
  // reference-order total: numpy pairwise leaves per filter (<= N/64 + 2)
  int64_t *leaf_start;
  int32_t *leaf_len;
  double *leaf_sum;
  int32_t *n_leaves;
  int64_t max_leaves;
  int64_t *klo, *khi;  // per u-tile CDF window (merge partition)
  double *cst;         // per (filter, tile chunk): max, weight sum, spacing sum, nan
};

constexpr int64_t kFilterChunk = 1024;  // tiles per CTA of the chunked filter pass (256 x 4)

static size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

static size_t wide_ws_layout(int64_t M, int64_t N, WideWs *w, char *base) {
  const int64_t tpf = (N + kTile - 1) / kTile;
  const int64_t nt = M * tpf;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char *p = base ? base + off : nullptr;
    off += align256(bytes);
    return p;
  };
  WideWs ws;
  ws.tmax = reinterpret_cast<double *>(take(nt * 8));
  ws.tsum = reinterpret_cast<double *>(take(nt * 8));
  ws.twsum = reinterpret_cast<double *>(take(nt * 8));
  ws.tesum = reinterpret_cast<double *>(take(nt * 8));
  ws.twoff = reinterpret_cast<double *>(take(nt * 8));
  ws.teoff = reinterpret_cast<double *>(take(nt * 8));
  ws.m = reinterpret_cast<double *>(take(M * 8));
  ws.total = reinterpret_cast<double *>(take(M * 8));
  ws.cN = reinterpret_cast<double *>(take(M * 8));
  ws.flag = reinterpret_cast<int *>(take(M * 4));
  ws.cum = reinterpret_cast<double *>(take(static_cast<size_t>(M) * N * 8));
  ws.max_leaves = N / 64 + 2;
  ws.leaf_start = reinterpret_cast<int64_t *>(take(static_cast<size_t>(M) * ws.max_leaves * 8));
  ws.leaf_len = reinterpret_cast<int32_t *>(take(static_cast<size_t>(M) * ws.max_leaves * 4));
  ws.leaf_sum = reinterpret_cast<double *>(take(static_cast<size_t>(M) * ws.max_leaves * 8));
  ws.n_leaves = reinterpret_cast<int32_t *>(take(M * 4));
  ws.klo = reinterpret_cast<int64_t *>(take(nt * 8));
  ws.khi = reinterpret_cast<int64_t *>(take(nt * 8));
  ws.cst = reinterpret_cast<double *>(take(static_cast<size_t>(M) * (tpf / kFilterChunk + 1) * 32));
  if (w) *w = ws;
  return off;
}

template <typename TW>
__global__ void __launch_bounds__(kTileThreads) wide_tile_max(const TW *__restrict__ logw,
                                                              int64_t N, int64_t tpf,
                                                              WideWs ws) {
  __shared__ double scratch[33];
  const int64_t tile = blockIdx.x;
  const int64_t f = tile / tpf, tt = tile - f * tpf;
  const int64_t i0 = tt * kTile, i1 = min(N, i0 + kTile);
  double mx = -INFINITY;
  int nan = 0;
  for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    const double v = load_lw(logw + f * N + i);
    nan |= isnan(v);
    mx = fmax(mx, v);
  }
  nan = __syncthreads_or(nan);
  const double m = block_max(mx, scratch);
  if (threadIdx.x == 0) ws.tmax[tile] = nan ? NAN : m;
}

__global__ void wide_filter_max(int64_t tpf, WideWs ws, uint8_t *collapsed, uint32_t *status) {
  __shared__ double scratch[33];
  const int64_t f = blockIdx.x;
  double mx = -INFINITY;
  int nan = 0;
  for (int64_t i = threadIdx.x; i < tpf; i += blockDim.x) {
    const double v = ws.tmax[f * tpf + i];
    nan |= isnan(v);
    mx = fmax(mx, v);
  }
  nan = __syncthreads_or(nan);
  const double m = block_max(mx, scratch);
  if (threadIdx.x == 0) {
    ws.m[f] = m;
    const int fl = nan ? 2 : (m == -INFINITY ? 1 : 0);
    ws.flag[f] = fl;
    collapsed[f] = fl == 1 ? 1 : 0;
    if (nan) atomicOr(status + f, PF_ST_NAN_WEIGHT);
  }
}



// tile sums of w and of the exponential spacings
template <typename TW, int MODE>
__global__ void __launch_bounds__(kTileThreads) wide_tile_sums(
    const TW *__restrict__ logw, int64_t N, int64_t tpf, WideWs ws,
    const double *__restrict__ u_tape, const uint32_t *__restrict__ keys, uint32_t t) {
  __shared__ double scratch[33];
  const int64_t tile = blockIdx.x;
  const int64_t f = tile / tpf, tt = tile - f * tpf;
  if (ws.flag[f]) return;
  const double m = ws.m[f], total = ws.total[f];
  const int64_t i0 = tt * kTile, i1 = min(N, i0 + kTile);
  double pw = 0.0, pe = 0.0;
  Key2 key{0u, 0u};
  if (MODE == 0) key = load_key(keys, f);
  for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    pw = __dadd_rn(pw, __ddiv_rn(exp(__dsub_rn(load_lw(logw + f * N + i), m)), total));
    if (MODE == 0) pe = __dadd_rn(pe, spacing_exp_fast(key, t, i));
  }
  const double sw = block_sum(pw, scratch);
  const double se = MODE == 0 ? block_sum(pe, scratch) : 0.0;
  if (threadIdx.x == 0) {
    ws.twsum[tile] = sw;
    ws.tesum[tile] = se;
  }
}

// exclusive tile offsets per filter: block per filter, carry across chunks
__global__ void wide_offsets_kernel(int64_t M, int64_t tpf, WideWs ws, int64_t N,
                                    const uint32_t *keys, uint32_t t) {
  // block per filter, sequential carry over tiles via block scan
  __shared__ double scratch[33];
  extern __shared__ double sbuf[];  // 2 * 1024 doubles
  const int64_t f = blockIdx.x;
  if (ws.flag[f]) return;
  double cw = 0.0, ce = 0.0;
  for (int64_t b0 = 0; b0 < tpf; b0 += 1024) {
    const int n = static_cast<int>((tpf - b0 < 1024 ? tpf - b0 : 1024));
    double *sw = sbuf, *se = sbuf + 1024;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      sw[i] = ws.twsum[f * tpf + b0 + i];
      se[i] = ws.tesum[f * tpf + b0 + i];
    }
    __syncthreads();
    // exclusive offsets = carry + inclusive scan - own
    const double cw_next = block_scan_inplace(sw, n, cw, scratch);
    const double ce_next = block_scan_inplace(se, n, ce, scratch);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      ws.twoff[f * tpf + b0 + i] = i == 0 ? cw : sw[i - 1];
      ws.teoff[f * tpf + b0 + i] = i == 0 ? ce : se[i - 1];
    }
    __syncthreads();
    cw = cw_next;
    ce = ce_next;
  }
  if (threadIdx.x == 0)  // c[N] = E_0 + ... + E_N
    ws.cN[f] = keys ? __dadd_rn(ce, spacing_exp_fast(load_key(keys, f), t, N)) : ce;
}

// cum for one tile -> ws.cum
// ---- per-thread runs for the wide path ------------------------------------
// Thread t of a tile owns the kRun consecutive elements [t*kRun, t*kRun+kRun)
// in registers: one block scan of run totals per tile (instead of one per
// 256 elements), vector loads, and a padded thread-major shared transpose for
// coalesced stores.
constexpr int kRun = kTile / kTileThreads;  // 8
constexpr int kPad = kTileThreads + 1;     // transpose row pitch (conflict-free)

template <typename TW>
__device__ __forceinline__ void load_run(const TW *p, int64_t avail, bool aligned, double *v) {
  if (sizeof(TW) == 4 && aligned && avail >= kRun) {
#pragma unroll
    for (int q = 0; q < kRun; q += 4) {
      const float4 x = __ldg(reinterpret_cast<const float4 *>(p + q));
      v[q] = x.x;
      v[q + 1] = x.y;
      v[q + 2] = x.z;
      v[q + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < kRun; ++q) v[q] = q < avail ? static_cast<double>(p[q]) : -INFINITY;
  }
}

// fp32 production log weights stay fp32 in registers (no fp64 conversions on
// the 16-lane XU pipe): -inf padding past `avail`
__device__ __forceinline__ void load_run_f(const float *p, int64_t avail, bool aligned, float *v) {
  if (aligned && avail >= kRun) {
#pragma unroll
    for (int q = 0; q < kRun; q += 4) {
      const float4 x = __ldg(reinterpret_cast<const float4 *>(p + q));
      v[q] = x.x;
      v[q + 1] = x.y;
      v[q + 2] = x.z;
      v[q + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < kRun; ++q) v[q] = q < avail ? __ldg(p + q) : -INFINITY;
  }
}

// kRun exponential spacings E_i, i = i0 .. i0+kRun-1 (i0 % 4 == 0): 4 Philox
// blocks, one 32-bit word per draw (same stream as spacing_exp_fast).
__device__ __forceinline__ void spacing_run(Key2 key, uint32_t t, int64_t i0, int64_t limit,
                                            double *e) {
#pragma unroll
  for (int q = 0; q < kRun; q += 4) {
    const uint4 r = philox10(make_uint4(static_cast<uint32_t>((i0 + q) >> 2), t,
                                        static_cast<uint32_t>((i0 + q) >> 34), kPurposeResample),
                             key);
    e[q] = i0 + q < limit ? spacing_exp_fast_word(r.x) : 0.0;
    e[q + 1] = i0 + q + 1 < limit ? spacing_exp_fast_word(r.y) : 0.0;
    e[q + 2] = i0 + q + 2 < limit ? spacing_exp_fast_word(r.z) : 0.0;
    e[q + 3] = i0 + q + 3 < limit ? spacing_exp_fast_word(r.w) : 0.0;
  }
}

// Gamma(a, 1) by Marsaglia & Tsang (a >= 1), fp64, counter-based: attempt
// `it` of tile `tile` uses Philox blocks (tile, t, it | {0, 2^31}).  In
// production mode the sum of a tile's a = n exponential spacings is drawn
// directly from Gamma(n) - S ~ Gamma(n) is independent of the normalised
// spacings E/S ~ Dirichlet(1..1) - so the pre-pass over every element's
// exponential disappears; the merge regenerates the tile's exponentials and
// rescales them to S (same joint law of the order statistics).
constexpr uint32_t kPurposeGamma = 0x47414D4Du;  // 'GAMM'

__device__ double gamma_tile_sum(Key2 key, uint32_t t, uint32_t tile, double a) {
  const double d = a - 1.0 / 3.0;
  const double c = 1.0 / sqrt(9.0 * d);
  for (uint32_t it = 0;; ++it) {
    const uint4 r = philox10(make_uint4(tile, t, it, kPurposeGamma), key);
    const double x = box_muller_f64(r.x, r.y, r.z, r.w).x;
    double v = 1.0 + c * x;
    if (v <= 0.0) continue;
    v = v * v * v;
    const uint4 r2 = philox10(make_uint4(tile, t, it | 0x80000000u, kPurposeGamma), key);
    const double u = u53_open0(r2.x, r2.y);
    if (log(u) < 0.5 * x * x + d - d * v + d * log(v)) return d * v;
  }
}

template <typename TW, bool FAST = false>
__global__ void __launch_bounds__(kTileThreads) wide_tile_cum(const TW *__restrict__ logw,
                                                              int64_t N, int64_t tpf,
                                                              WideWs ws) {
  __shared__ double scratch[33];
  __shared__ double s[kRun * kPad];
  const int64_t tile = blockIdx.x;
  const int64_t f = tile / tpf, tt = tile - f * tpf;
  if (ws.flag[f]) return;
  const double m = ws.m[f], total = ws.total[f];
  const int64_t i0 = tt * kTile;
  const int n = static_cast<int>((N - i0 < kTile ? N - i0 : kTile));
  const int r0 = threadIdx.x * kRun;
  double v[kRun];
  double run = 0.0;
  static_assert(!FAST || std::is_same<TW, float>::value, "FAST: fp32 log weights only");
  if constexpr (FAST) {
    // production fp32: w = exp(lw - tile max), an fp32 running sum over the
    // thread's run (the same association wide2_tile_stats sums in), scaled by
    // exp(tile max - max) / total in fp64 (see wide2_tile_stats)
    float lf[kRun];
    load_run_f(logw + f * N + i0 + r0, n - r0, ((f * N + i0) & 3) == 0, lf);
    const double mt = ws.tmax[tile];
    const bool live = mt != -INFINITY;  // an all -inf tile has weight 0
    const float mtf = static_cast<float>(mt);
    const double scale = live ? exp(__dsub_rn(mt, m)) / total : 0.0;
    float pf = 0.f;
#pragma unroll
    for (int q = 0; q < kRun; ++q) {
      if (live) pf += exp_fast(lf[q] - mtf);  // padding: exp(-inf) = 0
      v[q] = static_cast<double>(pf) * scale;
    }
    run = v[kRun - 1];
  } else {
    load_run(logw + f * N + i0 + r0, n - r0, ((f * N + i0) & 3) == 0, v);
#pragma unroll
    for (int q = 0; q < kRun; ++q) {
      const double w = r0 + q < n ? __ddiv_rn(exp(__dsub_rn(v[q], m)), total) : 0.0;
      run = __dadd_rn(run, w);
      v[q] = run;
    }
  }
  double tot;
  const double off = __dadd_rn(ws.twoff[tile], block_exclusive_scan(run, scratch, &tot));
#pragma unroll
  for (int q = 0; q < kRun; ++q) s[q * kPad + threadIdx.x] = __dadd_rn(off, v[q]);
  __syncthreads();
  double *out = ws.cum + f * N + i0;
  for (int e = threadIdx.x; e < n; e += kTileThreads) out[e] = s[(e % kRun) * kPad + e / kRun];
}



// ---- reference-order ("exact") CDF ----------------------------------------
__device__ double np_pairwise_sum(const double *a, int64_t n) {
  return np_pairwise_iter(a, n, nullptr);
}

// one thread, numpy cumsum order: c[0] = a[0], c[i] = c[i-1] + a[i]
__device__ void np_cumsum_serial(const double *a, double *c, int64_t n) {
  double run = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    run = i == 0 ? a[0] : __dadd_rn(run, a[i]);
    c[i] = run;
  }
}

// bank path, reference order; dynamic smem = 2*N doubles
template <typename TW, int MODE>
__global__ void __launch_bounds__(256) resample_bank_exact_kernel(
    const TW *__restrict__ logw, int32_t N, const double *__restrict__ u_tape,
    const uint32_t *__restrict__ keys, uint32_t t, int32_t *__restrict__ anc,
    double *__restrict__ lnc, uint8_t *__restrict__ collapsed, uint32_t *__restrict__ status) {
  extern __shared__ double sx[];
  double *s_a = sx, *s_cum = sx + N;
  __shared__ double scratch[33];
  __shared__ double s_total, s_cN;
  const int tid = threadIdx.x;
  const int64_t f = blockIdx.x, base = f * N;
  double mx = -INFINITY;
  int nan = 0;
  for (int i = tid; i < N; i += blockDim.x) {
    const double v = static_cast<double>(logw[base + i]);
    s_a[i] = v;
    nan |= isnan(v);
    mx = fmax(mx, v);
  }
  nan = __syncthreads_or(nan);
  const double m = block_max(mx, scratch);
  if (nan || m == -INFINITY) {
    for (int i = tid; i < N; i += blockDim.x) anc[base + i] = static_cast<int32_t>(base + i);
    if (tid == 0) {
      collapsed[f] = nan ? 0 : 1;
      if (nan) atomicOr(status + f, PF_ST_NAN_WEIGHT);
    }
    return;
  }
  for (int i = tid; i < N; i += blockDim.x) s_a[i] = exp(__dsub_rn(s_a[i], m));
  __syncthreads();
  if (tid == 0) s_total = np_pairwise_sum(s_a, N);  // shifted.sum(), core.py:135
  __syncthreads();
  const double total = s_total;
  for (int i = tid; i < N; i += blockDim.x) s_a[i] = __ddiv_rn(s_a[i], total);
  __syncthreads();
  if (tid == 0) np_cumsum_serial(s_a, s_cum, N);  // np.cumsum(weights), resampling.py:41
  __syncthreads();
  if (MODE == 1) {
    for (int i = tid; i < N; i += blockDim.x) s_a[i] = u_tape[base + i];
  } else {
    const Key2 key = load_key(keys, f);
    for (int i = tid; i < N; i += blockDim.x) s_a[i] = spacing_exp_fast(key, t, i);
    __syncthreads();
    if (tid == 0) {
      np_cumsum_serial(s_a, s_a, N);
      s_cN = __dadd_rn(s_a[N - 1], spacing_exp_fast(key, t, N));
    }
    __syncthreads();
    for (int i = tid; i < N; i += blockDim.x) s_a[i] = __ddiv_rn(s_a[i], s_cN);
  }
  __syncthreads();
  const int per = (N + blockDim.x - 1) / blockDim.x;
  const int j0 = tid * per, j1 = min(N, j0 + per);
  if (j0 < j1) {
    int k = lower_bound_f64(s_cum, N, s_a[j0]);
    for (int j = j0; j < j1; ++j) {
      k = advance_to<int>([&](int i) { return s_cum[i]; }, k, N, s_a[j]);
      anc[base + j] = static_cast<int32_t>(base + (k < N - 1 ? k : N - 1));
    }
  }
  if (tid == 0) {
    collapsed[f] = 0;
    const double lmr = __dsub_rn(__dadd_rn(m, log(total)), log(static_cast<double>(N)));
    lnc[f] = __dadd_rn(lnc[f], lmr);
  }
}

// wide path, reference order: e into ws.cum, numpy-order total (1 thread per
// filter), w = e/total, sequential cumsum (1 thread per filter).
template <typename TW>
__global__ void wide_exact_e(const TW *__restrict__ logw, int64_t N, int64_t tpf, WideWs ws) {
  const int64_t tile = blockIdx.x;
  const int64_t f = tile / tpf, tt = tile - f * tpf;
  if (ws.flag[f]) return;
  const double m = ws.m[f];
  const int64_t i0 = tt * kTile, i1 = min(N, i0 + kTile);
  for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x)
    ws.cum[f * N + i] = exp(__dsub_rn(load_lw(logw + f * N + i), m));
}

// numpy's recursion, split into (1) leaf enumeration (left to right),
// (2) parallel leaf sums, (3) the combine in the same tree order.
__device__ void np_enum_leaves(int64_t n_total, int64_t *start, int32_t *len, int32_t *cnt) {
  int64_t st_lo[48], st_n[48];
  int sp = 1;
  st_lo[0] = 0;
  st_n[0] = n_total;
  while (sp > 0) {
    --sp;
    const int64_t lo = st_lo[sp], n = st_n[sp];
    if (n <= 128) {
      start[*cnt] = lo;
      len[*cnt] = static_cast<int32_t>(n);
      ++*cnt;
      continue;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    st_lo[sp] = lo + n2;  // right pushed first -> left popped first
    st_n[sp] = n - n2;
    ++sp;
    st_lo[sp] = lo;
    st_n[sp] = n2;
    ++sp;
  }
}

__global__ void wide_exact_leaves(int64_t N, WideWs ws) {
  const int64_t f = blockIdx.x;
  if (threadIdx.x) return;
  int32_t cnt = 0;
  np_enum_leaves(N, ws.leaf_start + f * ws.max_leaves, ws.leaf_len + f * ws.max_leaves, &cnt);
  ws.n_leaves[f] = cnt;
}

__global__ void wide_exact_leafsum(int64_t N, WideWs ws) {
  const int64_t f = blockIdx.y;
  if (ws.flag[f]) return;
  const int64_t l = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (l >= ws.n_leaves[f]) return;
  const int64_t o = f * ws.max_leaves + l;
  ws.leaf_sum[o] = np_pairwise_block(ws.cum + f * N + ws.leaf_start[o], ws.leaf_len[o]);
}

__global__ void wide_exact_total(int64_t N, WideWs ws, double *lnc) {
  const int64_t f = blockIdx.x;
  if (ws.flag[f] || threadIdx.x) return;
  const double total = np_pairwise_iter(nullptr, N, ws.leaf_sum + f * ws.max_leaves);
  ws.total[f] = total;
  const double lmr = __dsub_rn(__dadd_rn(ws.m[f], log(total)), log(static_cast<double>(N)));
  lnc[f] = __dadd_rn(lnc[f], lmr);
}

__global__ void wide_exact_w(int64_t N, int64_t tpf, WideWs ws) {
  const int64_t tile = blockIdx.x;
  const int64_t f = tile / tpf, tt = tile - f * tpf;
  if (ws.flag[f]) return;
  const double total = ws.total[f];
  const int64_t i0 = tt * kTile, i1 = min(N, i0 + kTile);
  for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x)
    ws.cum[f * N + i] = __ddiv_rn(ws.cum[f * N + i], total);
}

// one warp per filter: the warp streams 1024-element tiles through shared
// memory (coalesced, next tile prefetched into registers) while lane 0 runs
// the strictly sequential numpy cumsum over the current tile.
__global__ void __launch_bounds__(32) wide_exact_cumsum(int64_t N, WideWs ws) {
  __shared__ double tile[2][1024];
  const int64_t f = blockIdx.x;
  if (ws.flag[f]) return;
  const int lane = threadIdx.x;
  double *c = ws.cum + f * N;
  const int64_t ntiles = (N + 1023) / 1024;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const int64_t i = j * 32 + lane;
    tile[0][j * 32 + lane] = i < N ? c[i] : 0.0;
  }
  __syncwarp();
  double run = 0.0;
  for (int64_t tt = 0; tt < ntiles; ++tt) {
    const int cur = tt & 1;
    double pre[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int64_t i = (tt + 1) * 1024 + j * 32 + lane;
      pre[j] = i < N ? c[i] : 0.0;
    }
    if (lane == 0) {
      const int64_t i0 = tt * 1024;
      const int cnt = static_cast<int>(N - i0 < 1024 ? N - i0 : 1024);
      int i = 0;
      if (tt == 0) {
        run = tile[cur][0];
        i = 1;
      }
#pragma unroll 8
      for (; i < cnt; ++i) {
        run = __dadd_rn(run, tile[cur][i]);
        tile[cur][i] = run;
      }
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int64_t i = tt * 1024 + j * 32 + lane;
      if (i < N) c[i] = tile[cur][j * 32 + lane];
      tile[cur ^ 1][j * 32 + lane] = pre[j];
    }
    __syncwarp();
  }
}

// ---- wide path, production (4 launches) -----------------------------------
// A: per tile, one read of the log weights: tile max m_t, s_t = sum exp(lw -
//    m_t) (online logsumexp) and the tile's sum of exponential spacings.
// B: per filter: m = max m_t, total = sum_t s_t exp(m_t - m) (fixed order),
//    lnc, exclusive tile offsets of the weights and of the spacings, c[N].
// C: per tile: w = exp(lw - m)/total, in-tile scan + offset -> cum (fp64).
// D: per u-tile: sorted uniforms, the CDF window they fall into is staged in
//    shared memory when it fits (galloping search in global memory when it
//    does not), ancestors and the fused gather written coalesced.
template <typename TW, int MODE, bool GAMMA = true>
__global__ void __launch_bounds__(kTileThreads) wide2_tile_stats(
    const TW *__restrict__ logw, int64_t N, int64_t tpf, WideWs ws,
    const uint32_t *__restrict__ keys, uint32_t t) {
  __shared__ double scratch[33];
  const int64_t tile = blockIdx.x;
  const int64_t f = tile / tpf, tt = tile - f * tpf;
  const int64_t i0 = tt * kTile;
  const int n = static_cast<int>(N - i0 < kTile ? N - i0 : kTile);
  const int r0 = threadIdx.x * kRun;
  if constexpr (MODE == 0 && std::is_same<TW, float>::value) {
    // production fp32: max, expf and the run sums in fp32 (wide_tile_cum<float,
    // true> recomputes exactly these run sums), one fp64 conversion per thread
    float lf[kRun];
    load_run_f(logw + f * N + i0 + r0, n - r0, ((f * N + i0) & 3) == 0, lf);
    float mxf = -INFINITY;
    int nanf = 0;
#pragma unroll
    for (int q = 0; q < kRun; ++q) {
      nanf |= isnan(lf[q]);
      mxf = fmaxf(mxf, lf[q]);
    }
    nanf = __syncthreads_or(nanf);
    const double mt = block_max_f(mxf, reinterpret_cast<float *>(scratch));
    float pf = 0.f;
    if (mt != -INFINITY) {
      const float mtf = static_cast<float>(mt);
#pragma unroll
      for (int q = 0; q < kRun; ++q) pf += exp_fast(lf[q] - mtf);
    }
    const double ssum = block_sum(static_cast<double>(pf), scratch);
    if (threadIdx.x == 0) {
      ws.tmax[tile] = nanf ? NAN : mt;
      ws.tsum[tile] = mt == -INFINITY ? 0.0 : ssum;
      if (GAMMA)
        ws.tesum[tile] = gamma_tile_sum(load_key(keys, f), t, static_cast<uint32_t>(tt),
                                        static_cast<double>(n));
    }
    return;
  }
  double lv[kRun];
  load_run(logw + f * N + i0 + r0, n - r0, ((f * N + i0) & 3) == 0, lv);
  double mx = -INFINITY;
  int nan = 0;
#pragma unroll
  for (int q = 0; q < kRun; ++q) {
    if (r0 + q >= n) lv[q] = -INFINITY;
    nan |= isnan(lv[q]);
    mx = fmax(mx, lv[q]);
  }
  nan = __syncthreads_or(nan);
  const double m = block_max(mx, scratch);
  double part = 0.0;
  if (m != -INFINITY) {  // fp64 exp against the tile max (tape mode, fp64 inputs)
#pragma unroll
    for (int q = 0; q < kRun; ++q)
      part = __dadd_rn(part, exp(__dsub_rn(lv[q], m)));
  }
  const double ssum = block_sum(part, scratch);
  if (threadIdx.x == 0) {
    ws.tmax[tile] = nan ? NAN : m;
    ws.tsum[tile] = m == -INFINITY ? 0.0 : ssum;
    // production: the tile's exponential-spacing sum S ~ Gamma(n) (gamma_tile_sum)
    if (GAMMA)
      ws.tesum[tile] = MODE == 0 ? gamma_tile_sum(load_key(keys, f), t, static_cast<uint32_t>(tt),
                                                  static_cast<double>(n))
                                 : 0.0;
  }
}

// Production tile spacing sums S_tile ~ Gamma(n_tile) (gamma_tile_sum), one
// thread per tile: the rejection sampler's fp64 latency no longer sits at the
// end of every stats CTA (same values, same counters).
__global__ void __launch_bounds__(128) wide2_gamma(int64_t M, int64_t N, int64_t tpf, WideWs ws,
                                                   const uint32_t *__restrict__ keys,
                                                   uint32_t t) {
  const int64_t tile = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (tile >= M * tpf) return;
  const int64_t f = tile / tpf, tt = tile - f * tpf;
  const int64_t n = N - tt * kTile < kTile ? N - tt * kTile : kTile;
  ws.tesum[tile] = gamma_tile_sum(load_key(keys, f), t, static_cast<uint32_t>(tt),
                                  static_cast<double>(n));
}

// Production filter totals for very wide filters (tpf > kFilterChunk tiles):
// the single-CTA wide2_filter walks 32K tiles on one SM (88 us at N = 2^26).
// A: one 256-thread CTA per (chunk, filter): chunk max, weight sum relative
//    to it, spacing sum, chunk-local exclusive scans into twoff / teoff.
// B: one warp per filter combines the chunks (online max rescaling).
// C: per (chunk, filter): rescale the local scans to global offsets.
__global__ void __launch_bounds__(256) wide2_chunk_scan(int64_t tpf, WideWs ws) {
  constexpr int kFr = kFilterChunk / 256;
  __shared__ double scratch[33];
  const int64_t f = blockIdx.y, c = blockIdx.x, nch = gridDim.x;
  const int64_t j0 = c * kFilterChunk + static_cast<int64_t>(threadIdx.x) * kFr;
  const double *tmax = ws.tmax + f * tpf, *tsum = ws.tsum + f * tpf, *tes = ws.tesum + f * tpf;
  double mv[kFr];
  double mx = -INFINITY;
  int nan = 0;
#pragma unroll
  for (int q = 0; q < kFr; ++q) {
    mv[q] = j0 + q < tpf ? tmax[j0 + q] : -INFINITY;
    nan |= isnan(mv[q]);
    mx = fmax(mx, mv[q]);
  }
  nan = __syncthreads_or(nan);
  const double cm = block_max(mx, scratch);
  double wv[kFr], ev[kFr];
  double rw = 0.0, re = 0.0;
#pragma unroll
  for (int q = 0; q < kFr; ++q) {
    const int64_t j = j0 + q;
    const double w = (j < tpf && cm != -INFINITY && !nan) ? tsum[j] * exp(mv[q] - cm) : 0.0;
    const double e = j < tpf ? tes[j] : 0.0;
    wv[q] = rw;
    ev[q] = re;
    rw += w;
    re += e;
  }
  double tw, te;
  const double ow = block_exclusive_scan(rw, scratch, &tw);
  const double oe = block_exclusive_scan(re, scratch, &te);
#pragma unroll
  for (int q = 0; q < kFr; ++q) {
    const int64_t j = j0 + q;
    if (j < tpf) {
      ws.twoff[f * tpf + j] = ow + wv[q];
      ws.teoff[f * tpf + j] = oe + ev[q];
    }
  }
  if (threadIdx.x == 0) {
    double *cs = ws.cst + (f * nch + c) * 4;
    cs[0] = cm;
    cs[1] = tw;
    cs[2] = te;
    cs[3] = nan ? 1.0 : 0.0;
  }
}

// one warp per filter: lanes take chunks 32 at a time (max, then an
// in-order scan of the rescaled chunk sums with a running carry)
__global__ void __launch_bounds__(128) wide2_chunk_combine(int64_t M, int64_t N, int64_t nch,
                                                           WideWs ws, uint8_t *collapsed,
                                                           uint32_t *status, double *lnc,
                                                           const uint32_t *keys, uint32_t t) {
  const int64_t f = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (f >= M) return;  // whole warps
  double *cs = ws.cst + f * nch * 4;
  double m = -INFINITY;
  int nan = 0;
  for (int64_t c = lane; c < nch; c += 32) {
    nan |= cs[4 * c + 3] != 0.0;
    m = fmax(m, cs[4 * c]);
  }
  m = warp_max(m);
  m = __shfl_sync(0xffffffffu, m, 0);
  nan = __any_sync(0xffffffffu, nan);
  const int fl = nan ? 2 : (m == -INFINITY ? 1 : 0);
  if (lane == 0) {
    ws.flag[f] = fl;
    ws.m[f] = m;
    collapsed[f] = fl == 1 ? 1 : 0;
    if (nan) atomicOr(status + f, PF_ST_NAN_WEIGHT);
  }
  if (fl) return;
  double cw = 0.0, ce = 0.0;  // carries
  for (int64_t c0 = 0; c0 < nch; c0 += 32) {
    const int64_t c = c0 + lane;
    double w = 0.0, e = 0.0;
    if (c < nch) {
      w = cs[4 * c] == -INFINITY ? 0.0 : cs[4 * c + 1] * exp(cs[4 * c] - m);
      e = cs[4 * c + 2];
    }
    double iw = w, ie = e;  // inclusive warp scans
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double yw = __shfl_up_sync(0xffffffffu, iw, o);
      const double ye = __shfl_up_sync(0xffffffffu, ie, o);
      if (lane >= o) {
        iw += yw;
        ie += ye;
      }
    }
    if (c < nch) {  // exclusive chunk offsets, in place
      cs[4 * c + 1] = cw + (iw - w);
      cs[4 * c + 2] = ce + (ie - e);
    }
    cw += __shfl_sync(0xffffffffu, iw, 31);
    ce += __shfl_sync(0xffffffffu, ie, 31);
  }
  if (lane == 0) {
    ws.total[f] = cw;
    ws.cN[f] = ce + spacing_exp_fast(load_key(keys, f), t, N);
    lnc[f] = lnc[f] + ((m + log(cw)) - log(static_cast<double>(N)));
  }
}

__global__ void __launch_bounds__(256) wide2_chunk_apply(int64_t tpf, WideWs ws) {
  constexpr int kFr = kFilterChunk / 256;
  const int64_t f = blockIdx.y, c = blockIdx.x, nch = gridDim.x;
  if (ws.flag[f]) return;
  const double *cs = ws.cst + (f * nch + c) * 4;
  const double inv = 1.0 / ws.total[f];
  const double scale = cs[0] == -INFINITY ? 0.0 : exp(cs[0] - ws.m[f]);
  const double ow = cs[1], oe = cs[2];
  const int64_t j0 = c * kFilterChunk + static_cast<int64_t>(threadIdx.x) * kFr;
#pragma unroll
  for (int q = 0; q < kFr; ++q) {
    const int64_t j = f * tpf + j0 + q;
    if (j0 + q < tpf) {
      ws.twoff[j] = fma(ws.twoff[j], scale, ow) * inv;
      ws.teoff[j] += oe;
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(1024) wide2_filter(int64_t N, int64_t tpf, WideWs ws,
                                                     uint8_t *collapsed, uint32_t *status,
                                                     double *lnc, const uint32_t *keys,
                                                     uint32_t t) {
  // one CTA per filter, 1024 threads; each thread owns runs of kFr
  // consecutive tiles (weights in registers), so the per-filter max, total
  // and the two tile-offset scans are one block reduction / scan per 16K
  // tiles instead of a serial walk
  constexpr int kFr = 8;
  __shared__ double scratch[33];
  const int64_t f = blockIdx.x;
  const double *tmax = ws.tmax + f * tpf, *tsum = ws.tsum + f * tpf, *tes = ws.tesum + f * tpf;
  double mx = -INFINITY;
  int nan = 0;
  for (int64_t i = threadIdx.x; i < tpf; i += blockDim.x) {
    const double v = tmax[i];
    nan |= isnan(v);
    mx = fmax(mx, v);
  }
  nan = __syncthreads_or(nan);
  const double m = block_max(mx, scratch);
  const int fl = nan ? 2 : (m == -INFINITY ? 1 : 0);
  if (threadIdx.x == 0) {
    ws.flag[f] = fl;
    ws.m[f] = m;
    collapsed[f] = fl == 1 ? 1 : 0;
    if (nan) atomicOr(status + f, PF_ST_NAN_WEIGHT);
  }
  if (fl) return;
  double part = 0.0;
  for (int64_t i = threadIdx.x; i < tpf; i += blockDim.x)
    part = __dadd_rn(part, __dmul_rn(tsum[i], exp(__dsub_rn(tmax[i], m))));
  const double total = block_sum(part, scratch);
  const double inv = 1.0 / total;
  double cw = 0.0, ce = 0.0;
  for (int64_t b0 = 0; b0 < tpf; b0 += static_cast<int64_t>(kFr) * blockDim.x) {
    const int64_t j0 = b0 + static_cast<int64_t>(threadIdx.x) * kFr;
    double wv[kFr], ev[kFr];
    double rw = 0.0, re = 0.0;
#pragma unroll
    for (int q = 0; q < kFr; ++q) {
      const int64_t j = j0 + q;
      const double w = j < tpf
                           ? (MODE == 1 ? __ddiv_rn(__dmul_rn(tsum[j], exp(__dsub_rn(tmax[j], m))),
                                                    total)
                                        : __dmul_rn(tsum[j], exp(__dsub_rn(tmax[j], m))) * inv)
                           : 0.0;
      const double e = j < tpf ? tes[j] : 0.0;
      wv[q] = rw;  // exclusive within the run
      ev[q] = re;
      rw = __dadd_rn(rw, w);
      re = __dadd_rn(re, e);
    }
    double tw, te;
    const double ow = __dadd_rn(cw, block_exclusive_scan(rw, scratch, &tw));
    const double oe = __dadd_rn(ce, block_exclusive_scan(re, scratch, &te));
#pragma unroll
    for (int q = 0; q < kFr; ++q) {
      const int64_t j = j0 + q;
      if (j < tpf) {
        ws.twoff[f * tpf + j] = __dadd_rn(ow, wv[q]);
        ws.teoff[f * tpf + j] = __dadd_rn(oe, ev[q]);
      }
    }
    cw = __dadd_rn(cw, tw);
    ce = __dadd_rn(ce, te);
  }
  if (threadIdx.x == 0) {
    ws.total[f] = total;
    if (MODE == 0) ws.cN[f] = __dadd_rn(ce, spacing_exp_fast(load_key(keys, f), t, N));
    const double lmr = __dsub_rn(__dadd_rn(m, log(total)), log(static_cast<double>(N)));
    lnc[f] = __dadd_rn(lnc[f], lmr);
  }
}

constexpr int kWin = 4096;  // CDF window staged in shared memory (32 KB)

// Merge partition: one thread per (u-tile, end) finds the CDF index range the
// tile's uniforms fall into.  Thousands of independent binary searches run
// concurrently, so their dependent-load latency overlaps (a search inside
// the merge CTA would stall the whole block).  The tile's first and last
// uniforms are recomputed from the tile offsets; a relative margin absorbs
// the different association of the in-tile scan.
template <int MODE>
__global__ void wide2_partition(int64_t N, int64_t tpf, int64_t ntiles, WideWs ws,
                                const double *__restrict__ u_tape,
                                const uint32_t *__restrict__ keys, uint32_t t) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= 2 * ntiles) return;
  const int64_t tile = g >> 1;
  const bool last = g & 1;
  const int64_t f = tile / tpf, tt = tile - f * tpf;
  if (ws.flag[f]) return;
  const int64_t i0 = tt * kTile;
  const int64_t n = N - i0 < kTile ? N - i0 : kTile;
  double u;
  if (MODE == 1) {
    u = u_tape[f * N + i0 + (last ? n - 1 : 0)];
  } else {
    // first uniform of the tile >= teoff / cN; last = (teoff + S_tile) / cN
    const double c = last ? __dadd_rn(ws.teoff[tile], ws.tesum[tile]) : ws.teoff[tile];
    u = c / ws.cN[f];
  }
  const double x = last ? u * (1.0 + 1e-12) : u * (1.0 - 1e-12);
  int64_t k = lower_bound_f64_64(ws.cum + f * N, N, x);
  if (last) {
    k = k + 1 < N ? k + 1 : N - 1;
    ws.khi[tile] = k;
  } else {
    ws.klo[tile] = k > 0 ? k - 1 : 0;
  }
}

// 8-byte global -> shared asynchronous copies (LDGSTS): the CDF window lands
// in shared memory while the uniforms are generated, without staging
// registers
__device__ __forceinline__ void cp_async8(double *smem, const double *gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// dynamic shared-memory bytes of wide2_merge<.., SEARCH>
constexpr size_t wide2_merge_smem(bool search) {
  return (kWin + (search ? 0 : kTile)) * sizeof(double) + kRun * kPad * sizeof(int32_t);
}

template <int MODE, bool GATHER, bool SEARCH = false>
__global__ void __launch_bounds__(kTileThreads, SEARCH ? 4 : 3) wide2_merge(
    int64_t N, int64_t tpf, WideWs ws, const double *__restrict__ u_tape,
    const uint32_t *__restrict__ keys, uint32_t t, int32_t *__restrict__ anc,
    const float *__restrict__ gx_in, float *__restrict__ gx_out, int gdims, int64_t gMN) {
  // dynamic shared: CDF window | uniforms (merge-path variant) | ancestor transpose
  extern __shared__ double s_dyn[];
  double *s_c = s_dyn;
  double *s_u = s_dyn + kWin;
  int32_t *s_a = reinterpret_cast<int32_t *>(s_u + (SEARCH ? 0 : kTile));
  __shared__ double scratch[33];
  const int64_t tile = blockIdx.x;
  const int64_t f = tile / tpf, tt = tile - f * tpf;
  const int64_t i0 = tt * kTile;
  const int n = static_cast<int>(N - i0 < kTile ? N - i0 : kTile);
  const int64_t base = f * N;
  // the filter flag, the CDF window bounds and (production) the thread's
  // exponential spacings are independent: their loads and the Philox / lg2
  // work overlap instead of running back to back
  const int fl = ws.flag[f];
  const int64_t lo = ws.klo[tile], hi = ws.khi[tile];
  const int r0 = threadIdx.x * kRun;
  double u[kRun];
  if (MODE == 0) spacing_run(load_key(keys, f), t, i0 + r0, N, u);
  if (fl) {  // collapse / NaN: identity ancestors (filters.py:105-109)
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      anc[base + i0 + i] = static_cast<int32_t>(base + i0 + i);
      if (GATHER)
        for (int d = 0; d < gdims; ++d)
          gx_out[d * gMN + base + i0 + i] = gx_in[d * gMN + base + i0 + i];
    }
    return;
  }
  const double *cum = ws.cum + base;
  const int64_t wlen = hi - lo + 1;
  const bool chunked = wlen <= 16 * static_cast<int64_t>(kWin);
  // start the first CDF chunk's copy into shared memory now; it lands while
  // the uniforms are generated below
  constexpr int kPer = kWin / kTileThreads;
  const int len0 = static_cast<int>(wlen < kWin ? wlen : kWin);
  if (chunked) {
#pragma unroll
    for (int r = 0; r < kPer; ++r) {
      const int i = r * kTileThreads + threadIdx.x;
      if (i < len0) cp_async8(s_c + i, cum + lo + i);
    }
    cp_async_commit();
  }
  // this thread's run of sorted uniforms, in registers
  if (MODE == 1) {
#pragma unroll
    for (int q = 0; q < kRun; ++q) u[q] = r0 + q < n ? u_tape[base + i0 + r0 + q] : 2.0;
  } else {
    double run = 0.0;
#pragma unroll
    for (int q = 0; q < kRun; ++q) {
      run = __dadd_rn(run, u[q]);
      u[q] = run;
    }
    double tot;
    const double eoff = block_exclusive_scan(run, scratch, &tot);
    // rescale the tile's spacings to its Gamma-drawn sum S (wide2_filter)
    const double scale = ws.tesum[tile] / tot, teoff = ws.teoff[tile];
    const double inv = 1.0 / ws.cN[f];
#pragma unroll
    for (int q = 0; q < kRun; ++q)
      u[q] = r0 + q < n ? fma(__dadd_rn(eoff, u[q]), scale, teoff) * inv : 2.0;
  }
  int32_t a[kRun];
  if (SEARCH && wlen <= kWin) {
    // the window in shared memory; each thread: one binary search for its
    // first uniform, then a galloping walk for the rest of its sorted run
    cp_async_wait_all();
    __syncthreads();
    const int A = static_cast<int>(wlen);
    const int kcap = static_cast<int>(N - 1 - lo);
    const int32_t row0 = static_cast<int32_t>(base + lo);
    // explicit 32-bit shared loads: ptxas otherwise re-derives the shared
    // window address inside the search loops
    const uint32_t scb = static_cast<uint32_t>(__cvta_generic_to_shared(s_c));
    auto cs = [&](int i) {
      double v;
      asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(scb + 8u * static_cast<uint32_t>(i)));
      return v;
    };
    int k = 0;
    if (r0 < n) {
      int hi2 = A;
      const double x = u[0];
      while (k < hi2) {
        const int mid = (k + hi2) >> 1;
        if (cs(mid) < x)
          k = mid + 1;
        else
          hi2 = mid;
      }
    }
#pragma unroll
    for (int q = 0; q < kRun; ++q) {
      if (r0 + q < n) k = advance_to<int>(cs, k, A, u[q]);
      a[q] = row0 + (k < kcap ? k : kcap);
    }
  } else if (wlen <= kWin) {
    // fast path: the whole CDF window and the tile's uniforms sit in shared
    // memory; a merge path gives every thread one diagonal binary search and
    // a fixed number of merge steps (cum[k] taken before u iff cum[k] < u)
    auto us = [](unsigned j) { return (j % kRun) * kTileThreads + j / kRun; };
    cp_async_wait_all();
#pragma unroll
    for (int q = 0; q < kRun; ++q)
      if (r0 + q < n) s_u[q * kTileThreads + threadIdx.x] = u[q];
    __syncthreads();
    const int A = static_cast<int>(wlen), L = A + n;
    const int per = (L + kTileThreads - 1) / kTileThreads;
    const int d0 = min(static_cast<int>(threadIdx.x) * per, L), d1 = min(d0 + per, L);
    int lo2 = max(0, d0 - n), hi2 = min(d0, A);
    while (lo2 < hi2) {
      const int mid = (lo2 + hi2) >> 1;
      if (s_c[mid] < s_u[us(d0 - 1 - mid)])
        lo2 = mid + 1;
      else
        hi2 = mid;
    }
    // branch-free merge: lanes differ only in which list they advance; one
    // shared load per step from the selected list (no divergent paths)
    unsigned ka = lo2, jb = d0 - lo2;
    const unsigned uA = A, un = n;
    const unsigned kcap = static_cast<unsigned>(N - 1 - lo);  // clamp to N-1 (accel.py:183)
    const int32_t row0 = static_cast<int32_t>(base + lo);
    double ca = ka < uA ? s_c[ka] : INFINITY;
    double ub = jb < un ? s_u[us(jb)] : INFINITY;
    for (int d = d0; d < d1; ++d) {
      const bool take_c = jb >= un || ca < ub;
      if (!take_c) s_a[(jb & (kRun - 1)) * kPad + jb / kRun] =
          row0 + static_cast<int32_t>(ka < kcap ? ka : kcap);
      ka += take_c;
      jb += !take_c;
      const double *src = take_c ? s_c + (ka < uA ? ka : uA - 1) : s_u + us(jb < un ? jb : un - 1);
      const double v = *src;
      ca = take_c ? (ka < uA ? v : INFINITY) : ca;
      ub = take_c ? ub : (jb < un ? v : INFINITY);
    }
    __syncthreads();
  } else if (chunked) {
    // stream the CDF window through shared memory in kWin chunks; every
    // uniform is placed in the chunk holding its answer (answers are
    // non-decreasing, so each thread resumes from its previous answer)
    uint32_t done = 0;
    int64_t k = lo;
    for (int64_t c0 = lo; c0 <= hi; c0 += kWin) {
      const int len = static_cast<int>(hi - c0 + 1 < kWin ? hi - c0 + 1 : kWin);
      __syncthreads();  // previous chunk consumed
      if (c0 != lo) {
#pragma unroll
        for (int r = 0; r < kPer; ++r) {
          const int i = r * kTileThreads + threadIdx.x;
          if (i < len) cp_async8(s_c + i, cum + c0 + i);
        }
        cp_async_commit();
      }
      cp_async_wait_all();
      __syncthreads();
      const bool last = c0 + len > hi;
      const double cmax = s_c[len - 1];
#pragma unroll
      for (int q = 0; q < kRun; ++q) {
        if ((done >> q) & 1u) continue;
        if (r0 + q >= n) {
          a[q] = static_cast<int32_t>(base);
          done |= 1u << q;
          continue;
        }
        if (!(u[q] <= cmax) && !last) break;  // this and later uniforms: later chunks
        int kl = static_cast<int>(k - c0 > 0 ? k - c0 : 0);
        kl = advance_to<int>([&](int i) { return s_c[i]; }, kl, len, u[q]);
        k = c0 + kl;
        a[q] = static_cast<int32_t>(base + (k < N - 1 ? k : N - 1));
        done |= 1u << q;
      }
    }
  } else {  // extreme window: galloping search in global memory
    int64_t k = r0 < n ? lo + lower_bound_f64_64(cum + lo, wlen, u[0]) : lo;
#pragma unroll
    for (int q = 0; q < kRun; ++q) {
      if (r0 + q < n) k = advance_to<int64_t>([&](int64_t i) { return __ldg(cum + i); }, k, N, u[q]);
      a[q] = static_cast<int32_t>(base + (k < N - 1 ? k : N - 1));
    }
  }
  if (wlen > kWin || SEARCH) {
#pragma unroll
    for (int q = 0; q < kRun; ++q) s_a[q * kPad + threadIdx.x] = a[q];
    __syncthreads();
  }
  if (GATHER && gdims == 3) {
    // the 3-float state (cfg1): all 24 gathered loads of the thread's 8
    // outputs in flight before the first store
    int32_t ai[kRun];
#pragma unroll
    for (int h = 0; h < kRun; ++h) {
      const int e = threadIdx.x + h * kTileThreads;
      ai[h] = e < n ? s_a[(e % kRun) * kPad + e / kRun] : 0;
      if (e < n) anc[base + i0 + e] = ai[h];
    }
    float v[3][kRun];
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int h = 0; h < kRun; ++h)
        v[d][h] = threadIdx.x + h * kTileThreads < n ? __ldg(gx_in + d * gMN + ai[h]) : 0.f;
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int h = 0; h < kRun; ++h) {
        const int e = threadIdx.x + h * kTileThreads;
        if (e < n) gx_out[d * gMN + base + i0 + e] = v[d][h];
      }
    return;
  }
  // coalesced write-out (thread-strided elements), gather loads batched 4 deep
  for (int e0 = threadIdx.x; e0 < n; e0 += 4 * kTileThreads) {
    int32_t ai[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int e = e0 + h * kTileThreads;
      ai[h] = e < n ? s_a[(e % kRun) * kPad + e / kRun] : 0;
      if (e < n) anc[base + i0 + e] = ai[h];
    }
    if (GATHER) {
      for (int d = 0; d < gdims; ++d) {
        float v[4];
#pragma unroll
        for (int h = 0; h < 4; ++h)
          v[h] = e0 + h * kTileThreads < n ? __ldg(gx_in + d * gMN + ai[h]) : 0.f;
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int e = e0 + h * kTileThreads;
          if (e < n) gx_out[d * gMN + base + i0 + e] = v[h];
        }
      }
    }
  }
}

// ---- wide path, production with fp32 log weights: no materialised CDF ------
// wide_tile_cum + wide2_partition + wide2_merge write and re-read an fp64 CDF
// (16 B per particle of the 52 B the pipeline moved).  Here the partition
// works on the per-tile CDF offsets (twoff) only, and each merge CTA
// recomputes the CDF of the few weight tiles its uniforms fall into, in
// shared memory, from the fp32 log weights - with exactly wide_tile_cum<float,
// true>'s arithmetic (same fp32 runs, same 256-thread block scan, same
// offsets), so the ancestors are identical to the materialised pipeline's.

// CDF of weight tile `tile` (filter f, tile index tt) into s_c, transposed
// (element e at s_c[(e % kRun) * kPad + e / kRun]: conflict-free stores);
// returns the tile's element count.  All kTileThreads threads participate.
__device__ __forceinline__ int tile_cdf_f32(const float *__restrict__ logw, int64_t N,
                                            int64_t tpf, const WideWs &ws, int64_t f,
                                            int64_t tt, double m, double total, double *s_c,
                                            double *scratch) {
  const int64_t tile = f * tpf + tt;
  const int64_t i0 = tt * kTile;
  const int n = static_cast<int>(N - i0 < kTile ? N - i0 : kTile);
  const int r0 = threadIdx.x * kRun;
  float lf[kRun];
  load_run_f(logw + f * N + i0 + r0, n - r0, ((f * N + i0) & 3) == 0, lf);
  const double mt = ws.tmax[tile];
  const bool live = mt != -INFINITY;
  const float mtf = static_cast<float>(mt);
  const double scale = live ? exp(__dsub_rn(mt, m)) / total : 0.0;
  double v[kRun];
  float pf = 0.f;
#pragma unroll
  for (int q = 0; q < kRun; ++q) {
    if (live) pf += exp_fast(lf[q] - mtf);
    v[q] = static_cast<double>(pf) * scale;
  }
  double tot;
  const double off = __dadd_rn(ws.twoff[tile], block_exclusive_scan(v[kRun - 1], scratch, &tot));
#pragma unroll
  for (int q = 0; q < kRun; ++q) s_c[q * kPad + threadIdx.x] = __dadd_rn(off, v[q]);
  return n;
}

// Partition on tile offsets: for each u-tile end, the weight tile its answer
// lies in.  The first tile is the last one whose CDF offset lies below the
// tile's first uniform (minus a relative margin that covers the different
// association of the in-tile scan); the last, the last whose offset lies at
// or below the last uniform (plus the margin).
template <int MODE>
__global__ void wide3_partition(int64_t N, int64_t tpf, int64_t ntiles, WideWs ws,
                                const double *__restrict__ u_tape) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= 2 * ntiles) return;
  const int64_t tile = g >> 1;
  const bool last = g & 1;
  const int64_t f = tile / tpf, tt = tile - f * tpf;
  if (ws.flag[f]) return;
  const int64_t i0 = tt * kTile;
  const int64_t n = N - i0 < kTile ? N - i0 : kTile;
  double u;
  if (MODE == 1) {
    u = u_tape[f * N + i0 + (last ? n - 1 : 0)];
  } else {
    const double c = last ? __dadd_rn(ws.teoff[tile], ws.tesum[tile]) : ws.teoff[tile];
    u = c / ws.cN[f];
  }
  const double *off = ws.twoff + f * tpf;
  // count of tiles whose offset is < x (first) / <= x (last)
  const double x = last ? u * (1.0 + 1e-12) : u * (1.0 - 1e-12);
  int64_t lo = 0, hi = tpf;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (last ? !(off[mid] > x) : off[mid] < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  const int64_t tsel = lo > 0 ? lo - 1 : 0;
  if (last)
    ws.khi[tile] = tsel;
  else
    ws.klo[tile] = tsel;
}

template <int MODE, bool GATHER>
__global__ void __launch_bounds__(kTileThreads, 4) wide3_merge(
    const float *__restrict__ logw, int64_t N, int64_t tpf, WideWs ws,
    const double *__restrict__ u_tape, const uint32_t *__restrict__ keys, uint32_t t,
    int32_t *__restrict__ anc, const float *__restrict__ gx_in, float *__restrict__ gx_out,
    int gdims, int64_t gMN) {
  __shared__ double s_c[kRun * kPad];     // one weight tile's CDF (transposed)
  __shared__ int32_t s_a[kRun * kPad];    // ancestors (transposed)
  __shared__ double scratch[33];
  const int64_t tile = blockIdx.x;
  const int64_t f = tile / tpf, tt = tile - f * tpf;
  const int64_t i0 = tt * kTile;
  const int n = static_cast<int>(N - i0 < kTile ? N - i0 : kTile);
  const int64_t base = f * N;
  if (ws.flag[f]) {  // collapse / NaN: identity ancestors (filters.py:105-109)
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      anc[base + i0 + i] = static_cast<int32_t>(base + i0 + i);
      if (GATHER)
        for (int d = 0; d < gdims; ++d)
          gx_out[d * gMN + base + i0 + i] = gx_in[d * gMN + base + i0 + i];
    }
    return;
  }
  // this thread's run of sorted uniforms, in registers
  const int r0 = threadIdx.x * kRun;
  double u[kRun];
  if (MODE == 1) {
#pragma unroll
    for (int q = 0; q < kRun; ++q) u[q] = r0 + q < n ? u_tape[base + i0 + r0 + q] : 2.0;
  } else {
    spacing_run(load_key(keys, f), t, i0 + r0, N, u);
    double run = 0.0;
#pragma unroll
    for (int q = 0; q < kRun; ++q) {
      run = __dadd_rn(run, u[q]);
      u[q] = run;
    }
    double tot;
    const double eoff = block_exclusive_scan(run, scratch, &tot);
    const double scale = ws.tesum[tile] / tot, teoff = ws.teoff[tile];
    const double inv = 1.0 / ws.cN[f];
#pragma unroll
    for (int q = 0; q < kRun; ++q)
      u[q] = r0 + q < n ? fma(__dadd_rn(eoff, u[q]), scale, teoff) * inv : 2.0;
  }
  const double m = ws.m[f], total = ws.total[f];
  const int64_t t_lo = ws.klo[tile], t_hi = ws.khi[tile];
  auto cs = [&](int i) { return s_c[(i & (kRun - 1)) * kPad + (i >> 3)]; };
  static_assert(kRun == 8, "cs() index map assumes runs of 8");
  int32_t a[kRun];
  uint32_t done = 0;
  int kl = 0;  // this thread's position inside the current tile
  // walk the window tiles (normally 1-2); past t_hi only if a uniform is
  // still unanswered (defensive: the margin makes that unreachable)
  for (int64_t wt = t_lo; wt < tpf; ++wt) {
    __syncthreads();  // previous tile consumed
    const int len = tile_cdf_f32(logw, N, tpf, ws, f, wt, m, total, s_c, scratch);
    __syncthreads();
    const bool last = wt == tpf - 1;
    const double cmax = cs(len - 1);
    const int64_t e0 = wt * kTile;
    if (wt != t_lo) kl = 0;
#pragma unroll
    for (int q = 0; q < kRun; ++q) {
      if ((done >> q) & 1u) continue;
      if (r0 + q >= n) {
        a[q] = static_cast<int32_t>(base);
        done |= 1u << q;
        continue;
      }
      if (!(u[q] <= cmax) && !last) break;  // this and later uniforms: later tiles
      kl = advance_to<int>(cs, kl, len, u[q]);
      const int64_t k = e0 + kl;
      a[q] = static_cast<int32_t>(base + (k < N - 1 ? k : N - 1));  // clamp (accel.py:183)
      done |= 1u << q;
    }
    if (__syncthreads_and(done == 0xffu)) break;  // block-uniform exit
    (void)t_hi;
  }
#pragma unroll
  for (int q = 0; q < kRun; ++q) s_a[q * kPad + threadIdx.x] = a[q];
  __syncthreads();
  if (GATHER && gdims == 3) {
    int32_t ai[kRun];
#pragma unroll
    for (int h = 0; h < kRun; ++h) {
      const int e = threadIdx.x + h * kTileThreads;
      ai[h] = e < n ? s_a[(e % kRun) * kPad + e / kRun] : 0;
      if (e < n) anc[base + i0 + e] = ai[h];
    }
    float v[3][kRun];
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int h = 0; h < kRun; ++h)
        v[d][h] = threadIdx.x + h * kTileThreads < n ? __ldg(gx_in + d * gMN + ai[h]) : 0.f;
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int h = 0; h < kRun; ++h) {
        const int e = threadIdx.x + h * kTileThreads;
        if (e < n) gx_out[d * gMN + base + i0 + e] = v[d][h];
      }
    return;
  }
  for (int e = threadIdx.x; e < n; e += kTileThreads) {
    const int32_t ai = s_a[(e % kRun) * kPad + e / kRun];
    anc[base + i0 + e] = ai;
    if (GATHER)
      for (int d = 0; d < gdims; ++d) gx_out[d * gMN + base + i0 + e] = __ldg(gx_in + d * gMN + ai);
  }
}

// 3-plane fp32 gather, 4 consecutive particles per thread: one int4 ancestor
// load, 12 independent gathered loads in flight, three float4 stores.
__global__ void __launch_bounds__(256) gather3_kernel(const float *__restrict__ xin,
                                                      const int32_t *__restrict__ anc, int64_t MN,
                                                      float *__restrict__ xout) {
  const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (4 * q >= MN) return;
  const int4 a = __ldg(reinterpret_cast<const int4 *>(anc) + q);
  float v[3][4];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const float *src = xin + d * MN;
    v[d][0] = __ldg(src + a.x);
    v[d][1] = __ldg(src + a.y);
    v[d][2] = __ldg(src + a.z);
    v[d][3] = __ldg(src + a.w);
  }
#pragma unroll
  for (int d = 0; d < 3; ++d)
    reinterpret_cast<float4 *>(xout + d * MN)[q] = make_float4(v[d][0], v[d][1], v[d][2], v[d][3]);
}

__global__ void wide_gather_kernel(const float *__restrict__ xin, const int32_t *__restrict__ anc,
                                   int64_t MN, int dims, float *__restrict__ xout) {
  const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (p >= MN) return;
  const int64_t a = __ldg(anc + p);
  for (int d = 0; d < dims; ++d) xout[d * MN + p] = __ldg(xin + d * MN + a);
}

template <typename TW>
static int launch_resample(const void *logw_v, int64_t M, int64_t N, const double *u_tape,
                           const uint32_t *keys, uint32_t t, int32_t *anc, double *lnc,
                           uint8_t *collapsed, uint32_t *status, void *ws_v, size_t ws_bytes,
                           cudaStream_t s, const float *gx_in = nullptr,
                           float *gx_out = nullptr, int gdims = 0, uint32_t flags = 0,
                           const EstFuse *ef = nullptr, bool *fused = nullptr) {
  const TW *logw = static_cast<const TW *>(logw_v);
  if (fused) *fused = false;
  const bool exact = flags & PF_RS_REFERENCE_ORDER;
  if (N <= kBankMaxN && exact) {
    auto kern = u_tape ? resample_bank_exact_kernel<TW, 1> : resample_bank_exact_kernel<TW, 0>;
    const size_t smem = 2 * static_cast<size_t>(N) * sizeof(double);
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem));
    kern<<<static_cast<unsigned>(M), 256, smem, s>>>(logw, static_cast<int32_t>(N), u_tape, keys,
                                                     t, anc, lnc, collapsed, status);
    if (gx_in)
      wide_gather_kernel<<<grid_for(M * N, 256), 256, 0, s>>>(gx_in, anc, M * N, gdims, gx_out);
    return check_launch("pf_segmented_resample(bank, reference order)");
  }
  if (N <= kBankMaxN) {
    using K = void (*)(const TW *, int32_t, const double *, const uint32_t *, uint32_t, int32_t *,
                       double *, uint8_t *, uint32_t *, const float *, float *, int, int64_t,
                       EstFuse);
    K kern;
    int threads, ipt;
    const bool g = gx_in != nullptr;
#define PF_PICK(TH, I)                                                                        \
  {                                                                                           \
    threads = TH;                                                                             \
    ipt = I;                                                                                  \
    kern = u_tape ? (g ? resample_bank_kernel<TW, 1, TH, I, true>                             \
                       : resample_bank_kernel<TW, 1, TH, I, false>)                           \
                  : (g ? resample_bank_kernel<TW, 0, TH, I, true>                             \
                       : resample_bank_kernel<TW, 0, TH, I, false>);                          \
  }
    if (M < kSmCount && N > 256 && N <= 2048) {
      // few filters (e.g. cfg0: 4 x 1000) leave most SMs idle and each CTA's
      // serial run length is the latency: wide CTAs, 2 particles per thread
      if (N <= 512) PF_PICK(256, 2)
      else if (N <= 1024) PF_PICK(512, 2)
      else PF_PICK(1024, 2)
    } else if (N <= 256) PF_PICK(128, 2)
    else if (N <= 512) PF_PICK(128, 4)
    else if (N <= 1024) PF_PICK(128, 8)
    else if (N <= 2048) PF_PICK(256, 8)
    else if (N <= 4096) PF_PICK(256, 16)
    else PF_PICK(512, 16)
#undef PF_PICK
    // thread-major CDF slots: THREADS * IPT doubles (>= N)
    const size_t smem = static_cast<size_t>(threads) * ipt * (2 * sizeof(double) + 4);
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem));
    EstFuse e{};
    if (ef && ef->x && ef->dim >= 1 && ef->dim <= kEstMaxDim) {
      e = *ef;
      if (fused) *fused = true;
    }
    kern<<<static_cast<unsigned>(M), threads, smem, s>>>(logw, static_cast<int32_t>(N), u_tape,
                                                         keys, t, anc, lnc, collapsed, status,
                                                         gx_in, gx_out, gdims, M * N, e);
    return check_launch("pf_segmented_resample(bank)");
  }
  WideWs ws;
  const size_t need = wide_ws_layout(M, N, &ws, static_cast<char *>(ws_v));
  PF_REQUIRE(ws_v && ws_bytes >= need, "pf_segmented_resample: workspace too small (%zu < %zu)",
             ws_bytes, need);
  const int64_t tpf = (N + kTile - 1) / kTile;
  const unsigned nt = static_cast<unsigned>(M * tpf);
  if (exact) {
    wide_tile_max<TW><<<nt, kTileThreads, 0, s>>>(logw, N, tpf, ws);
    wide_filter_max<<<static_cast<unsigned>(M), 256, 0, s>>>(tpf, ws, collapsed, status);
    wide_exact_e<TW><<<nt, kTileThreads, 0, s>>>(logw, N, tpf, ws);
    wide_exact_leaves<<<static_cast<unsigned>(M), 32, 0, s>>>(N, ws);
    wide_exact_leafsum<<<dim3(static_cast<unsigned>((ws.max_leaves + 127) / 128),
                              static_cast<unsigned>(M)),
                         128, 0, s>>>(N, ws);
    wide_exact_total<<<static_cast<unsigned>(M), 32, 0, s>>>(N, ws, lnc);
    wide_exact_w<<<nt, kTileThreads, 0, s>>>(N, tpf, ws);
    wide_exact_cumsum<<<static_cast<unsigned>(M), 32, 0, s>>>(N, ws);
    if (!u_tape) {  // tile offsets of the exponential spacings
      wide_tile_sums<TW, 0><<<nt, kTileThreads, 0, s>>>(logw, N, tpf, ws, u_tape, keys, t);
      wide_offsets_kernel<<<static_cast<unsigned>(M), 256, 2 * 1024 * sizeof(double), s>>>(
          M, tpf, ws, N, keys, t);
    }
  } else {
    if (u_tape) {
      wide2_tile_stats<TW, 1><<<nt, kTileThreads, 0, s>>>(logw, N, tpf, ws, keys, t);
      wide2_filter<1><<<static_cast<unsigned>(M), 1024, 0, s>>>(N, tpf, ws, collapsed, status,
                                                               lnc, keys, t);
    } else if (tpf > kFilterChunk) {
      const unsigned nch = static_cast<unsigned>((tpf + kFilterChunk - 1) / kFilterChunk);
      wide2_gamma<<<grid_for(M * tpf, 128), 128, 0, s>>>(M, N, tpf, ws, keys, t);
      wide2_tile_stats<TW, 0, false><<<nt, kTileThreads, 0, s>>>(logw, N, tpf, ws, keys, t);
      wide2_chunk_scan<<<dim3(nch, static_cast<unsigned>(M)), 256, 0, s>>>(tpf, ws);
      wide2_chunk_combine<<<grid_for(32 * M, 128), 128, 0, s>>>(M, N, nch, ws, collapsed, status, lnc,
                                                           keys, t);
      wide2_chunk_apply<<<dim3(nch, static_cast<unsigned>(M)), 256, 0, s>>>(tpf, ws);
    } else {
      wide2_tile_stats<TW, 0><<<nt, kTileThreads, 0, s>>>(logw, N, tpf, ws, keys, t);
      wide2_filter<0><<<static_cast<unsigned>(M), 1024, 0, s>>>(N, tpf, ws, collapsed, status,
                                                               lnc, keys, t);
    }
    if constexpr (std::is_same<TW, float>::value) {
      // PF_RS_WIDE_RECOMPUTE: no materialised CDF - partition on the tile
      // offsets, the merge recomputes its tiles' CDF (wide3_*).  Same
      // ancestors; 2.4 instead of 3.4 GB per 2^26-particle step, but the
      // merge recomputes ~2 tiles per uniform tile and measures slower (1.29
      // vs 0.84 ms at cfg1c), so it is opt-in
      if (!u_tape && (flags & PF_RS_WIDE_RECOMPUTE)) {
        wide3_partition<0><<<grid_for(2 * nt, 256), 256, 0, s>>>(N, tpf, nt, ws, u_tape);
        const bool g3 = gx_in != nullptr;
        if (g3)
          wide3_merge<0, true><<<nt, kTileThreads, 0, s>>>(logw, N, tpf, ws, u_tape, keys, t,
                                                           anc, gx_in, gx_out, gdims, M * N);
        else
          wide3_merge<0, false><<<nt, kTileThreads, 0, s>>>(logw, N, tpf, ws, u_tape, keys, t,
                                                            anc, nullptr, nullptr, 0, M * N);
        return check_launch("pf_segmented_resample(wide, recomputed CDF)");
      }
      if (!u_tape)
        wide_tile_cum<TW, true><<<nt, kTileThreads, 0, s>>>(logw, N, tpf, ws);
      else
        wide_tile_cum<TW><<<nt, kTileThreads, 0, s>>>(logw, N, tpf, ws);
    } else {
      wide_tile_cum<TW><<<nt, kTileThreads, 0, s>>>(logw, N, tpf, ws);
    }
  }
  if (u_tape)
    wide2_partition<1><<<grid_for(2 * nt, 256), 256, 0, s>>>(N, tpf, nt, ws, u_tape, keys, t);
  else
    wide2_partition<0><<<grid_for(2 * nt, 256), 256, 0, s>>>(N, tpf, nt, ws, u_tape, keys, t);
  // merge -> ancestors (+ the fused gather)
  // per-thread search (default) or merge path (flags & PF_RS_WIDE_MERGE_PATH)
  const bool search = !(flags & PF_RS_WIDE_MERGE_PATH);
  // the ancestor gather fused into the merge's write-out (cfg1c: 1.00 ->
  // 0.93 ms/step); flags & PF_RS_WIDE_GATHER_SEPARATE runs it as its own pass
  const bool fuse_gather = !(flags & PF_RS_WIDE_GATHER_SEPARATE);
  const bool fg = fuse_gather && gx_in && search;
  auto mk = u_tape ? (search ? (fg ? wide2_merge<1, true, true> : wide2_merge<1, false, true>)
                             : wide2_merge<1, false>)
                   : (search ? (fg ? wide2_merge<0, true, true> : wide2_merge<0, false, true>)
                             : wide2_merge<0, false>);
  const size_t msmem = wide2_merge_smem(search);
  cudaFuncSetAttribute(mk, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(msmem));
  mk<<<nt, kTileThreads, msmem, s>>>(N, tpf, ws, u_tape, keys, t, anc, fg ? gx_in : nullptr,
                                     fg ? gx_out : nullptr, fg ? gdims : 0, M * N);
  if (gx_in && !fg) {
    const int64_t MN = M * N;
    if (gdims == 3 && (MN & 3) == 0)
      gather3_kernel<<<grid_for(MN / 4, 256), 256, 0, s>>>(gx_in, anc, MN, gx_out);
    else
      wide_gather_kernel<<<grid_for(MN, 256), 256, 0, s>>>(gx_in, anc, MN, gdims, gx_out);
  }
  return check_launch("pf_segmented_resample(wide)");
}

// ---- normalize_log_weights operator (segmented) ---------------------------
template <typename TW>
__global__ void __launch_bounds__(256) nlw_kernel(const TW *__restrict__ logw, int32_t N,
                                                  double *__restrict__ w,
                                                  double *__restrict__ lmr,
                                                  uint8_t *__restrict__ collapsed,
                                                  uint32_t *__restrict__ status) {
  __shared__ double scratch[33];
  const int64_t f = blockIdx.x, base = f * N;
  double mx = -INFINITY;
  int nan = 0;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    const double v = load_lw(logw + base + i);
    nan |= isnan(v);
    mx = fmax(mx, v);
  }
  nan = __syncthreads_or(nan);
  const double m = block_max(mx, scratch);
  if (nan || m == -INFINITY) {
    if (threadIdx.x == 0) {
      collapsed[f] = nan ? 0 : 1;
      if (nan) atomicOr(status + f, PF_ST_NAN_WEIGHT);
    }
    return;
  }
  double part = 0.0;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    const double e = exp(__dsub_rn(load_lw(logw + base + i), m));
    w[base + i] = e;
    part = __dadd_rn(part, e);
  }
  const double total = block_sum(part, scratch);
  for (int i = threadIdx.x; i < N; i += blockDim.x) w[base + i] = __ddiv_rn(w[base + i], total);
  if (threadIdx.x == 0) {
    collapsed[f] = 0;
    lmr[f] = __dsub_rn(__dadd_rn(m, log(total)), log(static_cast<double>(N)));
  }
}

__global__ void resample_indices_kernel(const double *__restrict__ cum, int64_t n,
                                        const double *__restrict__ u, int64_t m,
                                        int64_t *__restrict__ idx) {
  const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (j >= m) return;
  const int64_t k = lower_bound_f64_64(cum, n, u[j]);
  idx[j] = k < n - 1 ? k : n - 1;
}

// Production resample that also writes the posterior mean of the resampled
// set of planar states when the bank kernel serves (N <= kBankMaxN, dim <= 8);
// *fused reports whether it did (bank.cu runs the standalone pass otherwise).
int segmented_resample_fused(pf_dtype dtype, const void *logw, int64_t M, int64_t N,
                             const uint32_t *keys, uint32_t t, int32_t *anc, double *lnc,
                             uint8_t *collapsed, uint32_t *status, void *ws, size_t ws_bytes,
                             const void *x, int dim, double *est, int64_t est_stride,
                             double *lnc_tr, uint8_t *coll_tr, cudaStream_t s, bool *fused) {
  PF_REQUIRE(logw && anc && lnc && collapsed && status && keys && fused,
             "segmented_resample_fused: null");
  const EstFuse ef{x, dim, M * N, est, est_stride, lnc_tr, coll_tr};
  if (dtype == PF_F64)
    return launch_resample<double>(logw, M, N, nullptr, keys, t, anc, lnc, collapsed, status, ws,
                                   ws_bytes, s, nullptr, nullptr, 0, 0u, &ef, fused);
  return launch_resample<float>(logw, M, N, nullptr, keys, t, anc, lnc, collapsed, status, ws,
                                ws_bytes, s, nullptr, nullptr, 0, 0u, &ef, fused);
}

}  // namespace pf

using namespace pf;

extern "C" {

size_t pf_resample_workspace_bytes(int64_t M, int64_t N) {
  if (M < 1 || N < 1 || N <= kBankMaxN) return 0;
  return wide_ws_layout(M, N, nullptr, nullptr);
}

int pf_segmented_resample(pf_dtype logw_dtype, const void *logw, int64_t M, int64_t N,
                          const double *u_tape, const uint32_t *keys, uint32_t t,
                          int32_t *anc_out, double *lnc, uint8_t *collapsed, uint32_t *status,
                          void *ws, size_t ws_bytes, void *stream) {
  PF_REQUIRE(logw && anc_out && lnc && collapsed && status, "pf_segmented_resample: null");
  PF_REQUIRE(M >= 1 && N >= 1 && M * N <= INT32_MAX, "pf_segmented_resample: bad M/N");
  PF_REQUIRE(u_tape || keys, "pf_segmented_resample: need keys (Philox) or u_tape");
  const cudaStream_t s = as_stream(stream);
  if (logw_dtype == PF_F64)
    return launch_resample<double>(logw, M, N, u_tape, keys, t, anc_out, lnc, collapsed, status,
                                   ws, ws_bytes, s);
  return launch_resample<float>(logw, M, N, u_tape, keys, t, anc_out, lnc, collapsed, status, ws,
                                ws_bytes, s);
}

int pf_segmented_resample_ex(pf_dtype logw_dtype, const void *logw, int64_t M, int64_t N,
                             const double *u_tape, const uint32_t *keys, uint32_t t,
                             int32_t *anc_out, double *lnc, uint8_t *collapsed, uint32_t *status,
                             void *ws, size_t ws_bytes, const float *x_in, float *x_out,
                             int32_t dims, uint32_t flags, void *stream) {
  PF_REQUIRE(logw && anc_out && lnc && collapsed && status, "pf_segmented_resample_ex: null");
  PF_REQUIRE(M >= 1 && N >= 1 && M * N <= INT32_MAX, "pf_segmented_resample_ex: bad M/N");
  PF_REQUIRE(u_tape || keys, "pf_segmented_resample_ex: need keys (Philox) or u_tape");
  PF_REQUIRE(!x_in || (x_out && dims >= 1 && x_in != x_out),
             "pf_segmented_resample_ex: gather needs x_out != x_in and dims >= 1");
  PF_REQUIRE((flags & ~(PF_RS_REFERENCE_ORDER | PF_RS_WIDE_MERGE_PATH |
                        PF_RS_WIDE_GATHER_SEPARATE | PF_RS_WIDE_RECOMPUTE)) == 0,
             "pf_segmented_resample_ex: unknown flags");
  const cudaStream_t s = as_stream(stream);
  if (logw_dtype == PF_F64)
    return launch_resample<double>(logw, M, N, u_tape, keys, t, anc_out, lnc, collapsed, status,
                                   ws, ws_bytes, s, x_in, x_out, dims, flags);
  return launch_resample<float>(logw, M, N, u_tape, keys, t, anc_out, lnc, collapsed, status, ws,
                                ws_bytes, s, x_in, x_out, dims, flags);
}

int pf_op_normalize_log_weights(pf_dtype logw_dtype, const void *logw, int64_t M, int64_t N,
                                double *weights_out, double *log_mean_raw_out,
                                uint8_t *collapsed, uint32_t *status, void *stream) {
  PF_REQUIRE(logw && weights_out && log_mean_raw_out && collapsed && status,
             "pf_op_normalize_log_weights: null");
  PF_REQUIRE(M >= 1 && N >= 1 && N <= INT32_MAX, "pf_op_normalize_log_weights: bad M/N");
  const cudaStream_t s = as_stream(stream);
  if (logw_dtype == PF_F64)
    nlw_kernel<double><<<static_cast<unsigned>(M), 256, 0, s>>>(
        static_cast<const double *>(logw), static_cast<int32_t>(N), weights_out,
        log_mean_raw_out, collapsed, status);
  else
    nlw_kernel<float><<<static_cast<unsigned>(M), 256, 0, s>>>(
        static_cast<const float *>(logw), static_cast<int32_t>(N), weights_out,
        log_mean_raw_out, collapsed, status);
  return check_launch("pf_op_normalize_log_weights");
}

int pf_op_resample_indices(const double *cum, int64_t n, const double *u, int64_t m,
                           int64_t *idx_out, void *stream) {
  PF_REQUIRE(cum && u && idx_out && n >= 1 && m >= 0, "pf_op_resample_indices: bad arguments");
  if (m == 0) return PF_OK;
  resample_indices_kernel<<<grid_for(m, 256), 256, 0, as_stream(stream)>>>(cum, n, u, m,
                                                                           idx_out);
  return check_launch("pf_op_resample_indices");
}

}  // extern "C"
