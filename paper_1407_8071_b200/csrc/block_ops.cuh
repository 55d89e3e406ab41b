// Block-level deterministic reductions and scans (fp64) in shared memory.
// Fixed association order for a given (n, blockDim): results are
// bit-reproducible run to run and independent of scheduling.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace pf {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ int warp_or(int v) { return __any_sync(0xffffffffu, v); }

// Block reduce (sum) of one value per thread; result broadcast to all.
// `scratch` >= 33 doubles of shared memory.
__device__ __forceinline__ double block_sum(double v, double *scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  // every warp reduces the warp partials (same order as a single warp would):
  // no divergent shuffle section, no second barrier
  double x = lane < nw ? scratch[lane] : 0.0;
  x = warp_sum(x);
  const double r = __shfl_sync(0xffffffffu, x, 0);
  __syncthreads();  // scratch reusable
  return r;
}

__device__ __forceinline__ double block_max(double v, double *scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_max(v);
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  double x = lane < nw ? scratch[lane] : -INFINITY;
  x = warp_max(x);
  const double r = __shfl_sync(0xffffffffu, x, 0);
  __syncthreads();
  return r;
}

// fp32 block max (scratch >= 32 floats); every warp reduces the partials
__device__ __forceinline__ float block_max_f(float v, float *scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  float x = lane < nw ? scratch[lane] : -INFINITY;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
  __syncthreads();
  return x;
}

__device__ __forceinline__ int block_or(int v, double *scratch) {
  return __syncthreads_or(v);
}

// In-place inclusive scan of s[0..n) (shared memory) in rounds of blockDim
// elements, starting from `carry`.  Returns carry + sum(s).  `scratch` >= 33
// doubles.  Every thread must call it.
__device__ __forceinline__ double block_scan_inplace(double *s, int n, double carry,
                                                     double *scratch) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  for (int b0 = 0; b0 < n; b0 += blockDim.x) {
    const int i = b0 + tid;
    double v = i < n ? s[i] : 0.0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v = __dadd_rn(v, u);
    }
    if (lane == 31) scratch[warp] = v;
    __syncthreads();
    double x = lane < nw ? scratch[lane] : 0.0;  // every warp scans the warp totals
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double u = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x = __dadd_rn(x, u);
    }
    const double wprev = __shfl_sync(0xffffffffu, x, warp > 0 ? warp - 1 : 0);
    const double wtot = __shfl_sync(0xffffffffu, x, nw - 1);
    const double off = warp > 0 ? __dadd_rn(carry, wprev) : carry;
    if (i < n) s[i] = __dadd_rn(off, v);
    carry = __dadd_rn(carry, wtot);
    __syncthreads();
  }
  return carry;
}

// Smallest k in [0, n) with a[k] >= x (n if none): np.searchsorted 'left'.
__device__ __forceinline__ int lower_bound_f64(const double *a, int n, double x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

__device__ __forceinline__ int64_t lower_bound_f64_64(const double *a, int64_t n, double x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(a + mid) < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

}  // namespace pf
