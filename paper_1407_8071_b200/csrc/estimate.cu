// Per-filter posterior mean of the resampled particle set.
//
// Reference: run_filter records posterior_mean(state) after every step
// (filters.py:188) = weights @ particles (core.py:154-156) with uniform
// weights 1/N over the resampled set propagated[idx] (filters.py:111), i.e.
// (1/N) * sum_j x[anc[j]].  On a collapsed step anc is the identity
// (filters.py:107-109).  Accumulation is fp64 in a fixed order, so the
// estimate is bit-reproducible and independent of the launch geometry.
#include "block_ops.cuh"
#include "common.cuh"

namespace pf {

constexpr int kSmallDim = 8;

template <typename T>
__global__ void __launch_bounds__(256) estimate_small_kernel(
    const T *__restrict__ x, int64_t sp, int64_t sd, int dim, const int32_t *__restrict__ anc,
    int32_t N, double invN, double *__restrict__ est, int64_t est_stride) {
  __shared__ double scratch[33];
  const int64_t f = blockIdx.x;
  double acc[kSmallDim];
#pragma unroll
  for (int d = 0; d < kSmallDim; ++d) acc[d] = 0.0;
  for (int j = threadIdx.x; j < N; j += blockDim.x) {
    const int64_t p = __ldg(anc + f * N + j);
#pragma unroll
    for (int d = 0; d < kSmallDim; ++d)
      if (d < dim) acc[d] = __dadd_rn(acc[d], static_cast<double>(x[p * sp + d * sd]));
  }
  for (int d = 0; d < dim; ++d) {
    const double s = block_sum(acc[d], scratch);
    if (threadIdx.x == 0) est[f * est_stride + d] = __dmul_rn(s, invN);
  }
}

// 32 dims per block (lanes), 8 warps split the particles; warp partials are
// combined in warp order.
template <typename T>
__global__ void __launch_bounds__(256) estimate_wide_kernel(
    const T *__restrict__ x, int64_t sp, int64_t sd, int dim, const int32_t *__restrict__ anc,
    int32_t N, double invN, double *__restrict__ est, int64_t est_stride) {
  __shared__ double part[8][32];
  const int64_t f = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int d = blockIdx.y * 32 + lane;
  double acc = 0.0;
  if (d < dim) {
    const int32_t *a = anc + f * N;
    int j = warp;
    for (; j + 24 < N; j += 32) {  // 4 independent loads in flight
      const int64_t p0 = __ldg(a + j), p1 = __ldg(a + j + 8), p2 = __ldg(a + j + 16),
                    p3 = __ldg(a + j + 24);
      const double v0 = x[p0 * sp + d * sd], v1 = x[p1 * sp + d * sd];
      const double v2 = x[p2 * sp + d * sd], v3 = x[p3 * sp + d * sd];
      acc = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(acc, v0), v1), v2), v3);
    }
    for (; j < N; j += 8) acc = __dadd_rn(acc, static_cast<double>(x[__ldg(a + j) * sp + d * sd]));
  }
  part[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && d < dim) {
    double s = part[0][lane];
    for (int w = 1; w < 8; ++w) s = __dadd_rn(s, part[w][lane]);
    est[f * est_stride + d] = __dmul_rn(s, invN);
  }
}

}  // namespace pf

using namespace pf;

extern "C" {

int pf_filter_estimate_strided(pf_dtype dtype, const void *x, int64_t stride_p, int64_t stride_d,
                               int32_t dim, const int32_t *anc, int64_t M, int64_t N,
                               double *est_out, int64_t est_stride, void *stream) {
  PF_REQUIRE(x && anc && est_out && dim >= 1 && M >= 1 && N >= 1 && M * N <= INT32_MAX &&
                 est_stride >= dim,
             "pf_filter_estimate: bad arguments");
  const cudaStream_t s = as_stream(stream);
  const double invN = 1.0 / static_cast<double>(N);  // uniform_weights value, core.py:112-113
  const int32_t n32 = static_cast<int32_t>(N);
  if (dim <= kSmallDim) {
    if (dtype == PF_F64)
      estimate_small_kernel<double><<<static_cast<unsigned>(M), 256, 0, s>>>(
          static_cast<const double *>(x), stride_p, stride_d, dim, anc, n32, invN, est_out, est_stride);
    else
      estimate_small_kernel<float><<<static_cast<unsigned>(M), 256, 0, s>>>(
          static_cast<const float *>(x), stride_p, stride_d, dim, anc, n32, invN, est_out, est_stride);
  } else {
    const dim3 grid(static_cast<unsigned>(M), static_cast<unsigned>((dim + 31) / 32));
    if (dtype == PF_F64)
      estimate_wide_kernel<double><<<grid, 256, 0, s>>>(static_cast<const double *>(x), stride_p,
                                                        stride_d, dim, anc, n32, invN, est_out, est_stride);
    else
      estimate_wide_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float *>(x), stride_p,
                                                       stride_d, dim, anc, n32, invN, est_out, est_stride);
  }
  return check_launch("pf_filter_estimate");
}

int pf_filter_estimate(pf_dtype dtype, const void *x, int64_t stride_p, int64_t stride_d,
                       int32_t dim, const int32_t *anc, int64_t M, int64_t N, double *est_out,
                       void *stream) {
  return pf_filter_estimate_strided(dtype, x, stride_p, stride_d, dim, anc, M, N, est_out, dim,
                                    stream);
}

}  // extern "C"
