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

// Wide filters with few dimensions (M=1 x N=2^22 Lorenz: one 256-thread CTA
// per filter would walk 16K gathered particles per thread): each filter is
// split into fixed chunks of kEstChunk particles, one CTA per (chunk, filter)
// sums its chunk (threads strided, warp shuffle tree, warps in order), and a
// second pass adds the chunk partials in chunk order.  The order depends on N
// only, so results stay bit-reproducible and independent of M and the GPU
// count.
constexpr int64_t kEstChunk = 16384;
constexpr int64_t kEstChunkMinN = 65536;  // below: one CTA per filter

template <typename T>
__global__ void __launch_bounds__(256) estimate_chunk_kernel(
    const T *__restrict__ x, int64_t sp, int64_t sd, int dim, const int32_t *__restrict__ anc,
    int32_t N, int32_t nch, double *__restrict__ part) {
  __shared__ double s_w[8][kSmallDim];
  const int64_t f = blockIdx.y;
  const int c = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t j0 = static_cast<int64_t>(c) * kEstChunk;
  const int64_t j1 = j0 + kEstChunk < N ? j0 + kEstChunk : N;
  double acc[kSmallDim];
#pragma unroll
  for (int d = 0; d < kSmallDim; ++d) acc[d] = 0.0;
  const int32_t *a = anc + f * N;
  for (int64_t j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
    const int64_t p = __ldg(a + j);
#pragma unroll
    for (int d = 0; d < kSmallDim; ++d)
      if (d < dim) acc[d] = __dadd_rn(acc[d], static_cast<double>(__ldg(x + p * sp + d * sd)));
  }
#pragma unroll
  for (int d = 0; d < kSmallDim; ++d) {
    double v = acc[d];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, o));
    if (lane == 0) s_w[warp][d] = v;
  }
  __syncthreads();
  if (threadIdx.x < dim) {
    double sum = s_w[0][threadIdx.x];
    for (int w = 1; w < 8; ++w) sum = __dadd_rn(sum, s_w[w][threadIdx.x]);
    part[(f * nch + c) * dim + threadIdx.x] = sum;
  }
}

__global__ void estimate_combine_kernel(const double *__restrict__ part, int64_t M, int32_t nch,
                                        int dim, double invN, double *__restrict__ est,
                                        int64_t est_stride) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= M * dim) return;
  const int64_t f = g / dim;
  const int d = static_cast<int>(g - f * dim);
  double s = 0.0;
  for (int c = 0; c < nch; ++c) s = __dadd_rn(s, part[(f * nch + c) * dim + d]);
  est[f * est_stride + d] = __dmul_rn(s, invN);
}

static int32_t est_chunks(int64_t N, int32_t dim) {
  return (dim <= kSmallDim && N >= kEstChunkMinN)
             ? static_cast<int32_t>((N + kEstChunk - 1) / kEstChunk)
             : 0;
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

size_t pf_estimate_workspace_bytes(int64_t M, int64_t N, int32_t dim) {
  if (M < 1 || N < 1 || dim < 1) return 0;
  return static_cast<size_t>(M) * est_chunks(N, dim) * dim * sizeof(double);
}

int pf_filter_estimate_ws(pf_dtype dtype, const void *x, int64_t stride_p, int64_t stride_d,
                          int32_t dim, const int32_t *anc, int64_t M, int64_t N, double *est_out,
                          int64_t est_stride, void *ws, size_t ws_bytes, void *stream) {
  const int32_t nch = est_chunks(N, dim);
  if (nch == 0)
    return pf_filter_estimate_strided(dtype, x, stride_p, stride_d, dim, anc, M, N, est_out,
                                      est_stride, stream);
  PF_REQUIRE(x && anc && est_out && M >= 1 && M * N <= INT32_MAX && est_stride >= dim,
             "pf_filter_estimate_ws: bad arguments");
  PF_REQUIRE(ws && ws_bytes >= pf_estimate_workspace_bytes(M, N, dim),
             "pf_filter_estimate_ws: workspace too small (%zu < %zu)", ws_bytes,
             pf_estimate_workspace_bytes(M, N, dim));
  const cudaStream_t s = as_stream(stream);
  double *part = static_cast<double *>(ws);
  const dim3 grid(static_cast<unsigned>(nch), static_cast<unsigned>(M));
  const int32_t n32 = static_cast<int32_t>(N);
  if (dtype == PF_F64)
    estimate_chunk_kernel<double><<<grid, 256, 0, s>>>(static_cast<const double *>(x), stride_p,
                                                       stride_d, dim, anc, n32, nch, part);
  else
    estimate_chunk_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float *>(x), stride_p,
                                                      stride_d, dim, anc, n32, nch, part);
  estimate_combine_kernel<<<grid_for(M * dim, 128), 128, 0, s>>>(
      part, M, nch, dim, 1.0 / static_cast<double>(N), est_out, est_stride);
  return check_launch("pf_filter_estimate_ws");
}

int pf_filter_estimate(pf_dtype dtype, const void *x, int64_t stride_p, int64_t stride_d,
                       int32_t dim, const int32_t *anc, int64_t M, int64_t N, double *est_out,
                       void *stream) {
  return pf_filter_estimate_strided(dtype, x, stride_p, stride_d, dim, anc, M, N, est_out, dim,
                                    stream);
}

}  // extern "C"
