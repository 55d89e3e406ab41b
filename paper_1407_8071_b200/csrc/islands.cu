// Island-level kernels of the double bootstrap (filters.py:201-313): the
// islands are the bank's filters, so only the island bookkeeping is new.
//
//  * pf_island_accumulate - log_weights[m] += lnc_new[m] - lnc_old[m]
//                           (dbf_step, filters.py:253-256)
//  * pf_island_copy       - whole-island resampling by island indices: the
//                           ancestors, lnc and collapse flag of island idx[m]
//                           become island m's (filters.py:258-263).  States are
//                           never copied: the next propagate gathers them
//                           through the composed ancestors.
//  * pf_island_pool       - pooled_estimate (filters.py:229-234): normalised
//                           island weights (numpy order) times the islands'
//                           posterior means, summed over islands in order
//  * pf_island_trace      - log of the island average of exp(lnc)
//                           (filters.py:301-303)
#include "common.cuh"
#include "npsum.cuh"

#include <algorithm>

namespace pf {

__global__ void island_accumulate_kernel(double *__restrict__ lw, const double *__restrict__ lnc,
                                         const double *__restrict__ lnc_old, int64_t M) {
  const int64_t m = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (m < M) lw[m] = __dadd_rn(lw[m], __dsub_rn(lnc[m], lnc_old[m]));
}

// idx[m] are row indices of a 1-segment resample over the M islands.
__global__ void island_copy_kernel(const int32_t *__restrict__ idx,
                                   const int32_t *__restrict__ anc_in, int32_t *__restrict__ anc_out,
                                   int64_t M, int32_t N) {
  const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (q >= M * N) return;
  const int64_t m = q / N;
  const int64_t j = q - m * N;
  anc_out[q] = anc_in[static_cast<int64_t>(idx[m]) * N + j];
}

__global__ void island_scalars_kernel(const int32_t *__restrict__ idx,
                                      const double *__restrict__ lnc_in,
                                      double *__restrict__ lnc_out,
                                      const uint8_t *__restrict__ coll_in,
                                      uint8_t *__restrict__ coll_out, double *__restrict__ lw,
                                      int64_t M) {
  const int64_t m = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (m >= M) return;
  lnc_out[m] = lnc_in[idx[m]];
  coll_out[m] = coll_in[idx[m]];
  lw[m] = 0.0;
}

// probs = exp(lw - max) / sum (numpy pairwise sum), then per dimension
// est = probs[0]*e_0; est = est + probs[m]*e_m.  Every block recomputes the
// probabilities into shared memory (M <= kMaxIslands).
constexpr int kMaxIslands = 4096;

__global__ void __launch_bounds__(256) island_pool_kernel(const double *__restrict__ est,
                                                          int64_t est_stride, int64_t M,
                                                          int64_t dim,
                                                          const double *__restrict__ lw,
                                                          double *__restrict__ out) {
  __shared__ double s_p[kMaxIslands];
  __shared__ double s_max, s_total;
  if (threadIdx.x == 0) {
    double mx = lw[0];
    for (int64_t m = 1; m < M; ++m) mx = fmax(mx, lw[m]);
    s_max = mx;
  }
  __syncthreads();
  for (int64_t m = threadIdx.x; m < M; m += blockDim.x) s_p[m] = exp(__dsub_rn(lw[m], s_max));
  __syncthreads();
  if (threadIdx.x < 32) {
    const double tot = np_pairwise_warp(s_p, static_cast<int>(M), threadIdx.x);
    if (threadIdx.x == 0) s_total = tot;
  }
  __syncthreads();
  for (int64_t m = threadIdx.x; m < M; m += blockDim.x) s_p[m] = __ddiv_rn(s_p[m], s_total);
  __syncthreads();
  const int64_t d = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (d >= dim) return;
  double acc = __dmul_rn(s_p[0], est[d]);
  for (int64_t m = 1; m < M; ++m) acc = __dadd_rn(acc, __dmul_rn(s_p[m], est[m * est_stride + d]));
  out[d] = acc;
}

// m + log(sum(exp(lnc - m))) - log(M)
__global__ void island_trace_kernel(const double *__restrict__ lnc, int64_t M,
                                    double *__restrict__ out) {
  __shared__ double s_e[kMaxIslands];
  __shared__ double s_max;
  if (threadIdx.x == 0) {
    double mx = lnc[0];
    for (int64_t m = 1; m < M; ++m) mx = fmax(mx, lnc[m]);
    s_max = mx;
  }
  __syncthreads();
  for (int64_t m = threadIdx.x; m < M; m += blockDim.x) s_e[m] = exp(__dsub_rn(lnc[m], s_max));
  __syncthreads();
  if (threadIdx.x < 32) {
    const double tot = np_pairwise_warp(s_e, static_cast<int>(M), threadIdx.x);
    if (threadIdx.x == 0)
      out[0] = __dsub_rn(__dadd_rn(s_max, log(tot)), log(static_cast<double>(M)));
  }
}

}  // namespace pf

using namespace pf;

extern "C" {

int pf_island_accumulate(double *log_weights, const double *lnc, const double *lnc_old,
                         int64_t M, void *stream) {
  PF_REQUIRE(log_weights && lnc && lnc_old && M >= 1, "pf_island_accumulate: bad arguments");
  island_accumulate_kernel<<<grid_for(M, 256), 256, 0, as_stream(stream)>>>(log_weights, lnc,
                                                                            lnc_old, M);
  return check_launch("pf_island_accumulate");
}

int pf_island_copy(const int32_t *idx, int32_t *anc, double *lnc, uint8_t *collapsed,
                   double *log_weights, int64_t M, int64_t N, int32_t *anc_tmp,
                   double *lnc_tmp, uint8_t *coll_tmp, void *stream) {
  PF_REQUIRE(idx && anc && lnc && collapsed && log_weights && anc_tmp && lnc_tmp && coll_tmp &&
                 M >= 1 && N >= 1 && M * N <= INT32_MAX,
             "pf_island_copy: bad arguments");
  const cudaStream_t s = as_stream(stream);
  island_copy_kernel<<<grid_for(M * N, 256), 256, 0, s>>>(idx, anc, anc_tmp, M,
                                                          static_cast<int32_t>(N));
  island_scalars_kernel<<<grid_for(M, 256), 256, 0, s>>>(idx, lnc, lnc_tmp, collapsed, coll_tmp,
                                                         log_weights, M);
  if (cudaMemcpyAsync(anc, anc_tmp, M * N * sizeof(int32_t), cudaMemcpyDeviceToDevice, s) !=
          cudaSuccess ||
      cudaMemcpyAsync(lnc, lnc_tmp, M * sizeof(double), cudaMemcpyDeviceToDevice, s) !=
          cudaSuccess ||
      cudaMemcpyAsync(collapsed, coll_tmp, M, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return check_launch("pf_island_copy(copy back)");
  return check_launch("pf_island_copy");
}

int pf_island_pool(const double *est, int64_t est_stride, int64_t M, int64_t dim,
                   const double *log_weights, double *out, void *stream) {
  PF_REQUIRE(est && log_weights && out && M >= 1 && M <= kMaxIslands && dim >= 1 &&
                 est_stride >= dim,
             "pf_island_pool: bad arguments (1 <= M <= %d)", kMaxIslands);
  island_pool_kernel<<<grid_for(dim, 256), 256, 0, as_stream(stream)>>>(est, est_stride, M, dim,
                                                                        log_weights, out);
  return check_launch("pf_island_pool");
}

int pf_island_trace(const double *lnc, int64_t M, double *out, void *stream) {
  PF_REQUIRE(lnc && out && M >= 1 && M <= kMaxIslands, "pf_island_trace: bad arguments");
  island_trace_kernel<<<1, 256, 0, as_stream(stream)>>>(lnc, M, out);
  return check_launch("pf_island_trace");
}

}  // extern "C"
