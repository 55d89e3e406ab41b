// Auxiliary particle filter glue (filters.py:115-154, apf_step).
//
// One APF interval on the bank reuses every bootstrap kernel:
//   1. noise-free propagate + weight -> first-stage log weights lambda
//      (transition_point_prediction, lorenz63.py:57-60 / fhn.py:194-197)
//   2. pf_apf_first_stage_prepare: a filter whose lambda are all -inf falls
//      back to lambda = 0 (uniform first stage, log_mean_first = 0,
//      filters.py:136-140) and is flagged
//   3. segmented resample on lambda -> first-stage ancestors anc1
//   4. pf_compose_ancestors: state rows of the chosen ancestors
//   5. propagate + weight with noise from those rows
//   6. pf_apf_second_stage_weights: log_w -= lambda[anc1] (filters.py:143)
//   7. segmented resample on log_w -> final ancestors
//   8. pf_apf_finish: a second-stage collapse keeps the lnc from before the
//      step (filters.py:146-148); the step is flagged if either stage
//      collapsed.
#include "block_ops.cuh"
#include "common.cuh"

namespace pf {

template <typename T>
__global__ void apf_prepare_kernel(T *__restrict__ lam, int32_t N, uint8_t *__restrict__ coll1) {
  __shared__ double scratch[33];
  const int64_t f = blockIdx.x, base = f * N;
  double mx = -INFINITY;
  int nan = 0;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    const double x = static_cast<double>(lam[base + i]);
    nan |= isnan(x);
    mx = fmax(mx, x);  // fmax drops NaN: tracked separately
  }
  const double m = block_max(mx, scratch);
  // np.max is NaN as soon as one lambda is (core.py:127-133): then lambda is
  // left untouched so the first-stage resampler flags it (ValueError), even
  // when every other value is -inf
  const bool any_nan = __syncthreads_or(nan) != 0;
  const bool collapse = !any_nan && m == -INFINITY;
  if (collapse)
    for (int i = threadIdx.x; i < N; i += blockDim.x) lam[base + i] = T(0);
  if (threadIdx.x == 0) coll1[f] = collapse ? 1 : 0;
}

__global__ void compose_kernel(const int32_t *__restrict__ outer, const int32_t *__restrict__ inner,
                               int64_t MN, int32_t *__restrict__ out) {
  const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (j >= MN) return;
  const int32_t a = __ldg(outer + j);
  out[j] = inner ? __ldg(inner + a) : a;
}

template <typename T>
__global__ void second_stage_kernel(T *__restrict__ logw, const T *__restrict__ lam,
                                    const int32_t *__restrict__ anc1, int64_t MN) {
  const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (j >= MN) return;
  logw[j] = Ar<T>::sub(logw[j], lam[__ldg(anc1 + j)]);
}

__global__ void apf_finish_kernel(double *__restrict__ lnc, const double *__restrict__ lnc_before,
                                  uint8_t *__restrict__ collapsed,
                                  const uint8_t *__restrict__ coll1, int64_t M) {
  const int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (f >= M) return;
  if (collapsed[f]) lnc[f] = lnc_before[f];
  collapsed[f] = collapsed[f] | coll1[f];
}

}  // namespace pf

using namespace pf;

extern "C" {

int pf_apf_first_stage_prepare(pf_dtype dtype, void *lam, int64_t M, int64_t N, uint8_t *coll1,
                               void *stream) {
  PF_REQUIRE(lam && coll1 && M >= 1 && N >= 1 && N <= INT32_MAX,
             "pf_apf_first_stage_prepare: bad arguments");
  const cudaStream_t s = as_stream(stream);
  if (dtype == PF_F64)
    apf_prepare_kernel<double><<<static_cast<unsigned>(M), 256, 0, s>>>(
        static_cast<double *>(lam), static_cast<int32_t>(N), coll1);
  else
    apf_prepare_kernel<float><<<static_cast<unsigned>(M), 256, 0, s>>>(
        static_cast<float *>(lam), static_cast<int32_t>(N), coll1);
  return check_launch("pf_apf_first_stage_prepare");
}

int pf_compose_ancestors(const int32_t *outer, const int32_t *inner, int64_t MN, int32_t *out,
                         void *stream) {
  PF_REQUIRE(outer && out && MN >= 1 && outer != out, "pf_compose_ancestors: bad arguments");
  compose_kernel<<<grid_for(MN, 256), 256, 0, as_stream(stream)>>>(outer, inner, MN, out);
  return check_launch("pf_compose_ancestors");
}

int pf_apf_second_stage_weights(pf_dtype dtype, void *logw, const void *lam, const int32_t *anc1,
                                int64_t MN, void *stream) {
  PF_REQUIRE(logw && lam && anc1 && MN >= 1, "pf_apf_second_stage_weights: bad arguments");
  const cudaStream_t s = as_stream(stream);
  if (dtype == PF_F64)
    second_stage_kernel<double><<<grid_for(MN, 256), 256, 0, s>>>(
        static_cast<double *>(logw), static_cast<const double *>(lam), anc1, MN);
  else
    second_stage_kernel<float><<<grid_for(MN, 256), 256, 0, s>>>(
        static_cast<float *>(logw), static_cast<const float *>(lam), anc1, MN);
  return check_launch("pf_apf_second_stage_weights");
}

int pf_apf_finish(double *lnc, const double *lnc_before, uint8_t *collapsed,
                  const uint8_t *collapsed_first, int64_t M, void *stream) {
  PF_REQUIRE(lnc && lnc_before && collapsed && collapsed_first && M >= 1,
             "pf_apf_finish: bad arguments");
  apf_finish_kernel<<<grid_for(M, 128), 128, 0, as_stream(stream)>>>(lnc, lnc_before, collapsed,
                                                                     collapsed_first, M);
  return check_launch("pf_apf_finish");
}

}  // extern "C"
