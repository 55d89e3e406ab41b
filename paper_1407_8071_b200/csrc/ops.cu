// Hook-level resampling helpers in the reference's floating-point order
// (resampling.py:21-72): the CDF cum = np.cumsum(w) and the order statistics
// np.cumsum(Exp(1) x (n+1))[:n] / c[n] are strictly sequential sums in numpy,
// so they are reproduced with a sequential device scan (one warp streams
// 1024-element tiles through shared memory while lane 0 adds); systematic
// thresholds (i + r) / n are elementwise.  The bank path never uses these
// (its resampler builds the CDF per filter, resample.cu).
#include "common.cuh"

namespace pf {

__global__ void __launch_bounds__(32) seq_cumsum_kernel(const double *__restrict__ a, int64_t n,
                                                        double *__restrict__ out) {
  __shared__ double tile[1024];
  const int lane = threadIdx.x;
  const int64_t ntiles = (n + 1023) / 1024;
  double pre[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const int64_t i = j * 32 + lane;
    pre[j] = i < n ? a[i] : 0.0;
  }
  double run = 0.0;
  for (int64_t tt = 0; tt < ntiles; ++tt) {
#pragma unroll
    for (int j = 0; j < 32; ++j) tile[j * 32 + lane] = pre[j];
    // prefetch the next tile while lane 0 scans this one
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int64_t i = (tt + 1) * 1024 + j * 32 + lane;
      pre[j] = i < n ? a[i] : 0.0;
    }
    __syncwarp();
    if (lane == 0) {
      const int64_t i0 = tt * 1024;
      const int cnt = static_cast<int>(n - i0 < 1024 ? n - i0 : 1024);
      for (int i = 0; i < cnt; ++i) {
        run = (tt == 0 && i == 0) ? tile[0] : __dadd_rn(run, tile[i]);
        tile[i] = run;
      }
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int64_t i = tt * 1024 + j * 32 + lane;
      if (i < n) out[i] = tile[j * 32 + lane];
    }
    __syncwarp();
  }
}

__global__ void spacing_divide_kernel(const double *__restrict__ c, int64_t n,
                                      double *__restrict__ u) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) u[i] = __ddiv_rn(c[i], c[n]);
}

__global__ void systematic_kernel(double r, int64_t n, double *__restrict__ u) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) u[i] = __ddiv_rn(__dadd_rn(static_cast<double>(i), r), static_cast<double>(n));
}

}  // namespace pf

using namespace pf;

extern "C" {

int pf_op_cumsum(const double *a, int64_t n, double *out, void *stream) {
  PF_REQUIRE(a && out && n >= 1, "pf_op_cumsum: bad arguments");
  seq_cumsum_kernel<<<1, 32, 0, as_stream(stream)>>>(a, n, out);
  return check_launch("pf_op_cumsum");
}

int pf_op_spacing_uniforms(const double *e, int64_t n_out, double *work, double *u,
                           void *stream) {
  PF_REQUIRE(e && work && u && n_out >= 1, "pf_op_spacing_uniforms: bad arguments");
  const cudaStream_t s = as_stream(stream);
  seq_cumsum_kernel<<<1, 32, 0, s>>>(e, n_out + 1, work);
  spacing_divide_kernel<<<grid_for(n_out, 256), 256, 0, s>>>(work, n_out, u);
  return check_launch("pf_op_spacing_uniforms");
}

int pf_op_systematic_uniforms(double r, int64_t n_out, double *u, void *stream) {
  PF_REQUIRE(u && n_out >= 1, "pf_op_systematic_uniforms: bad arguments");
  systematic_kernel<<<grid_for(n_out, 256), 256, 0, as_stream(stream)>>>(r, n_out, u);
  return check_launch("pf_op_systematic_uniforms");
}

}  // extern "C"
