// Library plumbing: error reporting, version, device query, Philox KAT,
// and the small generic kernels (row fill, plane gather, ensemble average).
#include <cstdarg>
#include <cstdio>

#include "common.cuh"
#include "philox.cuh"

namespace pf {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int check_launch(const char *what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return PF_ECUDA;
  }
  return PF_OK;
}

__global__ void philox_kat_kernel(const uint4 *ctr, const uint2 *key, uint4 *out, int64_t n) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const uint4 c = ctr[i];
  const Key2 k{key[i].x, key[i].y};
  uint4 r = philox10(c, k);
  // the hoisted form used by the lattice/Lorenz kernels must agree bit for
  // bit; a mismatch poisons the answer (the KAT test then fails)
  const uint4 h = philox10_t(philox_pre_t(c.x, c.z, c.w, k), philox_uni_t(c.x, c.w, k),
                             c.y ^ k.k0, k);
  if (h.x != r.x || h.y != r.y || h.z != r.z || h.w != r.w)
    r = make_uint4(~r.x, ~r.y, ~r.z, ~r.w);
  out[i] = r;
}

// FP32 peak probe: 8 independent FFMA chains per thread, 8 x 256-thread
// blocks per SM (64 warps), iters x 8 x 2 flop per thread; the result is
// stored only if impossible so the chains stay live.
__global__ void __launch_bounds__(256) fma_chain_kernel(float *sink, int64_t iters) {
  float a[8];
  const float m = 1.0000001f, c = 1e-7f * static_cast<float>(threadIdx.x & 7);
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = static_cast<float>(threadIdx.x + i);
  for (int64_t k = 0; k < iters; ++k) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], m, c);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == -1.0f) sink[threadIdx.x] = s;
}

template <typename T>
__global__ void fill_rows_kernel(T *x, int64_t total, int64_t row_len, const double *row) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    x[i] = static_cast<T>(row[i % row_len]);
}

template <typename T>
__global__ void gather_planes_kernel(const T *__restrict__ xin, const int32_t *__restrict__ anc,
                                     int64_t MN, int32_t dims, T *__restrict__ xout) {
  const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (p >= MN) return;
  const int64_t src = anc[p];
  for (int d = 0; d < dims; ++d) xout[d * MN + p] = xin[d * MN + src];
}

// Left-to-right sum over filters then divide (ensemble.py:68-73).
__global__ void ensemble_average_kernel(const double *__restrict__ est, int64_t T, int64_t M,
                                        int64_t dim, double *__restrict__ out) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= T * dim) return;
  const int64_t t = g / dim, d = g - t * dim;
  const double *e = est + t * M * dim + d;
  double acc = e[0];
  for (int64_t m = 1; m < M; ++m) acc = __dadd_rn(acc, e[m * dim]);
  out[g] = __ddiv_rn(acc, static_cast<double>(M));
}

}  // namespace pf

using namespace pf;

extern "C" {

const char *pf_last_error(void) { return g_err; }

int pf_version(void) { return 10000; }

int pf_device_sm_count(int *out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return PF_ECUDA;
  if (cudaDeviceGetAttribute(out, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return PF_ECUDA;
  return PF_OK;
}

int pf_probe_fp32_fma(float *sink, int64_t iters, void *stream) {
  PF_REQUIRE(sink && iters >= 1, "pf_probe_fp32_fma: bad arguments");
  int sms = kSmCount;
  pf_device_sm_count(&sms);
  fma_chain_kernel<<<sms * 8, 256, 0, as_stream(stream)>>>(sink, iters);
  return check_launch("pf_probe_fp32_fma");
}

int pf_philox_kat(const uint32_t *ctr, const uint32_t *key, uint32_t *out, int64_t n,
                  void *stream) {
  PF_REQUIRE(n >= 0 && (n == 0 || (ctr && key && out)), "pf_philox_kat: bad arguments");
  if (n == 0) return PF_OK;
  philox_kat_kernel<<<grid_for(n, 128), 128, 0, as_stream(stream)>>>(
      reinterpret_cast<const uint4 *>(ctr), reinterpret_cast<const uint2 *>(key),
      reinterpret_cast<uint4 *>(out), n);
  return check_launch("pf_philox_kat");
}

int pf_fill_rows(pf_dtype dtype, void *x, int64_t MN, int64_t row_len, const double *row,
                 void *stream) {
  PF_REQUIRE(x && row && MN >= 1 && row_len >= 1, "pf_fill_rows: bad arguments");
  const int64_t total = MN * row_len;
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(grid_for(total, 256), 148 * 16));
  if (dtype == PF_F64)
    fill_rows_kernel<double><<<grid, 256, 0, as_stream(stream)>>>(static_cast<double *>(x), total,
                                                                  row_len, row);
  else
    fill_rows_kernel<float><<<grid, 256, 0, as_stream(stream)>>>(static_cast<float *>(x), total,
                                                                 row_len, row);
  return check_launch("pf_fill_rows");
}

int pf_gather_planes(pf_dtype dtype, const void *x_in, const int32_t *anc, int64_t MN,
                     int32_t dims, void *x_out, void *stream) {
  PF_REQUIRE(x_in && anc && x_out && MN >= 1 && dims >= 1, "pf_gather_planes: bad arguments");
  if (dtype == PF_F64)
    gather_planes_kernel<double><<<grid_for(MN, 256), 256, 0, as_stream(stream)>>>(
        static_cast<const double *>(x_in), anc, MN, dims, static_cast<double *>(x_out));
  else
    gather_planes_kernel<float><<<grid_for(MN, 256), 256, 0, as_stream(stream)>>>(
        static_cast<const float *>(x_in), anc, MN, dims, static_cast<float *>(x_out));
  return check_launch("pf_gather_planes");
}

int pf_ensemble_average(const double *est, int64_t T, int64_t M, int64_t dim, double *out,
                        void *stream) {
  PF_REQUIRE(est && out && T >= 1 && M >= 1 && dim >= 1, "pf_ensemble_average: bad arguments");
  ensemble_average_kernel<<<grid_for(T * dim, 128), 128, 0, as_stream(stream)>>>(est, T, M, dim,
                                                                                 out);
  return check_launch("pf_ensemble_average");
}

}  // extern "C"
