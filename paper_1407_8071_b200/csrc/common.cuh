// Shared helpers for libpfbank (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdio>
#include <string>

#include "pfbank.h"

namespace pf {

void set_error(const char *fmt, ...);

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// Map the last launch error to a status code.
int check_launch(const char *what);

#define PF_REQUIRE(cond, ...)            \
  do {                                   \
    if (!(cond)) {                       \
      ::pf::set_error(__VA_ARGS__);      \
      return PF_EINVAL;                  \
    }                                    \
  } while (0)

constexpr int kSmCount = 148;

// Philox counter "purpose" words (fourth counter lane).
enum : uint32_t {
  kPurposePrior = 0x50524952u,      // 'PRIR'
  kPurposeLorenz = 0x4C4F525Au,     // 'LORZ'
  kPurposeFhn = 0x46484E5Fu,        // 'FHN_'
  kPurposeResample = 0x52534D50u,   // 'RSMP'
};

// ---- exact-order fp64 arithmetic: no FMA contraction, IEEE RN -------------
// The reference computes in numpy float64 with one rounding per operation;
// these wrappers keep nvcc from fusing a*b+c so the fp64 kernels reproduce
// the reference bit-for-bit on identical inputs.
template <typename T> struct Ar;
template <> struct Ar<double> {
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double fma(double a, double b, double c) {
    return __dadd_rn(__dmul_rn(a, b), c);
  }
};
// fp32 production arithmetic: contraction allowed (FFMA).
template <> struct Ar<float> {
  static __device__ __forceinline__ float add(float a, float b) { return a + b; }
  static __device__ __forceinline__ float sub(float a, float b) { return a - b; }
  static __device__ __forceinline__ float mul(float a, float b) { return a * b; }
  static __device__ __forceinline__ float fma(float a, float b, float c) { return fmaf(a, b, c); }
};

__device__ __forceinline__ bool finite_val(float x) { return isfinite(x); }
__device__ __forceinline__ bool finite_val(double x) { return isfinite(x); }

// production resample + fused posterior mean of planar states (resample.cu,
// used by the native bank driver bank.cu)
int segmented_resample_fused(pf_dtype dtype, const void *logw, int64_t M, int64_t N,
                             const uint32_t *keys, uint32_t t, int32_t *anc, double *lnc,
                             uint8_t *collapsed, uint32_t *status, void *ws, size_t ws_bytes,
                             const void *x, int dim, double *est, int64_t est_stride,
                             double *lnc_tr, uint8_t *coll_tr, cudaStream_t s, bool *fused);

// multi-GPU exchange (comm.cu): all-reduce(sum) of count doubles at buf on
// the communicator's side stream, ordered after the work enqueued on s
int comm_allreduce_after(pf_comm *c, double *buf, int64_t count, cudaStream_t s);

inline unsigned grid_for(int64_t n, int block) {
  return static_cast<unsigned>((n + block - 1) / block);
}

}  // namespace pf
