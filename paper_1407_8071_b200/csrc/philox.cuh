// Counter-based RNG: Philox4x32-10 (Salmon et al., SC'11) and the normal /
// exponential transforms used by the bank kernels.
//
// The reference draws from numpy PCG64 streams spawned per filter
// (ensemble.py:56-60) - inherently sequential.  On the GPU every draw is a
// pure function of (per-filter key, counter), so any thread can produce any
// draw, and results are independent of launch geometry and GPU count.
#pragma once

#include <stdint.h>

namespace pf {

struct Key2 {
  uint32_t k0, k1;
};

__device__ __forceinline__ uint4 philox10(uint4 c, Key2 k) {
  uint32_t k0 = k.k0, k1 = k.k1;
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const uint32_t lo0 = 0xD2511F53u * c.x;
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

__device__ __forceinline__ Key2 load_key(const uint32_t *keys, int64_t f) {
  const uint2 k = __ldg(reinterpret_cast<const uint2 *>(keys) + f);
  return Key2{k.x, k.y};
}

// ---- fp32 Box-Muller: two N(0,1) from two 32-bit words ---------------------
// radius from a 32-bit uniform in (0,1] (max |z| = sqrt(2*32*ln2) = 6.66),
// angle from the top 24 bits.  Fast-path MUFU instructions (lg2, sqrt,
// sin/cos); accuracy ~1e-6 relative, far below the Monte Carlo noise.
__device__ __forceinline__ float2 box_muller_f32(uint32_t a, uint32_t b) {
  const float u = fmaf(static_cast<float>(a), 2.3283064365386963e-10f, 1.1641532182693481e-10f);
  const float r = sqrtf(-1.3862943611198906f * __log2f(u));  // -2 ln u = -2 ln2 log2 u
  const float ang = static_cast<float>(b >> 8) * 5.9604644775390625e-08f;  // [0,1)
  float s, c;
  __sincosf(6.283185307179586f * ang, &s, &c);
  return make_float2(r * c, r * s);
}

// ---- fast fp32 Box-Muller on the MUFU approximations -----------------------
// lg2/sqrt/sin/cos .approx.ftz: ~2^-21 relative error, no denormal or
// special-case branches (the precise sqrtf/logf paths cost ~2x the issue
// slots).  The angle is centred on [-pi, pi) where sin/cos.approx are most
// accurate; the resulting sign flip is immaterial for a symmetric law.
__device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sin_approx(float x) {
  float y;
  asm("sin.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float cos_approx(float x) {
  float y;
  asm("cos.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float2 box_muller_fast(uint32_t a, uint32_t b) {
  const float u = fmaf(static_cast<float>(a), 2.3283064365386963e-10f, 1.1641532182693481e-10f);
  const float r = sqrt_approx(-1.3862943611198906f * lg2_approx(u));
  // angle from 23 random mantissa bits without an int->float conversion:
  // x in [2, 4) -> pi*x - 3*pi in [-pi, pi)
  const float x = __uint_as_float((b & 0x007fffffu) | 0x40000000u);
  const float ang = fmaf(x, 3.14159265358979f, -9.42477796076938f);
  return make_float2(r * cos_approx(ang), r * sin_approx(ang));
}

// Same draw with the constant sqrt(2 ln 2) left out of the radius (callers
// fold it into their noise scale): r' = sqrt(-log2 u), z = sqrt(2 ln 2) r'.
constexpr float kSqrt2Ln2 = 1.1774100225154747f;
__device__ __forceinline__ float2 box_muller_fast_unscaled(uint32_t a, uint32_t b) {
  const float u = fmaf(static_cast<float>(a), 2.3283064365386963e-10f, 1.1641532182693481e-10f);
  const float r = sqrt_approx(-lg2_approx(u));
  const float x = __uint_as_float((b & 0x007fffffu) | 0x40000000u);
  const float ang = fmaf(x, 3.14159265358979f, -9.42477796076938f);
  return make_float2(r * cos_approx(ang), r * sin_approx(ang));
}

// ---- fp64 transforms (53-bit uniforms) ------------------------------------
__device__ __forceinline__ double u53_open0(uint32_t hi, uint32_t lo) {
  // (v + 1) * 2^-53 in (0, 1] with v a 53-bit integer
  const uint64_t v = (static_cast<uint64_t>(hi) << 21) ^ static_cast<uint64_t>(lo >> 11);
  return static_cast<double>(v + 1ull) * 1.1102230246251565e-16;
}

__device__ __forceinline__ double exp1_f64(uint32_t hi, uint32_t lo) {
  return -log(u53_open0(hi, lo));
}

__device__ __forceinline__ double2 box_muller_f64(uint32_t a, uint32_t b, uint32_t c,
                                                  uint32_t d) {
  const double u = u53_open0(a, b);
  const double v = u53_open0(c, d);
  const double r = sqrt(-2.0 * log(u));
  double s, co;
  sincospi(2.0 * v, &s, &co);
  return make_double2(r * co, r * s);
}

}  // namespace pf
