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

// Philox4x32 rounds: 10, the Random123 / cuRAND default this library specifies
// and its known-answer tests pin.  -DPF_PHILOX_ROUNDS=7 (the authors' minimum
// that passes BigCrush) exists only to measure what the 32x32 multiplies cost
// (dispatch-slot bound); such a build fails the
// known-answer tests by design.
#ifndef PF_PHILOX_ROUNDS
#define PF_PHILOX_ROUNDS 10
#endif
constexpr int kPhiloxRounds = PF_PHILOX_ROUNDS;
static_assert(kPhiloxRounds >= 4 && kPhiloxRounds <= 10, "hoisted rounds 1-3 + key schedule");

__device__ __forceinline__ uint4 philox10(uint4 c, Key2 k) {
  uint32_t k0 = k.k0, k1 = k.k1;
#pragma unroll
  for (int i = 0; i < kPhiloxRounds; ++i) {
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

// 32x32 -> 64 product as one IMAD.WIDE.U32 (ptxas otherwise may split the
// lo/hi halves into IMAD + IMAD.HI, two issue slots).
__device__ __forceinline__ void mulhilo(uint32_t m, uint32_t a, uint32_t &lo, uint32_t &hi) {
  uint64_t p;
  asm("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(a), "r"(m));
  asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(p));
}

// Philox4x32-10 for a counter (c0, c1, c2, c3) with c0 block-uniform and
// fixed (FH-N: particle index; Lorenz: observation time), c1 the uniform word
// that changes inside the loop (FH-N: Euler step; Lorenz: draw index), c2
// fixed per thread (FH-N: node pair; Lorenz: particle) and c3 the purpose.
// philox_pre_t hoists everything of rounds 1-3 that does not depend on c1
// (3 words per thread and draw index); philox10_t is bit-identical to
// philox10(make_uint4(c0, c1, c2, c3), k).
struct PhiloxPreT {
  uint32_t h1;        // hi(M1 c2)                      (round 1, X1 = h1 ^ c1 ^ k0)
  uint32_t lo3, hi3;  // lo/hi(M0 X2), X2 independent of c1 (round 3)
};
struct PhiloxUni {    // block-uniform, c1-independent words (uniform registers)
  uint32_t w1k1;      // W1 ^ (k1 + C1)         (round 2, Z2 = hi(M0 X1) ^ W1 ^ k1')
  uint32_t y2k0;      // Y2 ^ (k0 + 2 C0)       (round 3, X3 = hi(M1 Z2) ^ Y2 ^ k0'')
};

__device__ __forceinline__ PhiloxUni philox_uni_t(uint32_t c0, uint32_t c3, Key2 k) {
  const uint32_t w1 = 0xD2511F53u * c0;
  const uint32_t z1 = __umulhi(0xD2511F53u, c0) ^ c3 ^ k.k1;
  const uint32_t y2 = 0xCD9E8D57u * z1;
  return PhiloxUni{w1 ^ (k.k1 + 0xBB67AE85u), y2 ^ (k.k0 + 2u * 0x9E3779B9u)};
}

__device__ __forceinline__ PhiloxPreT philox_pre_t(uint32_t c0, uint32_t c2, uint32_t c3,
                                                   Key2 k) {
  const uint32_t z1 = __umulhi(0xD2511F53u, c0) ^ c3 ^ k.k1;
  const uint32_t y1 = 0xCD9E8D57u * c2;
  const uint32_t x2 = __umulhi(0xCD9E8D57u, z1) ^ y1 ^ (k.k0 + 0x9E3779B9u);
  PhiloxPreT pre;
  pre.h1 = __umulhi(0xCD9E8D57u, c2);
  mulhilo(0xD2511F53u, x2, pre.lo3, pre.hi3);
  return pre;
}

// c1k0 = c1 ^ k0 (per step, uniform)
__device__ __forceinline__ uint4 philox10_t(const PhiloxPreT &pre, const PhiloxUni &u,
                                            uint32_t c1k0, Key2 k) {
  uint32_t lo, hi;
  // round 1 -> X1; round 2: Z2, W2
  const uint32_t x1 = pre.h1 ^ c1k0;
  mulhilo(0xD2511F53u, x1, lo, hi);
  const uint32_t z2 = hi ^ u.w1k1, w2 = lo;
  // round 3 (key k + 2C)
  mulhilo(0xCD9E8D57u, z2, lo, hi);
  uint4 c = make_uint4(hi ^ u.y2k0, lo, pre.hi3 ^ w2 ^ (k.k1 + 2u * 0xBB67AE85u), pre.lo3);
  uint32_t k0 = k.k0 + 2u * 0x9E3779B9u, k1 = k.k1 + 2u * 0xBB67AE85u;
#pragma unroll
  for (int i = 3; i < kPhiloxRounds; ++i) {
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
    uint32_t lo0, hi0, lo1, hi1;
    mulhilo(0xD2511F53u, c.x, lo0, hi0);
    mulhilo(0xCD9E8D57u, c.z, lo1, hi1);
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
  }
  return c;
}

// The Philox key schedule k + i*C (i = 0..9) computed once per thread (for a
// block-uniform key the compiler can keep it in uniform registers).
struct PhiloxKeys {
  uint32_t k0[10], k1[10];
};
__device__ __forceinline__ PhiloxKeys philox_round_keys(Key2 k) {
  PhiloxKeys r;
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    r.k0[i] = k.k0 + static_cast<uint32_t>(i) * 0x9E3779B9u;
    r.k1[i] = k.k1 + static_cast<uint32_t>(i) * 0xBB67AE85u;
  }
  return r;
}

// philox10_t with a precomputed key schedule (bit-identical)
__device__ __forceinline__ uint4 philox10_t(const PhiloxPreT &pre, const PhiloxUni &u,
                                            uint32_t c1k0, const PhiloxKeys &rk) {
  uint32_t lo, hi;
  const uint32_t x1 = pre.h1 ^ c1k0;
  mulhilo(0xD2511F53u, x1, lo, hi);
  const uint32_t z2 = hi ^ u.w1k1, w2 = lo;
  mulhilo(0xCD9E8D57u, z2, lo, hi);
  uint4 c = make_uint4(hi ^ u.y2k0, lo, pre.hi3 ^ w2 ^ rk.k1[2], pre.lo3);
#pragma unroll
  for (int i = 3; i < kPhiloxRounds; ++i) {
    uint32_t lo0, hi0, lo1, hi1;
    mulhilo(0xD2511F53u, c.x, lo0, hi0);
    mulhilo(0xCD9E8D57u, c.z, lo1, hi1);
    c = make_uint4(hi1 ^ c.y ^ rk.k0[i], lo1, hi0 ^ c.w ^ rk.k1[i], lo0);
  }
  return c;
}

__device__ __forceinline__ Key2 load_key(const uint32_t *keys, int64_t f) {
  const uint2 k = __ldg(reinterpret_cast<const uint2 *>(keys) + f);
  return Key2{k.x, k.y};
}

// ---- fp32 Box-Muller, accurate libm form (generic kernels) ------------------
// The same map from two 32-bit words to two N(0,1) as box_muller_rad_trig
// below - radius from u = (a + 1/2) 2^-32 in (0,1) (max |z| = 6.66), angle
// pi*x - 3*pi from the low 23 bits of b (x in [2,4)) - but with accurate
// logf/sqrtf/sincosf instead of the MUFU approximations, so a generic kernel
// reproduces the fast kernels' draws to ~1e-6 and can check them.
__device__ __forceinline__ float2 box_muller_ref_f32(uint32_t a, uint32_t b) {
  const float u = fmaf(static_cast<float>(a), 2.3283064365386963e-10f, 1.1641532182693481e-10f);
  const float r = sqrtf(-2.0f * logf(u));
  const float x = __uint_as_float((b & 0x007fffffu) | 0x40000000u);
  const float ang = fmaf(x, 3.14159265358979f, -9.42477796076938f);
  float s, c;
  sincosf(ang, &s, &c);
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

// Box-Muller with the caller's noise scale folded into the radius: returns
// r' = sqrt(log2(u) * s2) with s2 = -(2 ln 2) s^2 and the trig factors, so
// that s*z0 = r'*c0 and s*z1 = r'*s1 (one FFMA per increment at the caller).
__device__ __forceinline__ void box_muller_rad_trig(uint32_t a, uint32_t b, float s2,
                                                    float &rad, float &c0, float &s1) {
  const float u = fmaf(static_cast<float>(a), 2.3283064365386963e-10f, 1.1641532182693481e-10f);
  rad = sqrt_approx(lg2_approx(u) * s2);
  const float x = __uint_as_float((b & 0x007fffffu) | 0x40000000u);
  const float ang = fmaf(x, 3.14159265358979f, -9.42477796076938f);
  c0 = cos_approx(ang);
  s1 = sin_approx(ang);
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
