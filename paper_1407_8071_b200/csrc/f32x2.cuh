// Packed fp32 pairs on sm_100a: FFMA2 / FADD2 / FMUL2 (PTX fma/add/mul
// .rn.f32x2) execute two independent IEEE fp32 operations per lane in ONE
// issue slot.  Each lane rounds exactly like the scalar fmaf / + / * (no FTZ,
// no contraction), so a kernel restated on pairs is bit-identical to its
// scalar form; what changes is the instruction count of issue-bound kernels.
// A pair built from one scalar (f2_bcast) is folded by ptxas into a
// broadcast ".F32" operand (constant bank / uniform register): no copies.
#pragma once

namespace pf {

typedef unsigned long long f2_t;  // {lo, hi} = two fp32 lanes

__device__ __forceinline__ f2_t f2_pack(float lo, float hi) {
  f2_t d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(lo), "f"(hi));
  return d;
}
__device__ __forceinline__ f2_t f2_bcast(float s) { return f2_pack(s, s); }
__device__ __forceinline__ float f2_lo(f2_t a) {
  float lo;
  asm("{\n .reg .f32 h;\n mov.b64 {%0, h}, %1;\n}" : "=f"(lo) : "l"(a));
  return lo;
}
__device__ __forceinline__ float f2_hi(f2_t a) {
  float hi;
  asm("{\n .reg .f32 l;\n mov.b64 {l, %0}, %1;\n}" : "=f"(hi) : "l"(a));
  return hi;
}
// a * b + c per lane, one rounding
__device__ __forceinline__ f2_t f2_fma(f2_t a, f2_t b, f2_t c) {
  f2_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f2_t f2_add(f2_t a, f2_t b) {
  f2_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2_t f2_mul(f2_t a, f2_t b) {
  f2_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

}  // namespace pf
