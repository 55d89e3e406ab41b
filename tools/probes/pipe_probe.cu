// Issue/pipe throughput probe for the instruction mix of the Philox +
// Box-Muller + Euler kernels (fhn_fast_kernel, lorenz_fast_kernel).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_probe pipe_probe.cu
//   ./pipe_probe
//
// Each kernel runs 8 independent dependency chains per thread at full
// occupancy (148 SMs x 8 blocks x 256 threads), so the result is the
// throughput bound of the instruction form, reported as warp instructions
// per clock per SM sub-partition (SMSP) at the measured SM clock.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kChains = 8;

#define CHAINS(body)                      \
  _Pragma("unroll") for (int c = 0; c < kChains; ++c) { body; }

__global__ void k_ffma_reg(float *out, float a, float b) {
  float x[kChains];
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x + c;
  float aa = a + threadIdx.x * 1e-9f, bb = b;
  for (int i = 0; i < kIters; ++i) {
    CHAINS(asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(aa), "f"(bb)));
  }
  float s = 0;
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1.2345f) out[0] = s;
}

__global__ void k_ffma_imm(float *out, float a, float b) {
  float x[kChains];
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x + c;
  float bb = b + threadIdx.x * 1e-9f;
  for (int i = 0; i < kIters; ++i) {
    CHAINS(asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFFE, %1;" : "+f"(x[c]) : "f"(bb)));
  }
  float s = 0;
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1.2345f) out[0] = s;
}

// multiplier from the kernel parameter (constant bank operand)
__global__ void k_ffma_cbank(float *out, float a, float b) {
  float x[kChains];
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x + c;
  float bb = b + threadIdx.x * 1e-9f;
  for (int i = 0; i < kIters; ++i) {
    CHAINS(x[c] = fmaf(x[c], a, bb));
  }
  float s = 0;
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1.2345f) out[0] = s;
}

__global__ void k_imad_wide(float *out, uint32_t a, uint32_t b) {
  uint32_t x[kChains];
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 7 + c;
  for (int i = 0; i < kIters; ++i) {
    CHAINS({
      uint64_t p;
      asm volatile("mul.wide.u32 %0, %1, 3528531795;" : "=l"(p) : "r"(x[c]));
      x[c] = static_cast<uint32_t>(p >> 32) ^ static_cast<uint32_t>(p);
    });
  }
  uint32_t s = 0;
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345u) out[0] = s;
}

__global__ void k_imad_hi(float *out, uint32_t a, uint32_t b) {
  uint32_t x[kChains];
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 7 + c;
  for (int i = 0; i < kIters; ++i) {
    CHAINS(asm volatile("mul.hi.u32 %0, %0, 3528531795;" : "+r"(x[c])));
  }
  uint32_t s = 0;
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345u) out[0] = s;
}

__global__ void k_imad_lo(float *out, uint32_t a, uint32_t b) {
  uint32_t x[kChains];
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 7 + c;
  for (int i = 0; i < kIters; ++i) {
    CHAINS(asm volatile("mul.lo.u32 %0, %0, 3528531795;" : "+r"(x[c])));
  }
  uint32_t s = 0;
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345u) out[0] = s;
}

__global__ void k_lop3(float *out, uint32_t a, uint32_t b) {
  uint32_t x[kChains];
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 7 + c;
  uint32_t aa = a ^ threadIdx.x, bb = b;
  for (int i = 0; i < kIters; ++i) {
    CHAINS(asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(aa), "r"(bb)));
  }
  uint32_t s = 0;
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345u) out[0] = s;
}

// FFMA (reg) interleaved 1:1 with LOP3 (alu): dual-pipe issue
__global__ void k_mix_ffma_lop3(float *out, uint32_t a, uint32_t b) {
  float x[kChains / 2];
  uint32_t y[kChains / 2];
  for (int c = 0; c < kChains / 2; ++c) {
    x[c] = threadIdx.x + c;
    y[c] = threadIdx.x * 3 + c;
  }
  float fa = 1.0000001f + threadIdx.x * 1e-9f, fb = 1e-7f;
  uint32_t aa = a ^ threadIdx.x, bb = b;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains / 2; ++c) {
      asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(fa), "f"(fb));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(y[c]) : "r"(aa), "r"(bb));
    }
  }
  float s = 0;
  for (int c = 0; c < kChains / 2; ++c) s += x[c] + y[c];
  if (s == 1.2345f) out[0] = s;
}

// IMAD.WIDE interleaved 1:1 with LOP3
__global__ void k_mix_imadw_lop3(float *out, uint32_t a, uint32_t b) {
  uint32_t x[kChains / 2], y[kChains / 2];
  for (int c = 0; c < kChains / 2; ++c) {
    x[c] = threadIdx.x + c;
    y[c] = threadIdx.x * 3 + c;
  }
  uint32_t aa = a ^ threadIdx.x, bb = b;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains / 2; ++c) {
      uint64_t p;
      asm volatile("mul.wide.u32 %0, %1, 3528531795;" : "=l"(p) : "r"(x[c]));
      x[c] = static_cast<uint32_t>(p >> 32) + static_cast<uint32_t>(p);
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(y[c]) : "r"(aa), "r"(bb));
    }
  }
  uint32_t s = 0;
  for (int c = 0; c < kChains / 2; ++c) s += x[c] + y[c];
  if (s == 12345u) out[0] = s;
}

__global__ void k_mufu_lg2(float *out, float a, float b) {
  float x[kChains];
  for (int c = 0; c < kChains; ++c) x[c] = 2.f + threadIdx.x + c;
  for (int i = 0; i < kIters; ++i) {
    CHAINS(asm volatile("lg2.approx.ftz.f32 %0, %0;" : "+f"(x[c])));
  }
  float s = 0;
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1.2345f) out[0] = s;
}

__global__ void k_mufu_sin(float *out, float a, float b) {
  float x[kChains];
  for (int c = 0; c < kChains; ++c) x[c] = 0.1f * (threadIdx.x + c);
  for (int i = 0; i < kIters; ++i) {
    CHAINS(asm volatile("sin.approx.ftz.f32 %0, %0;" : "+f"(x[c])));
  }
  float s = 0;
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1.2345f) out[0] = s;
}

__global__ void k_i2f(float *out, uint32_t a, uint32_t b) {
  uint32_t x[kChains];
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 7 + c;
  for (int i = 0; i < kIters; ++i) {
    CHAINS({
      float f;
      asm volatile("cvt.rn.f32.u32 %0, %1;" : "=f"(f) : "r"(x[c]));
      x[c] = __float_as_uint(f);
    });
  }
  uint32_t s = 0;
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345u) out[0] = s;
}

// HFMA2 on packed halves (fma pipe, 2 ops per lane)
__global__ void k_fmul_reg(float *out, float a, float b) {
  float x[kChains];
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x + c;
  float aa = a + threadIdx.x * 1e-9f;
  for (int i = 0; i < kIters; ++i) {
    CHAINS(asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(x[c]) : "f"(aa)));
  }
  float s = 0;
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1.2345f) out[0] = s;
}

__global__ void k_fadd_reg(float *out, float a, float b) {
  float x[kChains];
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x + c;
  float aa = a + threadIdx.x * 1e-9f;
  for (int i = 0; i < kIters; ++i) {
    CHAINS(asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(x[c]) : "f"(aa)));
  }
  float s = 0;
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1.2345f) out[0] = s;
}


// packed fp32 pairs (sm_100a FFMA2 / FADD2 / FMUL2): 2 lane-ops per issue
__global__ void k_ffma2_reg(float *out, float a, float b) {
  unsigned long long x[kChains];
  for (int c = 0; c < kChains; ++c) {
    const float f = threadIdx.x + c;
    asm("mov.b64 %0, {%1, %1};" : "=l"(x[c]) : "f"(f));
  }
  unsigned long long aa, bb;
  const float fa = a + threadIdx.x * 1e-9f;
  asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(fa));
  asm("mov.b64 %0, {%1, %1};" : "=l"(bb) : "f"(b));
  for (int i = 0; i < kIters; ++i) {
    CHAINS(asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[c]) : "l"(aa), "l"(bb)));
  }
  float s = 0;
  for (int c = 0; c < kChains; ++c) s += __uint_as_float(static_cast<uint32_t>(x[c]));
  if (s == 1.2345f) out[0] = s;
}

// FFMA2 with a scalar (broadcast) multiplier from the constant bank
__global__ void k_ffma2_bcast(float *out, float a, float b) {
  unsigned long long x[kChains];
  for (int c = 0; c < kChains; ++c) {
    const float f = threadIdx.x + c;
    asm("mov.b64 %0, {%1, %1};" : "=l"(x[c]) : "f"(f));
  }
  unsigned long long aa, bb;
  asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(a));
  asm("mov.b64 %0, {%1, %1};" : "=l"(bb) : "f"(b));
  for (int i = 0; i < kIters; ++i) {
    CHAINS(asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[c]) : "l"(aa), "l"(bb)));
  }
  float s = 0;
  for (int c = 0; c < kChains; ++c) s += __uint_as_float(static_cast<uint32_t>(x[c]));
  if (s == 1.2345f) out[0] = s;
}

__global__ void k_fadd2_reg(float *out, float a, float b) {
  unsigned long long x[kChains];
  for (int c = 0; c < kChains; ++c) {
    const float f = threadIdx.x + c;
    asm("mov.b64 %0, {%1, %1};" : "=l"(x[c]) : "f"(f));
  }
  unsigned long long aa;
  const float fa = a + threadIdx.x * 1e-9f;
  asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(fa));
  for (int i = 0; i < kIters; ++i) {
    CHAINS(asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(x[c]) : "l"(aa)));
  }
  float s = 0;
  for (int c = 0; c < kChains; ++c) s += __uint_as_float(static_cast<uint32_t>(x[c]));
  if (s == 1.2345f) out[0] = s;
}

// FFMA2 interleaved 1:1 with IMAD.WIDE (both fma-pipe families)
__global__ void k_mix_ffma2_imadw(float *out, float a, float b) {
  unsigned long long x[kChains / 2];
  uint32_t y[kChains / 2];
  unsigned long long aa, bb;
  const float fa = a + threadIdx.x * 1e-9f;
  asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(fa));
  asm("mov.b64 %0, {%1, %1};" : "=l"(bb) : "f"(b));
  for (int c = 0; c < kChains / 2; ++c) {
    const float f = threadIdx.x + c;
    asm("mov.b64 %0, {%1, %1};" : "=l"(x[c]) : "f"(f));
    y[c] = threadIdx.x * 3 + c;
  }
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains / 2; ++c) {
      asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[c]) : "l"(aa), "l"(bb));
      uint64_t p;
      asm volatile("mul.wide.u32 %0, %1, 3528531795;" : "=l"(p) : "r"(y[c]));
      y[c] = static_cast<uint32_t>(p >> 32) + static_cast<uint32_t>(p);
    }
  }
  float s = 0;
  for (int c = 0; c < kChains / 2; ++c) s += __uint_as_float(static_cast<uint32_t>(x[c])) + y[c];
  if (s == 1.2345f) out[0] = s;
}


// MUFU.LG2 with NW IMAD.WIDE per MUFU on independent chains: do the XU pipe
// (8 clocks per warp MUFU) and the FMA-heavy pipe (4 clocks per warp
// IMAD.WIDE) overlap?  NW = 2 is the ratio of the Philox + Box-Muller
// kernels (8 + 8 clocks per group if they overlap, 16 if they serialise).
template <int NW>
__global__ void k_mix_mufu_imadw(float *out, float a, float b) {
  float x[4];
  uint32_t y[4][NW > 0 ? NW : 1];
  for (int c = 0; c < 4; ++c) {
    x[c] = 2.f + threadIdx.x + c;
    for (int w = 0; w < NW; ++w) y[c][w] = threadIdx.x * 3 + c + 17 * w;
  }
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      asm volatile("lg2.approx.ftz.f32 %0, %0;" : "+f"(x[c]));
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        uint64_t p;
        asm volatile("mul.wide.u32 %0, %1, 3528531795;" : "=l"(p) : "r"(y[c][w]));
        y[c][w] = static_cast<uint32_t>(p >> 32) ^ static_cast<uint32_t>(p);
      }
    }
  }
  float s = 0;
  for (int c = 0; c < 4; ++c) {
    s += x[c];
    for (int w = 0; w < NW; ++w) s += y[c][w];
  }
  if (s == 1.2345f) out[0] = s;
}

// The production kernels' per-step instruction mix on independent chains,
// per group: MU MUFU, 2 IMAD.WIDE each followed by the xor of its halves,
// NX more LOP3, NF FFMA.  fhn_cm_kernel issues MUFU : IMAD.WIDE : LOP3 :
// FFMA/FADD/FMUL = 24 : 49 : 67 : 96 per thread-step (1 : 2 : 3 : 4),
// lorenz_fast_kernel 6 : 12 : 15 : 20 (1 : 2 : 2.5 : 3.3): the issue rate the
// mix reaches without barriers, shared memory or dependent chains, at full
// occupancy and at the FH-N kernel's 4 warps per SMSP.
template <int MU, int NX, int NF>
__global__ void k_mix_fhn(float *out, float a, float b) {
  float x[4], f[4][NF > 0 ? NF : 1];
  uint32_t y[4][2], z[4];
  const float fa = 1.0000001f + threadIdx.x * 1e-9f, fb = 1e-7f;
  for (int c = 0; c < 4; ++c) {
    x[c] = 2.f + threadIdx.x + c;
    z[c] = threadIdx.x * 5 + c;
    for (int w = 0; w < 2; ++w) y[c][w] = threadIdx.x * 3 + c + 17 * w;
    for (int w = 0; w < NF; ++w) f[c][w] = threadIdx.x + c + w;
  }
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (MU) asm volatile("lg2.approx.ftz.f32 %0, %0;" : "+f"(x[c]));
#pragma unroll
      for (int w = 0; w < 2; ++w) {
        uint64_t p;
        asm volatile("mul.wide.u32 %0, %1, 3528531795;" : "=l"(p) : "r"(y[c][w]));
        y[c][w] = static_cast<uint32_t>(p >> 32) ^ static_cast<uint32_t>(p);
#pragma unroll
        for (int q = w * NF / 2; q < (w + 1) * NF / 2; ++q)
          asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[c][q]) : "f"(fa), "f"(fb));
      }
#pragma unroll
      for (int q = 0; q < NX; ++q)
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(z[c]) : "r"(y[c][0]), "r"(y[c][1]));
    }
  }
  float s = 0;
  for (int c = 0; c < 4; ++c) {
    s += x[c] + z[c];
    for (int w = 0; w < 2; ++w) s += y[c][w];
    for (int w = 0; w < NF; ++w) s += f[c][w];
  }
  if (s == 1.2345f) out[0] = s;
}

// groups of `ops` instructions, 4 groups per iteration; blocks_per_sm sets
// the occupancy (256-thread blocks)
template <typename K>
void run_mix(const char *name, K kern, int ops, int blocks_per_sm, float *out, int sms,
             double clk_ghz) {
  const int blocks = sms * blocks_per_sm, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(out, 1.f, 1.f);
  cudaEventRecord(e0);
  for (int r = 0; r < 3; ++r) kern<<<blocks, threads>>>(out, 1.f, 1.f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double groups = 3.0 * blocks * (threads / 32) * double(kIters) * 4;
  const double clk_per_group = (ms * 1e-3) * (clk_ghz * 1e9) * (sms * 4) / groups;
  printf("%-22s %2d warps/SMSP %8.3f ms  %6.2f clk/group/SMSP  %.3f warp-inst/clk/SMSP (%d per group)\n",
         name, blocks_per_sm * 2, ms, clk_per_group, ops / clk_per_group, ops);
}

template <typename K, typename A>
void run(const char *name, K kern, A a, A b, float *out, int sms, double clk_ghz) {
  const int blocks = sms * 8, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(out, a, b);
  cudaEventRecord(e0);
  for (int r = 0; r < 3; ++r) kern<<<blocks, threads>>>(out, a, b);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warp_inst = 3.0 * blocks * (threads / 32) * double(kIters) * kChains;
  const double per_smsp_clk = warp_inst / (ms * 1e-3) / (sms * 4) / (clk_ghz * 1e9);
  printf("%-18s %8.3f ms  %.3f warp-inst/clk/SMSP (main op)\n", name, ms, per_smsp_clk);
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  const double ghz = clk_khz / 1e6;
  printf("SMs %d, max SM clock %.3f GHz (rates assume the max clock)\n", sms, ghz);
  float *out;
  cudaMalloc(&out, 64);
  run("ffma_reg", k_ffma_reg, 1.0000001f, 1e-7f, out, sms, ghz);
  run("ffma_imm", k_ffma_imm, 1.0000001f, 1e-7f, out, sms, ghz);
  run("ffma_cbank", k_ffma_cbank, 1.0000001f, 1e-7f, out, sms, ghz);
  run("ffma2_reg", k_ffma2_reg, 1.0000001f, 1e-7f, out, sms, ghz);
  run("ffma2_bcast", k_ffma2_bcast, 1.0000001f, 1e-7f, out, sms, ghz);
  run("fadd2_reg", k_fadd2_reg, 1e-7f, 1e-7f, out, sms, ghz);
  run("mix_ffma2_imadw", k_mix_ffma2_imadw, 1.0000001f, 1e-7f, out, sms, ghz);
  run("fmul_reg", k_fmul_reg, 1.0000001f, 1e-7f, out, sms, ghz);
  run("fadd_reg", k_fadd_reg, 1e-7f, 1e-7f, out, sms, ghz);
  run("imad_wide_imm", k_imad_wide, 3u, 5u, out, sms, ghz);
  run("imad_hi_imm", k_imad_hi, 3u, 5u, out, sms, ghz);
  run("imad_lo_imm", k_imad_lo, 3u, 5u, out, sms, ghz);
  run("lop3", k_lop3, 3u, 5u, out, sms, ghz);
  run("mix_ffma_lop3", k_mix_ffma_lop3, 3u, 5u, out, sms, ghz);
  run("mix_imadw_lop3", k_mix_imadw_lop3, 3u, 5u, out, sms, ghz);
  run("mufu_lg2", k_mufu_lg2, 1.f, 1.f, out, sms, ghz);
  run("mufu_sin", k_mufu_sin, 1.f, 1.f, out, sms, ghz);
  run("i2f_u32", k_i2f, 3u, 5u, out, sms, ghz);
  // mixes: instructions per group incl. the xor of each multiply
  run_mix("mufu_only", k_mix_mufu_imadw<0>, 1, 8, out, sms, ghz);
  run_mix("mufu+1imadw", k_mix_mufu_imadw<1>, 3, 8, out, sms, ghz);
  run_mix("mufu+2imadw", k_mix_mufu_imadw<2>, 5, 8, out, sms, ghz);
  run_mix("mufu+4imadw", k_mix_mufu_imadw<4>, 9, 8, out, sms, ghz);
  run_mix("fhn_mix 1:2:3:4", k_mix_fhn<1, 1, 4>, 10, 8, out, sms, ghz);
  run_mix("fhn_mix 1:2:3:4", k_mix_fhn<1, 1, 4>, 10, 2, out, sms, ghz);
  run_mix("fhn_mix 1:2:3:4", k_mix_fhn<1, 1, 4>, 10, 1, out, sms, ghz);
  run_mix("lorenz_mix 1:2:3:3", k_mix_fhn<1, 1, 3>, 9, 8, out, sms, ghz);
  run_mix("mix 1:2:3:0 (no FFMA)", k_mix_fhn<1, 1, 0>, 6, 8, out, sms, ghz);
  run_mix("mix 1:2:3:2", k_mix_fhn<1, 1, 2>, 8, 8, out, sms, ghz);
  run_mix("mix 0:2:3:4 (no MUFU)", k_mix_fhn<0, 1, 4>, 9, 8, out, sms, ghz);
  run_mix("mix 0:2:3:8 (no MUFU)", k_mix_fhn<0, 1, 8>, 13, 8, out, sms, ghz);
  run_mix("mix 1:2:3:8", k_mix_fhn<1, 1, 8>, 14, 8, out, sms, ghz);
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
