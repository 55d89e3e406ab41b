// Philox4x32-10 issue-rate probe: variants of the round's 32x32->64 multiply.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o philox_probe philox_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mulhi_asm(uint32_t a, uint32_t b) {
  uint32_t r;
  asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t mullo_asm(uint32_t a, uint32_t b) {
  uint32_t r;
  asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

template <int V>
__device__ __forceinline__ uint4 philox(uint4 c, uint32_t k0, uint32_t k1, uint32_t m0 = 0,
                                        uint32_t m1 = 0) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    uint32_t lo0, hi0, lo1, hi1;
    if (V == 0) {
      lo0 = 0xD2511F53u * c.x; hi0 = __umulhi(0xD2511F53u, c.x);
      lo1 = 0xCD9E8D57u * c.z; hi1 = __umulhi(0xCD9E8D57u, c.z);
    } else if (V == 2) {  // lo from a runtime copy of the multiplier: no IMAD.WIDE fusion
      lo0 = m0 * c.x; hi0 = __umulhi(0xD2511F53u, c.x);
      lo1 = m1 * c.z; hi1 = __umulhi(0xCD9E8D57u, c.z);
    } else {
      lo0 = mullo_asm(0xD2511F53u, c.x); hi0 = mulhi_asm(0xD2511F53u, c.x);
      lo1 = mullo_asm(0xCD9E8D57u, c.z); hi1 = mulhi_asm(0xCD9E8D57u, c.z);
    }
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

template <int V, int ILP>
__global__ void __launch_bounds__(256) probe(uint32_t *out, int iters, uint32_t k0, uint32_t k1,
                                             uint32_t m0, uint32_t m1) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int e = 0; e < ILP; ++e) {
      const uint4 r = philox<V>(make_uint4(j, it, e, 7u), k0, k1, m0, m1);
      acc ^= r.x ^ r.y ^ r.z ^ r.w;
    }
  }
  out[j] = acc;
}

template <int V, int ILP>
void run(const char *name, uint32_t *d, int blocks) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 4096 / ILP;
  probe<V, ILP><<<blocks, 256>>>(d, iters, 1, 2, 0xD2511F53u, 0xCD9E8D57u);
  cudaEventRecord(a);
  probe<V, ILP><<<blocks, 256>>>(d, iters, 1, 2, 0xD2511F53u, 0xCD9E8D57u);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double n = double(blocks) * 256 * iters * ILP;
  printf("%-14s %8.3f ms  %.3e philox/s  %.2f philox/clk/SM (1.965 GHz)\n", name, ms, n / (ms * 1e-3),
         n / (ms * 1e-3) / 148 / 1.965e9);
}

int main() {
  uint32_t *d;
  const int blocks = 148 * 8 * 4;
  cudaMalloc(&d, blocks * 256 * 4);
  run<0, 1>("wide ilp1", d, blocks);
  run<0, 2>("wide ilp2", d, blocks);
  run<1, 1>("split ilp1", d, blocks);
  run<1, 2>("split ilp2", d, blocks);
  run<2, 1>("hi+lo ilp1", d, blocks);
  run<2, 2>("hi+lo ilp2", d, blocks);
  run<0, 1>("wide ilp1", d, blocks);
  // correctness: variants agree
  return 0;
}
