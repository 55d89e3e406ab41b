// Stochastically forced FitzHugh-Nagumo network: the paper's lattice model
// (models/fhn.py:85-207).
//
// One transition = ONE lattice Euler step (fhn.py:153-189):
//   1. stimulus region  R = {nodes whose own or a 4-neighbour's U lies in
//      (u_minus, u_plus)}                                   (fhn.py:52-67)
//   2. with probability stim_prob (one uniform per particle) a new stimulus
//      at the rank-th region cell, rank = int(u_sel * |R|) in row-major
//      order, plus its von Neumann neighbours               (fhn.py:157-168)
//   3. drive = forcing_mask * forcing(t) + stim_amp * [stimulus in the last
//      stim_hold steps]                                      (fhn.py:149-151, 170-174)
//   4. accel.fhn_euler_block with sig_sqdt * N(0,1) noise    (accel.py:110-129)
//   5. history shift Q <- [q_new, Q(t-1) .. ]                (fhn.py:188)
// then the zone log-likelihood (fhn.py:199-207) in the epilogue.
//
// Layout: per particle p the voltage and recovery planes
// x[p*2*nodes + {0, nodes} + node] (fp32 or fp64) and the stimulus history
// as a bit field q[p*nodes + node] (bit k = Q(t-k)), so the reference's
// (2 + stim_hold) * J^2 float64 row (221 KB at J = 32) is 12 B/node in fp32.
//
// One CTA owns one particle per iteration of a persistent loop: U is staged
// in shared memory for the 4-neighbour stencil and the region test, V and
// the history bits stream through registers with vectorised loads, and the
// ancestor gather is fused into the load (filters.py:111).  The region /
// cell search only runs for the ~stim_prob of particles that fire
// (CTA-uniform branch).  fp64 uses the exact-order Ar<double> arithmetic and
// is bit-identical to the reference on identical draws.
#include "bulk.cuh"
#include "common.cuh"
#include "npsum.cuh"
#include "philox.cuh"

#include <algorithm>
#include <cstdlib>
#include <cstring>

namespace pf {

enum : uint32_t {
  kPurposeNetNoise = 0x464E4E5Au,  // 'FNNZ'
  kPurposeNetStim = 0x464E5354u,   // 'FNST'
};

struct NetConsts {
  int J, nodes, n_obs, stochastic;
  uint32_t hist_mask, recent_mask;
  double dt, coupling, a3, a2, a1, a0, b0, b1, b2;
  double u_minus, u_plus, stim_prob, stim_amp, forcing, sig, obs_coef;
};

// numpy Generator.random(): (v >> 11) * 2^-53 in [0, 1)
__device__ __forceinline__ double u53_closed0(uint32_t hi, uint32_t lo) {
  const uint64_t v = (static_cast<uint64_t>(hi) << 21) ^ static_cast<uint64_t>(lo >> 11);
  return static_cast<double>(v) * 1.1102230246251565e-16;
}

// Production normals: Philox block g covers 4 nodes (fp32: two MUFU
// Box-Muller pairs) or 2 nodes (fp64: one precise pair), independent of the
// vector width a launch uses.
template <typename T> struct NetNoise;
template <> struct NetNoise<float> {
  static constexpr int kGroup = 4;
  static __device__ __forceinline__ void draw(Key2 k, uint32_t j, uint32_t t, uint32_t g,
                                              float *z) {
    const uint4 r = philox10(make_uint4(j, t, g, kPurposeNetNoise), k);
    const float2 a = box_muller_fast(r.x, r.y), b = box_muller_fast(r.z, r.w);
    z[0] = a.x;
    z[1] = a.y;
    z[2] = b.x;
    z[3] = b.y;
  }
};
template <> struct NetNoise<double> {
  static constexpr int kGroup = 2;
  static __device__ __forceinline__ void draw(Key2 k, uint32_t j, uint32_t t, uint32_t g,
                                              double *z) {
    const uint4 r = philox10(make_uint4(j, t, g, kPurposeNetNoise), k);
    const double2 a = box_muller_f64(r.x, r.y, r.z, r.w);
    z[0] = a.x;
    z[1] = a.y;
  }
};

template <typename T, int G> struct VecIO;
template <typename T> struct VecIO<T, 1> {
  static __device__ __forceinline__ void load(const T *p, T *v) { v[0] = p[0]; }
  static __device__ __forceinline__ void store(T *p, const T *v) { p[0] = v[0]; }
  static __device__ __forceinline__ void loadq(const uint32_t *p, uint32_t *v) { v[0] = p[0]; }
  static __device__ __forceinline__ void storeq(uint32_t *p, const uint32_t *v) { p[0] = v[0]; }
};
template <> struct VecIO<float, 4> {
  static __device__ __forceinline__ void load(const float *p, float *v) {
    const float4 a = *reinterpret_cast<const float4 *>(p);
    v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w;
  }
  static __device__ __forceinline__ void store(float *p, const float *v) {
    *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
  static __device__ __forceinline__ void loadq(const uint32_t *p, uint32_t *v) {
    const uint4 a = *reinterpret_cast<const uint4 *>(p);
    v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w;
  }
  static __device__ __forceinline__ void storeq(uint32_t *p, const uint32_t *v) {
    *reinterpret_cast<uint4 *>(p) = make_uint4(v[0], v[1], v[2], v[3]);
  }
};
template <> struct VecIO<double, 2> {
  static __device__ __forceinline__ void load(const double *p, double *v) {
    const double2 a = *reinterpret_cast<const double2 *>(p);
    v[0] = a.x, v[1] = a.y;
  }
  static __device__ __forceinline__ void store(double *p, const double *v) {
    *reinterpret_cast<double2 *>(p) = make_double2(v[0], v[1]);
  }
  static __device__ __forceinline__ void loadq(const uint32_t *p, uint32_t *v) {
    const uint2 a = *reinterpret_cast<const uint2 *>(p);
    v[0] = a.x, v[1] = a.y;
  }
  static __device__ __forceinline__ void storeq(uint32_t *p, const uint32_t *v) {
    *reinterpret_cast<uint2 *>(p) = make_uint2(v[0], v[1]);
  }
};

// MODE 0 = Philox draws, MODE 1 = tape: stim_tape (M, 2, N) [fire, select]
// uniforms and z_tape (M, N, nodes) standard normals, fp64.
// G = nodes per thread and vector access (nodes % G == 0).
template <typename T, int MODE, int G>
__global__ void __launch_bounds__(256) fhnnet_step_kernel(
    const T *__restrict__ xin, const uint32_t *__restrict__ qin, const int32_t *__restrict__ anc,
    T *__restrict__ xout, uint32_t *__restrict__ qout, const double *__restrict__ fmask,
    const double *__restrict__ y, const int32_t *__restrict__ obs_idx, T *__restrict__ logw,
    int64_t MN, int32_t N, NetConsts c, const uint32_t *__restrict__ keys, uint32_t t,
    const double *__restrict__ stim_tape, const double *__restrict__ z_tape,
    uint32_t *__restrict__ status) {
  using A = Ar<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *s_u = reinterpret_cast<T *>(smem_raw);               // [nodes] U(t-1)
  T *s_un = s_u + c.nodes;                                // [nodes] U(t)
  double *s_sq = reinterpret_cast<double *>(s_un + c.nodes);  // [n_obs] residual^2
  uint32_t *s_mask = reinterpret_cast<uint32_t *>(s_sq + c.n_obs);  // region bits
  __shared__ int s_fire, s_cell, s_bad;
  __shared__ double s_sel;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int words = (c.nodes + 31) >> 5;
  const int groups = c.nodes / G;
  const T dt = T(c.dt);

  for (int64_t p = blockIdx.x; p < MN; p += gridDim.x) {
    const int64_t f = p / N;
    const uint32_t j = static_cast<uint32_t>(p - f * N);
    const int64_t src = anc ? static_cast<int64_t>(__ldg(anc + p)) : p;
    const T *xs = xin + src * 2 * static_cast<int64_t>(c.nodes);
    const uint32_t *qs = qin + src * static_cast<int64_t>(c.nodes);
    Key2 key{0u, 0u};
    if (MODE == 0 && c.stochastic) key = load_key(keys, f);

    if (tid == 0) {
      // rng.random(n) twice: fire, then cell select (fhn.py:158-159)
      int fire = 0;
      double sel = 0.0;
      if (c.stochastic) {
        double uf;
        if (MODE == 1) {
          uf = stim_tape[(f * 2) * N + j];
          sel = stim_tape[(f * 2 + 1) * N + j];
        } else {
          const uint4 r = philox10(make_uint4(j, t, 0u, kPurposeNetStim), key);
          uf = u53_closed0(r.x, r.y);
          sel = u53_closed0(r.z, r.w);
        }
        fire = uf < c.stim_prob;
      }
      s_fire = fire;
      s_sel = sel;
      s_cell = -1;
      s_bad = 0;
    }
    for (int n = tid; n < c.nodes; n += blockDim.x) s_u[n] = xs[n];
    __syncthreads();

    if (s_fire) {  // CTA-uniform: rare (stim_prob per particle-step)
      const T lo = T(c.u_minus), hi = T(c.u_plus);
      for (int base = 0; base < c.nodes; base += blockDim.x) {
        const int n = base + tid;
        bool in_region = false;
        if (n < c.nodes) {
          const int i = n / c.J, jj = n - i * c.J;
          auto inside = [&](T u) { return u > lo && u < hi; };
          in_region = inside(s_u[n]) || (i > 0 && inside(s_u[n - c.J])) ||
                      (i < c.J - 1 && inside(s_u[n + c.J])) || (jj > 0 && inside(s_u[n - 1])) ||
                      (jj < c.J - 1 && inside(s_u[n + 1]));
        }
        const uint32_t bits = __ballot_sync(0xffffffffu, in_region);
        if (lane == 0 && ((base >> 5) + warp) < words) s_mask[(base >> 5) + warp] = bits;
      }
      __syncthreads();
      if (warp == 0) {
        int count = 0;
        for (int w0 = 0; w0 < words; w0 += 32) {
          const uint32_t m = (w0 + lane < words) ? s_mask[w0 + lane] : 0u;
          count += __reduce_add_sync(0xffffffffu, __popc(m));
        }
        if (count > 0) {
          // rank = int(u_sel * counts); cell = argmax(cumsum(region) > rank)
          int rank = static_cast<int>(__dmul_rn(s_sel, static_cast<double>(count)));
          int before = 0;
          for (int w0 = 0; w0 < words; w0 += 32) {
            const uint32_t m = (w0 + lane < words) ? s_mask[w0 + lane] : 0u;
            const int pc = __popc(m);
            int incl = pc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int v = __shfl_up_sync(0xffffffffu, incl, o);
              if (lane >= o) incl += v;
            }
            const int excl = before + incl - pc;
            if (pc > 0 && excl <= rank && rank < before + incl) {
              int r = rank - excl;
              uint32_t mm = m;
              while (r-- > 0) mm &= mm - 1;  // drop the lowest set bits
              s_cell = (w0 + lane) * 32 + (__ffs(mm) - 1);
            }
            before += __shfl_sync(0xffffffffu, incl, 31);
          }
        }
      }
      __syncthreads();
    }

    const int cell = s_cell;
    const int ci = cell >= 0 ? cell / c.J : -4, cj = cell >= 0 ? cell - (cell / c.J) * c.J : -4;
    const T *vs = xs + c.nodes;
    T *xd = xout + p * 2 * static_cast<int64_t>(c.nodes);
    uint32_t *qd = qout + p * static_cast<int64_t>(c.nodes);
    bool fin = true;
    for (int g = tid; g < groups; g += blockDim.x) {
      const int n0 = g * G;
      T v[G], z[G], un[G], vn[G];
      uint32_t q[G], qn_out[G];
      VecIO<T, G>::load(vs + n0, v);
      VecIO<T, G>::loadq(qs + n0, q);
#pragma unroll
      for (int e = 0; e < G; ++e) z[e] = T(0);
      if (c.stochastic) {
        if (MODE == 1) {
          const double *zt = z_tape + p * static_cast<int64_t>(c.nodes) + n0;
#pragma unroll
          for (int e = 0; e < G; ++e) z[e] = T(zt[e]);
        } else {
          constexpr int NG = NetNoise<T>::kGroup;
          if (G % NG == 0) {
#pragma unroll
            for (int h = 0; h < G / NG; ++h)
              NetNoise<T>::draw(key, j, t, static_cast<uint32_t>(n0 / NG + h), z + h * NG);
          } else {
#pragma unroll
            for (int e = 0; e < G; ++e) {
              T zz[NG];
              NetNoise<T>::draw(key, j, t, static_cast<uint32_t>((n0 + e) / NG), zz);
              z[e] = zz[(n0 + e) % NG];
            }
          }
        }
      }
#pragma unroll
      for (int e = 0; e < G; ++e) {
        const int n = n0 + e;
        const int i = n / c.J, jj = n - i * c.J;
        const T u = s_u[n];
        // neighbour sum in the reference order: up, down, left, right
        T nb = T(0);
        if (i > 0) nb = A::add(nb, s_u[n - c.J]);
        if (i < c.J - 1) nb = A::add(nb, s_u[n + c.J]);
        if (jj > 0) nb = A::add(nb, s_u[n - 1]);
        if (jj < c.J - 1) nb = A::add(nb, s_u[n + 1]);
        const bool qnew = (i == ci && (jj == cj || jj == cj - 1 || jj == cj + 1)) ||
                          (jj == cj && (i == ci - 1 || i == ci + 1));
        const T psi = (qnew || (q[e] & c.recent_mask)) ? T(c.stim_amp) : T(0);
        const T drive = A::add(A::mul(T(__ldg(fmask + n)), T(c.forcing)), psi);
        const T p3 =
            A::add(A::mul(A::add(A::mul(A::add(A::mul(T(c.a3), u), T(c.a2)), u), T(c.a1)), u),
                   T(c.a0));
        const T t1 = A::add(u, A::mul(dt, A::sub(p3, v[e])));
        const T t2 = A::add(t1, A::mul(dt, A::add(A::mul(T(c.coupling), nb), drive)));
        un[e] = A::add(t2, A::mul(T(c.sig), z[e]));
        vn[e] = A::add(v[e], A::mul(dt, A::add(A::add(A::mul(T(c.b0), u), A::mul(T(c.b1), v[e])),
                                               T(c.b2))));
        fin = fin && finite_val(un[e]) && finite_val(vn[e]);
        qn_out[e] = ((q[e] << 1) | (qnew ? 1u : 0u)) & c.hist_mask;
        s_un[n] = un[e];
      }
      VecIO<T, G>::store(xd + n0, un);
      VecIO<T, G>::store(xd + c.nodes + n0, vn);
      VecIO<T, G>::storeq(qd + n0, qn_out);
    }
    if (!fin) s_bad = 1;
    __syncthreads();

    if (logw) {
      for (int i = tid; i < c.n_obs; i += blockDim.x) {
        const double r = __dsub_rn(y[i], static_cast<double>(s_un[__ldg(obs_idx + i)]));
        s_sq[i] = __dmul_rn(r, r);
      }
      __syncthreads();
      if (warp == 0) {
        // reference order for a filter of N >= 2 particles; fp32 keeps the tree
        const double sum = np_rows_sum(s_sq, c.n_obs, sizeof(T) == 8 && N >= 2, lane);
        if (lane == 0) logw[p] = T(__dmul_rn(c.obs_coef, sum));
      }
    }
    if (tid == 0 && s_bad) atomicOr(status + f, PF_ST_DIVERGED);
    __syncthreads();
  }
}

// Reference rows (n, (2 + hold) * nodes) fp64 <-> device planes + bits.
template <typename T>
__global__ void fhnnet_pack_kernel(const double *__restrict__ rows, int64_t n, int nodes,
                                   int hold, T *__restrict__ x, uint32_t *__restrict__ q) {
  const int64_t dim = static_cast<int64_t>(2 + hold) * nodes;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
       e < n * nodes; e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t p = e / nodes;
    const int node = static_cast<int>(e - p * nodes);
    const double *r = rows + p * dim;
    x[p * 2 * nodes + node] = T(r[node]);
    x[p * 2 * nodes + nodes + node] = T(r[nodes + node]);
    uint32_t bits = 0;
    for (int k = 0; k < hold; ++k) bits |= (r[(2 + k) * static_cast<int64_t>(nodes) + node] != 0.0 ? 1u : 0u) << k;
    q[p * nodes + node] = bits;
  }
}

template <typename T>
__global__ void fhnnet_unpack_kernel(const T *__restrict__ x, const uint32_t *__restrict__ q,
                                     const int32_t *__restrict__ anc, int64_t n, int nodes,
                                     int hold, double *__restrict__ rows) {
  const int64_t dim = static_cast<int64_t>(2 + hold) * nodes;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
       e < n * nodes; e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t p = e / nodes;
    const int node = static_cast<int>(e - p * nodes);
    const int64_t s = anc ? static_cast<int64_t>(anc[p]) : p;
    double *r = rows + p * dim;
    r[node] = static_cast<double>(x[s * 2 * nodes + node]);
    r[nodes + node] = static_cast<double>(x[s * 2 * nodes + nodes + node]);
    const uint32_t bits = q[s * nodes + node];
    for (int k = 0; k < hold; ++k)
      r[(2 + k) * static_cast<int64_t>(nodes) + node] = ((bits >> k) & 1u) ? 1.0 : 0.0;
  }
}

// Posterior mean of the history indicators over the resampled set:
// est[f*stride + k*nodes + node] = (1/N) * #{j : bit k of q[anc[f*N+j]][node]}.
__global__ void __launch_bounds__(256) bits_estimate_kernel(
    const uint32_t *__restrict__ q, int nodes, int nbits, const int32_t *__restrict__ anc,
    int32_t N, double invN, double *__restrict__ est, int64_t stride) {
  const int64_t f = blockIdx.x;
  const int node = blockIdx.y * blockDim.x + threadIdx.x;
  if (node >= nodes) return;
  uint32_t cnt[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) cnt[k] = 0;
  const int32_t *a = anc + f * N;
  for (int jj = 0; jj < N; ++jj) {
    const uint32_t b = __ldg(q + static_cast<int64_t>(__ldg(a + jj)) * nodes + node);
    if (b) {
#pragma unroll
      for (int k = 0; k < 32; ++k) cnt[k] += (b >> k) & 1u;
    }
  }
  double *e = est + f * stride;
#pragma unroll
  for (int k = 0; k < 32; ++k)
    if (k < nbits) e[static_cast<int64_t>(k) * nodes + node] = __dmul_rn(double(cnt[k]), invN);
}

// ---- fp32 production kernel: particle rows streamed by bulk copies ---------
// Warp-specialised: one producer warp streams each particle's gathered
// ancestor rows (U|V 8 B/node, history 4 B/node) into an S-stage shared
// ring with cp.async.bulk (completion on full[s]) and publishes the
// particle's per-step scalars with it (filter, index, Philox key, stimulus
// draws); CW compute warps walk the same particle sequence
// p = blockIdx.x + i*gridDim.x and release the stage through empty[s] (one
// arrival per warp) - no CTA-wide barrier on the common path.  Each compute
// thread owns the same 4-node group of every particle, so its lattice
// position, boundary flags, forcing term and observation bits are computed
// once per launch and live in registers.  Results leave as 16-B stores from
// registers; the zone likelihood is summed per warp and the last warp to
// finish a particle combines the partials in warp order (deterministic).
struct NetMeta {
  int64_t p, f;
  uint32_t j, fire;
  uint32_t k0, k1;
  double sel;
};

// NF: noise-free transition (transition_point_prediction, fhn.py:191-197): no
// new stimulus, zero increments, no draws.
// bulk-copy ring depth of the fast kernel; `net` workload ms per interval
// (propagate kernel), A/B on one box: 2 stages 1.283, 3 stages 1.272,
// 4 stages 1.372, 5 stages 1.500 (the ring's shared memory comes out of L1)
#ifndef PF_NET_STAGES
#define PF_NET_STAGES 3
#endif
template <int CW, int S, bool NF = false>
__global__ void __launch_bounds__((CW + 1) * 32, CW >= 8 ? 4 : CW >= 4 ? 6 : CW >= 2 ? 8 : 12) fhnnet_fast_kernel(
    const float *__restrict__ xin, const uint32_t *__restrict__ qin,
    const int32_t *__restrict__ anc, float *__restrict__ xout, uint32_t *__restrict__ qout,
    const double *__restrict__ fmask, const double *__restrict__ y,
    const int32_t *__restrict__ obs_idx, float *__restrict__ logw, int64_t MN, int32_t N,
    NetConsts c, const uint32_t *__restrict__ keys, uint32_t t, uint32_t *__restrict__ status) {
  using A = Ar<float>;
  constexpr int kCompute = CW * 32;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int nodes = c.nodes;
  const uint32_t stage_bytes = static_cast<uint32_t>(nodes) * 12u;
  double *s_y = reinterpret_cast<double *>(smem_raw + S * stage_bytes);  // y at observed nodes
  uint32_t *s_mask = reinterpret_cast<uint32_t *>(s_y + nodes);        // stimulus region bits
  __shared__ __align__(8) uint64_t full[S], empty[S];
  __shared__ NetMeta meta[S];
  __shared__ double s_part[S][CW];
  __shared__ int s_cnt[S];
  __shared__ int s_cell;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int words = (nodes + 31) >> 5;
  const int groups = nodes >> 2;
  const int J = c.J;

  if (tid == 0) {
    for (int k = 0; k < S; ++k) {
      mbar_init(&full[k], 1);
      mbar_init(&empty[k], CW);
      s_cnt[k] = 0;
    }
    mbar_fence_init();
  }
  if (logw)
    for (int i = tid; i < c.n_obs; i += blockDim.x) s_y[__ldg(obs_idx + i)] = y[i];
  __syncthreads();

  const int64_t first = blockIdx.x, stride = gridDim.x;
  const int64_t count = first < MN ? (MN - 1 - first) / stride + 1 : 0;

  if (warp == CW) {  // ---- producer warp
    if (lane == 0) {
      for (int64_t i = 0; i < count; ++i) {
        const int k = static_cast<int>(i % S);
        if (i >= S) mbar_wait(&empty[k], static_cast<uint32_t>(((i / S) - 1) & 1));
        const int64_t p = first + i * stride;
        const int64_t f = p / N;
        const uint32_t j = static_cast<uint32_t>(p - f * N);
        NetMeta &m = meta[k];
        m.p = p;
        m.f = f;
        m.j = j;
        if (NF) {
          m.fire = 0;
          m.sel = 0.0;
          m.k0 = m.k1 = 0u;
        } else {
          const Key2 key = load_key(keys, f);
          // stimulus draws (fhn.py:158-159): fire, then cell select
          const uint4 r = philox10(make_uint4(j, t, 0u, kPurposeNetStim), key);
          m.fire = u53_closed0(r.x, r.y) < c.stim_prob;
          m.sel = u53_closed0(r.z, r.w);
          m.k0 = key.k0;
          m.k1 = key.k1;
        }
        const int64_t src = anc ? static_cast<int64_t>(__ldg(anc + p)) : p;
        unsigned char *st = smem_raw + k * stage_bytes;
        mbar_arrive_expect_tx(&full[k], stage_bytes);  // release: meta visible with the data
        bulk_g2s(st, xin + src * 2 * static_cast<int64_t>(nodes), 8u * nodes, &full[k]);
        bulk_g2s(st + 8 * nodes, qin + src * static_cast<int64_t>(nodes), 4u * nodes,
                 &full[k]);
      }
    }
    return;
  }

  // ---- compute warps: loop-invariant per-thread geometry
  const int g = tid;  // node group (4 nodes, one lattice row)
  const bool active = g < groups;
  const int n0 = 4 * (active ? g : 0);
  const int r = n0 / J, c0 = n0 - r * J;
  const bool has_up = r > 0, has_dn = r < J - 1, has_l = c0 > 0, has_r = c0 + 4 < J;
  float drv[4];
#pragma unroll
  for (int e = 0; e < 4; ++e)
    drv[e] = active ? A::mul(float(__ldg(fmask + n0 + e)), float(c.forcing)) : 0.f;
  uint32_t obits = 0;
  if (logw && active)
    for (int i = 0; i < c.n_obs; ++i) {
      const int o = __ldg(obs_idx + i) - n0;
      if (o >= 0 && o < 4) obits |= 1u << o;
    }
  const float dt = float(c.dt), fa3 = float(c.a3), fa2 = float(c.a2), fa1 = float(c.a1),
              fa0 = float(c.a0), fb0 = float(c.b0), fb1 = float(c.b1), fb2 = float(c.b2),
              fcpl = float(c.coupling), famp = float(c.stim_amp);
  const float fsig = float(c.sig) * kSqrt2Ln2;  // normals from box_muller_fast_unscaled

  for (int64_t i = 0; i < count; ++i) {
    const int k = static_cast<int>(i % S);
    mbar_wait(&full[k], static_cast<uint32_t>((i / S) & 1));
    const NetMeta m = meta[k];
    const float *su = reinterpret_cast<const float *>(smem_raw + k * stage_bytes);
    const float *sv = su + nodes;
    const uint32_t *sq = reinterpret_cast<const uint32_t *>(su + 2 * nodes);

    int ci = -4, cj = -4;
    if (m.fire) {  // uniform over the compute warps, rare: named barrier 1
      const float lo = float(c.u_minus), hi = float(c.u_plus);
      auto inside = [&](float u) { return u > lo && u < hi; };
      for (int base = 0; base < nodes; base += kCompute) {
        const int n = base + tid;
        bool in_region = false;
        if (n < nodes) {
          const int rr = n / J, cc = n - rr * J;
          in_region = inside(su[n]) || (rr > 0 && inside(su[n - J])) ||
                      (rr < J - 1 && inside(su[n + J])) || (cc > 0 && inside(su[n - 1])) ||
                      (cc < J - 1 && inside(su[n + 1]));
        }
        const uint32_t bits = __ballot_sync(0xffffffffu, in_region);
        if (lane == 0 && (base >> 5) + warp < words) s_mask[(base >> 5) + warp] = bits;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kCompute) : "memory");
      if (warp == 0) {
        int cnt = 0;
        for (int w0 = 0; w0 < words; w0 += 32)
          cnt += __reduce_add_sync(0xffffffffu,
                                   __popc(w0 + lane < words ? s_mask[w0 + lane] : 0u));
        int found = -1;
        if (cnt > 0) {
          const int rank = static_cast<int>(__dmul_rn(m.sel, static_cast<double>(cnt)));
          int before = 0;
          for (int w0 = 0; w0 < words; w0 += 32) {
            const uint32_t mw = w0 + lane < words ? s_mask[w0 + lane] : 0u;
            const int pc = __popc(mw);
            int incl = pc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int v = __shfl_up_sync(0xffffffffu, incl, o);
              if (lane >= o) incl += v;
            }
            if (pc > 0 && before + incl - pc <= rank && rank < before + incl) {
              uint32_t mm = mw;
              for (int q = rank - (before + incl - pc); q > 0; --q) mm &= mm - 1;
              found = (w0 + lane) * 32 + (__ffs(mm) - 1);
            }
            before += __shfl_sync(0xffffffffu, incl, 31);
          }
          found = __reduce_max_sync(0xffffffffu, found);
        }
        if (lane == 0) s_cell = found;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kCompute) : "memory");
      const int cell = s_cell;  // rewritten only after another bar.sync 1
      if (cell >= 0) {
        ci = cell / J;
        cj = cell - ci * J;
      }
    }

    double part = 0.0;
    if (active) {
      const float4 u4 = *reinterpret_cast<const float4 *>(su + n0);
      const float4 v4 = *reinterpret_cast<const float4 *>(sv + n0);
      const uint4 q4 = *reinterpret_cast<const uint4 *>(sq + n0);
      const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 up = has_up ? *reinterpret_cast<const float4 *>(su + n0 - J) : zero4;
      const float4 dn = has_dn ? *reinterpret_cast<const float4 *>(su + n0 + J) : zero4;
      const float left = has_l ? su[n0 - 1] : 0.f;
      const float right = has_r ? su[n0 + 4] : 0.f;
      float2 za = make_float2(0.f, 0.f), zb = za;
      if (!NF) {
        const uint4 rr = philox10(make_uint4(m.j, t, static_cast<uint32_t>(g), kPurposeNetNoise),
                                  Key2{m.k0, m.k1});
        za = box_muller_fast_unscaled(rr.x, rr.y);
        zb = box_muller_fast_unscaled(rr.z, rr.w);
      }
      const float uu[6] = {left, u4.x, u4.y, u4.z, u4.w, right};
      const float upv[4] = {up.x, up.y, up.z, up.w}, dnv[4] = {dn.x, dn.y, dn.z, dn.w};
      const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
      const float z[4] = {za.x, za.y, zb.x, zb.y};
      const uint32_t qq[4] = {q4.x, q4.y, q4.z, q4.w};
      float un[4], vn[4];
      uint32_t qn[4];
      float big = 0.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int cc = c0 + e;
        const float u = uu[e + 1];
        // reference neighbour order up, down, left, right; a missing
        // neighbour contributes an exact +0 (x + 0 == x)
        const float nb = A::add(A::add(A::add(upv[e], dnv[e]), uu[e]), uu[e + 2]);
        const bool qnew = (r == ci && (cc == cj || cc == cj - 1 || cc == cj + 1)) ||
                          (cc == cj && (r == ci - 1 || r == ci + 1));
        const float psi = (qnew || (qq[e] & c.recent_mask)) ? famp : 0.0f;
        const float drive = A::add(drv[e], psi);
        const float p3 =
            A::add(A::mul(A::add(A::mul(A::add(A::mul(fa3, u), fa2), u), fa1), u), fa0);
        const float t1 = A::add(u, A::mul(dt, A::sub(p3, vv[e])));
        const float t2 = A::add(t1, A::mul(dt, A::add(A::mul(fcpl, nb), drive)));
        un[e] = A::add(t2, A::mul(fsig, z[e]));
        vn[e] = A::add(vv[e], A::mul(dt, A::add(A::add(A::mul(fb0, u), A::mul(fb1, vv[e])), fb2)));
        big = fmaxf(big, fmaxf(fabsf(un[e]), fabsf(vn[e])));
        qn[e] = ((qq[e] << 1) | (qnew ? 1u : 0u)) & c.hist_mask;
      }
      float *xd = xout + m.p * 2 * static_cast<int64_t>(nodes);
      uint32_t *qd = qout + m.p * static_cast<int64_t>(nodes);
      *reinterpret_cast<float4 *>(xd + n0) = make_float4(un[0], un[1], un[2], un[3]);
      *reinterpret_cast<float4 *>(xd + nodes + n0) = make_float4(vn[0], vn[1], vn[2], vn[3]);
      *reinterpret_cast<uint4 *>(qd + n0) = make_uint4(qn[0], qn[1], qn[2], qn[3]);
      // fmaxf drops NaN operands, so test the values themselves too
      if (!(big <= 3.402823466e38f) || un[0] != un[0] || un[1] != un[1] || un[2] != un[2] ||
          un[3] != un[3] || vn[0] != vn[0] || vn[1] != vn[1] || vn[2] != vn[2] ||
          vn[3] != vn[3])
        atomicOr(status + m.f, PF_ST_DIVERGED);
      if (obits) {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (obits & (1u << e)) {
            const double d = s_y[n0 + e] - static_cast<double>(un[e]);
            part = fma(d, d, part);
          }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_down_sync(0xffffffffu, part, o);
    if (lane == 0) {
      if (logw) {
        s_part[k][warp] = part;
        __threadfence_block();
        if (atomicAdd(&s_cnt[k], 1) == CW - 1) {  // last warp: combine in warp order
          __threadfence_block();
          double sum = 0.0;
#pragma unroll
          for (int w = 0; w < CW; ++w) sum += s_part[k][w];
          logw[m.p] = static_cast<float>(c.obs_coef * sum);
          s_cnt[k] = 0;
        }
      }
      // this warp is done with stage k - including its s_part / s_cnt slot,
      // so no warp can reach item i+S (same stage) before item i's combine
      // has read and reset them
      mbar_arrive(&empty[k]);
    }
  }
}

template <int CW, int S, bool NF = false>
static int launch_net_fast(const NetConsts &c, const void *x_in, const uint32_t *q_in,
                           const int32_t *anc, void *x_out, uint32_t *q_out, const double *fmask,
                           const double *y, const int32_t *obs_idx, void *logw, int64_t MN,
                           int32_t N, const uint32_t *keys, uint32_t t, uint32_t *status,
                           cudaStream_t s) {
  const size_t smem = static_cast<size_t>(S) * c.nodes * 12 + static_cast<size_t>(c.nodes) * 8 +
                      static_cast<size_t>((c.nodes + 31) / 32) * 4;
  auto kern = fhnnet_fast_kernel<CW, S, NF>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, (CW + 1) * 32, smem);
  if (per_sm < 1) per_sm = 1;
  int sms = kSmCount, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t grid = std::min<int64_t>(MN, static_cast<int64_t>(sms) * per_sm);
  kern<<<static_cast<unsigned>(grid), (CW + 1) * 32, smem, s>>>(
      static_cast<const float *>(x_in), q_in, anc, static_cast<float *>(x_out), q_out, fmask, y,
      obs_idx, static_cast<float *>(logw), MN, N, c, keys, t, status);
  return check_launch("pf_fhnnet_step(fast)");
}

static int net_fast_warps(const NetConsts &c) {
  const int groups = c.nodes / 4;
  return groups <= 32 ? 1 : groups <= 64 ? 2 : groups <= 128 ? 4 : groups <= 256 ? 8 : 0;
}

// The bulk-copy kernel serves fp32 Philox steps on lattices with J % 4 == 0
// and J <= 32 (one 4-node group per compute thread).
// flags & PF_KERNEL_GENERIC (pf_fhnnet_step_ex) forces the generic kernel
// (comparison tests).
static bool net_fast_ok(const NetConsts &c, pf_dtype dtype, bool tape, uint32_t flags) {
  if (dtype != PF_F32 || tape || c.J % 4 != 0 || net_fast_warps(c) == 0)
    return false;
  return !(flags & PF_KERNEL_GENERIC);
}

// Zone log-likelihood of stored rows (fhn.py:199-207), one warp per row:
// out[r] = -0.5/obs_var * sum_i (y[i] - x[r*stride + idx[i]])^2 in the
// reference's order (np_rows_sum).
template <typename T>
__global__ void __launch_bounds__(128) zone_loglik_kernel(const T *__restrict__ x, int64_t n,
                                                          int64_t stride,
                                                          const int32_t *__restrict__ idx,
                                                          int n_obs, const double *__restrict__ y,
                                                          double coef, double *__restrict__ out) {
  extern __shared__ double s_sq_all[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double *s_sq = s_sq_all + static_cast<int64_t>(warp) * n_obs;
  for (int64_t r = blockIdx.x * 4 + warp; r < n; r += static_cast<int64_t>(gridDim.x) * 4) {
    for (int i = lane; i < n_obs; i += 32) {
      const double d = __dsub_rn(y[i], static_cast<double>(x[r * stride + __ldg(idx + i)]));
      s_sq[i] = __dmul_rn(d, d);
    }
    __syncwarp();
    const double sum = np_rows_sum(s_sq, n_obs, n >= 2, lane);
    if (lane == 0) out[r] = __dmul_rn(coef, sum);
    __syncwarp();
  }
}

static NetConsts make_net_consts(const pf_fhnnet_params *p, uint32_t t) {
  NetConsts c;
  c.J = p->J;
  c.nodes = p->J * p->J;
  c.n_obs = p->n_obs;
  c.stochastic = p->stochastic;
  c.hist_mask = p->stim_hold >= 32 ? 0xffffffffu : ((1u << p->stim_hold) - 1u);
  c.recent_mask = (1u << (p->stim_hold - 1)) - 1u;  // Q(t-1) .. Q(t-hold+1)
  c.dt = p->dt;
  c.coupling = p->coupling;
  c.a3 = p->cubic[0];
  c.a2 = p->cubic[1];
  c.a1 = p->cubic[2];
  c.a0 = p->cubic[3];
  c.b0 = p->beta[0];
  c.b1 = p->beta[1];
  c.b2 = p->beta[2];
  c.u_minus = p->u_minus;
  c.u_plus = p->u_plus;
  c.stim_prob = p->stim_prob;
  c.stim_amp = p->stim_amp;
  // forcing_value (fhn.py:149-151): amp if mod(t*dt, period) <= width; np.mod
  // of positive operands is the exact IEEE fmod
  const double s = static_cast<double>(t) * p->dt;
  c.forcing = std::fmod(s, p->forcing_period) <= p->forcing_width ? p->forcing_amp : 0.0;
  c.sig = p->sig_sqdt;
  c.obs_coef = -0.5 / p->obs_var;
  return c;
}

template <typename T, int MODE, int G>
static int launch_net(const NetConsts &c, const void *x_in, const uint32_t *q_in,
                      const int32_t *anc, void *x_out, uint32_t *q_out, const double *fmask,
                      const double *y, const int32_t *obs_idx, void *logw, int64_t MN, int32_t N,
                      const uint32_t *keys, uint32_t t, const double *stim_tape,
                      const double *z_tape, uint32_t *status, cudaStream_t s) {
  const int groups = c.nodes / G;
  const int threads = std::min(256, std::max(32, (groups + 31) / 32 * 32));
  const size_t smem = 2 * static_cast<size_t>(c.nodes) * sizeof(T) +
                      static_cast<size_t>(c.n_obs) * sizeof(double) +
                      static_cast<size_t>((c.nodes + 31) / 32) * sizeof(uint32_t);
  auto kern = fhnnet_step_kernel<T, MODE, G>;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  if (per_sm < 1) per_sm = 1;
  int sms = kSmCount, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t grid = std::min<int64_t>(MN, static_cast<int64_t>(sms) * per_sm);
  kern<<<static_cast<unsigned>(grid), threads, smem, s>>>(
      static_cast<const T *>(x_in), q_in, anc, static_cast<T *>(x_out), q_out, fmask, y, obs_idx,
      static_cast<T *>(logw), MN, N, c, keys, t, stim_tape, z_tape, status);
  return check_launch("pf_fhnnet_step");
}

template <typename T, int MODE>
static int dispatch_vec(const NetConsts &c, const void *x_in, const uint32_t *q_in,
                        const int32_t *anc, void *x_out, uint32_t *q_out, const double *fmask,
                        const double *y, const int32_t *obs_idx, void *logw, int64_t MN,
                        int32_t N, const uint32_t *keys, uint32_t t, const double *stim_tape,
                        const double *z_tape, uint32_t *status, cudaStream_t s) {
  constexpr int GV = sizeof(T) == 4 ? 4 : 2;
  if (c.nodes % GV == 0)
    return launch_net<T, MODE, GV>(c, x_in, q_in, anc, x_out, q_out, fmask, y, obs_idx, logw, MN,
                                   N, keys, t, stim_tape, z_tape, status, s);
  return launch_net<T, MODE, 1>(c, x_in, q_in, anc, x_out, q_out, fmask, y, obs_idx, logw, MN, N,
                                keys, t, stim_tape, z_tape, status, s);
}

}  // namespace pf

using namespace pf;

extern "C" {

int pf_fhnnet_step(const pf_fhnnet_params *p, pf_dtype dtype, const void *x_in,
                   const uint32_t *q_in, const int32_t *anc, void *x_out, uint32_t *q_out,
                   const double *forcing_mask, const double *y, const int32_t *obs_idx,
                   void *logw_out, int64_t M, int64_t N, const uint32_t *keys, uint32_t t,
                   const double *stim_tape, const double *z_tape, uint32_t *status,
                   void *stream) {
  return pf_fhnnet_step_ex(p, dtype, x_in, q_in, anc, x_out, q_out, forcing_mask, y, obs_idx,
                           logw_out, M, N, keys, t, stim_tape, z_tape, status, 0u, stream);
}

int pf_fhnnet_step_ex(const pf_fhnnet_params *p, pf_dtype dtype, const void *x_in,
                      const uint32_t *q_in, const int32_t *anc, void *x_out, uint32_t *q_out,
                      const double *forcing_mask, const double *y, const int32_t *obs_idx,
                      void *logw_out, int64_t M, int64_t N, const uint32_t *keys, uint32_t t,
                      const double *stim_tape, const double *z_tape, uint32_t *status,
                      uint32_t flags, void *stream) {
  PF_REQUIRE(p && x_in && q_in && x_out && q_out && forcing_mask && status,
             "pf_fhnnet_step: null argument");
  PF_REQUIRE(p->J >= 1 && p->stim_hold >= 1 && p->stim_hold <= 32,
             "pf_fhnnet_step: need J >= 1 and 1 <= stim_hold <= 32");
  PF_REQUIRE(M >= 1 && N >= 1 && M * N <= INT32_MAX, "pf_fhnnet_step: bad M, N");
  PF_REQUIRE(!logw_out || (y && obs_idx && p->n_obs >= 1 && p->obs_var > 0),
             "pf_fhnnet_step: likelihood needs y, obs_idx, n_obs >= 1, obs_var > 0");
  PF_REQUIRE(!p->stochastic || (stim_tape ? z_tape != nullptr : (keys && !z_tape)),
             "pf_fhnnet_step: stochastic steps need keys or both tapes");
  const NetConsts c = make_net_consts(p, t);
  const size_t smem = 2 * static_cast<size_t>(c.nodes) * (dtype == PF_F64 ? 8 : 4) +
                      static_cast<size_t>(c.n_obs) * 8 + (c.nodes + 31) / 32 * 4;
  PF_REQUIRE(smem <= 200 * 1024, "pf_fhnnet_step: lattice too large (J=%d)", p->J);
  const cudaStream_t s = as_stream(stream);
  const int64_t MN = M * N;
  const int32_t n32 = static_cast<int32_t>(N);
  const bool tape = p->stochastic && stim_tape;
  if (net_fast_ok(c, dtype, tape, flags)) {
#define PF_NET_FAST(CW)                                                                       \
  return c.stochastic                                                                        \
             ? launch_net_fast<CW, PF_NET_STAGES>(c, x_in, q_in, anc, x_out, q_out, forcing_mask, y,      \
                                      obs_idx, logw_out, MN, n32, keys, t, status, s)        \
             : launch_net_fast<CW, PF_NET_STAGES, true>(c, x_in, q_in, anc, x_out, q_out, forcing_mask, y, \
                                            obs_idx, logw_out, MN, n32, keys, t, status, s)
    switch (net_fast_warps(c)) {
      case 1: PF_NET_FAST(1);
      case 2: PF_NET_FAST(2);
      case 4: PF_NET_FAST(4);
      default: PF_NET_FAST(8);
    }
#undef PF_NET_FAST
  }
  if (dtype == PF_F64)
    return tape ? dispatch_vec<double, 1>(c, x_in, q_in, anc, x_out, q_out, forcing_mask, y,
                                          obs_idx, logw_out, MN, n32, keys, t, stim_tape, z_tape,
                                          status, s)
                : dispatch_vec<double, 0>(c, x_in, q_in, anc, x_out, q_out, forcing_mask, y,
                                          obs_idx, logw_out, MN, n32, keys, t, nullptr, nullptr,
                                          status, s);
  return tape ? dispatch_vec<float, 1>(c, x_in, q_in, anc, x_out, q_out, forcing_mask, y, obs_idx,
                                       logw_out, MN, n32, keys, t, stim_tape, z_tape, status, s)
              : dispatch_vec<float, 0>(c, x_in, q_in, anc, x_out, q_out, forcing_mask, y, obs_idx,
                                       logw_out, MN, n32, keys, t, nullptr, nullptr, status, s);
}

int pf_fhnnet_pack(pf_dtype dtype, const double *rows, int64_t n, int32_t nodes, int32_t hold,
                   void *x, uint32_t *q, void *stream) {
  PF_REQUIRE(rows && x && q && n >= 0 && nodes >= 1 && hold >= 1 && hold <= 32,
             "pf_fhnnet_pack: bad arguments");
  if (n == 0) return PF_OK;
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>((n * nodes + 255) / 256, 4096));
  if (dtype == PF_F64)
    fhnnet_pack_kernel<double><<<grid, 256, 0, as_stream(stream)>>>(
        rows, n, nodes, hold, static_cast<double *>(x), q);
  else
    fhnnet_pack_kernel<float><<<grid, 256, 0, as_stream(stream)>>>(
        rows, n, nodes, hold, static_cast<float *>(x), q);
  return check_launch("pf_fhnnet_pack");
}

int pf_fhnnet_unpack(pf_dtype dtype, const void *x, const uint32_t *q, const int32_t *anc,
                     int64_t n, int32_t nodes, int32_t hold, double *rows, void *stream) {
  PF_REQUIRE(rows && x && q && n >= 0 && nodes >= 1 && hold >= 1 && hold <= 32,
             "pf_fhnnet_unpack: bad arguments");
  if (n == 0) return PF_OK;
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>((n * nodes + 255) / 256, 4096));
  if (dtype == PF_F64)
    fhnnet_unpack_kernel<double><<<grid, 256, 0, as_stream(stream)>>>(
        static_cast<const double *>(x), q, anc, n, nodes, hold, rows);
  else
    fhnnet_unpack_kernel<float><<<grid, 256, 0, as_stream(stream)>>>(
        static_cast<const float *>(x), q, anc, n, nodes, hold, rows);
  return check_launch("pf_fhnnet_unpack");
}

int pf_zone_loglik(pf_dtype dtype, const void *x, int64_t n, int64_t row_stride,
                   const int32_t *obs_idx, int32_t n_obs, const double *y, double obs_var,
                   double *out, void *stream) {
  PF_REQUIRE(x && obs_idx && y && out && n >= 0 && n_obs >= 1 && obs_var > 0 &&
                 static_cast<size_t>(n_obs) * 8 * 4 <= 200 * 1024,
             "pf_zone_loglik: bad arguments");
  if (n == 0) return PF_OK;
  const size_t smem = static_cast<size_t>(n_obs) * 8 * 4;
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>((n + 3) / 4, 65535));
  const double coef = -0.5 / obs_var;
  if (dtype == PF_F64) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(zone_loglik_kernel<double>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    zone_loglik_kernel<double><<<grid, 128, smem, as_stream(stream)>>>(
        static_cast<const double *>(x), n, row_stride, obs_idx, n_obs, y, coef, out);
  } else {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(zone_loglik_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem));
    zone_loglik_kernel<float><<<grid, 128, smem, as_stream(stream)>>>(
        static_cast<const float *>(x), n, row_stride, obs_idx, n_obs, y, coef, out);
  }
  return check_launch("pf_zone_loglik");
}

int pf_bits_estimate(const uint32_t *q, int32_t nodes, int32_t nbits, const int32_t *anc,
                     int64_t M, int64_t N, double *est, int64_t est_stride, void *stream) {
  PF_REQUIRE(q && anc && est && nodes >= 1 && nbits >= 1 && nbits <= 32 && M >= 1 && N >= 1 &&
                 M * N <= INT32_MAX && est_stride >= static_cast<int64_t>(nbits) * nodes,
             "pf_bits_estimate: bad arguments");
  const dim3 grid(static_cast<unsigned>(M), static_cast<unsigned>((nodes + 255) / 256));
  bits_estimate_kernel<<<grid, 256, 0, as_stream(stream)>>>(
      q, nodes, nbits, anc, static_cast<int32_t>(N), 1.0 / static_cast<double>(N), est,
      est_stride);
  return check_launch("pf_bits_estimate");
}

}  // extern "C"
