// Stochastic Lorenz-63 bank kernels.
//
//  * pf_lorenz_prior            - bf_init / Lorenz63Model.sample_prior
//                                 (filters.py:87-94, lorenz63.py:42-44)
//  * pf_lorenz_propagate_weight - bf_step propagate + weight
//                                 (filters.py:103-104, lorenz63.py:46-65,
//                                 accel.py:60-102), ancestor gather fused
//                                 into the load (filters.py:111)
//  * pf_op_lorenz_euler_block   - the accel.lorenz_euler_block operator
//
// One thread owns one particle and keeps its 3-vector in registers for all
// n_sub Euler substeps of an observation interval; the only HBM traffic is
// the gathered load (3 values), the store (3 values) and the log-weight.
// Production mode generates the Gaussian increments in-register with
// Philox4x32-10 + Box-Muller; tape mode reads the reference's exact draws.
#include "common.cuh"
#include "philox.cuh"

#include <cstdlib>
#include <cstring>
#include <type_traits>

namespace pf {

struct LorenzConsts {
  double s, r, b, dt, dts, sq, ns, two_obs_var;
  int n_sub;
  float f_dt, f_ndts, f_r, f_nb, f_cz;  // fp32 production constants (host-folded)
  float f_s2;                           // -(2 ln 2) * (sqrt(dt) * noise_scale)^2
};

// One Euler-Maruyama substep in the reference's evaluation order
// (accel.py:73-75).  For double every op rounds once (bit-exact with the
// numpy/numba twins); for float nvcc contracts to FFMA.
template <typename T>
__device__ __forceinline__ void lorenz_substep(T &x1, T &x2, T &x3, T z1, T z2, T z3,
                                               const LorenzConsts &c) {
  using A = Ar<T>;
  const T dt = T(c.dt), dts = T(c.dts), sq = T(c.sq), ns = T(c.ns);
  const T r = T(c.r), b = T(c.b);
  const T n1 = A::add(A::sub(x1, A::mul(dts, A::sub(x1, x2))), A::mul(sq, A::mul(ns, z1)));
  const T n2 = A::add(A::add(x2, A::mul(dt, A::sub(A::sub(A::mul(r, x1), x2), A::mul(x1, x3)))),
                      A::mul(sq, A::mul(ns, z2)));
  const T n3 = A::add(A::add(x3, A::mul(dt, A::sub(A::mul(x1, x2), A::mul(b, x3)))),
                      A::mul(sq, A::mul(ns, z3)));
  x1 = n1;
  x2 = n2;
  x3 = n3;
}

// fp64 production substep (Philox draws, so there is no reference bit pattern
// to reproduce): the fp32 production form in double - fused multiply-adds,
// 11 instead of 23 fp64 operations and a 4- instead of 6-deep dependency
// chain per substep.  Tape (oracle) mode and the L1 operator keep
// lorenz_substep's exact reference order.
__device__ __forceinline__ void lorenz_substep_fma(double &x1, double &x2, double &x3, double z1,
                                                   double z2, double z3, const LorenzConsts &c) {
  const double cz = c.sq * c.ns;
  const double n1 = fma(cz, z1, fma(-c.dts, x1 - x2, x1));
  const double t2 = fma(-x1, x3, fma(c.r, x1, -x2));
  const double n2 = fma(cz, z2, fma(c.dt, t2, x2));
  const double t3 = fma(-c.b, x3, x1 * x2);
  const double n3 = fma(cz, z3, fma(c.dt, t3, x3));
  x1 = n1;
  x2 = n2;
  x3 = n3;
}

// fp32 production substep: constants pre-folded (sq*ns), explicit FFMA.
__device__ __forceinline__ void lorenz_substep_fast(float &x1, float &x2, float &x3, float z1,
                                                    float z2, float z3, float dt, float ndts,
                                                    float r, float nb, float cz) {
  const float n1 = fmaf(cz, z1, fmaf(ndts, x1 - x2, x1));
  const float t2 = fmaf(-x1, x3, fmaf(r, x1, -x2));
  const float n2 = fmaf(cz, z2, fmaf(dt, t2, x2));
  const float t3 = fmaf(nb, x3, x1 * x2);
  const float n3 = fmaf(cz, z3, fmaf(dt, t3, x3));
  x1 = n1;
  x2 = n2;
  x3 = n3;
}

// log-likelihood, lorenz63.py:62-65 (obs_dim 1) / SURVEY §8a-A8 (obs_dim 2)
template <typename T>
__device__ __forceinline__ T lorenz_loglik(T x1, T x3, const double *y, int obs_dim,
                                           double two_obs_var) {
  using A = Ar<T>;
  if (obs_dim == 1) {
    const T r0 = A::sub(T(y[0]), x1);
    return -A::mul(r0, r0) / T(two_obs_var);
  }
  const T r0 = A::sub(T(y[0]), x1);
  const T r1 = A::sub(T(y[1]), x3);
  return -A::add(A::mul(r0, r0), A::mul(r1, r1)) / T(two_obs_var);
}

template <typename T>
__global__ void lorenz_prior_kernel(T *__restrict__ x, int64_t MN, int32_t N, double m0,
                                    double m1, double m2, double sd,
                                    const uint32_t *__restrict__ keys,
                                    const double *__restrict__ tape) {
  const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (p >= MN) return;
  double z0, z1, z2;
  if (tape) {
    z0 = tape[p * 3 + 0];
    z1 = tape[p * 3 + 1];
    z2 = tape[p * 3 + 2];
  } else {
    const int64_t f = p / N;
    const uint32_t j = static_cast<uint32_t>(p - f * N);
    const Key2 key = load_key(keys, f);
    const uint4 a = philox10(make_uint4(j, 0u, 0u, kPurposePrior), key);
    const uint4 b = philox10(make_uint4(j, 0u, 1u, kPurposePrior), key);
    const double2 g0 = box_muller_f64(a.x, a.y, a.z, a.w);
    const double2 g1 = box_muller_f64(b.x, b.y, b.z, b.w);
    z0 = g0.x;
    z1 = g0.y;
    z2 = g1.x;
  }
  // mean + sqrt(var) * z  (lorenz63.py:44), one rounding per op
  x[p] = static_cast<T>(__dadd_rn(m0, __dmul_rn(sd, z0)));
  x[MN + p] = static_cast<T>(__dadd_rn(m1, __dmul_rn(sd, z1)));
  x[2 * MN + p] = static_cast<T>(__dadd_rn(m2, __dmul_rn(sd, z2)));
}

// ---- propagate + weight -------------------------------------------------
// MODE 0: Philox; MODE 1: tape (M, n_sub, N, 3) fp64.
template <typename T, int MODE>
__global__ void __launch_bounds__(256) lorenz_pw_kernel(
    const T *__restrict__ xin, const int32_t *__restrict__ anc, T *__restrict__ xout,
    const double *__restrict__ y, T *__restrict__ logw, int64_t MN, int32_t N, int obs_dim,
    LorenzConsts c, const uint32_t *__restrict__ keys, uint32_t t,
    const double *__restrict__ tape, uint32_t *__restrict__ status) {
  const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (p >= MN) return;
  const int64_t src = anc ? static_cast<int64_t>(__ldg(anc + p)) : p;
  T x1 = xin[src], x2 = xin[MN + src], x3 = xin[2 * MN + src];
  const int64_t f = p / N;
  const int32_t j = static_cast<int32_t>(p - f * N);

  if (MODE == 1) {
    const double *z = tape + (f * c.n_sub * static_cast<int64_t>(N) + j) * 3;
    const int64_t kstride = static_cast<int64_t>(N) * 3;
    for (int k = 0; k < c.n_sub; ++k) {
      const double *zk = z + k * kstride;
      lorenz_substep<T>(x1, x2, x3, T(zk[0]), T(zk[1]), T(zk[2]), c);
    }
  } else {
    // fp64 Philox: 2 substeps = 6 normals = 3 Philox blocks (fp64 Box-Muller)
    const Key2 key = load_key(keys, f);
    for (int k0 = 0; k0 < c.n_sub; k0 += 2) {
      double z[6];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const uint4 rr = philox10(
            make_uint4(static_cast<uint32_t>(j), t, static_cast<uint32_t>((k0 >> 1) * 3 + q),
                       kPurposeLorenz),
            key);
        const double2 g = box_muller_f64(rr.x, rr.y, rr.z, rr.w);
        z[2 * q] = g.x;
        z[2 * q + 1] = g.y;
      }
      if constexpr (std::is_same<T, double>::value) {
        lorenz_substep_fma(x1, x2, x3, z[0], z[1], z[2], c);
        if (k0 + 1 < c.n_sub) lorenz_substep_fma(x1, x2, x3, z[3], z[4], z[5], c);
      } else {
        lorenz_substep<T>(x1, x2, x3, T(z[0]), T(z[1]), T(z[2]), c);
        if (k0 + 1 < c.n_sub) lorenz_substep<T>(x1, x2, x3, T(z[3]), T(z[4]), T(z[5]), c);
      }
    }
  }

  if (!(finite_val(x1) && finite_val(x2) && finite_val(x3)))
    atomicOr(status + f, PF_ST_DIVERGED);
  xout[p] = x1;
  xout[MN + p] = x2;
  xout[2 * MN + p] = x3;
  logw[p] = lorenz_loglik<T>(x1, x3, y, obs_dim, c.two_obs_var);
}

// fp32 production kernel (Philox): constants host-folded, unpredicated
// 4-substep chunks (12 normals = 3 Philox blocks = 6 Box-Muller pairs).  The
// noise scale is folded into each pair's radius (cz*z = r'*cos with
// r' = sqrt(-log2(u) * 2 ln2 * cz^2)), so an increment costs one FFMA.
// UKEY: every block lies inside one filter (N % 256 == 0), so the filter id,
// its Philox key and the key schedule are block-uniform (uniform registers);
// same draws and arithmetic as UKEY=false.
template <bool UKEY>
__global__ void __launch_bounds__(256) lorenz_fast_kernel(
    const float *__restrict__ xin, const int32_t *__restrict__ anc, float *__restrict__ xout,
    const double *__restrict__ y, float *__restrict__ logw, int64_t MN, int32_t N, int obs_dim,
    LorenzConsts c, const uint32_t *__restrict__ keys, uint32_t t,
    uint32_t *__restrict__ status) {
  int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const bool live = p < MN;
  if (!UKEY && !live) p = MN - 1;  // tail: recompute the last particle, no store
  const int64_t f = UKEY ? (static_cast<int64_t>(blockIdx.x) * 256) / N : p / N;
  const uint32_t j = static_cast<uint32_t>(p - f * N);
  const Key2 key = load_key(keys, f);
  // counter (t, draw index, particle, purpose): only the uniform draw index
  // changes inside the loop, rounds 1-3 are mostly hoisted (philox10_t)
  const PhiloxPreT pre = philox_pre_t(t, j, kPurposeLorenz, key);
  const PhiloxUni uni = philox_uni_t(t, kPurposeLorenz, key);
  const PhiloxKeys rk = philox_round_keys(key);
  const int64_t src = anc ? static_cast<int64_t>(__ldg(anc + p)) : p;
  float x1 = xin[src], x2 = xin[MN + src], x3 = xin[2 * MN + src];
  const float dt = c.f_dt, ndts = c.f_ndts, r = c.f_r, nb = c.f_nb, s2 = c.f_s2;
  // Software-pipelined chunks of 4 substeps: the Philox blocks of chunk k+1
  // are generated in the same basic block as chunk k's Box-Muller transforms
  // (MUFU-heavy) and Euler steps (FFMA), so the integer, XU and FMA work
  // interleave instead of arriving in bursts.
  const int nch = (c.n_sub + 3) >> 2;
  auto draws = [&](int k4, uint4 *rr) {
#pragma unroll
    for (int q = 0; q < 3; ++q)
      rr[q] = philox10_t(pre, uni, static_cast<uint32_t>(k4 * 3 + q) ^ key.k0, rk);
  };
  auto chunk = [&](const uint4 *rr, int left) {
    float rad[6], tr[12];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      box_muller_rad_trig(rr[q].x, rr[q].y, s2, rad[2 * q], tr[4 * q], tr[4 * q + 1]);
      box_muller_rad_trig(rr[q].z, rr[q].w, s2, rad[2 * q + 1], tr[4 * q + 2], tr[4 * q + 3]);
    }
    auto sub = [&](int n0) {  // normals n0..n0+2: pair n/2, trig factor n
      const float n1 = fmaf(rad[n0 >> 1], tr[n0], fmaf(ndts, x1 - x2, x1));
      const float t2 = fmaf(-x1, x3, fmaf(r, x1, -x2));
      const float m2 = fmaf(rad[(n0 + 1) >> 1], tr[n0 + 1], fmaf(dt, t2, x2));
      const float t3 = fmaf(nb, x3, x1 * x2);
      const float m3 = fmaf(rad[(n0 + 2) >> 1], tr[n0 + 2], fmaf(dt, t3, x3));
      x1 = n1;
      x2 = m2;
      x3 = m3;
    };
    if (left >= 4) {
#pragma unroll
      for (int q = 0; q < 4; ++q) sub(3 * q);
    } else {
#pragma unroll
      for (int q = 0; q < 3; ++q)
        if (q < left) sub(3 * q);
    }
  };
  if (nch > 0) {
    // two draw buffers in ping-pong (the loop is unrolled by two chunks, so
    // no register copies between chunks); only the last chunk can be partial
    uint4 ra[3], rb[3];
    draws(0, ra);
    int k4 = 0;
    for (; k4 + 2 < nch; k4 += 2) {
      draws(k4 + 1, rb);
      chunk(ra, 4);
      draws(k4 + 2, ra);
      chunk(rb, 4);
    }
    const int last = c.n_sub - 4 * (nch - 1);
    if (k4 + 1 < nch) {
      draws(k4 + 1, rb);
      chunk(ra, 4);
      chunk(rb, last);
    } else {
      chunk(ra, last);
    }
  }
  if (!live) return;
  if (!(isfinite(x1) && isfinite(x2) && isfinite(x3))) atomicOr(status + f, PF_ST_DIVERGED);
  xout[p] = x1;
  xout[MN + p] = x2;
  xout[2 * MN + p] = x3;
  logw[p] = lorenz_loglik<float>(x1, x3, y, obs_dim, c.two_obs_var);
}

// Noise-free interval (the auxiliary filter's point prediction,
// lorenz63.py:57-60): the same substep arithmetic with zero increments and no
// draws at all.  FAST=true uses the fp32 production substep (bit-identical
// to lorenz_fast_kernel with zero noise scale: fma(0, z, v) == v), else the
// exact-order substep of lorenz_pw_kernel.
template <typename T, bool FAST>
__global__ void __launch_bounds__(256) lorenz_det_kernel(
    const T *__restrict__ xin, const int32_t *__restrict__ anc, T *__restrict__ xout,
    const double *__restrict__ y, T *__restrict__ logw, int64_t MN, int32_t N, int obs_dim,
    LorenzConsts c, uint32_t *__restrict__ status) {
  const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (p >= MN) return;
  const int64_t src = anc ? static_cast<int64_t>(__ldg(anc + p)) : p;
  T x1 = xin[src], x2 = xin[MN + src], x3 = xin[2 * MN + src];
  for (int k = 0; k < c.n_sub; ++k) {
    if constexpr (FAST)
      lorenz_substep_fast(x1, x2, x3, 0.f, 0.f, 0.f, c.f_dt, c.f_ndts, c.f_r, c.f_nb, c.f_cz);
    else
      lorenz_substep<T>(x1, x2, x3, T(0), T(0), T(0), c);
  }
  if (!(finite_val(x1) && finite_val(x2) && finite_val(x3)))
    atomicOr(status + p / N, PF_ST_DIVERGED);
  xout[p] = x1;
  xout[MN + p] = x2;
  xout[2 * MN + p] = x3;
  logw[p] = lorenz_loglik<T>(x1, x3, y, obs_dim, c.two_obs_var);
}

// fp64 production kernel for SMALL banks (BASELINE cfg0: 4 x 1000 particles):
// a warp per K particles (K = 2 in production).  The Gaussian increments do not depend on the
// state, so the 32 lanes generate a chunk of substeps' normals in parallel
// (same Philox counters and fp64 Box-Muller as lorenz_pw_kernel<double,0>:
// block b of a substep pair yields normals 2b, 2b+1 of the flat sequence)
// into shared memory, and lane 0 runs the exact-order substep chain.  With
// one thread per particle the 4000-particle bank occupied 16 SMs and was
// bound by the serial RNG latency.  Results are bit-identical.
constexpr int kSmallChunk = 64;  // substeps per generated chunk (even)
constexpr int64_t kSmallBank = 1 << 15;  // particles: below this, a warp per particle

// K particles per warp: the lanes generate all K particles' normals of a
// chunk (K * 3 * chunk/2 Philox blocks) and lanes 0..K-1 then run the K
// exact-order chains side by side.  A chain is a serial sequence of fp64
// warp instructions; with one particle per warp each of them occupied the
// fp64 pipe for a whole warp slot while 31 lanes idled (ncu: fp64 pipe 67 %
// busy, the chain 55 % of the instructions), so K chains per warp divide
// that cost by K while the generation stays fully parallel.
template <int K>
__global__ void __launch_bounds__(32 * (8 / K)) lorenz_small_kernel(
    const double *__restrict__ xin, const int32_t *__restrict__ anc, double *__restrict__ xout,
    const double *__restrict__ y, double *__restrict__ logw, int64_t MN, int32_t N, int obs_dim,
    LorenzConsts c, const uint32_t *__restrict__ keys, uint32_t t,
    uint32_t *__restrict__ status) {
  constexpr int W = 8 / K;  // warps per block (shared memory: K * 8 chunk buffers)
  __shared__ double s_z[W][K][3 * kSmallChunk];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t p0 = (blockIdx.x * static_cast<int64_t>(W) + w) * K;
  if (p0 >= MN) return;
  // this lane's chain (lanes 0..K-1) and its particle
  const int64_t p = p0 + lane;
  const bool chain = lane < K && p < MN;
  double x1 = 0.0, x2 = 0.0, x3 = 0.0;
  if (chain) {
    const int64_t src = anc ? static_cast<int64_t>(__ldg(anc + p)) : p;
    x1 = xin[src];
    x2 = xin[MN + src];
    x3 = xin[2 * MN + src];
  }
  for (int k0 = 0; k0 < c.n_sub; k0 += kSmallChunk) {
    const int nk = c.n_sub - k0 < kSmallChunk ? c.n_sub - k0 : kSmallChunk;
    const int nblocks = ((nk + 1) / 2) * 3;  // 3 Philox blocks per substep pair
    __syncwarp();
    for (int bb = lane; bb < K * nblocks; bb += 32) {
      const int kk = bb / nblocks, b = bb - kk * nblocks;
      const int64_t q = p0 + kk;
      if (q >= MN) continue;
      const int64_t f = q / N;
      const uint32_t j = static_cast<uint32_t>(q - f * N);
      const uint32_t gb = static_cast<uint32_t>((k0 >> 1) * 3 + b);  // global block index
      const uint4 rr = philox10(make_uint4(j, t, gb, kPurposeLorenz), load_key(keys, f));
      const double2 g = box_muller_f64(rr.x, rr.y, rr.z, rr.w);
      s_z[w][kk][2 * b] = g.x;
      s_z[w][kk][2 * b + 1] = g.y;
    }
    __syncwarp();
    if (chain) {
      const double *z = s_z[w][lane];
      for (int k = 0; k < nk; ++k)
        lorenz_substep_fma(x1, x2, x3, z[3 * k], z[3 * k + 1], z[3 * k + 2], c);
    }
  }
  if (chain) {
    const int64_t f = p / N;
    if (!(finite_val(x1) && finite_val(x2) && finite_val(x3))) atomicOr(status + f, PF_ST_DIVERGED);
    xout[p] = x1;
    xout[MN + p] = x2;
    xout[2 * MN + p] = x3;
    logw[p] = lorenz_loglik<double>(x1, x3, y, obs_dim, c.two_obs_var);
  }
}

// accel.lorenz_euler_block: states (n,3) row-major, noise (n_sub, n, 3)
__global__ void lorenz_block_op_kernel(const double *__restrict__ st,
                                       const double *__restrict__ nz, int64_t n,
                                       LorenzConsts c, double *__restrict__ out) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  double x1 = st[3 * i], x2 = st[3 * i + 1], x3 = st[3 * i + 2];
  for (int k = 0; k < c.n_sub; ++k) {
    const double *z = nz + (k * n + i) * 3;
    lorenz_substep<double>(x1, x2, x3, z[0], z[1], z[2], c);
  }
  out[3 * i] = x1;
  out[3 * i + 1] = x2;
  out[3 * i + 2] = x3;
}

static LorenzConsts make_consts(const pf_lorenz_params *p) {
  LorenzConsts c;
  c.s = p->s;
  c.r = p->r;
  c.b = p->b;
  c.dt = p->dt;
  c.dts = p->dt * p->s;  // (dt * s), accel.py:73
  c.sq = std::sqrt(p->dt);
  c.ns = p->noise_scale;
  c.two_obs_var = 2.0 * p->obs_var;
  c.n_sub = p->n_sub;
  c.f_dt = static_cast<float>(c.dt);
  c.f_ndts = static_cast<float>(-c.dts);
  c.f_r = static_cast<float>(c.r);
  c.f_nb = static_cast<float>(-c.b);
  c.f_cz = static_cast<float>(c.sq * c.ns) * kSqrt2Ln2;
  c.f_s2 = static_cast<float>(-2.0 * std::log(2.0) * (c.sq * c.ns) * (c.sq * c.ns));
  return c;
}

}  // namespace pf

using namespace pf;

extern "C" {

int pf_lorenz_prior(pf_dtype dtype, void *x, int64_t M, int64_t N, const double *mean3_host,
                    double prior_sd, const uint32_t *keys, const double *z_tape,
                    void *stream) {
  PF_REQUIRE(x && mean3_host && M >= 1 && N >= 1, "pf_lorenz_prior: bad arguments");
  PF_REQUIRE(z_tape || keys, "pf_lorenz_prior: need keys (Philox) or z_tape");
  PF_REQUIRE(N <= INT32_MAX && M * N <= INT32_MAX, "pf_lorenz_prior: M*N exceeds int32 range");
  const int64_t MN = M * N;
  const cudaStream_t s = as_stream(stream);
  if (dtype == PF_F64)
    lorenz_prior_kernel<double><<<grid_for(MN, 256), 256, 0, s>>>(
        static_cast<double *>(x), MN, static_cast<int32_t>(N), mean3_host[0], mean3_host[1],
        mean3_host[2], prior_sd, keys, z_tape);
  else
    lorenz_prior_kernel<float><<<grid_for(MN, 256), 256, 0, s>>>(
        static_cast<float *>(x), MN, static_cast<int32_t>(N), mean3_host[0], mean3_host[1],
        mean3_host[2], prior_sd, keys, z_tape);
  return check_launch("pf_lorenz_prior");
}

int pf_lorenz_propagate_weight(const pf_lorenz_params *p, pf_dtype dtype, const void *x_in,
                               const int32_t *anc, void *x_out, const double *y,
                               void *logw_out, int64_t M, int64_t N, const uint32_t *keys,
                               uint32_t t, const double *z_tape, uint32_t *status,
                               void *stream) {
  return pf_lorenz_propagate_weight_ex(p, dtype, x_in, anc, x_out, y, logw_out, M, N, keys, t,
                                       z_tape, status, 0u, stream);
}

// flags & PF_KERNEL_GENERIC keeps one thread per particle for small fp64
// banks too (comparison tests of the warp-per-particle kernel).
int pf_lorenz_propagate_weight_ex(const pf_lorenz_params *p, pf_dtype dtype, const void *x_in,
                                  const int32_t *anc, void *x_out, const double *y,
                                  void *logw_out, int64_t M, int64_t N, const uint32_t *keys,
                                  uint32_t t, const double *z_tape, uint32_t *status,
                                  uint32_t flags, void *stream) {
  PF_REQUIRE(p && x_in && x_out && y && logw_out && status, "pf_lorenz_propagate_weight: null");
  PF_REQUIRE(M >= 1 && N >= 1 && M * N <= INT32_MAX, "pf_lorenz_propagate_weight: bad M/N");
  PF_REQUIRE(p->n_sub >= 0, "substeps must be >= 0");
  PF_REQUIRE(p->obs_dim == 1 || p->obs_dim == 2, "obs_dim must be 1 or 2");
  PF_REQUIRE(z_tape || keys, "need keys (Philox) or z_tape");
  PF_REQUIRE(x_in != x_out, "x_in and x_out must not alias");
  const LorenzConsts c = make_consts(p);
  const int64_t MN = M * N;
  const cudaStream_t s = as_stream(stream);
  const unsigned grid = grid_for(MN, 256);
  const int32_t n32 = static_cast<int32_t>(N);
  if (p->noise_scale == 0.0 && p->n_sub > 0) {  // point prediction: no draws
    if (dtype == PF_F64)
      lorenz_det_kernel<double, false><<<grid, 256, 0, s>>>(
          static_cast<const double *>(x_in), anc, static_cast<double *>(x_out), y,
          static_cast<double *>(logw_out), MN, n32, p->obs_dim, c, status);
    else if (z_tape)
      lorenz_det_kernel<float, false><<<grid, 256, 0, s>>>(
          static_cast<const float *>(x_in), anc, static_cast<float *>(x_out), y,
          static_cast<float *>(logw_out), MN, n32, p->obs_dim, c, status);
    else
      lorenz_det_kernel<float, true><<<grid, 256, 0, s>>>(
          static_cast<const float *>(x_in), anc, static_cast<float *>(x_out), y,
          static_cast<float *>(logw_out), MN, n32, p->obs_dim, c, status);
    return check_launch("pf_lorenz_propagate_weight(noise-free)");
  }
  if (dtype == PF_F64) {
    auto *xi = static_cast<const double *>(x_in);
    auto *xo = static_cast<double *>(x_out);
    auto *lw = static_cast<double *>(logw_out);
    if (z_tape)
      lorenz_pw_kernel<double, 1><<<grid, 256, 0, s>>>(xi, anc, xo, y, lw, MN, n32, p->obs_dim,
                                                       c, keys, t, z_tape, status);
    else if (MN <= kSmallBank && !(flags & PF_KERNEL_GENERIC))
      // two particles per warp: cfg0 propagate 19.8 -> 15.4 us (one: 19.8, four: 15.9)
      lorenz_small_kernel<2><<<grid_for(MN, 8), 128, 0, s>>>(xi, anc, xo, y, lw, MN, n32,
                                                             p->obs_dim, c, keys, t, status);
    else
      lorenz_pw_kernel<double, 0><<<grid, 256, 0, s>>>(xi, anc, xo, y, lw, MN, n32, p->obs_dim,
                                                       c, keys, t, z_tape, status);
  } else {
    auto *xi = static_cast<const float *>(x_in);
    auto *xo = static_cast<float *>(x_out);
    auto *lw = static_cast<float *>(logw_out);
    if (z_tape)
      lorenz_pw_kernel<float, 1><<<grid, 256, 0, s>>>(xi, anc, xo, y, lw, MN, n32, p->obs_dim,
                                                      c, keys, t, z_tape, status);
    else if (N % 256 == 0)  // occupancy 4-8 blocks/SM measured equal (issue-bound)
      lorenz_fast_kernel<true><<<grid, 256, 0, s>>>(xi, anc, xo, y, lw, MN, n32, p->obs_dim, c,
                                                    keys, t, status);
    else
      lorenz_fast_kernel<false><<<grid, 256, 0, s>>>(xi, anc, xo, y, lw, MN, n32, p->obs_dim, c,
                                                     keys, t, status);
  }
  return check_launch("pf_lorenz_propagate_weight");
}

int pf_op_lorenz_euler_block(const double *states, const double *noise, int64_t n,
                             int64_t n_sub, double dt, double s, double r, double b,
                             double *out, void *stream) {
  PF_REQUIRE(states && out && n >= 1 && n_sub >= 0 && (noise || n_sub == 0),
             "pf_op_lorenz_euler_block: bad arguments");
  pf_lorenz_params p{s, r, b, dt, 1.0, 1.0, static_cast<int32_t>(n_sub), 1};
  LorenzConsts c = make_consts(&p);
  lorenz_block_op_kernel<<<grid_for(n, 128), 128, 0, as_stream(stream)>>>(states, noise, n, c,
                                                                           out);
  return check_launch("pf_op_lorenz_euler_block");
}

}  // extern "C"
