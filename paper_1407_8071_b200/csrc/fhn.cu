// FitzHugh-Nagumo lattice kernels.
//
//  * pf_fhn_interval       - one observation interval of the bank: n_sub
//                            lattice Euler steps (accel.py:110-129 per step)
//                            + Gaussian electrode log-likelihood
//                            (fhn.py:199-207), ancestor gather fused into
//                            the load (filters.py:111).
//  * pf_op_fhn_euler_block - the accel.fhn_euler_block operator (fp64).
//
// Design: one CTA owns one particle for the whole interval.
// The lattice (rows x cols, v and w) lives in registers - each thread owns a
// vertical strip of R rows of one column - and v is exchanged through a
// double-buffered shared-memory plane for the 5-point stencil, one barrier
// per Euler step.  HBM sees the particle once per interval (gathered load +
// store), i.e. 50x less traffic than streaming every Euler step, which
// turns the kernel from HBM-bound into issue-bound (RNG dominated).
#include "common.cuh"
#include <type_traits>
#include "bulk.cuh"
#include "philox.cuh"
#include "f32x2.cuh"

namespace pf {

constexpr int kFhnRows = 6;  // rows per thread (even: Philox pairs rows)

struct FhnConsts {
  int rows, cols, n_sub, n_obs, nseg, nodes;
  double dt, coupling, a3, a2, a1, a0, b0, b1, b2, sig_v, sig_w, degree_drive, obs_coef;
};

// One node update in the reference order (accel.py:121-128) plus w-noise.
template <typename T>
__device__ __forceinline__ void fhn_node(T u, T w, T nb, T negdeg, T zv, T zw,
                                         const FhnConsts &c, T &u_new, T &w_new) {
  using A = Ar<T>;
  const T dt = T(c.dt);
  const T p3 = A::add(A::mul(A::add(A::mul(A::add(A::mul(T(c.a3), u), T(c.a2)), u), T(c.a1)), u),
                      T(c.a0));
  const T drive = A::mul(negdeg, u);
  const T t1 = A::add(u, A::mul(dt, A::sub(p3, w)));
  const T t2 = A::add(t1, A::mul(dt, A::add(A::mul(T(c.coupling), nb), drive)));
  u_new = A::add(t2, A::mul(T(c.sig_v), zv));
  const T wn = A::add(w, A::mul(dt, A::add(A::add(A::mul(T(c.b0), u), A::mul(T(c.b1), w)), T(c.b2))));
  w_new = A::add(wn, A::mul(T(c.sig_w), zw));
}

// MODE 0 = Philox, MODE 1 = tape (M, n_sub, 2, N, nodes) fp64.
template <typename T, int MODE>
__global__ void __launch_bounds__(256) fhn_interval_kernel(
    const T *__restrict__ xin, const int32_t *__restrict__ anc, T *__restrict__ xout,
    const double *__restrict__ y, const int32_t *__restrict__ obs_idx, T *__restrict__ logw,
    int64_t MN, int32_t N, FhnConsts c, const uint32_t *__restrict__ keys, uint32_t t,
    const double *__restrict__ tape, uint32_t *__restrict__ status) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *vs = reinterpret_cast<T *>(smem_raw);  // [2][nodes]
  __shared__ double red[8];
  __shared__ int bad;

  const int tid = threadIdx.x;
  const int seg = tid / c.cols;
  const int col = tid - seg * c.cols;
  const bool active = seg < c.nseg;
  const int row0 = seg * kFhnRows;

  for (int64_t p = blockIdx.x; p < MN; p += gridDim.x) {
    const int64_t f = p / N;
    const int32_t j = static_cast<int32_t>(p - f * N);
    const int64_t src = anc ? static_cast<int64_t>(__ldg(anc + p)) : p;
    const T *xs = xin + src * 2 * static_cast<int64_t>(c.nodes);
    if (tid == 0) bad = 0;

    T v[kFhnRows], w[kFhnRows], negdeg[kFhnRows];
#pragma unroll
    for (int r = 0; r < kFhnRows; ++r) {
      const int row = row0 + r;
      v[r] = T(0);
      w[r] = T(0);
      negdeg[r] = T(0);
      if (active && row < c.rows) {
        const int node = row * c.cols + col;
        v[r] = xs[node];
        w[r] = xs[c.nodes + node];
        const int deg = (row > 0) + (row < c.rows - 1) + (col > 0) + (col < c.cols - 1);
        negdeg[r] = T(c.degree_drive * deg);
        vs[node] = v[r];
      }
    }
    __syncthreads();

    Key2 key{0u, 0u};
    if (MODE == 0) key = load_key(keys, f);
    const uint32_t step0 = (t - 1u) * static_cast<uint32_t>(c.n_sub);
    int buf = 0;
    for (int k = 0; k < c.n_sub; ++k) {
      const T *cur = vs + buf * c.nodes;
      T *nxt = vs + (buf ^ 1) * c.nodes;
      if (active) {
        T zv[kFhnRows], zw[kFhnRows];
        if (MODE == 0) {
          // one Philox block = (zv, zw) for a pair of rows of this column
#pragma unroll
          for (int q = 0; q < kFhnRows / 2; ++q) {
            const uint32_t node_pair =
                static_cast<uint32_t>(((row0 >> 1) + q) * c.cols + col);
            const uint4 rr = philox10(make_uint4(static_cast<uint32_t>(j), step0 + k, node_pair,
                                                 kPurposeFhn),
                                      key);
            if (sizeof(T) == 4) {
              // the fast kernel's draw layout, evaluated with accurate
              // libm functions: words (x, y) -> v increments of rows 2q,
              // 2q+1 (cos, sin), words (z, w) -> their w increments
              const float2 gv = box_muller_ref_f32(rr.x, rr.y);
              const float2 gw = box_muller_ref_f32(rr.z, rr.w);
              zv[2 * q] = T(gv.x);
              zv[2 * q + 1] = T(gv.y);
              zw[2 * q] = T(gw.x);
              zw[2 * q + 1] = T(gw.y);
            } else {
              const double2 g0 = box_muller_f64(rr.x, rr.y, rr.z, rr.w);
              const uint4 r2 = philox10(make_uint4(static_cast<uint32_t>(j), step0 + k,
                                                   node_pair | 0x80000000u, kPurposeFhn),
                                        key);
              const double2 g1 = box_muller_f64(r2.x, r2.y, r2.z, r2.w);
              zv[2 * q] = T(g0.x);
              zw[2 * q] = T(g0.y);
              zv[2 * q + 1] = T(g1.x);
              zw[2 * q + 1] = T(g1.y);
            }
          }
        } else {
          const int64_t base =
              ((f * c.n_sub + k) * 2 * static_cast<int64_t>(N) + j) * c.nodes;
          const int64_t wofs = static_cast<int64_t>(N) * c.nodes;
#pragma unroll
          for (int r = 0; r < kFhnRows; ++r) {
            const int row = row0 + r;
            zv[r] = T(0);
            zw[r] = T(0);
            if (row < c.rows) {
              zv[r] = T(tape[base + row * c.cols + col]);
              zw[r] = T(tape[base + wofs + row * c.cols + col]);
            }
          }
        }
        T vn[kFhnRows], wn[kFhnRows];
#pragma unroll
        for (int r = 0; r < kFhnRows; ++r) {
          const int row = row0 + r;
          vn[r] = v[r];
          wn[r] = w[r];
          if (row < c.rows) {
            // neighbour sum in the reference order: up, down, left, right
            T nb = T(0);
            if (row > 0) nb = Ar<T>::add(nb, r > 0 ? v[r - 1] : cur[(row - 1) * c.cols + col]);
            if (row < c.rows - 1)
              nb = Ar<T>::add(nb, r < kFhnRows - 1 ? v[r + 1] : cur[(row + 1) * c.cols + col]);
            if (col > 0) nb = Ar<T>::add(nb, cur[row * c.cols + col - 1]);
            if (col < c.cols - 1) nb = Ar<T>::add(nb, cur[row * c.cols + col + 1]);
            fhn_node<T>(v[r], w[r], nb, negdeg[r], zv[r], zw[r], c, vn[r], wn[r]);
            nxt[row * c.cols + col] = vn[r];
          }
        }
#pragma unroll
        for (int r = 0; r < kFhnRows; ++r) {
          v[r] = vn[r];
          w[r] = wn[r];
        }
      }
      __syncthreads();
      buf ^= 1;
    }

    // ---- epilogue: divergence, store, electrode log-likelihood ----------
    bool fin = true;
    T *xd = xout + p * 2 * static_cast<int64_t>(c.nodes);
#pragma unroll
    for (int r = 0; r < kFhnRows; ++r) {
      const int row = row0 + r;
      if (active && row < c.rows) {
        const int node = row * c.cols + col;
        fin = fin && finite_val(v[r]) && finite_val(w[r]);
        xd[node] = v[r];
        xd[c.nodes + node] = w[r];
      }
    }
    if (!fin) bad = 1;
    const T *fin_v = vs + buf * c.nodes;
    if (tid == 0 && N >= 2) {
      // a filter of N >= 2 particles: np.sum(resid*resid, axis=1) over the
      // column-major fancy-indexed block is a sequential sum (npsum.cuh)
      double res = 0.0;
      for (int i = 0; i < c.n_obs; ++i) {
        const double rsd = __dsub_rn(y[i], double(fin_v[obs_idx[i]]));
        const double sq = __dmul_rn(rsd, rsd);
        res = i == 0 ? sq : __dadd_rn(res, sq);
      }
      red[0] = res;
    } else if (tid < 32 && N < 2) {
      // a single particle: contiguous row, numpy pairwise order for n <= 128
      // (8 strided accumulators, then ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)),
      // then the remainder).
      const int n = c.n_obs;
      const int lane = tid;
      double acc = 0.0;
      const int nblk = n - (n % 8);
      if (n >= 8 && lane < 8) {
        for (int i = lane; i < nblk; i += 8) {
          const double rsd = __dsub_rn(y[i], double(fin_v[obs_idx[i]]));
          const double sq = __dmul_rn(rsd, rsd);
          acc = (i == lane) ? sq : __dadd_rn(acc, sq);
        }
      }
      // combine ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))
      const double o1 = __shfl_down_sync(0xffffffffu, acc, 1);
      const double s01 = __dadd_rn(acc, o1);  // lanes 0,2,4,6 hold pairs
      const double o2 = __shfl_down_sync(0xffffffffu, s01, 2);
      const double s0123 = __dadd_rn(s01, o2);  // lanes 0,4
      const double o4 = __shfl_down_sync(0xffffffffu, s0123, 4);
      if (lane == 0) {
        double res;
        int i;
        if (n >= 8) {
          res = __dadd_rn(s0123, o4);
          i = nblk;
        } else {
          res = 0.0;
          i = 0;
        }
        for (; i < n; ++i) {
          const double rsd = __dsub_rn(y[i], double(fin_v[obs_idx[i]]));
          res = __dadd_rn(res, __dmul_rn(rsd, rsd));
        }
        red[0] = res;
      }
    }
    __syncthreads();
    if (tid == 0) {
      logw[p] = T(__dmul_rn(c.obs_coef, red[0]));
      if (bad) atomicOr(status + f, PF_ST_DIVERGED);
    }
    __syncthreads();
  }
}

// ---- fp32 production kernel (Philox, Neumann Laplacian) --------------------
// Same dynamics, restated for throughput (tolerance-checked, not bit-exact):
//  * shared plane padded with a ghost ring holding the mirrored boundary
//    value ("ghost = self"), so the 5-point stencil has no boundary
//    predicates: coupling*nb - deg*u == coupling*(sum of 4 padded nbrs - 4u)
//    when degree_drive == -coupling (BASELINE cfg3/cfg4);
//  * constants pre-folded into FFMA form; MUFU-approx Box-Muller;
//  * register budget for 4 resident CTAs/SM (32 warps) to hide the
//    dependent Philox/MUFU latencies.
struct FhnFast {
  int rows, cols, n_sub, n_obs, nseg, nodes;
  float a3, a2, a1, a0;       // u + dt*cubic(u) - 4*dt*coupling*u, folded into one cubic
  float dt, dtc, dtc4;        // dt, dt*coupling, 4*dt*coupling
  float wc, uc, c0;           // w' = wc*w + uc*u + c0  (1+dt*b1, dt*b0, dt*b2)
  float sig_v, sig_w;
  double obs_coef;
};

// Lattice geometry is compile-time (ROWS x COLS, R rows per thread) so every
// shared-memory access is base register + immediate.  TAPE=true reads the
// standard normals from an fp64 tape (parity tests of this exact kernel).
// PP particles are advanced together by the same threads (independent
// dependency chains -> more ILP per warp, one barrier per Euler step for
// all PP particles).
// Row pitch of the shared v plane: no ghost columns (edge threads read
// themselves, Neumann "ghost = self"), and chosen so that a warp spanning two
// strips (rows R apart) hits 32 distinct banks: R*W - COLS == 0 (mod 32)
// (30x50, R=6: W = 51).
__host__ __device__ constexpr int fhn_pitch(int cols, int r) {
  for (int w = cols; w < cols + 32; ++w)
    if ((r * w - cols) % 32 == 0) return w;
  return cols;
}

template <int ROWS, int COLS, int R, bool TAPE, int MINB, int PP, bool NF = false>
__global__ void __launch_bounds__(256, MINB) fhn_fast_kernel(
    const float *__restrict__ xin, const int32_t *__restrict__ anc, float *__restrict__ xout,
    const double *__restrict__ y, const int32_t *__restrict__ obs_idx, float *__restrict__ logw,
    int64_t MN, int32_t N, FhnFast c, const uint32_t *__restrict__ keys, uint32_t t,
    const double *__restrict__ tape, uint32_t *__restrict__ status) {
  constexpr int W = fhn_pitch(COLS, R);
  constexpr int P = (ROWS + 2) * W;  // + a spare row above and below
  constexpr int NSEG = (ROWS + R - 1) / R;
  constexpr int NODES = ROWS * COLS;
  static_assert(R % 2 == 0, "rows per thread must be even (Philox row pairs)");
  extern __shared__ __align__(16) float vsp[];  // [PP][2][P]
  __shared__ double red[PP];
  __shared__ int bad[PP];
  const int tid = threadIdx.x;
  const int seg = tid / COLS;
  const int col = tid - seg * COLS;
  const bool active = seg < NSEG;
  const int row0 = seg * R;
  // horizontal neighbours; an edge column reads itself (ghost = self)
  const int lo = col == 0 ? 0 : -1;
  const int ro = col == COLS - 1 ? 0 : 1;
  const int base = (row0 + 1) * W + col;  // this thread's first cell

  for (int64_t pb = static_cast<int64_t>(blockIdx.x) * PP; pb < MN;
       pb += static_cast<int64_t>(gridDim.x) * PP) {
    float v[PP][R], w[PP][R];
    int64_t fe[PP];
    uint32_t je[PP];
    Key2 key[PP];
#pragma unroll
    for (int e = 0; e < PP; ++e) {
      const int64_t p = pb + e < MN ? pb + e : MN - 1;  // tail: recompute the last (no store)
      fe[e] = p / N;
      je[e] = static_cast<uint32_t>(p - fe[e] * N);
      const int64_t src = anc ? static_cast<int64_t>(__ldg(anc + p)) : p;
      const float *xs = xin + src * 2 * static_cast<int64_t>(NODES);
      if (tid == 0) bad[e] = 0;
      key[e] = Key2{0u, 0u};
      if (!TAPE && !NF) key[e] = load_key(keys, fe[e]);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        v[e][r] = 0.f;
        w[e][r] = 0.f;
        if (active && row0 + r < ROWS) {
          const int node = (row0 + r) * COLS + col;
          v[e][r] = __ldg(xs + node);
          w[e][r] = __ldg(xs + NODES + node);
          vsp[e * 2 * P + base + r * W] = v[e][r];
        }
      }
    }
    __syncthreads();

    // Philox: the per-thread, step-independent part of each row pair's
    // counter (je, step, node_pair, purpose) is hoisted out of the Euler
    // loop (philox_pre_t); each pair's two Box-Muller draws give the v
    // increments of rows 2q, 2q+1 (radius scaled by sig_v) and the w
    // increments (radius scaled by sig_w): one FFMA per increment.
    const float s2v = -1.3862943611198906f * c.sig_v * c.sig_v;
    const float s2w = -1.3862943611198906f * c.sig_w * c.sig_w;
    PhiloxPreT pre[PP][R / 2];
    PhiloxUni uni[PP];
    PhiloxKeys rk[PP];
    if (!TAPE && !NF) {
#pragma unroll
      for (int e = 0; e < PP; ++e) {
        uni[e] = philox_uni_t(je[e], kPurposeFhn, key[e]);
        rk[e] = philox_round_keys(key[e]);
#pragma unroll
        for (int q = 0; q < R / 2; ++q)
          pre[e][q] = philox_pre_t(je[e], static_cast<uint32_t>(((row0 >> 1) + q) * COLS + col),
                                   kPurposeFhn, key[e]);
      }
    }
    const uint32_t step0 = (t - 1u) * static_cast<uint32_t>(c.n_sub);
    // one Euler step from plane PAR to plane PAR^1 (parity static: every
    // shared address is base + immediate)
    auto euler = [&](int k, auto par_c) {
      constexpr int PAR = decltype(par_c)::value;
      if (active) {
#pragma unroll
        for (int e = 0; e < PP; ++e) {
          const float *cur = vsp + e * 2 * P + PAR * P + base;
          float *nxt = vsp + e * 2 * P + (PAR ^ 1) * P + base;
          // old value of the row above this strip (the top row: itself)
          float up = row0 == 0 ? v[e][0] : cur[-W];
          const uint32_t c1k0 = (step0 + k) ^ key[e].k0;
#pragma unroll
          for (int q = 0; q < R / 2; ++q) {
            // v increment of row 2q+h = av * tv[h], w increment = aw * tw[h]
            float av, aw, tv[2], tw[2];
            if (TAPE) {
              const int64_t b0 =
                  ((fe[e] * c.n_sub + k) * 2 * static_cast<int64_t>(N) + je[e]) * NODES +
                  (row0 + 2 * q) * COLS + col;
              const int64_t wo = static_cast<int64_t>(N) * NODES;
              const bool ok1 = row0 + 2 * q + 1 < ROWS;
              av = c.sig_v;
              aw = c.sig_w;
              tv[0] = float(tape[b0]);
              tw[0] = float(tape[b0 + wo]);
              tv[1] = ok1 ? float(tape[b0 + COLS]) : 0.f;
              tw[1] = ok1 ? float(tape[b0 + wo + COLS]) : 0.f;
            } else if (NF) {  // noise-free lookahead: no draws (0 * 0 adds an exact 0)
              av = aw = tv[0] = tv[1] = tw[0] = tw[1] = 0.f;
            } else {
              const uint4 rr = philox10_t(pre[e][q], uni[e], c1k0, rk[e]);
              box_muller_rad_trig(rr.x, rr.y, s2v, av, tv[0], tv[1]);
              box_muller_rad_trig(rr.z, rr.w, s2w, aw, tw[0], tw[1]);
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int r = 2 * q + h;
              if (row0 + r < ROWS) {
                const float *cell = cur + r * W;
                const float u = v[e][r];
                const float dn = row0 + r == ROWS - 1 ? u : (r < R - 1 ? v[e][r + 1] : cell[W]);
                const float nb = ((up + dn) + cell[lo]) + cell[ro];
                // u + dt(p3(u) - w) + dt*coupling*(nb - 4u) + sig_v*zv, with
                // u + dt p3(u) - 4 dt coupling u one host-folded cubic
                float un = fmaf(fmaf(fmaf(c.a3, u, c.a2), u, c.a1), u, c.a0);
                un = fmaf(-c.dt, w[e][r], un);
                un = fmaf(c.dtc, nb, un);
                un = fmaf(av, tv[h], un);
                w[e][r] = fmaf(aw, tw[h], fmaf(c.wc, w[e][r], fmaf(c.uc, u, c.c0)));
                nxt[r * W] = un;
                up = u;
                v[e][r] = un;
              }
            }
          }
        }
      }
      __syncthreads();
    };
    int k = 0;
    for (; k + 1 < c.n_sub; k += 2) {
      euler(k, std::integral_constant<int, 0>{});
      euler(k + 1, std::integral_constant<int, 1>{});
    }
    if (k < c.n_sub) euler(k, std::integral_constant<int, 0>{});

    // epilogue: divergence flag, store, electrode log-likelihood
#pragma unroll
    for (int e = 0; e < PP; ++e) {
      if (pb + e >= MN) continue;
      const int64_t p = pb + e;
      bool fin = true;
      float *xd = xout + p * 2 * static_cast<int64_t>(NODES);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (active && row0 + r < ROWS) {
          const int node = (row0 + r) * COLS + col;
          fin = fin && isfinite(v[e][r]) && isfinite(w[e][r]);
          xd[node] = v[e][r];
          xd[NODES + node] = w[e][r];
        }
      }
      if (!fin) bad[e] = 1;
    }
    if (tid < 32 * PP) {
      const int e = tid >> 5, lane = tid & 31;
      const float *fv = vsp + e * 2 * P + (c.n_sub & 1) * P;
      double acc = 0.0;
      for (int i = lane; i < c.n_obs; i += 32) {
        const int n = __ldg(obs_idx + i);
        const int rr = n / COLS;
        const double rsd = __ldg(y + i) - static_cast<double>(fv[(rr + 1) * W + (n - rr * COLS)]);
        acc = fma(rsd, rsd, acc);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
      if (lane == 0) red[e] = acc;
    }
    __syncthreads();
    if (tid < PP && pb + tid < MN) {
      logw[pb + tid] = static_cast<float>(c.obs_coef * red[tid]);
      if (bad[tid]) atomicOr(status + fe[tid], PF_ST_DIVERGED);
    }
    __syncthreads();
  }
}

// ---- production kernel with column-major strip slots (fp32, Philox) --------
// fhn_fast_kernel's decomposition, RNG and arithmetic, bit for bit, with the
// shared v plane laid out so that every neighbour read is vectorised: each
// (strip, column) owns an 8-float slot [R=6 rows | up halo | down halo] at
// col * kCmPitch + seg * 8 (32-byte aligned; pitch 44 = 12 mod 32 makes the
// quarter-warp 128-bit accesses conflict-free).  Per Euler step a thread
// reads its left and right neighbours' strips with LDS.128 + LDS.64 each and
// its vertical neighbours from its own halo (LDS.64), writes its new strip
// with STS.128 + STS.64 and its boundary rows into the adjacent strips'
// halos: 5 loads + 4 stores instead of 14 + 6.
// PF_FHN_SPLIT: the per-step CTA barrier of fhn_cm_kernel as an mbarrier
// arrive / wait pair with the last PF_FHN_SPLIT of the next step's three
// Philox blocks generated in between (register-only work that hides the
// skew between the warps).  cfg4 ms per interval, A/B on one box: classic
// __syncthreads (-1) 37.45; 0 blocks 37.94; 1 block 36.96; 2 blocks 37.21;
// all 3 (no Philox interleaved with the Box-Muller MUFUs any more) 37.56.
#ifndef PF_FHN_SPLIT
#define PF_FHN_SPLIT 1
#endif
constexpr int kCmPitch = 44;
__host__ __device__ constexpr int cm_plane(int cols) { return cols * kCmPitch + 64; }

template <int ROWS, int COLS, int R, int MINB, bool X2, bool PIPE = true>
__global__ void __launch_bounds__(256, MINB) fhn_cm_kernel(
    const float *__restrict__ xin, const int32_t *__restrict__ anc, float *__restrict__ xout,
    const double *__restrict__ y, const int32_t *__restrict__ obs_idx, float *__restrict__ logw,
    int64_t MN, int32_t N, FhnFast c, const uint32_t *__restrict__ keys, uint32_t t,
    uint32_t *__restrict__ status) {
  static_assert(R == 6 && ROWS % R == 0, "6-row strips tiling the lattice");
  constexpr int NSEG = ROWS / R;
  static_assert(NSEG * 8 <= kCmPitch, "strip slots must fit the column pitch");
  constexpr int P = cm_plane(COLS);  // plane stride: the slots + the idle threads' scratch
  constexpr int NODES = ROWS * COLS;
  static_assert(256 - NSEG * COLS >= 0 && (256 - NSEG * COLS) * 8 <= P - COLS * kCmPitch,
                "idle threads' scratch slots");
  extern __shared__ __align__(16) float cms[];  // [2][P] planes, then the electrode tables
  __shared__ double red[8];                     // per-warp electrode sums
  __shared__ int badw[8];                       // per-warp divergence flags
  __shared__ uint32_t s_zero;
  const int tid = threadIdx.x;
  if (tid == 0) s_zero = 0;  // ordered before any read by the first prologue barrier
#if PF_FHN_SPLIT >= 0
  __shared__ __align__(8) uint64_t s_mbar;
  if (tid == 0) {
    mbar_init(&s_mbar, 256);
    mbar_fence_init();
  }
  uint32_t phase = 0;
#endif
  const int seg = tid / COLS;
  const int col = tid - seg * COLS;
  const bool active = seg < NSEG;
  const int row0 = seg * R;
  // The 256 - NSEG*COLS idle threads run every Euler step too, on zeros in
  // a scratch slot of their own past the lattice (neighbours = themselves,
  // halos inside the slot): the step needs no `active` branch (BSSY/BSYNC
  // reconvergence per step).
  const int own = active ? col * kCmPitch + seg * 8 : COLS * kCmPitch + (tid - NSEG * COLS) * 8;
  const int lft = !active ? own : (col == 0 ? col : col - 1) * kCmPitch + seg * 8;  // ghost = self at the edges
  const int rgt = !active ? own : (col == COLS - 1 ? col : col + 1) * kCmPitch + seg * 8;
  const bool top = seg == 0, bottom = seg == NSEG - 1;
  // halo targets: the down halo of the strip above / up halo of the strip
  // below; the top / bottom strip writes its edge row into its own halo, so
  // the Neumann ghost = self needs no select when the halos are read back
  const int h_above = !active || top ? own + 6 : own - 1;
  const int h_below = !active || bottom ? own + 7 : own + 14;
  const float s2v = -1.3862943611198906f * c.sig_v * c.sig_v;
  const float s2w = -1.3862943611198906f * c.sig_w * c.sig_w;
  const uint32_t step0 = (t - 1u) * static_cast<uint32_t>(c.n_sub);

  // a strip's new values into plane `pl`: its slot + the adjacent halos
  auto put = [&](float *pl, const float *vv) {
    *reinterpret_cast<float4 *>(pl + own) = make_float4(vv[0], vv[1], vv[2], vv[3]);
    *reinterpret_cast<float2 *>(pl + own + 4) = make_float2(vv[4], vv[5]);
    pl[h_above] = vv[0];
    pl[h_below] = vv[5];
  };

  // Electrode log-likelihood, fhn.py:207 (-0.5/obs_var * sum (y - v)^2), taken
  // from the registers of the thread that owns each observed node: the
  // observation is the same for every particle of the launch, so each thread
  // tabulates once per CTA, per strip row r, the number of electrodes on its
  // node (cnt_r), -2 * the sum of their y (nb_r) and, over its strip, the sum
  // of y^2 (cy): its share of the sum is cy + sum_r v_r (cnt_r v_r + nb_r)
  // (fp64; duplicated electrodes allowed).  All warps share the epilogue
  // instead of one warp walking the electrodes over the shared plane while
  // the other seven wait at a barrier (~3 % of cfg4's stall samples).
  double *s_nb = reinterpret_cast<double *>(cms + 2 * P);  // [R][256]
  double *s_cnt = s_nb + R * 256;                           // [R][256]
  double *s_cy = s_cnt + R * 256;                           // [256]
  uint32_t *s_msk = reinterpret_cast<uint32_t *>(s_cy + 256);  // [256] rows with electrodes
  {
    double cy = 0.0;
    uint32_t msk = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      s_nb[r * 256 + tid] = 0.0;
      s_cnt[r * 256 + tid] = 0.0;
    }
    if (active) {
      for (int i = 0; i < c.n_obs; ++i) {
        const int n = __ldg(obs_idx + i);
        const int rr = n / COLS;
        if (n - rr * COLS == col && rr >= row0 && rr < row0 + R) {
          const double yv = __ldg(y + i);
          s_nb[(rr - row0) * 256 + tid] -= 2.0 * yv;
          s_cnt[(rr - row0) * 256 + tid] += 1.0;
          cy = fma(yv, yv, cy);
          msk |= 1u << (rr - row0);
        }
      }
    }
    s_cy[tid] = cy;
    s_msk[tid] = msk;  // read back by this thread only: no barrier
  }
  // this thread's share of the electrode sum and the divergence flag of the
  // new state, reduced per warp into red / badw (all 256 threads call it)
  auto ll_part = [&](const float *vv, const float *ww) {
    double acc = 0.0;
    bool fin = true;
    if (active) {
      const uint32_t msk = s_msk[tid];
      if (msk) {
        acc = s_cy[tid];
#pragma unroll
        for (int r = 0; r < R; ++r)
          if ((msk >> r) & 1u) {
            const double x = vv[r];
            acc = fma(x, fma(s_cnt[r * 256 + tid], x, s_nb[r * 256 + tid]), acc);
          }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) fin = fin && isfinite(vv[r]) && isfinite(ww[r]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    const bool all_fin = __all_sync(0xffffffffu, fin);
    if ((tid & 31) == 0) {
      red[tid >> 5] = acc;
      badw[tid >> 5] = all_fin ? 0 : 1;
    }
  };

  for (int64_t p = blockIdx.x; p < MN; p += gridDim.x) {
    const int64_t f = p / N;
    const uint32_t j = static_cast<uint32_t>(p - f * N);
    const int64_t src = anc ? static_cast<int64_t>(__ldg(anc + p)) : p;
    const float *xs = xin + src * 2 * static_cast<int64_t>(NODES);
    const Key2 key = load_key(keys, f);
    float v[R], w[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      v[r] = 0.f;
      w[r] = 0.f;
      if (active) {
        const int node = (row0 + r) * COLS + col;
        v[r] = __ldg(xs + node);
        w[r] = __ldg(xs + NODES + node);
      }
    }
    put(cms, v);
    __syncthreads();

    PhiloxPreT pre[R / 2];
    const PhiloxUni uni = philox_uni_t(j, kPurposeFhn, key);
    const PhiloxKeys rk = philox_round_keys(key);
#pragma unroll
    for (int q = 0; q < R / 2; ++q)
      pre[q] = philox_pre_t(j, static_cast<uint32_t>(((row0 >> 1) + q) * COLS + col), kPurposeFhn,
                            key);
    // X2: the same per-lane arithmetic on packed row pairs (2q, 2q+1) -
    // FFMA2/FADD2/FMUL2, bit-identical to the scalar form, ~25 fewer issue
    // slots per thread-step (PF_KERNEL_PACKED; not faster, see the launcher).  The vertical sums up+dn stay scalar FADDs whose
    // results land directly in pair registers (no register moves).
    f2_t vp[R / 2], wp[R / 2];
    if constexpr (X2) {
#pragma unroll
      for (int q = 0; q < R / 2; ++q) {
        vp[q] = f2_pack(v[2 * q], v[2 * q + 1]);
        wp[q] = f2_pack(w[2 * q], w[2 * q + 1]);
      }
    }
    const f2_t s2vw = f2_pack(s2v, s2w);
    // PIPE: every Euler step's Philox words are generated one step ahead,
    // in the same basic block as the previous step's MUFU Box-Muller and FMA
    // stencil, so that ptxas interleaves the FMA-heavy (IMAD.WIDE) and XU
    // streams instead of running all Philox rounds, then all MUFU, between
    // two barriers (cfg4 40.1 -> 39.0 ms; issue-active 60.5 -> 64.4 %).  The
    // last step's lookahead is discarded (a guard would split the block:
    // 41.8 ms).  Carrying the Box-Muller factors one step ahead as well
    // (18 floats instead of 12 words) measured 42.3 ms.
    uint4 rpipe[R / 2];
    if constexpr (PIPE) {
#pragma unroll
      for (int q = 0; q < R / 2; ++q) rpipe[q] = philox10_t(pre[q], uni, step0 ^ key.k0, rk);
    }
    auto euler = [&](int k, auto par_c, auto last_c) {
      constexpr int PAR = decltype(par_c)::value;
      // LAST: the interval's final step generates no lookahead words and
      // skips the barrier (the epilogue's __syncthreads orders its plane
      // reads before the next particle's prologue stores)
      constexpr bool LAST = decltype(last_c)::value;
      // The next step's Philox counter goes through a volatile shared load
      // of 0 issued after this step's barrier.  With the step body free of
      // branches, ptxas would otherwise hoist the lookahead Philox of both
      // unrolled steps into the first (128 registers; 39.7 ms per cfg4
      // interval instead of 37.7).
#if PF_FHN_SPLIT >= 0
      if constexpr (!X2 && PIPE) {
        // split barrier: arrive once the new strip is stored, generate the
        // last PF_FHN_SPLIT blocks of the next step's Philox words (no shared
        // data), then wait
        uint32_t knext = 0;
        if constexpr (!LAST) {
          // (no volatile-zero fence here: the barrier wait between two steps
          // already keeps ptxas from hoisting the next lookahead; 36.33 vs
          // 36.50 ms with the fence)
          knext = (step0 + k + 1) ^ key.k0;
        }
        const float *cur = cms + PAR * P;
        float *nxt = cms + (PAR ^ 1) * P;
        const float4 l4 = *reinterpret_cast<const float4 *>(cur + lft);
        const float2 l2 = *reinterpret_cast<const float2 *>(cur + lft + 4);
        const float4 r4 = *reinterpret_cast<const float4 *>(cur + rgt);
        const float2 r2 = *reinterpret_cast<const float2 *>(cur + rgt + 4);
        const float2 hl = *reinterpret_cast<const float2 *>(cur + own + 6);
        const float L[R] = {l4.x, l4.y, l4.z, l4.w, l2.x, l2.y};
        const float Rt[R] = {r4.x, r4.y, r4.z, r4.w, r2.x, r2.y};
        float up = hl.x;
        const float dn_last = hl.y;
        float vn[R];
#pragma unroll
        for (int q = 0; q < R / 2; ++q) {
          float av, aw, tv[2], tw[2];
          const uint4 rr = rpipe[q];
          if (!LAST && q < R / 2 - PF_FHN_SPLIT) rpipe[q] = philox10_t(pre[q], uni, knext, rk);
          box_muller_rad_trig(rr.x, rr.y, s2v, av, tv[0], tv[1]);
          box_muller_rad_trig(rr.z, rr.w, s2w, aw, tw[0], tw[1]);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = 2 * q + h;
            const float u = v[r];
            const float dn = r < R - 1 ? v[r + 1] : dn_last;
            const float nb = ((up + dn) + L[r]) + Rt[r];
            float un = fmaf(fmaf(fmaf(c.a3, u, c.a2), u, c.a1), u, c.a0);
            un = fmaf(-c.dt, w[r], un);
            un = fmaf(c.dtc, nb, un);
            un = fmaf(av, tv[h], un);
            w[r] = fmaf(aw, tw[h], fmaf(c.wc, w[r], fmaf(c.uc, u, c.c0)));
            vn[r] = un;
            up = u;
          }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = vn[r];
        put(nxt, v);
        if constexpr (LAST) return;
        mbar_arrive(&s_mbar);
        uint32_t zero2;
        asm volatile("ld.volatile.shared.u32 %0, [%1];"
                     : "=r"(zero2)
                     : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(&s_zero))));
        const uint32_t kn = (step0 + k + 1 + zero2) ^ key.k0;
#pragma unroll
        for (int q = R / 2 - PF_FHN_SPLIT; q < R / 2; ++q) rpipe[q] = philox10_t(pre[q], uni, kn, rk);
        // no suspend hint: the barrier completes within a few hundred clocks
        // (36.88 vs 36.93 ms with NANOSLEEP.SYNCS in the retry path)
        mbar_wait_short(&s_mbar, phase);
        phase ^= 1u;
        return;
      }
#endif
      uint32_t zero;
      asm volatile("ld.volatile.shared.u32 %0, [%1];"
                   : "=r"(zero)
                   : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(&s_zero))));
      const uint32_t knext = (step0 + k + 1 + zero) ^ key.k0;
      if constexpr (X2) {
        {
          const float *cur = cms + PAR * P;
          float *nxt = cms + (PAR ^ 1) * P;
          const ulonglong2 l4 = *reinterpret_cast<const ulonglong2 *>(cur + lft);
          const f2_t l2 = *reinterpret_cast<const f2_t *>(cur + lft + 4);
          const ulonglong2 r4 = *reinterpret_cast<const ulonglong2 *>(cur + rgt);
          const f2_t r2 = *reinterpret_cast<const f2_t *>(cur + rgt + 4);
          const float2 hl = *reinterpret_cast<const float2 *>(cur + own + 6);
          const f2_t L2[R / 2] = {l4.x, l4.y, l2};
          const f2_t R2[R / 2] = {r4.x, r4.y, r2};
          float vs[R];
#pragma unroll
          for (int q = 0; q < R / 2; ++q) {
            vs[2 * q] = f2_lo(vp[q]);
            vs[2 * q + 1] = f2_hi(vp[q]);
          }
          const float up0 = hl.x;
          const float dn5 = hl.y;
          // up + dn of every row (row r: v[r-1] + v[r+1]), packed per pair
          f2_t S[R / 2];
#pragma unroll
          for (int q = 0; q < R / 2; ++q) {
            const float u0 = q == 0 ? up0 : vs[2 * q - 1];
            const float d1 = q == R / 2 - 1 ? dn5 : vs[2 * q + 2];
            S[q] = f2_pack(u0 + vs[2 * q + 1], vs[2 * q] + d1);
          }
          const uint32_t c1k0 = (step0 + k) ^ key.k0;
          f2_t vn[R / 2];
#pragma unroll
          for (int q = 0; q < R / 2; ++q) {
            uint4 rr;
            if constexpr (PIPE) {
              rr = rpipe[q];
              rpipe[q] = philox10_t(pre[q], uni, knext, rk);
            } else {
              rr = philox10_t(pre[q], uni, c1k0, rk);
            }
            // box_muller_rad_trig on the v words (x, y) and the w words (z, w)
            const f2_t uu = f2_fma(f2_pack(static_cast<float>(rr.x), static_cast<float>(rr.z)),
                                   f2_bcast(2.3283064365386963e-10f),
                                   f2_bcast(1.1641532182693481e-10f));
            const f2_t lg = f2_mul(f2_pack(lg2_approx(f2_lo(uu)), lg2_approx(f2_hi(uu))), s2vw);
            const float av = sqrt_approx(f2_lo(lg)), aw = sqrt_approx(f2_hi(lg));
            const f2_t xx = f2_pack(__uint_as_float((rr.y & 0x007fffffu) | 0x40000000u),
                                    __uint_as_float((rr.w & 0x007fffffu) | 0x40000000u));
            const f2_t ang =
                f2_fma(xx, f2_bcast(3.14159265358979f), f2_bcast(-9.42477796076938f));
            const f2_t tv = f2_pack(cos_approx(f2_lo(ang)), sin_approx(f2_lo(ang)));
            const f2_t tw = f2_pack(cos_approx(f2_hi(ang)), sin_approx(f2_hi(ang)));
            const f2_t u = vp[q];
            const f2_t nb = f2_add(f2_add(S[q], L2[q]), R2[q]);
            f2_t un = f2_fma(f2_fma(f2_fma(f2_bcast(c.a3), u, f2_bcast(c.a2)), u, f2_bcast(c.a1)),
                             u, f2_bcast(c.a0));
            un = f2_fma(f2_bcast(-c.dt), wp[q], un);
            un = f2_fma(f2_bcast(c.dtc), nb, un);
            un = f2_fma(f2_bcast(av), tv, un);
            wp[q] = f2_fma(f2_bcast(aw), tw,
                           f2_fma(f2_bcast(c.wc), wp[q], f2_fma(f2_bcast(c.uc), u, f2_bcast(c.c0))));
            vn[q] = un;
          }
#pragma unroll
          for (int q = 0; q < R / 2; ++q) vp[q] = vn[q];
          // three 8-byte stores: a 16-byte store would pin vp[0], vp[1] to
          // one register quad and cost register moves every step
#pragma unroll
          for (int q = 0; q < R / 2; ++q)
            asm volatile("st.volatile.shared.b64 [%0], %1;" ::"r"(
                             static_cast<uint32_t>(__cvta_generic_to_shared(nxt + own + 2 * q))),
                         "l"(vp[q])
                         : "memory");
          nxt[h_above] = f2_lo(vp[0]);
          nxt[h_below] = f2_hi(vp[R / 2 - 1]);
        }
        __syncthreads();
        return;
      }
      {
        const float *cur = cms + PAR * P;
        float *nxt = cms + (PAR ^ 1) * P;
        const float4 l4 = *reinterpret_cast<const float4 *>(cur + lft);
        const float2 l2 = *reinterpret_cast<const float2 *>(cur + lft + 4);
        const float4 r4 = *reinterpret_cast<const float4 *>(cur + rgt);
        const float2 r2 = *reinterpret_cast<const float2 *>(cur + rgt + 4);
        const float2 hl = *reinterpret_cast<const float2 *>(cur + own + 6);
        const float L[R] = {l4.x, l4.y, l4.z, l4.w, l2.x, l2.y};
        const float Rt[R] = {r4.x, r4.y, r4.z, r4.w, r2.x, r2.y};
        float up = hl.x;
        const float dn_last = hl.y;
        const uint32_t c1k0 = (step0 + k) ^ key.k0;
        float vn[R];
#pragma unroll
        for (int q = 0; q < R / 2; ++q) {
          float av, aw, tv[2], tw[2];
          uint4 rr;
          if constexpr (PIPE) {
            rr = rpipe[q];  // generated during the previous step
            rpipe[q] = philox10_t(pre[q], uni, knext, rk);
          } else {
            rr = philox10_t(pre[q], uni, c1k0, rk);
          }
          box_muller_rad_trig(rr.x, rr.y, s2v, av, tv[0], tv[1]);
          box_muller_rad_trig(rr.z, rr.w, s2w, aw, tw[0], tw[1]);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = 2 * q + h;
            const float u = v[r];
            const float dn = r < R - 1 ? v[r + 1] : dn_last;
            const float nb = ((up + dn) + L[r]) + Rt[r];
            float un = fmaf(fmaf(fmaf(c.a3, u, c.a2), u, c.a1), u, c.a0);
            un = fmaf(-c.dt, w[r], un);
            un = fmaf(c.dtc, nb, un);
            un = fmaf(av, tv[h], un);
            w[r] = fmaf(aw, tw[h], fmaf(c.wc, w[r], fmaf(c.uc, u, c.c0)));
            vn[r] = un;
            up = u;
          }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = vn[r];
        put(nxt, v);
      }
      __syncthreads();
    };
    // unrolled by four (37.4 vs 37.7 ms per cfg4 interval unrolled by two;
    // passing the Box-Muller noise scale through the fence as well: 38.5);
    // the final step is peeled (no lookahead, no barrier); with the split
    // barrier: unrolled by two 37.18, by four 36.33, by eight 36.23 ms
    using P0 = std::integral_constant<int, 0>;
    using P1 = std::integral_constant<int, 1>;
    constexpr std::false_type more{};
    constexpr std::true_type last{};
    const int n1 = c.n_sub - 1;
    int k = 0;
    for (; k + 7 < n1; k += 8) {
      euler(k, P0{}, more);
      euler(k + 1, P1{}, more);
      euler(k + 2, P0{}, more);
      euler(k + 3, P1{}, more);
      euler(k + 4, P0{}, more);
      euler(k + 5, P1{}, more);
      euler(k + 6, P0{}, more);
      euler(k + 7, P1{}, more);
    }
    for (; k + 3 < n1; k += 4) {
      euler(k, P0{}, more);
      euler(k + 1, P1{}, more);
      euler(k + 2, P0{}, more);
      euler(k + 3, P1{}, more);
    }
    for (; k + 1 < n1; k += 2) {
      euler(k, P0{}, more);
      euler(k + 1, P1{}, more);
    }
    if (k < n1) {
      euler(k, P0{}, more);
      ++k;
    }
    if (k < c.n_sub) {
      if (k & 1)
        euler(k, P1{}, last);
      else
        euler(k, P0{}, last);
    }
    if constexpr (X2) {
#pragma unroll
      for (int q = 0; q < R / 2; ++q) {
        v[2 * q] = f2_lo(vp[q]);
        v[2 * q + 1] = f2_hi(vp[q]);
        w[2 * q] = f2_lo(wp[q]);
        w[2 * q + 1] = f2_hi(wp[q]);
      }
    }

    // epilogue: per-warp electrode shares and flags, one barrier, the state,
    // the log weight (red / badw are next written after the next particle's
    // prologue barrier)
    ll_part(v, w);
    __syncthreads();
    if (active) {
      float *xd = xout + p * 2 * static_cast<int64_t>(NODES);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int node = (row0 + r) * COLS + col;
        xd[node] = v[r];
        xd[NODES + node] = w[r];
      }
    }
    if (tid == 0) {
      double acc = red[0];
      int bad = badw[0];
#pragma unroll
      for (int i = 1; i < 8; ++i) {
        acc += red[i];
        bad |= badw[i];
      }
      logw[p] = static_cast<float>(c.obs_coef * acc);
      if (bad) atomicOr(status + f, PF_ST_DIVERGED);
    }
  }
}

template <int ROWS, int COLS, int MINB, bool X2, bool PIPE = true>
static int launch_fhn_cm(const FhnFast &fc, const void *x_in, const int32_t *anc, void *x_out,
                         const double *y, const int32_t *obs_idx, void *logw, int64_t MN,
                         int32_t N, const uint32_t *keys, uint32_t t, uint32_t *status,
                         cudaStream_t s) {
  // two v planes + the electrode tables (2 x kFhnRows x 256 + 256 doubles, 256 masks)
  constexpr size_t smem = 2 * static_cast<size_t>(cm_plane(COLS)) * sizeof(float) +
                          (2 * kFhnRows + 1) * 256 * sizeof(double) + 256 * sizeof(uint32_t);
  auto kern = fhn_cm_kernel<ROWS, COLS, kFhnRows, MINB, X2, PIPE>;
  static const int per_sm = [] {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(fhn_cm_kernel<ROWS, COLS, kFhnRows, MINB, X2, PIPE>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fhn_cm_kernel<ROWS, COLS, kFhnRows, MINB, X2, PIPE>,
                                                  256, smem);
    return n < 1 ? 1 : n;
  }();
  int sms = kSmCount, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t grid = std::min<int64_t>(MN, static_cast<int64_t>(sms) * per_sm);
  kern<<<static_cast<unsigned>(grid), 256, smem, s>>>(
      static_cast<const float *>(x_in), anc, static_cast<float *>(x_out), y, obs_idx,
      static_cast<float *>(logw), MN, N, fc, keys, t, status);
  return check_launch("pf_fhn_interval(column-major)");
}

// accel.fhn_euler_block (general form, fp64, per-node drive), one thread per
// node, reference order.
__global__ void fhn_block_op_kernel(const double *__restrict__ U, const double *__restrict__ V,
                                    const double *__restrict__ drive,
                                    const double *__restrict__ noise, int64_t total, int J1,
                                    int J2, FhnConsts c, double *__restrict__ un,
                                    double *__restrict__ vn) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= total) return;
  const int64_t plane = static_cast<int64_t>(J1) * J2;
  const int64_t p = g / plane;
  const int rem = static_cast<int>(g - p * plane);
  const int i = rem / J2, j = rem - (rem / J2) * J2;
  const double *Up = U + p * plane;
  using A = Ar<double>;
  double nb = 0.0;
  if (i > 0) nb = A::add(nb, Up[(i - 1) * J2 + j]);
  if (i < J1 - 1) nb = A::add(nb, Up[(i + 1) * J2 + j]);
  if (j > 0) nb = A::add(nb, Up[i * J2 + j - 1]);
  if (j < J2 - 1) nb = A::add(nb, Up[i * J2 + j + 1]);
  const double u = U[g], v = V[g];
  const double p3 = A::add(A::mul(A::add(A::mul(A::add(A::mul(c.a3, u), c.a2), u), c.a1), u), c.a0);
  const double t1 = A::add(u, A::mul(c.dt, A::sub(p3, v)));
  const double t2 = A::add(t1, A::mul(c.dt, A::add(A::mul(c.coupling, nb), drive[g])));
  un[g] = A::add(t2, A::mul(c.sig_v, noise[g]));
  vn[g] = A::add(v, A::mul(c.dt, A::add(A::add(A::mul(c.b0, u), A::mul(c.b1, v)), c.b2)));
}

static FhnConsts make_consts(const pf_fhn_params *p) {
  FhnConsts c;
  c.rows = p->rows;
  c.cols = p->cols;
  c.n_sub = p->n_sub;
  c.n_obs = p->n_obs;
  c.nseg = (p->rows + kFhnRows - 1) / kFhnRows;
  c.nodes = p->rows * p->cols;
  c.dt = p->dt;
  c.coupling = p->coupling;
  c.a3 = p->cubic[0];
  c.a2 = p->cubic[1];
  c.a1 = p->cubic[2];
  c.a0 = p->cubic[3];
  c.b0 = p->beta[0];
  c.b1 = p->beta[1];
  c.b2 = p->beta[2];
  c.sig_v = p->sig_v;
  c.sig_w = p->sig_w;
  c.degree_drive = p->degree_drive;
  c.obs_coef = -0.5 / p->obs_var;  // fhn.py:207: -0.5 / obs_var * sum
  return c;
}

template <typename T, int MODE>
static int launch_fhn(const FhnConsts &c, const void *x_in, const int32_t *anc, void *x_out,
                      const double *y, const int32_t *obs_idx, void *logw, int64_t MN,
                      int32_t N, const uint32_t *keys, uint32_t t, const double *tape,
                      uint32_t *status, cudaStream_t s) {
  const int threads = ((c.nseg * c.cols + 31) / 32) * 32;
  const size_t smem = 2 * static_cast<size_t>(c.nodes) * sizeof(T);
  auto kern = fhn_interval_kernel<T, MODE>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  if (per_sm < 1) per_sm = 1;
  int sms = kSmCount;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t grid = std::min<int64_t>(MN, static_cast<int64_t>(sms) * per_sm * 16);
  kern<<<static_cast<unsigned>(grid), threads, smem, s>>>(
      static_cast<const T *>(x_in), anc, static_cast<T *>(x_out), y, obs_idx,
      static_cast<T *>(logw), MN, N, c, keys, t, tape, status);
  return check_launch("pf_fhn_interval");
}

template <int ROWS, int COLS, bool TAPE, int MINB, int PP, bool NF = false, int R = kFhnRows>
static int launch_fhn_fast_t(const FhnFast &fc, const void *x_in, const int32_t *anc, void *x_out,
                             const double *y, const int32_t *obs_idx, void *logw, int64_t MN,
                             int32_t N, const uint32_t *keys, uint32_t t, const double *tape,
                             uint32_t *status, cudaStream_t s) {
  constexpr int threads = (((ROWS + R - 1) / R * COLS) + 31) / 32 * 32;
  static_assert(threads <= 256, "lattice too large for the fast kernel");
  const size_t smem = PP * 2 * static_cast<size_t>((ROWS + 2) * fhn_pitch(COLS, R)) * sizeof(float);
  auto kern = fhn_fast_kernel<ROWS, COLS, R, TAPE, MINB, PP, NF>;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  if (per_sm < 1) per_sm = 1;
  int sms = kSmCount, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t grid =
      std::min<int64_t>((MN + PP - 1) / PP, static_cast<int64_t>(sms) * per_sm);
  kern<<<static_cast<unsigned>(grid), threads, smem, s>>>(
      static_cast<const float *>(x_in), anc, static_cast<float *>(x_out), y, obs_idx,
      static_cast<float *>(logw), MN, N, fc, keys, t, tape, status);
  return check_launch("pf_fhn_interval(fast)");
}

// The fp32 fast path covers lattices with a compiled geometry; others use
// the generic kernel.
static bool fhn_fast_supported(const pf_fhn_params *p) {
  return p->rows == 30 && p->cols == 50 && p->degree_drive == -p->coupling;
}


static int launch_fhn_fast(const FhnConsts &c, const void *x_in, const int32_t *anc, void *x_out,
                           const double *y, const int32_t *obs_idx, void *logw, int64_t MN,
                           int32_t N, const uint32_t *keys, uint32_t t, const double *tape,
                           uint32_t *status, cudaStream_t s, uint32_t flags) {
  FhnFast fc;
  fc.rows = c.rows;
  fc.cols = c.cols;
  fc.n_sub = c.n_sub;
  fc.n_obs = c.n_obs;
  fc.nseg = c.nseg;
  fc.nodes = c.nodes;
  fc.a3 = float(c.dt * c.a3);
  fc.a2 = float(c.dt * c.a2);
  fc.a1 = float(1.0 + c.dt * c.a1 - 4.0 * c.dt * c.coupling);
  fc.a0 = float(c.dt * c.a0);
  fc.dt = float(c.dt);
  fc.dtc = float(c.dt * c.coupling);
  fc.dtc4 = float(4.0 * c.dt * c.coupling);
  fc.wc = float(1.0 + c.dt * c.b1);
  fc.uc = float(c.dt * c.b0);
  fc.c0 = float(c.dt * c.b2);
  fc.sig_v = float(c.sig_v);
  fc.sig_w = float(c.sig_w);
  fc.obs_coef = c.obs_coef;
  if (tape)
    return launch_fhn_fast_t<30, 50, true, 3, 1>(fc, x_in, anc, x_out, y, obs_idx, logw, MN, N,
                                                 keys, t, tape, status, s);
  // one particle per CTA, 2 CTAs/SM: the Philox key schedule, the hoisted
  // rounds and the next step's Philox words stay in registers (119).  cfg4:
  // 39.0 ms/interval for the column-major kernel with the Philox lookahead
  // (DESIGN §3); at 3 CTAs/SM ptxas rematerialises the round keys every step
  // (80 registers, 44.6 ms; 43.1 vs 41.8 ms for the row-major kernel before
  // the lookahead), 4 CTAs/SM and two particles per CTA measured slower too.
  // The noise-free lookahead variant has no draws (56 registers; its
  // column-major form measured 15.4 vs 14.1 ms).
  if (c.sig_v == 0.0 && c.sig_w == 0.0)  // the auxiliary filter's point prediction
    return launch_fhn_fast_t<30, 50, false, 3, 1, true>(fc, x_in, anc, x_out, y, obs_idx, logw,
                                                        MN, N, keys, t, tape, status, s);
  if (flags & PF_KERNEL_ALT)  // the row-major plane variant (same draws and arithmetic)
    return launch_fhn_fast_t<30, 50, false, 2, 1>(fc, x_in, anc, x_out, y, obs_idx, logw, MN, N,
                                                  keys, t, tape, status, s);
  // PF_KERNEL_PACKED: the same arithmetic on FFMA2/FADD2/FMUL2 pairs
  // (bit-identical, ~10 % fewer warp instructions per cfg4 launch, but 39.4
  // vs 39.0 ms: a packed op holds both FMA pipes, so the Philox IMAD.WIDE
  // on the heavy pipe waits more; without the Philox lookahead 40.5 vs 40.3
  // ms, math-pipe throttle 6.6 -> 12.5 % of stalls, profiles/r02_exp_fhn_ffma2.txt)
  if (flags & PF_KERNEL_PACKED)
    return launch_fhn_cm<30, 50, 2, true>(fc, x_in, anc, x_out, y, obs_idx, logw, MN, N, keys, t,
                                          status, s);
  return launch_fhn_cm<30, 50, 2, false>(fc, x_in, anc, x_out, y, obs_idx, logw, MN, N, keys, t,
                                         status, s);
}

}  // namespace pf

using namespace pf;

extern "C" {

int pf_fhn_interval(const pf_fhn_params *p, pf_dtype dtype, const void *x_in,
                    const int32_t *anc, void *x_out, const double *y, const int32_t *obs_idx,
                    void *logw_out, int64_t M, int64_t N, const uint32_t *keys, uint32_t t,
                    const double *z_tape, uint32_t *status, void *stream) {
  return pf_fhn_interval_ex(p, dtype, x_in, anc, x_out, y, obs_idx, logw_out, M, N, keys, t,
                            z_tape, status, 0u, stream);
}

int pf_fhn_interval_ex(const pf_fhn_params *p, pf_dtype dtype, const void *x_in,
                       const int32_t *anc, void *x_out, const double *y, const int32_t *obs_idx,
                       void *logw_out, int64_t M, int64_t N, const uint32_t *keys, uint32_t t,
                       const double *z_tape, uint32_t *status, uint32_t flags, void *stream) {
  PF_REQUIRE(p && x_in && x_out && y && obs_idx && logw_out && status, "pf_fhn_interval: null");
  PF_REQUIRE(M >= 1 && N >= 1 && M * N <= INT32_MAX, "pf_fhn_interval: bad M/N");
  PF_REQUIRE(p->rows >= 1 && p->cols >= 1 && p->n_sub >= 0, "pf_fhn_interval: bad lattice");
  PF_REQUIRE(p->n_obs >= 1 && p->n_obs <= 128, "pf_fhn_interval: need 1 <= n_obs <= 128");
  PF_REQUIRE(t >= 1, "pf_fhn_interval: t is 1-based");
  PF_REQUIRE(z_tape || keys, "pf_fhn_interval: need keys (Philox) or z_tape");
  PF_REQUIRE(x_in != x_out, "pf_fhn_interval: x_in and x_out must not alias");
  const FhnConsts c = make_consts(p);
  PF_REQUIRE(c.nseg * c.cols <= 256, "pf_fhn_interval: lattice too large for one CTA (%d threads)",
             c.nseg * c.cols);
  const int64_t MN = M * N;
  const int32_t n32 = static_cast<int32_t>(N);
  const cudaStream_t s = as_stream(stream);
  if (dtype == PF_F32 && fhn_fast_supported(p) && !(flags & PF_KERNEL_GENERIC))
    return launch_fhn_fast(c, x_in, anc, x_out, y, obs_idx, logw_out, MN, n32, keys, t, z_tape,
                           status, s, flags);
  if (dtype == PF_F64)
    return z_tape ? launch_fhn<double, 1>(c, x_in, anc, x_out, y, obs_idx, logw_out, MN, n32,
                                          keys, t, z_tape, status, s)
                  : launch_fhn<double, 0>(c, x_in, anc, x_out, y, obs_idx, logw_out, MN, n32,
                                          keys, t, z_tape, status, s);
  return z_tape ? launch_fhn<float, 1>(c, x_in, anc, x_out, y, obs_idx, logw_out, MN, n32, keys,
                                       t, z_tape, status, s)
                : launch_fhn<float, 0>(c, x_in, anc, x_out, y, obs_idx, logw_out, MN, n32, keys,
                                       t, z_tape, status, s);
}

int pf_op_fhn_euler_block(const double *U, const double *V, const double *drive,
                          const double *noise, int64_t n, int32_t J1, int32_t J2, double dt,
                          double coupling, const double *cubic4_host,
                          const double *beta3_host, double sig_sqdt, double *u_new,
                          double *v_new, void *stream) {
  PF_REQUIRE(U && V && drive && noise && u_new && v_new && cubic4_host && beta3_host,
             "pf_op_fhn_euler_block: null");
  PF_REQUIRE(n >= 1 && J1 >= 1 && J2 >= 1, "pf_op_fhn_euler_block: bad shape");
  pf_fhn_params p{};
  p.rows = J1;
  p.cols = J2;
  p.n_sub = 1;
  p.n_obs = 1;
  p.dt = dt;
  p.coupling = coupling;
  for (int i = 0; i < 4; ++i) p.cubic[i] = cubic4_host[i];
  for (int i = 0; i < 3; ++i) p.beta[i] = beta3_host[i];
  p.sig_v = sig_sqdt;
  p.sig_w = 0.0;
  p.degree_drive = 0.0;
  p.obs_var = 1.0;
  const FhnConsts c = make_consts(&p);
  const int64_t total = n * J1 * static_cast<int64_t>(J2);
  fhn_block_op_kernel<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(
      U, V, drive, noise, total, J1, J2, c, u_new, v_new);
  return check_launch("pf_op_fhn_euler_block");
}

}  // extern "C"
