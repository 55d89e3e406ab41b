// Small-state oracle models of the reference's verification suite:
//
//  * finite-state HMM (models/hmm.py:19-77): prior / transition by inverse-CDF
//    on a uniform (searchsorted-right on the cumulative prior, count of
//    cumulative row entries <= u), exact log-emission weights;
//  * linear-Gaussian model (models/linear_gaussian.py:18-95):
//    x' = x A^T + z L_q^T, log-likelihood with its normalising constant.
//
// Both keep the state as dim planes x[d*M*N + p] (one thread per particle,
// ancestor gather fused into the load) so the bank's resampler and estimator
// are shared with Lorenz-63.  fp64 evaluates every product and sum in the
// reference's order with one rounding each; tape mode reads the reference's
// exact uniforms / normals.
#include "common.cuh"
#include "philox.cuh"

namespace pf {

enum : uint32_t {
  kPurposeHmm = 0x484D4D5Fu,  // 'HMM_'
  kPurposeLgm = 0x4C474D5Fu,  // 'LGM_'
};

constexpr int kLgmMaxDim = 8;

// numpy Generator.random(): (v >> 11) * 2^-53 in [0, 1)
__device__ __forceinline__ double u53_random(uint4 r) {
  const uint64_t v = (static_cast<uint64_t>(r.x) << 21) ^ static_cast<uint64_t>(r.y >> 11);
  return static_cast<double>(v) * 1.1102230246251565e-16;
}

template <typename T>
__global__ void hmm_prior_kernel(T *__restrict__ x, int64_t MN, int32_t N, int K,
                                 const double *__restrict__ cum_prior,
                                 const uint32_t *__restrict__ keys,
                                 const double *__restrict__ tape) {
  const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (p >= MN) return;
  const int64_t f = p / N;
  const uint32_t j = static_cast<uint32_t>(p - f * N);
  const double u = tape ? tape[p]
                        : u53_random(philox10(make_uint4(j, 0u, 0u, kPurposePrior),
                                              load_key(keys, f)));
  // searchsorted(cum_prior, u, side="right"), clamped (hmm.py:57-60)
  int s = 0;
  for (int k = 0; k < K; ++k) s += cum_prior[k] <= u;
  x[p] = T(s < K - 1 ? s : K - 1);
}

template <typename T>
__global__ void hmm_step_kernel(const T *__restrict__ xin, const int32_t *__restrict__ anc,
                                T *__restrict__ xout, const double *__restrict__ y,
                                T *__restrict__ logw, int64_t MN, int32_t N, int K, int S,
                                const double *__restrict__ cum_rows,
                                const double *__restrict__ log_emission,
                                const uint32_t *__restrict__ keys, uint32_t t,
                                const double *__restrict__ tape) {
  const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (p >= MN) return;
  const int64_t f = p / N;
  const uint32_t j = static_cast<uint32_t>(p - f * N);
  const int64_t src = anc ? static_cast<int64_t>(anc[p]) : p;
  const int s = static_cast<int>(xin[src]);
  const double u = tape ? tape[p]
                        : u53_random(philox10(make_uint4(j, t, 0u, kPurposeHmm),
                                              load_key(keys, f)));
  // (u >= cum_row).sum(), clamped (hmm.py:62-68)
  int nxt = 0;
  for (int k = 0; k < K; ++k) nxt += u >= cum_rows[s * K + k];
  nxt = nxt < K - 1 ? nxt : K - 1;
  xout[p] = T(nxt);
  if (logw) {
    const int sym = static_cast<int>(y[0]);
    logw[p] = T(log_emission[nxt * S + sym]);  // log(emission[state, sym]) (hmm.py:70-72)
  }
}

__global__ void hmm_loglik_kernel(const double *__restrict__ x, int64_t n, int S,
                                  const double *__restrict__ y,
                                  const double *__restrict__ log_emission,
                                  double *__restrict__ out) {
  const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (q >= n) return;
  out[q] = log_emission[static_cast<int>(x[q]) * S + static_cast<int>(y[0])];
}

// LGM: noise-free (point prediction) when noise_free != 0.
template <typename T>
__device__ __forceinline__ void lgm_normals(Key2 key, uint32_t j, uint32_t t, int dx,
                                            const double *tape_row, double *z) {
  if (tape_row) {
    for (int d = 0; d < dx; ++d) z[d] = tape_row[d];
    return;
  }
  for (int d = 0; d < dx; d += 2) {
    const uint4 r = philox10(make_uint4(j, t, static_cast<uint32_t>(d >> 1), kPurposeLgm), key);
    const double2 g = box_muller_f64(r.x, r.y, r.z, r.w);
    z[d] = g.x;
    if (d + 1 < dx) z[d + 1] = g.y;
  }
}

// y = v @ M^T for a row vector v (matmul order: sum over the inner index
// left to right)
__device__ __forceinline__ double row_dot(const double *v, const double *Mrow, int n) {
  double acc = __dmul_rn(v[0], Mrow[0]);
  for (int k = 1; k < n; ++k) acc = __dadd_rn(acc, __dmul_rn(v[k], Mrow[k]));
  return acc;
}

template <typename T>
__global__ void lgm_prior_kernel(T *__restrict__ x, int64_t MN, int32_t N, int dx,
                                 const double *__restrict__ mean, const double *__restrict__ L,
                                 const uint32_t *__restrict__ keys,
                                 const double *__restrict__ tape) {
  const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (p >= MN) return;
  const int64_t f = p / N;
  const uint32_t j = static_cast<uint32_t>(p - f * N);
  double z[kLgmMaxDim];
  lgm_normals<T>(tape ? Key2{0u, 0u} : load_key(keys, f), j, 0u, dx, tape ? tape + p * dx : nullptr,
                 z);
  // prior_mean + z @ L0^T (linear_gaussian.py:66-68)
  for (int i = 0; i < dx; ++i) x[i * MN + p] = T(__dadd_rn(mean[i], row_dot(z, L + i * dx, dx)));
}

template <typename T>
__global__ void lgm_step_kernel(const T *__restrict__ xin, const int32_t *__restrict__ anc,
                                T *__restrict__ xout, const double *__restrict__ y,
                                T *__restrict__ logw, int64_t MN, int32_t N, int dx, int dy,
                                const double *__restrict__ A, const double *__restrict__ Lq,
                                const double *__restrict__ H, const double *__restrict__ P,
                                double logconst, int noise_free,
                                const uint32_t *__restrict__ keys, uint32_t t,
                                const double *__restrict__ tape, uint32_t *__restrict__ status) {
  const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (p >= MN) return;
  const int64_t f = p / N;
  const uint32_t j = static_cast<uint32_t>(p - f * N);
  const int64_t src = anc ? static_cast<int64_t>(anc[p]) : p;
  double xv[kLgmMaxDim], xn[kLgmMaxDim];
  for (int d = 0; d < dx; ++d) xv[d] = static_cast<double>(xin[d * MN + src]);
  bool fin = true;
  if (noise_free) {
    // x_prev @ A^T (linear_gaussian.py:74-75)
    for (int i = 0; i < dx; ++i) xn[i] = row_dot(xv, A + i * dx, dx);
  } else {
    double z[kLgmMaxDim];
    lgm_normals<T>(tape ? Key2{0u, 0u} : load_key(keys, f), j, t, dx,
                   tape ? tape + p * dx : nullptr, z);
    // x_prev @ A^T + z @ Lq^T (linear_gaussian.py:70-72)
    for (int i = 0; i < dx; ++i)
      xn[i] = __dadd_rn(row_dot(xv, A + i * dx, dx), row_dot(z, Lq + i * dx, dx));
  }
  for (int i = 0; i < dx; ++i) {
    const T v = T(xn[i]);
    fin = fin && finite_val(v);
    xout[i * MN + p] = v;
  }
  if (!fin) atomicOr(status + f, PF_ST_DIVERGED);
  if (logw) {
    // resid = y - x @ H^T; quad = einsum("ni,ij,nj->n", r, P, r);
    // logconst - 0.5 * quad (linear_gaussian.py:77-82)
    double r[kLgmMaxDim];
    for (int i = 0; i < dy; ++i) {
      double xs[kLgmMaxDim];
      for (int d = 0; d < dx; ++d) xs[d] = static_cast<double>(T(xn[d]));
      r[i] = __dsub_rn(y[i], row_dot(xs, H + i * dx, dx));
    }
    double quad = 0.0;
    for (int i = 0; i < dy; ++i)
      for (int k = 0; k < dy; ++k) quad = __dadd_rn(quad, __dmul_rn(__dmul_rn(r[i], P[i * dy + k]), r[k]));
    logw[p] = T(__dsub_rn(logconst, __dmul_rn(0.5, quad)));
  }
}

// Stored-state log-likelihood (LinearGaussianModel.log_likelihood hook):
// states given as planes x[d*n + r], fp64.
__global__ void lgm_loglik_kernel(const double *__restrict__ x, int64_t n, int dx, int dy,
                                  const double *__restrict__ y, const double *__restrict__ H,
                                  const double *__restrict__ P, double logconst,
                                  double *__restrict__ out) {
  const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (q >= n) return;
  double xs[kLgmMaxDim], r[kLgmMaxDim];
  for (int d = 0; d < dx; ++d) xs[d] = x[d * n + q];
  for (int i = 0; i < dy; ++i) r[i] = __dsub_rn(y[i], row_dot(xs, H + i * dx, dx));
  double quad = 0.0;
  for (int i = 0; i < dy; ++i)
    for (int k = 0; k < dy; ++k) quad = __dadd_rn(quad, __dmul_rn(__dmul_rn(r[i], P[i * dy + k]), r[k]));
  out[q] = __dsub_rn(logconst, __dmul_rn(0.5, quad));
}

}  // namespace pf

using namespace pf;

extern "C" {

int pf_hmm_prior(const pf_hmm_params *h, pf_dtype dtype, void *x, int64_t M, int64_t N,
                 const uint32_t *keys, const double *u_tape, void *stream) {
  PF_REQUIRE(h && x && h->K >= 1 && h->cum_prior && M >= 1 && N >= 1 && M * N <= INT32_MAX,
             "pf_hmm_prior: bad arguments");
  PF_REQUIRE(u_tape || keys, "pf_hmm_prior: need keys (Philox) or u_tape");
  const int64_t MN = M * N;
  const cudaStream_t s = as_stream(stream);
  if (dtype == PF_F64)
    hmm_prior_kernel<double><<<grid_for(MN, 256), 256, 0, s>>>(
        static_cast<double *>(x), MN, static_cast<int32_t>(N), h->K, h->cum_prior, keys, u_tape);
  else
    hmm_prior_kernel<float><<<grid_for(MN, 256), 256, 0, s>>>(
        static_cast<float *>(x), MN, static_cast<int32_t>(N), h->K, h->cum_prior, keys, u_tape);
  return check_launch("pf_hmm_prior");
}

int pf_hmm_propagate_weight(const pf_hmm_params *h, pf_dtype dtype, const void *x_in,
                            const int32_t *anc, void *x_out, const double *y, void *logw_out,
                            int64_t M, int64_t N, const uint32_t *keys, uint32_t t,
                            const double *u_tape, uint32_t *status, void *stream) {
  PF_REQUIRE(h && x_in && x_out && h->K >= 1 && h->S >= 1 && h->cum_rows && h->log_emission &&
                 M >= 1 && N >= 1 && M * N <= INT32_MAX,
             "pf_hmm_propagate_weight: bad arguments");
  PF_REQUIRE(u_tape || keys, "pf_hmm_propagate_weight: need keys (Philox) or u_tape");
  PF_REQUIRE(!logw_out || y, "pf_hmm_propagate_weight: weights need y");
  (void)status;
  const int64_t MN = M * N;
  const cudaStream_t s = as_stream(stream);
  if (dtype == PF_F64)
    hmm_step_kernel<double><<<grid_for(MN, 256), 256, 0, s>>>(
        static_cast<const double *>(x_in), anc, static_cast<double *>(x_out), y,
        static_cast<double *>(logw_out), MN, static_cast<int32_t>(N), h->K, h->S, h->cum_rows,
        h->log_emission, keys, t, u_tape);
  else
    hmm_step_kernel<float><<<grid_for(MN, 256), 256, 0, s>>>(
        static_cast<const float *>(x_in), anc, static_cast<float *>(x_out), y,
        static_cast<float *>(logw_out), MN, static_cast<int32_t>(N), h->K, h->S, h->cum_rows,
        h->log_emission, keys, t, u_tape);
  return check_launch("pf_hmm_propagate_weight");
}

int pf_hmm_loglik(const pf_hmm_params *h, const double *x, int64_t n, const double *y,
                  double *out, void *stream) {
  PF_REQUIRE(h && x && y && out && n >= 0 && h->log_emission, "pf_hmm_loglik: bad arguments");
  if (n == 0) return PF_OK;
  hmm_loglik_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(x, n, h->S, y,
                                                                     h->log_emission, out);
  return check_launch("pf_hmm_loglik");
}

int pf_lgm_prior(const pf_lgm_params *g, pf_dtype dtype, void *x, int64_t M, int64_t N,
                 const uint32_t *keys, const double *z_tape, void *stream) {
  PF_REQUIRE(g && x && g->dx >= 1 && g->dx <= kLgmMaxDim && g->prior_mean && g->chol_p0 &&
                 M >= 1 && N >= 1 && M * N <= INT32_MAX,
             "pf_lgm_prior: bad arguments (dim_x <= %d)", kLgmMaxDim);
  PF_REQUIRE(z_tape || keys, "pf_lgm_prior: need keys (Philox) or z_tape");
  const int64_t MN = M * N;
  const cudaStream_t s = as_stream(stream);
  if (dtype == PF_F64)
    lgm_prior_kernel<double><<<grid_for(MN, 256), 256, 0, s>>>(
        static_cast<double *>(x), MN, static_cast<int32_t>(N), g->dx, g->prior_mean, g->chol_p0,
        keys, z_tape);
  else
    lgm_prior_kernel<float><<<grid_for(MN, 256), 256, 0, s>>>(
        static_cast<float *>(x), MN, static_cast<int32_t>(N), g->dx, g->prior_mean, g->chol_p0,
        keys, z_tape);
  return check_launch("pf_lgm_prior");
}

int pf_lgm_propagate_weight(const pf_lgm_params *g, pf_dtype dtype, const void *x_in,
                            const int32_t *anc, void *x_out, const double *y, void *logw_out,
                            int64_t M, int64_t N, const uint32_t *keys, uint32_t t,
                            const double *z_tape, uint32_t *status, void *stream) {
  PF_REQUIRE(g && x_in && x_out && status && g->dx >= 1 && g->dx <= kLgmMaxDim && g->dy >= 1 &&
                 g->dy <= kLgmMaxDim && g->A && g->chol_q && M >= 1 && N >= 1 &&
                 M * N <= INT32_MAX,
             "pf_lgm_propagate_weight: bad arguments (dims <= %d)", kLgmMaxDim);
  PF_REQUIRE(g->noise_free || z_tape || keys,
             "pf_lgm_propagate_weight: need keys (Philox) or z_tape");
  PF_REQUIRE(!logw_out || (y && g->H && g->obs_prec),
             "pf_lgm_propagate_weight: weights need y, H and a positive-definite obs_cov");
  const int64_t MN = M * N;
  const cudaStream_t s = as_stream(stream);
  if (dtype == PF_F64)
    lgm_step_kernel<double><<<grid_for(MN, 256), 256, 0, s>>>(
        static_cast<const double *>(x_in), anc, static_cast<double *>(x_out), y,
        static_cast<double *>(logw_out), MN, static_cast<int32_t>(N), g->dx, g->dy, g->A,
        g->chol_q, g->H, g->obs_prec, g->obs_logconst, g->noise_free, keys, t, z_tape, status);
  else
    lgm_step_kernel<float><<<grid_for(MN, 256), 256, 0, s>>>(
        static_cast<const float *>(x_in), anc, static_cast<float *>(x_out), y,
        static_cast<float *>(logw_out), MN, static_cast<int32_t>(N), g->dx, g->dy, g->A,
        g->chol_q, g->H, g->obs_prec, g->obs_logconst, g->noise_free, keys, t, z_tape, status);
  return check_launch("pf_lgm_propagate_weight");
}

int pf_lgm_loglik(const pf_lgm_params *g, const double *x, int64_t n, const double *y,
                  double *out, void *stream) {
  PF_REQUIRE(g && x && y && out && n >= 0 && g->dx >= 1 && g->dx <= kLgmMaxDim && g->dy >= 1 &&
                 g->dy <= kLgmMaxDim && g->H && g->obs_prec,
             "pf_lgm_loglik: bad arguments");
  if (n == 0) return PF_OK;
  lgm_loglik_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(
      x, n, g->dx, g->dy, y, g->H, g->obs_prec, g->obs_logconst, out);
  return check_launch("pf_lgm_loglik");
}

}  // extern "C"
