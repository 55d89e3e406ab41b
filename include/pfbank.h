/*
 * pfbank.h - C ABI of the B200-native particle-filter bank (libpfbank.so).
 *
 * Drop-in boundary for the hot path of the reference `parpf`
 * (arXiv 1407.8071): a bank of M independent bootstrap particle filters
 * with N particles each.  The reference is pure Python; its "FFI" for this
 * path is the module-level kernel rebinding in parpf/accel.py:206-213 plus
 * the Python entry points it feeds.  Each entry point below cites the
 * reference interface it replaces (paths relative to
 * /root/reference/pkg/src/parpf/).
 *
 * Conventions
 *  - All array pointers are DEVICE pointers owned by the caller
 *    (e.g. PyTorch CUDA tensors); parameter structs and `mean3`-style small
 *    vectors marked "host" are host pointers.  Nothing is allocated inside,
 *    nothing synchronises the host.  Every call is stream-ordered on
 *    `stream` (a cudaStream_t passed as void*; NULL = legacy default).
 *  - Return codes: PF_OK (0); PF_EINVAL for bad arguments (the Python layer
 *    raises ValueError, matching core.py:127-133, resampling.py:12-17,
 *    filters.py:90-91, ensemble.py:87-90); PF_ECUDA for a CUDA launch error
 *    (RuntimeError).  pf_last_error() returns a thread-local message.
 *  - Per-filter runtime outcomes are device flags, not return codes:
 *    status[f] |= PF_ST_DIVERGED (non-finite state: the reference raises
 *    NumericalDivergenceError, lorenz63.py:48-49 / fhn.py:186-187),
 *    status[f] |= PF_ST_NAN_WEIGHT (core.py:132-133 ValueError);
 *    collapsed[f] = 1 on total weight underflow (core.py:130-131 ->
 *    filters.py:105-109: uniform weights, lnc unchanged, identity ancestors).
 *  - Particle layouts (row index p = f*N + i, filter-major):
 *      Lorenz : three planes x[d*M*N + p], d = 0..2   (T = float|double)
 *      FH-N   : rows x[p*2*nodes + {0: v block, nodes: w block} + node]
 *  - Randomness: production mode draws Philox4x32-10 keyed by a per-filter
 *    64-bit key keys[2f], keys[2f+1] with counters built from
 *    (particle, time, draw, purpose), so results do not depend on how
 *    filters are sharded over GPUs.  Oracle ("tape") mode instead reads
 *    caller-supplied standard normals / sorted uniforms (fp64), which lets
 *    the test harness feed the reference's exact draws.
 */
#ifndef PFBANK_H
#define PFBANK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PF_OK 0
#define PF_EINVAL (-22)
#define PF_ECUDA (-5)

#define PF_ST_DIVERGED 1u
#define PF_ST_NAN_WEIGHT 2u

typedef enum pf_dtype { PF_F32 = 0, PF_F64 = 1 } pf_dtype;

/* Stochastic Lorenz-63 (models/lorenz63.py:22-69 + BASELINE cfg0/cfg2
 * adapter).  obs_dim = 1 observes x1 (stock Lorenz63Model.log_likelihood,
 * lorenz63.py:62-65); obs_dim = 2 observes (x1, x3). */
typedef struct pf_lorenz_params {
  double s, r, b, dt;
  double noise_scale; /* multiplies the N(0,1) draws before the sqrt(dt) scaling */
  double obs_var;
  int32_t n_sub;   /* Euler substeps per observation interval */
  int32_t obs_dim; /* 1 or 2 */
} pf_lorenz_params;

/* Lattice FitzHugh-Nagumo in the reference kernel's general form
 * (accel.py:110-129): u' = u + dt(p3(u) - w) + dt(coupling*nb + drive)
 * + sig_v*z; w' = w + dt(b0 u + b1 w + b2) [+ sig_w*z'], with
 * drive = degree_drive * deg(i,j) * u (degree_drive = -1 gives the Neumann
 * 5-point Laplacian of BASELINE cfg3/cfg4).  Observation: Gaussian on u at
 * `n_obs` electrode nodes (fhn.py:199-207). */
typedef struct pf_fhn_params {
  int32_t rows, cols, n_sub, n_obs;
  double dt, coupling;
  double cubic[4]; /* a3, a2, a1, a0 */
  double beta[3];  /* b0, b1, b2 */
  double sig_v, sig_w;
  double degree_drive;
  double obs_var;
} pf_fhn_params;

/* Stochastically forced FH-N network, the paper's lattice model
 * (models/fhn.py:85-207): J x J nodes, ONE Euler step per transition with
 * drive = forcing_mask * forcing(t) + stim_amp * [stimulus in the last
 * stim_hold steps], random stimuli behind travelling waves (stim_prob per
 * particle-step at a uniformly chosen cell of the (u_minus, u_plus) region,
 * plus its von Neumann neighbours).  Device layout per particle p: U, V planes
 * x[p*2*J*J + {0, J*J} + node] and the stimulus history as bits
 * q[p*J*J + node] (bit k = Q(t-k), so stim_hold <= 32). */
typedef struct pf_fhnnet_params {
  int32_t J, stim_hold, n_obs;
  int32_t stochastic; /* 0 = transition_point_prediction (fhn.py:191-197): no new
                         stimulus, no noise; forcing and latched stimuli apply */
  double dt, coupling;
  double cubic[4]; /* a3, a2, a1, a0 */
  double beta[3];  /* b0, b1, b2 */
  double u_minus, u_plus;
  double stim_prob, stim_amp;
  double forcing_amp, forcing_period, forcing_width;
  double sig_sqdt; /* sqrt(dyn_var) * sqrt(dt) */
  double obs_var;
} pf_fhnnet_params;

/* Finite-state HMM (models/hmm.py:19-77).  Device tables: cum_prior (K),
 * cum_rows (K*K, row-wise cumsum of the transition matrix), log_emission
 * (K*S) = log(emission).  States are stored as floating-point indices. */
typedef struct pf_hmm_params {
  int32_t K, S;
  const double *cum_prior, *cum_rows, *log_emission; /* device */
} pf_hmm_params;

/* Linear-Gaussian model (models/linear_gaussian.py:18-95), dim_x, dim_y <= 8.
 * Device row-major matrices: A (dx*dx), chol_q (dx*dx), H (dy*dx),
 * obs_prec (dy*dy), prior_mean (dx), chol_p0 (dx*dx). */
typedef struct pf_lgm_params {
  int32_t dx, dy;
  int32_t noise_free; /* transition_point_prediction (linear_gaussian.py:74-75) */
  int32_t reserved;
  const double *A, *chol_q, *H, *obs_prec, *prior_mean, *chol_p0; /* device */
  double obs_logconst; /* -0.5 (dy log 2pi + log det obs_cov) */
} pf_lgm_params;

/* ---- library ------------------------------------------------------- */
const char *pf_last_error(void);
int pf_version(void);
int pf_device_sm_count(int *out);

/* FP32 peak probe (measurement helper for bench.py's Lorenz roofline): one
   launch of SMs x 8 blocks x 256 threads, each running 8 independent FFMA chains
   for iters x 16 steps = 256 * iters flop per thread.  Time it with events. */
int pf_probe_fp32_fma(float *sink, int64_t iters, void *stream);

/* Philox4x32-10 known-answer helper: out[4] for ctr[4], key[2] (device).
   Also evaluates the kernels' hoisted form (philox10_t) and returns the
   complemented words if the two ever differ. */
int pf_philox_kat(const uint32_t *ctr, const uint32_t *key, uint32_t *out, int64_t n, void *stream);

/* ---- L1 operator drop-ins (accel.py) --------------------------------- */
/* accel.lorenz_euler_block (accel.py:60-102): states (n,3), noise
 * (n_sub,n,3), fp64, reference evaluation order, no FMA -> bit-exact. */
int pf_op_lorenz_euler_block(const double *states, const double *noise, int64_t n,
                             int64_t n_sub, double dt, double s, double r, double b,
                             double *out, void *stream);

/* accel.fhn_euler_block (accel.py:110-167) for (n, J1, J2) fp64 lattices
 * (rectangular allowed, unlike the reference jit twin accel.py:135). */
int pf_op_fhn_euler_block(const double *U, const double *V, const double *drive,
                          const double *noise, int64_t n, int32_t J1, int32_t J2, double dt,
                          double coupling, const double *cubic4_host,
                          const double *beta3_host, double sig_sqdt, double *u_new,
                          double *v_new, void *stream);

/* accel.resample_indices (accel.py:175-203): smallest k with cum[k] >= u,
 * clamped to n-1; int64 out. */
int pf_op_resample_indices(const double *cum, int64_t n, const double *u, int64_t m,
                           int64_t *idx_out, void *stream);

/* core.normalize_log_weights (core.py:116-138) for M segments of N.
 * weights_out (M*N) fp64, log_mean_raw_out (M) fp64; collapsed[f] set
 * on total underflow (weights untouched), status NaN flag on NaN. */
int pf_op_normalize_log_weights(pf_dtype logw_dtype, const void *logw, int64_t M, int64_t N,
                                double *weights_out, double *log_mean_raw_out,
                                uint8_t *collapsed, uint32_t *status, void *stream);

/* Hook-level resampling helpers in numpy's order (resampling.py:21-72):
 * out = np.cumsum(a) (sequential); u = cumsum(e)[:n_out] / cumsum(e)[n_out]
 * for e of length n_out + 1 (work: n_out + 1 doubles); systematic thresholds
 * u_i = (i + r) / n_out. */
int pf_op_cumsum(const double *a, int64_t n, double *out, void *stream);
int pf_op_spacing_uniforms(const double *e, int64_t n_out, double *work, double *u,
                           void *stream);
int pf_op_systematic_uniforms(double r, int64_t n_out, double *u, void *stream);

/* Explicit ancestor gather of a 3-plane state (filters.py:111 / cfg1):
 * x_out[d][p] = x_in[d][anc[p]]. */
int pf_gather_planes(pf_dtype dtype, const void *x_in, const int32_t *anc, int64_t MN,
                     int32_t dims, void *x_out, void *stream);

/* ---- L2-L4 bank kernels --------------------------------------------- */
/* bf_init prior (filters.py:87-94 + lorenz63.py:42-44): x = mean + sd*z,
 * z from Philox (purpose PRIOR) or z_tape (M,N,3) fp64. */
int pf_lorenz_prior(pf_dtype dtype, void *x, int64_t M, int64_t N, const double *mean3_host,
                    double prior_sd, const uint32_t *keys, const double *z_tape,
                    void *stream);

/* Broadcast one fp64 state row to every particle (deterministic priors,
 * fhn.py:144-147 and the cfg3/4 stimulated point mass). */
int pf_fill_rows(pf_dtype dtype, void *x, int64_t MN, int64_t row_len, const double *row,
                 void *stream);

/* bf_step propagate + weight (filters.py:103-104; lorenz63.py:46-65):
 * x_out[p] = EM^{n_sub}(x_in[anc[p]]) (anc NULL = identity), logw_out[p] =
 * log-likelihood of y (device, obs_dim doubles) at observation time t.
 * z_tape (M, n_sub, N, 3) fp64 or NULL (Philox). */
int pf_lorenz_propagate_weight(const pf_lorenz_params *p, pf_dtype dtype, const void *x_in,
                               const int32_t *anc, void *x_out, const double *y,
                               void *logw_out, int64_t M, int64_t N, const uint32_t *keys,
                               uint32_t t, const double *z_tape, uint32_t *status,
                               void *stream);

/* Kernel selection for the *_ex entry points (per call; no process-wide
 * state).  0 = the production choice.  PF_KERNEL_GENERIC forces the generic
 * (runtime-geometry, accurate-libm) kernel instead of the specialised fast
 * one, with the same Philox counters and draw layout - the comparison tests
 * pin the fast kernels against it. */
#define PF_KERNEL_GENERIC 1u
/* PF_KERNEL_ALT: the production kernel's alternative layout where one exists
 * (FH-N lattice: the row-major shared plane instead of column-major strip
 * slots) - bit-identical results, kept for comparison. */
#define PF_KERNEL_ALT 2u
/* PF_KERNEL_PACKED: the production kernel issued on packed fp32 pairs
 * (sm_100a FFMA2/FADD2/FMUL2: 10 % fewer instructions for the FH-N lattice)
 * - bit-identical results; measured slower (FFMA2 occupies the FMA-heavy
 * pipe the Philox IMAD.WIDE needs), kept for comparison. */
#define PF_KERNEL_PACKED 4u
int pf_lorenz_propagate_weight_ex(const pf_lorenz_params *p, pf_dtype dtype, const void *x_in,
                                  const int32_t *anc, void *x_out, const double *y,
                                  void *logw_out, int64_t M, int64_t N, const uint32_t *keys,
                                  uint32_t t, const double *z_tape, uint32_t *status,
                                  uint32_t flags, void *stream);

/* One FH-N observation interval: n_sub lattice Euler steps with the particle
 * resident in shared memory/registers, ancestor gather fused into the load,
 * electrode log-likelihood fused into the epilogue.
 * z_tape (M, n_sub, 2, N, rows*cols) fp64 or NULL (Philox). */
int pf_fhn_interval(const pf_fhn_params *p, pf_dtype dtype, const void *x_in,
                    const int32_t *anc, void *x_out, const double *y, const int32_t *obs_idx,
                    void *logw_out, int64_t M, int64_t N, const uint32_t *keys, uint32_t t,
                    const double *z_tape, uint32_t *status, void *stream);
int pf_fhn_interval_ex(const pf_fhn_params *p, pf_dtype dtype, const void *x_in,
                       const int32_t *anc, void *x_out, const double *y, const int32_t *obs_idx,
                       void *logw_out, int64_t M, int64_t N, const uint32_t *keys, uint32_t t,
                       const double *z_tape, uint32_t *status, uint32_t flags, void *stream);

/* normalize_log_weights + multinomial_resample_indices for M segments
 * (core.py:116-138, resampling.py:21-43, accel.py:175-203):
 * per-filter max / exp / sum in fp64, w = e/total, fp64 inclusive scan,
 * sorted uniforms (u_tape (M,N) fp64, or Philox exponential spacings with an
 * fp64 scan), merge -> anc_out[f*N + j] = f*N + k (int32, non-decreasing).
 * lnc[f] += m + log(total) - log(N) unless collapsed.  ws may be NULL when
 * pf_resample_workspace_bytes() returns 0. */
size_t pf_resample_workspace_bytes(int64_t M, int64_t N);
int pf_segmented_resample(pf_dtype logw_dtype, const void *logw, int64_t M, int64_t N,
                          const double *u_tape, const uint32_t *keys, uint32_t t,
                          int32_t *anc_out, double *lnc, uint8_t *collapsed, uint32_t *status,
                          void *ws, size_t ws_bytes, void *stream);

/* pf_segmented_resample with options (filters.py:111, resampling.py:29-43):
 *  - x_in/x_out/dims (nullable): fused ancestor gather of a planar fp32 state,
 *    x_out[d][p] = x_in[d][anc[p]] (BASELINE cfg1);
 *  - flags & PF_RS_REFERENCE_ORDER: build the CDF in the reference's exact
 *    floating-point order (numpy pairwise sum for the total, IEEE division,
 *    strictly sequential cumsum) so ancestors are bit-identical to the
 *    reference's for identical uniforms (oracle mode; slower). */
#define PF_RS_REFERENCE_ORDER 1u
/* Wide (N > 8192) production pipeline alternatives, same ancestors:
 * PF_RS_WIDE_MERGE_PATH merges by merge path instead of the per-thread
 * search; PF_RS_WIDE_GATHER_SEPARATE runs the ancestor gather as its own
 * pass instead of fusing it into the merge's write-out. */
#define PF_RS_WIDE_MERGE_PATH 2u
#define PF_RS_WIDE_GATHER_SEPARATE 4u
/* fp32 log weights, production: no materialised fp64 CDF - the merge
 * recomputes the CDF of the weight tiles its uniforms fall into (less HBM
 * traffic, more instructions; same ancestors). */
#define PF_RS_WIDE_RECOMPUTE 8u
int pf_segmented_resample_ex(pf_dtype logw_dtype, const void *logw, int64_t M, int64_t N,
                             const double *u_tape, const uint32_t *keys, uint32_t t,
                             int32_t *anc_out, double *lnc, uint8_t *collapsed, uint32_t *status,
                             void *ws, size_t ws_bytes, const float *x_in, float *x_out,
                             int32_t dims, uint32_t flags, void *stream);

/* posterior_mean of the resampled set (core.py:154-156 via filters.py:188):
 * est[f*dim + d] = (1/N) * sum_j x(anc[f*N+j], d) in a fixed order, fp64,
 * with element (p, d) at x[p*stride_p + d*stride_d]. */
int pf_filter_estimate(pf_dtype dtype, const void *x, int64_t stride_p, int64_t stride_d,
                       int32_t dim, const int32_t *anc, int64_t M, int64_t N, double *est_out,
                       void *stream);
/* The same estimate for wide filters with dim <= 8 (e.g. the centralised
 * M=1 x N=2^22 Lorenz filter): fixed chunks of 16384 particles summed by one
 * CTA each, then the chunk partials in chunk order - bit-reproducible,
 * independent of M and the GPU count.  ws: pf_estimate_workspace_bytes(M, N,
 * dim) bytes (0 -> the one-CTA-per-filter kernel, ws unused). */
size_t pf_estimate_workspace_bytes(int64_t M, int64_t N, int32_t dim);
int pf_filter_estimate_ws(pf_dtype dtype, const void *x, int64_t stride_p, int64_t stride_d,
                          int32_t dim, const int32_t *anc, int64_t M, int64_t N, double *est_out,
                          int64_t est_stride, void *ws, size_t ws_bytes, void *stream);

/* pf_filter_estimate writing filter f's row at est_out + f*est_stride. */
int pf_filter_estimate_strided(pf_dtype dtype, const void *x, int64_t stride_p, int64_t stride_d,
                               int32_t dim, const int32_t *anc, int64_t M, int64_t N,
                               double *est_out, int64_t est_stride, void *stream);

/* average_estimates (ensemble.py:68-73): out[t][d] = (e_0 + e_1 + ...) / M,
 * left to right over filters, fp64.  est is (T, M, dim), out is (T, dim). */
int pf_ensemble_average(const double *est, int64_t T, int64_t M, int64_t dim, double *out,
                        void *stream);

/* ---- FH-N network (models/fhn.py:85-207) ------------------------------- */
/* One transition of the network model for M*N particles (sample_transition
 * fhn.py:153-192, or transition_point_prediction when p->stochastic == 0):
 * x_out/q_out[p] = step(x_in/q_in[anc[p]]) (anc NULL = identity), and when
 * logw_out != NULL the zone log-likelihood of y (n_obs doubles at obs_idx,
 * fhn.py:199-207).  Draws: stim_tape (M, 2, N) fp64 [fire, select uniforms]
 * plus z_tape (M, N, J*J) fp64 normals (oracle mode), or Philox (both NULL). */
int pf_fhnnet_step(const pf_fhnnet_params *p, pf_dtype dtype, const void *x_in,
                   const uint32_t *q_in, const int32_t *anc, void *x_out, uint32_t *q_out,
                   const double *forcing_mask, const double *y, const int32_t *obs_idx,
                   void *logw_out, int64_t M, int64_t N, const uint32_t *keys, uint32_t t,
                   const double *stim_tape, const double *z_tape, uint32_t *status,
                   void *stream);
int pf_fhnnet_step_ex(const pf_fhnnet_params *p, pf_dtype dtype, const void *x_in,
                      const uint32_t *q_in, const int32_t *anc, void *x_out, uint32_t *q_out,
                      const double *forcing_mask, const double *y, const int32_t *obs_idx,
                      void *logw_out, int64_t M, int64_t N, const uint32_t *keys, uint32_t t,
                      const double *stim_tape, const double *z_tape, uint32_t *status,
                      uint32_t flags, void *stream);
/* Reference state rows (n, (2 + hold) * nodes) fp64 [U, V, Q(t) .. Q(t-hold+1)]
 * <-> device planes + history bits (fhn.py:122-138 unpack/pack).  Q entries
 * are indicators; any nonzero value packs as 1.  unpack gathers rows anc[p]
 * when anc != NULL. */
int pf_fhnnet_pack(pf_dtype dtype, const double *rows, int64_t n, int32_t nodes, int32_t hold,
                   void *x, uint32_t *q, void *stream);
int pf_fhnnet_unpack(pf_dtype dtype, const void *x, const uint32_t *q, const int32_t *anc,
                     int64_t n, int32_t nodes, int32_t hold, double *rows, void *stream);
/* Zone log-likelihood of stored states (fhn.py:199-207): out[r] (fp64) =
 * -0.5/obs_var * sum_i (y[i] - x[r*row_stride + obs_idx[i]])^2, numpy order. */
int pf_zone_loglik(pf_dtype dtype, const void *x, int64_t n, int64_t row_stride,
                   const int32_t *obs_idx, int32_t n_obs, const double *y, double obs_var,
                   double *out, void *stream);
/* posterior_mean of the history indicators over the resampled set:
 * est[f*est_stride + k*nodes + node] = (1/N) #{j : bit k of q[anc[f*N+j]][node]}. */
int pf_bits_estimate(const uint32_t *q, int32_t nodes, int32_t nbits, const int32_t *anc,
                     int64_t M, int64_t N, double *est, int64_t est_stride, void *stream);

/* ---- small-state verification models (models/hmm.py, linear_gaussian.py) */
/* State planes x[d*M*N + p].  HMM draws: one uniform per particle and step
 * (u_tape (M,N) fp64 in oracle mode); LGM draws: dim_x normals (z_tape
 * (M,N,dx) fp64).  logw_out NULL skips the weights. */
int pf_hmm_prior(const pf_hmm_params *h, pf_dtype dtype, void *x, int64_t M, int64_t N,
                 const uint32_t *keys, const double *u_tape, void *stream);
int pf_hmm_propagate_weight(const pf_hmm_params *h, pf_dtype dtype, const void *x_in,
                            const int32_t *anc, void *x_out, const double *y, void *logw_out,
                            int64_t M, int64_t N, const uint32_t *keys, uint32_t t,
                            const double *u_tape, uint32_t *status, void *stream);
int pf_lgm_prior(const pf_lgm_params *g, pf_dtype dtype, void *x, int64_t M, int64_t N,
                 const uint32_t *keys, const double *z_tape, void *stream);
int pf_lgm_propagate_weight(const pf_lgm_params *g, pf_dtype dtype, const void *x_in,
                            const int32_t *anc, void *x_out, const double *y, void *logw_out,
                            int64_t M, int64_t N, const uint32_t *keys, uint32_t t,
                            const double *z_tape, uint32_t *status, void *stream);
/* DiscreteHmm.log_likelihood of n stored fp64 states: log_emission[x[r], y[0]]. */
int pf_hmm_loglik(const pf_hmm_params *h, const double *x, int64_t n, const double *y,
                  double *out, void *stream);
/* LinearGaussianModel.log_likelihood of n stored fp64 states (planes x[d*n + r]). */
int pf_lgm_loglik(const pf_lgm_params *g, const double *x, int64_t n, const double *y,
                  double *out, void *stream);

/* ---- double bootstrap: islands = the bank's filters (filters.py:201-313) - */
/* log_weights[m] += lnc[m] - lnc_old[m]  (dbf_step, filters.py:253-256). */
int pf_island_accumulate(double *log_weights, const double *lnc, const double *lnc_old,
                         int64_t M, void *stream);
/* Whole-island resampling (filters.py:258-263): island m takes island
 * idx[m]'s ancestors (so the next propagate gathers its particles), lnc and
 * collapse flag; log_weights := 0.  idx comes from a 1-segment
 * pf_segmented_resample_ex over the M island log-weights; *_tmp are
 * caller-provided scratch of the same sizes. */
int pf_island_copy(const int32_t *idx, int32_t *anc, double *lnc, uint8_t *collapsed,
                   double *log_weights, int64_t M, int64_t N, int32_t *anc_tmp,
                   double *lnc_tmp, uint8_t *coll_tmp, void *stream);
/* pooled_estimate (filters.py:229-234): out[d] = sum_m p_m est[m*est_stride+d]
 * with p = softmax(log_weights) in numpy order; M <= 4096. */
int pf_island_pool(const double *est, int64_t est_stride, int64_t M, int64_t dim,
                   const double *log_weights, double *out, void *stream);
/* out[0] = max + log(sum exp(lnc - max)) - log(M)  (filters.py:301-303). */
int pf_island_trace(const double *lnc, int64_t M, double *out, void *stream);

/* ---- multi-GPU estimate exchange (NCCL) --------------------
 * Replaces the reference's fork pool + pickled per-filter estimates
 * (ensemble.py:96-108).  One communicator per process group; rank 0 makes
 * the id, the caller broadcasts it (torch.distributed), every rank calls
 * pf_comm_init concurrently.  NCCL is bound at run time (the libnccl.so.2
 * torch loaded); pf_comm_available() == 0 when it cannot be found.
 * All-reduces run on the communicator's side stream after an event of the
 * given stream; pf_comm_join makes `stream` wait for every exchange issued
 * so far (no host wait). */
#define PF_COMM_ID_BYTES 128
typedef struct pf_comm pf_comm;
int pf_comm_available(void);
int pf_comm_nccl_version(void);
int pf_comm_unique_id(uint8_t *id_out /* PF_COMM_ID_BYTES */);
int pf_comm_init(const uint8_t *id, int32_t nranks, int32_t rank, pf_comm **out);
int pf_comm_destroy(pf_comm *c);
/* in-place sum over ranks of count doubles, ordered after `stream`'s work;
 * `stream` waits for the result */
int pf_comm_allreduce_f64(pf_comm *c, double *buf, int64_t count, void *stream);
/* the per-observation exchanges of steps k0..k0+n_steps-1 of an estimate
 * trace est[k*step_stride .. +count) without running a bank (a rank that
 * owns no filters still joins every collective) */
int pf_comm_exchange_steps(pf_comm *c, double *est, int64_t step_stride, int64_t count,
                           int32_t k0, int32_t n_steps, void *stream);
int pf_comm_join(pf_comm *c, void *stream);

/* ---- native bank driver ------------------------------------------------ */
/* Production-mode (Philox) bootstrap bank: runs observations k0..k0+n-1 back
 * to back (propagate+weight, segmented resample, estimate, lnc/collapse trace
 * copies per observation) without returning to the host - the loop of
 * run_filter (filters.py:184-191) for every filter at once.  `cur` is the
 * index of the state buffer holding the current particles; after the call the
 * current buffer is cur ^ (n_steps & 1).  have_ancestors = 0 on the first
 * interval (the prior has no ancestors). */
#define PF_MODEL_LORENZ 0
#define PF_MODEL_FHN 1
#define PF_MODEL_FHNNET 2
#define PF_MODEL_HMM 3
#define PF_MODEL_LGM 4
/* Double bootstrap (filters.py:201-313) in the native driver, single process:
 * the bank's M filters are the islands.  After each interval's resample the
 * island log weights gain lnc - lnc_before (pf_island_accumulate); every
 * `period` intervals (t % period == 0) the islands are resampled by them
 * (one segment of M, island Philox key, time word t) and island m takes island
 * idx[m]'s ancestors, lnc and collapse flag (pf_island_copy) - before the
 * interval's estimate; after it, the pooled estimate row and the logmeanexp
 * trace entry (pf_island_pool / pf_island_trace). */
typedef struct pf_island_desc {
  int32_t period;
  const uint32_t *key; /* (2) island-level Philox key */
  double *lw;          /* (M) accumulated island log weights */
  double *lnc_old;     /* (M) scratch */
  int32_t *idx;        /* (M) scratch: selected islands */
  int32_t *anc_tmp;    /* (M*N) scratch */
  double *lnc_tmp;     /* (M) scratch */
  uint8_t *coll_tmp;   /* (M) scratch */
  double *s_lnc;       /* (1) island-resample outputs */
  uint8_t *s_coll;
  uint32_t *s_status;
  void *ws; /* pf_resample_workspace_bytes(1, M) bytes */
  size_t ws_bytes;
  double *pool;     /* (T, pool_dim): pooled estimate of observation k at pool + k*pool_dim */
  double *trace;    /* (T) */
  int32_t pool_dim; /* estimate columns pooled per island row (<= the row stride; the
                       FH-N network's rows carry the history-bit means after the state) */
} pf_island_desc;

typedef struct pf_bank_desc {
  int32_t model; /* PF_MODEL_* */
  pf_dtype dtype;
  int64_t M, N;
  const pf_lorenz_params *lorenz; /* host */
  const pf_fhn_params *fhn;       /* host */
  const int32_t *obs_idx;         /* FH-N electrodes */
  void *x[2];                     /* state double buffer */
  void *logw;
  int32_t *anc;
  double *lnc;
  uint8_t *collapsed;
  uint32_t *status;
  const uint32_t *keys;
  void *ws;
  size_t ws_bytes;
  const double *obs; /* (T, dim_y) */
  int32_t dim_y;
  double *est; /* step k's estimates at est + k*est_step_stride + est_offset */
  int64_t est_step_stride, est_offset, est_stride_p, est_stride_d;
  int32_t est_dim;
  double *lnc_trace;        /* (T, M) or NULL */
  uint8_t *collapsed_trace; /* (T, M) or NULL */
  float *prop_ms; /* host (n_steps) or NULL: propagate-kernel durations; the call then
                     waits for the last propagate to finish before returning */
  /* FH-N network only */
  const pf_fhnnet_params *fhnnet; /* host */
  uint32_t *q[2];                 /* stimulus-history double buffer */
  const double *forcing_mask;     /* (J*J) */
  int64_t est_stride_f; /* distance between filters' estimate rows (0 = est_dim) */
  int32_t est_bits;     /* > 0: history bit means written after the est_dim state means */
  const pf_hmm_params *hmm; /* host */
  const pf_lgm_params *lgm; /* host */
  float *step_ms; /* host (n_steps) or NULL: whole-interval durations (waits like prop_ms) */
  void **events;  /* host array of 4*n_steps caller-created timing cudaEvent_t, or NULL:
                     recorded at each interval's start, around its (main) propagate kernel
                     and at its end; nothing waits (the caller reads the times) */
  /* auxiliary particle filter (filters.py:115-154): variant = 1 runs apf_step per
   * interval with the noise-free params0 (same struct type as the model's) */
  int32_t variant;
  const void *params0;
  void *lam;           /* (M*N) first-stage log weights, logw dtype */
  int32_t *anc1;       /* (M*N) first-stage ancestors */
  int32_t *anc_comp;   /* (M*N) composed state rows */
  void *x_tmp;         /* lookahead states, like x[0] */
  uint32_t *q_tmp;     /* FH-N network lookahead history */
  double *lnc_before;  /* (M) */
  uint8_t *coll1;      /* (M) first-stage collapse flags */
  uint32_t kernel_flags; /* PF_KERNEL_* for the propagate launches (0 = production) */
  /* multi-GPU: after observation k's estimate, all-reduce the exch_count
   * doubles at est + k*est_step_stride (the disjoint-support (M_total, width)
   * block) over comm; NULL / 0 = single process */
  pf_comm *comm;
  int64_t exch_count;
  /* nonzero: pf_bank_run captures its intervals into one CUDA graph and
   * launches it when n_steps >= 32 (1: the default threshold) or >= use_graph
   * (> 1) - launch-bound small banks; shorter runs enqueue directly, since the
   * capture and instantiation cost ~0.5 ms; ignored with comm */
  int32_t use_graph;
  /* non-NULL: double bootstrap islands (variant 0, single process, no comm) */
  const pf_island_desc *islands;
} pf_bank_desc;
int pf_bank_run(const pf_bank_desc *d, int32_t k0, int32_t n_steps, int32_t cur,
                int32_t have_ancestors, void *stream);

/* The same intervals as pf_bank_run(d, k0, n_steps, cur, have_ancestors)
 * captured once (on `stream`) into an instantiated CUDA graph; each
 * pf_bank_graph_launch enqueues all of them.  The descriptor's buffers are
 * baked in; d->events (if any) are recorded by the graph; comm and
 * host-read timing (prop_ms/step_ms) are not allowed. */
typedef struct pf_bank_graph pf_bank_graph;
int pf_bank_graph_create(const pf_bank_desc *d, int32_t k0, int32_t n_steps, int32_t cur,
                         int32_t have_ancestors, void *stream, pf_bank_graph **out);
int pf_bank_graph_launch(pf_bank_graph *g, void *stream);
int pf_bank_graph_destroy(pf_bank_graph *g);

/* ---- auxiliary particle filter glue (filters.py:115-154) --------------- */
/* First stage: filters whose lambda are all -inf get lambda := 0 (uniform
 * first-stage weights, log_mean_first = 0, filters.py:136-140); coll1[f]=1. */
int pf_apf_first_stage_prepare(pf_dtype dtype, void *lam, int64_t M, int64_t N, uint8_t *coll1,
                               void *stream);
/* out[j] = inner ? inner[outer[j]] : outer[j]  (state rows of the chosen
 * first-stage ancestors: particles[ancestors] of filters.py:142). */
int pf_compose_ancestors(const int32_t *outer, const int32_t *inner, int64_t MN, int32_t *out,
                         void *stream);
/* logw[j] -= lam[anc1[j]]  (filters.py:143). */
int pf_apf_second_stage_weights(pf_dtype dtype, void *logw, const void *lam, const int32_t *anc1,
                                int64_t MN, void *stream);
/* After the second resampling: a second-stage collapse restores
 * lnc_before (filters.py:146-148); collapsed |= collapsed_first. */
int pf_apf_finish(double *lnc, const double *lnc_before, uint8_t *collapsed,
                  const uint8_t *collapsed_first, int64_t M, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* PFBANK_H */
