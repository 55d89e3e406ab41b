// Native bank driver: runs observation intervals back to back from C++.
//
// The per-observation loop of run_filter (filters.py:184-191) and the
// per-filter loop of run_ensemble (ensemble.py:96-99) collapse into one call
// that enqueues, for each observation t, the propagate+weight kernel, the
// segmented resample, the estimate and two trace copies - no host round trip
// and no Python in between, so launch-bound configurations (small banks)
// run at the device's launch rate.
#include "common.cuh"

#include <vector>

extern "C" int pf_lorenz_propagate_weight(const pf_lorenz_params *, pf_dtype, const void *,
                                          const int32_t *, void *, const double *, void *,
                                          int64_t, int64_t, const uint32_t *, uint32_t,
                                          const double *, uint32_t *, void *);
extern "C" int pf_fhnnet_step(const pf_fhnnet_params *, pf_dtype, const void *, const uint32_t *,
                              const int32_t *, void *, uint32_t *, const double *, const double *,
                              const int32_t *, void *, int64_t, int64_t, const uint32_t *,
                              uint32_t, const double *, const double *, uint32_t *, void *);
extern "C" int pf_fhn_interval(const pf_fhn_params *, pf_dtype, const void *, const int32_t *,
                               void *, const double *, const int32_t *, void *, int64_t, int64_t,
                               const uint32_t *, uint32_t, const double *, uint32_t *, void *);

using namespace pf;

extern "C" {

int pf_bank_run(const pf_bank_desc *d, int32_t k0, int32_t n_steps, int32_t cur,
                int32_t have_ancestors, void *stream) {
  PF_REQUIRE(d && n_steps >= 0 && k0 >= 0 && (cur == 0 || cur == 1), "pf_bank_run: bad arguments");
  PF_REQUIRE(d->model == PF_MODEL_LORENZ
                 ? d->lorenz != nullptr
                 : d->model == PF_MODEL_FHN
                       ? (d->fhn && d->obs_idx)
                       : d->model == PF_MODEL_FHNNET
                             ? (d->fhnnet && d->obs_idx && d->q[0] && d->q[1] && d->forcing_mask)
                             : d->model == PF_MODEL_HMM ? d->hmm != nullptr
                                                        : (d->model == PF_MODEL_LGM && d->lgm),
             "pf_bank_run: model descriptor missing");
  PF_REQUIRE(d->x[0] && d->x[1] && d->logw && d->anc && d->lnc && d->collapsed && d->status &&
                 d->keys && d->obs && d->est,
             "pf_bank_run: null buffer");
  const cudaStream_t s = as_stream(stream);
  const int64_t MN = d->M * d->N;
  // optional per-interval timing (events on the launch stream): start of the
  // interval, end of the propagate kernel (the dominant one), end of the interval
  struct Events {
    std::vector<cudaEvent_t> e;
    ~Events() {
      for (cudaEvent_t x : e) cudaEventDestroy(x);
    }
  } evs;
  cudaEvent_t *ev = nullptr;
  if (d->events && n_steps > 0) {
    // caller-owned, pre-created timing events: record only, no host wait
    ev = reinterpret_cast<cudaEvent_t *>(d->events);
  } else if ((d->prop_ms || d->step_ms) && n_steps > 0) {
    evs.e.resize(3 * static_cast<size_t>(n_steps));
    for (auto &x : evs.e) cudaEventCreate(&x);
    ev = evs.e.data();
  }
  // planar states (x[d*MN + p]): the estimate is fused into the resampler
  const bool planar = d->model == PF_MODEL_LORENZ || d->model == PF_MODEL_HMM ||
                      d->model == PF_MODEL_LGM;
  for (int32_t i = 0; i < n_steps; ++i) {
    const int32_t k = k0 + i;
    const uint32_t t = static_cast<uint32_t>(k + 1);
    const void *xin = d->x[cur];
    void *xout = d->x[cur ^ 1];
    const int32_t *anc = (have_ancestors || i > 0) ? d->anc : nullptr;
    const double *y = d->obs + static_cast<int64_t>(k) * d->dim_y;
    int rc;
    if (ev) cudaEventRecord(ev[3 * i], s);
    if (d->model == PF_MODEL_LORENZ)
      rc = pf_lorenz_propagate_weight(d->lorenz, d->dtype, xin, anc, xout, y, d->logw, d->M, d->N,
                                      d->keys, t, nullptr, d->status, stream);
    else if (d->model == PF_MODEL_HMM)
      rc = pf_hmm_propagate_weight(d->hmm, d->dtype, xin, anc, xout, y, d->logw, d->M, d->N,
                                   d->keys, t, nullptr, d->status, stream);
    else if (d->model == PF_MODEL_LGM)
      rc = pf_lgm_propagate_weight(d->lgm, d->dtype, xin, anc, xout, y, d->logw, d->M, d->N,
                                   d->keys, t, nullptr, d->status, stream);
    else if (d->model == PF_MODEL_FHNNET)
      rc = pf_fhnnet_step(d->fhnnet, d->dtype, xin, d->q[cur], anc, xout, d->q[cur ^ 1],
                          d->forcing_mask, y, d->obs_idx, d->logw, d->M, d->N, d->keys, t,
                          nullptr, nullptr, d->status, stream);
    else
      rc = pf_fhn_interval(d->fhn, d->dtype, xin, anc, xout, y, d->obs_idx, d->logw, d->M, d->N,
                           d->keys, t, nullptr, d->status, stream);
    if (ev) cudaEventRecord(ev[3 * i + 1], s);
    if (rc) return rc;
    double *est = d->est + static_cast<int64_t>(k) * d->est_step_stride + d->est_offset;
    const int64_t est_f0 = d->est_stride_f ? d->est_stride_f : d->est_dim;
    bool fused = false;
    if (planar && d->est_stride_p == 1 && d->est_stride_d == MN)
      rc = segmented_resample_fused(d->dtype, d->logw, d->M, d->N, d->keys, t, d->anc, d->lnc,
                                    d->collapsed, d->status, d->ws, d->ws_bytes, xout,
                                    d->est_dim, est, est_f0, s, &fused);
    else
      rc = pf_segmented_resample_ex(d->dtype, d->logw, d->M, d->N, nullptr, d->keys, t, d->anc,
                                    d->lnc, d->collapsed, d->status, d->ws, d->ws_bytes, nullptr,
                                    nullptr, 0, 0u, stream);
    if (rc) return rc;
    const int64_t est_f = est_f0;
    if (!fused) {
      rc = pf_filter_estimate_strided(d->dtype, xout, d->est_stride_p, d->est_stride_d,
                                      d->est_dim, d->anc, d->M, d->N, est, est_f, stream);
      if (rc) return rc;
    }
    if (d->model == PF_MODEL_FHNNET && d->est_bits > 0) {
      const int32_t nodes = d->fhnnet->J * d->fhnnet->J;
      rc = pf_bits_estimate(d->q[cur ^ 1], nodes, d->est_bits, d->anc, d->M, d->N,
                            est + d->est_dim, est_f, stream);
      if (rc) return rc;
    }
    if (d->lnc_trace &&
        cudaMemcpyAsync(d->lnc_trace + static_cast<int64_t>(k) * d->M, d->lnc,
                        d->M * sizeof(double), cudaMemcpyDeviceToDevice, s) != cudaSuccess)
      return check_launch("pf_bank_run(lnc trace)");
    if (d->collapsed_trace &&
        cudaMemcpyAsync(d->collapsed_trace + static_cast<int64_t>(k) * d->M, d->collapsed,
                        d->M * sizeof(uint8_t), cudaMemcpyDeviceToDevice, s) != cudaSuccess)
      return check_launch("pf_bank_run(collapse trace)");
    if (ev) cudaEventRecord(ev[3 * i + 2], s);
    cur ^= 1;
  }
  (void)MN;
  if (ev && !d->events) {
    cudaEventSynchronize(ev[3 * n_steps - 1]);
    for (int32_t i = 0; i < n_steps; ++i) {
      if (d->prop_ms) cudaEventElapsedTime(&d->prop_ms[i], ev[3 * i], ev[3 * i + 1]);
      if (d->step_ms) cudaEventElapsedTime(&d->step_ms[i], ev[3 * i], ev[3 * i + 2]);
    }
  }
  return check_launch("pf_bank_run");
}

}  // extern "C"
