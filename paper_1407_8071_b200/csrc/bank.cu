// Native bank driver: runs observation intervals back to back from C++.
//
// The per-observation loop of run_filter (filters.py:184-191) and the
// per-filter loop of run_ensemble (ensemble.py:96-99) collapse into one call
// that enqueues, for each observation t, the propagate+weight kernel, the
// segmented resample, the estimate and two trace copies - no host round trip
// and no Python in between, so launch-bound configurations (small banks)
// run at the device's launch rate.
#include "common.cuh"

#include <mutex>
#include <vector>

using namespace pf;

// One propagate+weight launch of the descriptor's model with the given
// (host) parameter struct - the bank's params or the auxiliary filter's
// noise-free params0.
static int bank_propagate(const pf_bank_desc *d, const void *params, const void *xin,
                          const uint32_t *qin, const int32_t *anc, void *xout, uint32_t *qout,
                          const double *y, void *logw, uint32_t t, void *stream) {
  switch (d->model) {
    case PF_MODEL_LORENZ:
      return pf_lorenz_propagate_weight_ex(static_cast<const pf_lorenz_params *>(params),
                                           d->dtype, xin, anc, xout, y, logw, d->M, d->N, d->keys,
                                           t, nullptr, d->status, d->kernel_flags, stream);
    case PF_MODEL_HMM:
      return pf_hmm_propagate_weight(static_cast<const pf_hmm_params *>(params), d->dtype, xin,
                                     anc, xout, y, logw, d->M, d->N, d->keys, t, nullptr,
                                     d->status, stream);
    case PF_MODEL_LGM:
      return pf_lgm_propagate_weight(static_cast<const pf_lgm_params *>(params), d->dtype, xin,
                                     anc, xout, y, logw, d->M, d->N, d->keys, t, nullptr,
                                     d->status, stream);
    case PF_MODEL_FHNNET:
      return pf_fhnnet_step_ex(static_cast<const pf_fhnnet_params *>(params), d->dtype, xin,
                               qin, anc, xout, qout, d->forcing_mask, y, d->obs_idx, logw, d->M,
                               d->N, d->keys, t, nullptr, nullptr, d->status, d->kernel_flags,
                               stream);
    default:
      return pf_fhn_interval_ex(static_cast<const pf_fhn_params *>(params), d->dtype, xin, anc,
                                xout, y, d->obs_idx, logw, d->M, d->N, d->keys, t, nullptr,
                                d->status, d->kernel_flags, stream);
  }
}

static const void *bank_params(const pf_bank_desc *d) {
  switch (d->model) {
    case PF_MODEL_LORENZ: return d->lorenz;
    case PF_MODEL_HMM: return d->hmm;
    case PF_MODEL_LGM: return d->lgm;
    case PF_MODEL_FHNNET: return d->fhnnet;
    default: return d->fhn;
  }
}

namespace {

int bank_validate(const pf_bank_desc *d, int32_t k0, int32_t n_steps, int32_t cur) {
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
  PF_REQUIRE(!d->islands ||
                 (d->variant == 0 && !d->comm && d->islands->period >= 1 && d->islands->key &&
                  d->islands->lw && d->islands->lnc_old && d->islands->idx &&
                  d->islands->anc_tmp && d->islands->lnc_tmp && d->islands->coll_tmp &&
                  d->islands->s_lnc && d->islands->s_coll && d->islands->s_status &&
                  d->islands->pool && d->islands->trace && d->islands->pool_dim >= 1 &&
                  (d->est_stride_f == 0 ? d->islands->pool_dim <= d->est_dim
                                        : d->islands->pool_dim <= d->est_stride_f)),
             "pf_bank_run: islands need variant 0, no comm and every island buffer");
  PF_REQUIRE(d->variant != 1 || (d->params0 && d->lam && d->anc1 && d->anc_comp && d->x_tmp &&
                                 d->lnc_before && d->coll1 &&
                                 (d->model != PF_MODEL_FHNNET || d->q_tmp)),
             "pf_bank_run: auxiliary variant needs params0 and the APF scratch buffers");
  return PF_OK;
}

// Enqueue observations k0..k0+n_steps-1 on stream s (directly, or into a
// graph being captured on s).  ev: NULL or 4 timing events per interval.
int bank_enqueue(const pf_bank_desc *d, int32_t k0, int32_t n_steps, int32_t cur,
                        int32_t have_ancestors, cudaStream_t s, cudaEvent_t *ev) {
  void *stream = s;
  const int64_t MN = d->M * d->N;
  // inside a graph capture a plain event record only orders captured work;
  // timing events must become external event-record nodes of the graph
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cap);
  const unsigned rec_flags =
      cap == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : cudaEventRecordDefault;
  const bool apf = d->variant == 1;
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
    if (ev) cudaEventRecordWithFlags(ev[4 * i], s, rec_flags);
    uint32_t *qin = d->q[cur], *qout = d->q[cur ^ 1];
    const int32_t *src_anc = anc;
    if (apf) {
      // first stage (filters.py:126-141): lambda = log p(y | noise-free prediction),
      // all -inf -> lambda = 0 (flagged), resample by lambda with a distinct
      // Philox time word, compose with the previous ancestors
      rc = bank_propagate(d, d->params0, xin, qin, anc, d->x_tmp, d->q_tmp, y, d->lam, t, stream);
      if (rc) return rc;
      rc = pf_apf_first_stage_prepare(d->dtype, d->lam, d->M, d->N, d->coll1, stream);
      if (rc) return rc;
      if (cudaMemcpyAsync(d->lnc_before, d->lnc, d->M * sizeof(double),
                          cudaMemcpyDeviceToDevice, s) != cudaSuccess)
        return check_launch("pf_bank_run(apf lnc)");
      rc = pf_segmented_resample_ex(d->dtype, d->lam, d->M, d->N, nullptr, d->keys,
                                    t | 0x80000000u, d->anc1, d->lnc, d->collapsed, d->status,
                                    d->ws, d->ws_bytes, nullptr, nullptr, 0, 0u, stream);
      if (rc) return rc;
      rc = pf_compose_ancestors(d->anc1, anc, MN, d->anc_comp, stream);
      if (rc) return rc;
      src_anc = d->anc_comp;
    }
    const pf_island_desc *isl = d->islands;
    if (isl && cudaMemcpyAsync(isl->lnc_old, d->lnc, d->M * sizeof(double),
                               cudaMemcpyDeviceToDevice, s) != cudaSuccess)
      return check_launch("pf_bank_run(island lnc)");
    if (ev) cudaEventRecordWithFlags(ev[4 * i + 1], s, rec_flags);
    rc = bank_propagate(d, bank_params(d), xin, qin, src_anc, xout, qout, y, d->logw, t, stream);
    if (!rc && apf)  // second stage weights log w - lambda[anc1] (filters.py:143)
      rc = pf_apf_second_stage_weights(d->dtype, d->logw, d->lam, d->anc1, MN, stream);
    if (ev) cudaEventRecordWithFlags(ev[4 * i + 2], s, rec_flags);
    if (rc) return rc;
    double *est = d->est + static_cast<int64_t>(k) * d->est_step_stride + d->est_offset;
    const int64_t est_f0 = d->est_stride_f ? d->est_stride_f : d->est_dim;
    bool fused = false;
    // planar states: estimate and both trace rows written by the resampler
    // itself (one launch per interval besides the propagate)
    double *lnc_row = d->lnc_trace ? d->lnc_trace + static_cast<int64_t>(k) * d->M : nullptr;
    uint8_t *coll_row =
        d->collapsed_trace ? d->collapsed_trace + static_cast<int64_t>(k) * d->M : nullptr;
    // (the auxiliary filter finishes lnc / collapse after the resample: its
    // trace rows are copied afterwards)
    // (islands: the estimate follows the island copy, so it is not fused)
    if (planar && d->est_stride_p == 1 && d->est_stride_d == MN && !isl)
      rc = segmented_resample_fused(d->dtype, d->logw, d->M, d->N, d->keys, t, d->anc, d->lnc,
                                    d->collapsed, d->status, d->ws, d->ws_bytes, xout,
                                    d->est_dim, est, est_f0, apf ? nullptr : lnc_row,
                                    apf ? nullptr : coll_row, s, &fused);
    else
      rc = pf_segmented_resample_ex(d->dtype, d->logw, d->M, d->N, nullptr, d->keys, t, d->anc,
                                    d->lnc, d->collapsed, d->status, d->ws, d->ws_bytes, nullptr,
                                    nullptr, 0, 0u, stream);
    if (rc) return rc;
    if (apf) {  // a second-stage collapse restores the pre-step lnc (filters.py:146-148)
      rc = pf_apf_finish(d->lnc, d->lnc_before, d->collapsed, d->coll1, d->M, stream);
      if (rc) return rc;
    }
    if (isl) {  // double bootstrap: island weights, and the island step (filters.py:245-265)
      rc = pf_island_accumulate(isl->lw, d->lnc, isl->lnc_old, d->M, stream);
      if (!rc && t % static_cast<uint32_t>(isl->period) == 0) {
        rc = pf_segmented_resample_ex(PF_F64, isl->lw, 1, d->M, nullptr, isl->key, t, isl->idx,
                                      isl->s_lnc, isl->s_coll, isl->s_status, isl->ws,
                                      isl->ws_bytes, nullptr, nullptr, 0, 0u, stream);
        if (!rc)
          rc = pf_island_copy(isl->idx, d->anc, d->lnc, d->collapsed, isl->lw, d->M, d->N,
                              isl->anc_tmp, isl->lnc_tmp, isl->coll_tmp, stream);
      }
      if (rc) return rc;
    }
    const int64_t est_f = est_f0;
    if (!fused) {
      // the resampler is done with the workspace: wide filters use it for
      // their chunked estimate partials
      rc = pf_filter_estimate_ws(d->dtype, xout, d->est_stride_p, d->est_stride_d, d->est_dim,
                                 d->anc, d->M, d->N, est, est_f, d->ws, d->ws_bytes, stream);
      if (rc) return rc;
    }
    if (d->model == PF_MODEL_FHNNET && d->est_bits > 0) {
      const int32_t nodes = d->fhnnet->J * d->fhnnet->J;
      rc = pf_bits_estimate(d->q[cur ^ 1], nodes, d->est_bits, d->anc, d->M, d->N,
                            est + d->est_dim, est_f, stream);
      if (rc) return rc;
    }
    // multi-GPU: this observation's disjoint-support estimate block, summed
    // over ranks on the communicator's side stream (overlaps the next interval)
    if (d->comm && d->exch_count > 0) {
      rc = comm_allreduce_after(d->comm, d->est + static_cast<int64_t>(k) * d->est_step_stride,
                                d->exch_count, s);
      if (rc) return rc;
    }
    if (isl) {  // pooled estimate and logmeanexp trace of observation k
      rc = pf_island_pool(est, est_f, d->M, isl->pool_dim, isl->lw,
                          isl->pool + static_cast<int64_t>(k) * isl->pool_dim, stream);
      if (!rc) rc = pf_island_trace(d->lnc, d->M, isl->trace + k, stream);
      if (rc) return rc;
    }
    const bool traced = fused && !apf;  // rows already written by the resampler
    if (!traced && lnc_row &&
        cudaMemcpyAsync(lnc_row, d->lnc, d->M * sizeof(double), cudaMemcpyDeviceToDevice, s) !=
            cudaSuccess)
      return check_launch("pf_bank_run(lnc trace)");
    if (!traced && coll_row &&
        cudaMemcpyAsync(coll_row, d->collapsed, d->M * sizeof(uint8_t), cudaMemcpyDeviceToDevice,
                        s) != cudaSuccess)
      return check_launch("pf_bank_run(collapse trace)");
    if (ev) cudaEventRecordWithFlags(ev[4 * i + 3], s, rec_flags);
    cur ^= 1;
  }
  (void)MN;
  return PF_OK;
}

}  // namespace

// An instantiated CUDA graph of n_steps intervals (launch-bound banks: one
// graph launch replaces ~4 launches per observation and their host costs).
constexpr int32_t kGraphMinSteps = 32;
struct pf_bank_graph {
  cudaGraphExec_t exec = nullptr;
  int32_t n_steps = 0;
};

namespace {

// Capture runs on a private stream (the caller's may be the legacy default
// stream, which cannot capture); capturing executes nothing, and the graph
// is launched on the caller's stream, so stream order is the caller's.
cudaStream_t capture_stream() {
  thread_local cudaStream_t cs[16] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 16) return nullptr;
  if (!cs[dev]) cudaStreamCreateWithFlags(&cs[dev], cudaStreamNonBlocking);
  return cs[dev];
}

int graph_capture(const pf_bank_desc *d, int32_t k0, int32_t n_steps, int32_t cur,
                  int32_t have_ancestors, cudaStream_t, cudaEvent_t *ev, pf_bank_graph **out) {
  *out = nullptr;
  cudaGetLastError();
  const cudaStream_t s = capture_stream();
  if (!s || cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed) != cudaSuccess)
    return check_launch("pf_bank_graph: begin capture");
  const int rc = bank_enqueue(d, k0, n_steps, cur, have_ancestors, s, ev);
  cudaGraph_t g = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(s, &g);
  if (rc != PF_OK) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  if (ce != cudaSuccess || !g) return check_launch("pf_bank_graph: end capture");
  auto *bg = new pf_bank_graph();
  bg->n_steps = n_steps;
  const cudaError_t ie = cudaGraphInstantiate(&bg->exec, g, 0);
  cudaGraphDestroy(g);
  if (ie != cudaSuccess) {
    delete bg;
    return check_launch("pf_bank_graph: instantiate");
  }
  *out = bg;
  return PF_OK;
}

// Executable graphs of pf_bank_run calls: destroyed once their completion
// event has fired (checked at the next call), never while still running.
struct Retired {
  cudaGraphExec_t exec;
  cudaEvent_t done;
};
std::mutex g_retired_mu;
std::vector<Retired> g_retired;

void retire(cudaGraphExec_t exec, cudaStream_t s) {
  cudaEvent_t e = nullptr;
  cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  cudaEventRecord(e, s);
  std::lock_guard<std::mutex> lk(g_retired_mu);
  g_retired.push_back({exec, e});
}

void reap() {
  std::lock_guard<std::mutex> lk(g_retired_mu);
  for (size_t i = 0; i < g_retired.size();) {
    if (cudaEventQuery(g_retired[i].done) == cudaSuccess) {
      cudaGraphExecDestroy(g_retired[i].exec);
      cudaEventDestroy(g_retired[i].done);
      g_retired[i] = g_retired.back();
      g_retired.pop_back();
    } else {
      ++i;
    }
  }
  cudaGetLastError();  // a pending (not ready) query is not an error
}

}  // namespace

extern "C" {

int pf_bank_run(const pf_bank_desc *d, int32_t k0, int32_t n_steps, int32_t cur,
                int32_t have_ancestors, void *stream) {
  const int vr = bank_validate(d, k0, n_steps, cur);
  if (vr != PF_OK) return vr;
  const cudaStream_t s = as_stream(stream);
  reap();
  // optional per-interval timing (events on the launch stream): start of the
  // interval, around the (main) propagate kernel - the dominant one - and the
  // end of the interval: 4 events per interval
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
    evs.e.resize(4 * static_cast<size_t>(n_steps));
    for (auto &x : evs.e) cudaEventCreate(&x);
    ev = evs.e.data();
  }
  int rc;
  // a graph pays its capture + instantiation (~0.5 ms) back only over a run
  // of intervals; short calls enqueue directly (measured: cfg0 shape)
  const int32_t min_graph = d->use_graph > 1 ? d->use_graph : kGraphMinSteps;
  if (d->use_graph && n_steps >= min_graph && !d->comm) {
    pf_bank_graph *g = nullptr;
    rc = graph_capture(d, k0, n_steps, cur, have_ancestors, s, ev, &g);
    if (rc != PF_OK) return rc;
    const cudaError_t le = cudaGraphLaunch(g->exec, s);
    retire(g->exec, s);
    delete g;
    if (le != cudaSuccess) return check_launch("pf_bank_run: graph launch");
  } else {
    rc = bank_enqueue(d, k0, n_steps, cur, have_ancestors, s, ev);
    if (rc != PF_OK) return rc;
  }
  if (ev && !d->events) {
    cudaEventSynchronize(ev[4 * n_steps - 1]);
    for (int32_t i = 0; i < n_steps; ++i) {
      if (d->prop_ms) cudaEventElapsedTime(&d->prop_ms[i], ev[4 * i + 1], ev[4 * i + 2]);
      if (d->step_ms) cudaEventElapsedTime(&d->step_ms[i], ev[4 * i], ev[4 * i + 3]);
    }
  }
  return check_launch("pf_bank_run");
}

int pf_bank_graph_create(const pf_bank_desc *d, int32_t k0, int32_t n_steps, int32_t cur,
                         int32_t have_ancestors, void *stream, pf_bank_graph **out) {
  PF_REQUIRE(out, "pf_bank_graph_create: null out");
  const int vr = bank_validate(d, k0, n_steps, cur);
  if (vr != PF_OK) return vr;
  PF_REQUIRE(n_steps >= 1 && !d->comm && !d->prop_ms && !d->step_ms,
             "pf_bank_graph_create: needs n_steps >= 1, no comm and no host-read timing");
  return graph_capture(d, k0, n_steps, cur, have_ancestors, as_stream(stream),
                       reinterpret_cast<cudaEvent_t *>(d->events), out);
}

int pf_bank_graph_launch(pf_bank_graph *g, void *stream) {
  PF_REQUIRE(g && g->exec, "pf_bank_graph_launch: null graph");
  if (cudaGraphLaunch(g->exec, as_stream(stream)) != cudaSuccess)
    return check_launch("pf_bank_graph_launch");
  return PF_OK;
}

int pf_bank_graph_destroy(pf_bank_graph *g) {
  if (!g) return PF_OK;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  delete g;
  return PF_OK;
}

}  // extern "C"
