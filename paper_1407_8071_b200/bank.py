"""The GPU filter bank: M independent bootstrap filters of N particles.

This replaces, for the whole bank at once, the reference's per-filter Python
loop run_filter -> bf_step (filters.py:97-112, 163-193) and the per-filter
task loop of run_ensemble (ensemble.py:76-111).  One observation interval
is three stream-ordered launches on device-resident state:

  1. propagate+weight  (pf_lorenz_propagate_weight | pf_fhn_interval):
     ancestor gather fused into the load, Euler-Maruyama steps in
     registers/shared memory, Gaussian log-likelihood in the epilogue;
  2. pf_segmented_resample: per-filter logsumexp, lnc update, collapse flag,
     fp64 CDF scan, sorted uniforms, merge -> ancestors;
  3. pf_filter_estimate: per-filter posterior mean of the resampled set.

The resampled particle set is never materialised: the next interval loads
x[anc[p]] directly (filters.py:111's ``propagated[idx]``).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib


@dataclass
class DrawTape:
    """Oracle-mode draws, indexed by GLOBAL filter id (rows).

    prior:    (M, N, 3) standard normals (Lorenz) or None (deterministic prior)
    noise:    per step k, (M, n_sub, N, 3) [Lorenz], (M, n_sub, 2, N, nodes)
              [FH-N lattice] or (M, N, nodes) [FH-N network] standard normals
    stim:     per step k, (M, 2, N) fire / select uniforms [FH-N network]
    uniforms: per step k, (M, N) sorted uniforms (rows of collapsed filters
              are ignored - the reference draws none for them)
    """

    prior: np.ndarray | None = None
    noise: list = field(default_factory=list)
    uniforms: list = field(default_factory=list)
    uniforms_first: list = field(default_factory=list)  # auxiliary filter, first stage
    stim: list = field(default_factory=list)  # FH-N network stimulus uniforms
    islands: dict = field(default_factory=dict)  # double bootstrap: t -> (1, M) uniforms


def _torch_dtype(dtype):
    import torch

    if dtype in (None, "float64", "f64", np.float64, torch.float64):
        return torch.float64
    if dtype in ("float32", "f32", np.float32, torch.float32):
        return torch.float32
    raise ValueError(f"unsupported dtype {dtype!r}")


class FilterBank:
    """M_local filters of one model on the current CUDA device."""

    def __init__(self, model, n_filters: int, n_particles: int, keys, n_steps: int, *,
                 dtype=None, tape: DrawTape | None = None, filter_offset: int = 0,
                 estimate: str = "full", est_buffer=None, est_row_offset: int = 0,
                 reference_order: bool = True, variant: str = "bootstrap",
                 kernel_flags: int = 0, graph: bool | None = None):
        import torch

        _lib.require_cuda()
        if n_filters < 1 or n_particles < 1:
            raise ValueError("n_filters and n_particles must be >= 1")
        if n_filters * n_particles > 2**31 - 1:
            raise ValueError("M*N per GPU must fit int32 particle indices")
        if model.kind not in ("lorenz", "fhn", "fhnnet", "hmm", "lgm"):
            raise ValueError(f"model kind {model.kind!r} has no GPU descriptor")
        if variant not in ("bootstrap", "auxiliary"):
            raise ValueError(f"unknown filter variant {variant!r}")
        self.variant = variant
        # _lib.PF_KERNEL_GENERIC: the propagate launches use the generic
        # kernels (comparison tests); 0 = production kernels
        self.kernel_flags = int(kernel_flags)
        self.model = model
        self.M, self.N = int(n_filters), int(n_particles)
        self.MN = self.M * self.N
        # launch-bound banks run their native records as one CUDA graph
        # (pf_bank_desc.use_graph); graph=None picks it for banks of up to
        # 2^20 particles, whose intervals are tens of microseconds
        self.use_graph = bool(graph) if graph is not None else self.MN <= (1 << 20)
        # graph=True: every run_native call of >= 2 intervals is one graph;
        # graph=None: runs of >= 32 intervals (shorter ones enqueue directly -
        # capture + instantiation cost ~0.5 ms)
        self.graph_min_steps = 2 if graph else 0
        self.T = int(n_steps)
        self.dtype = _torch_dtype(dtype)
        self.code = _lib.dtype_code(self.dtype)
        self.tape = tape
        self.offset = int(filter_offset)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        kw = dict(device=dev)

        from .models import estimate_width

        self.est_width = estimate_width(model, estimate)
        self.est_bits = 0
        self.q = [None, None]
        if model.kind in ("lorenz", "hmm", "lgm"):  # state planes x[d][p]
            self.x = [torch.empty((model.dim_x, self.MN), dtype=self.dtype, **kw)
                      for _ in range(2)]
            self.params = model.params()
            self.est_dim = model.dim_x
            self.est_strides = (1, self.MN)
        elif model.kind == "fhnnet":
            nodes = model.nodes
            self.x = [torch.empty((self.MN, 2 * nodes), dtype=self.dtype, **kw) for _ in range(2)]
            self.q = [torch.empty((self.MN, nodes), dtype=torch.int32, **kw) for _ in range(2)]
            self.params = model.params()
            self.obs_idx = torch.from_numpy(model.obs_indices.astype(np.int32)).to(dev)
            self.fmask = model.device_mask(dev)
            self.est_dim = 2 * nodes if estimate == "full" else nodes
            self.est_bits = model.stim_hold if estimate == "full" else 0
            self.est_strides = (2 * nodes, 1)
        else:
            self.x = [torch.empty((self.MN, model.dim_x), dtype=self.dtype, **kw)
                      for _ in range(2)]
            self.params = model.params()
            self.obs_idx = torch.from_numpy(model.obs_indices.astype(np.int32)).to(dev)
            self.est_dim = model.dim_x if estimate == "full" else model.nodes
            self.est_strides = (model.dim_x, 1)
        if estimate not in ("full", "projection"):
            raise ValueError("estimate must be 'full' or 'projection'")
        self.logw = torch.empty(self.MN, dtype=self.dtype, **kw)
        self.anc = torch.empty(self.MN, dtype=torch.int32, **kw)
        self.lnc = torch.zeros(self.M, dtype=torch.float64, **kw)
        self.collapsed = torch.zeros(self.M, dtype=torch.uint8, **kw)
        self.status = torch.zeros(self.M, dtype=torch.int32, **kw)
        k = np.ascontiguousarray(np.asarray(keys, dtype=np.uint32).reshape(self.M, 2))
        self.keys = torch.from_numpy(k.view(np.int32)).to(dev)
        # one scratch for the resampler and, after it, the chunked estimate
        # partials of wide filters (pf_filter_estimate_ws)
        ws = max(_lib.load().pf_resample_workspace_bytes(self.M, self.N),
                 _lib.load().pf_estimate_workspace_bytes(self.M, self.N, self.est_dim))
        self.ws_bytes = int(ws)
        self.ws = torch.empty(max(self.ws_bytes, 1), dtype=torch.uint8, **kw)
        if est_buffer is None:
            self.est = torch.empty((self.T, self.M, self.est_width), dtype=torch.float64, **kw)
            self.est_row = 0
        else:
            self.est = est_buffer
            self.est_row = int(est_row_offset)
        self.lnc_tr = torch.empty((self.T, self.M), dtype=torch.float64, **kw)
        self.coll_tr = torch.empty((self.T, self.M), dtype=torch.uint8, **kw)
        self.obs = None
        self.cur = 0
        self.steps_done = 0
        self.kernel_events = None  # optional (start, end) CUDA events around propagate
        # optional callable(k, t) run after resampling, before the estimate
        # (double bootstrap island selection, islands.py)
        self.post_resample = None
        # optional _lib.IslandDesc: the double bootstrap's island step inside
        # the native driver (islands.IslandBank.run)
        self.island_desc = None
        self._desc = None  # cached pf_bank_desc (buffers are fixed for the bank's lifetime)
        # oracle mode builds the CDF in the reference's exact order (bit-exact
        # ancestors); production mode uses the parallel scan
        self.rs_flags = _lib.PF_RS_REFERENCE_ORDER if (tape is not None and reference_order) else 0
        if variant == "auxiliary":  # apf_step scratch (filters.py:115-154)
            self.params0 = model.params(noise_free=True)
            self.lam = torch.empty(self.MN, dtype=self.dtype, **kw)
            self.anc1 = torch.empty(self.MN, dtype=torch.int32, **kw)
            self.anc_comp = torch.empty(self.MN, dtype=torch.int32, **kw)
            self.x_tmp = torch.empty_like(self.x[0])
            self.q_tmp = torch.empty_like(self.q[0]) if self.q[0] is not None else None
            self.lnc_before = torch.empty(self.M, dtype=torch.float64, **kw)
            self.coll1 = torch.empty(self.M, dtype=torch.uint8, **kw)

    # -- setup ----------------------------------------------------------------
    def load_observations(self, observations):
        import torch

        obs = np.atleast_2d(np.asarray(observations, dtype=np.float64))
        if obs.shape[1] != self.model.dim_y:
            raise ValueError(f"observations must have {self.model.dim_y} columns")
        if obs.shape[0] < self.T:
            raise ValueError("fewer observations than steps")
        self.obs = torch.from_numpy(np.ascontiguousarray(obs[: self.T])).to(self.device)
        self._desc = None

    def set_observation_buffer(self, obs_device):
        """Use a caller-owned (T, dim_y) float64 device tensor (bench/e2e)."""
        self.obs = obs_device
        self._desc = None

    def _rows(self):
        return slice(self.offset, self.offset + self.M)

    def init(self):
        """bf_init for every filter (filters.py:87-94)."""
        import torch

        s = _lib.stream_ptr()
        m = self.model
        if m.kind == "lorenz":
            mean, mean_p = _lib.host_f64(m.prior_mean)
            ztape = None
            if self.tape is not None:
                if self.tape.prior is None:
                    raise ValueError("tape has no prior draws")
                z = np.ascontiguousarray(self.tape.prior[self._rows()], dtype=np.float64)
                ztape = torch.from_numpy(z).to(self.device)
            _lib.call("pf_lorenz_prior", self.code, _lib.ptr(self.x[0]), self.M, self.N, mean_p,
                      m.prior_sd(), _lib.ptr(self.keys), _lib.ptr(ztape), s)
        elif m.kind in ("hmm", "lgm"):
            ztape = None
            if self.tape is not None:
                if self.tape.prior is None:
                    raise ValueError("tape has no prior draws")
                z = np.ascontiguousarray(self.tape.prior[self._rows()], dtype=np.float64)
                ztape = torch.from_numpy(z).to(self.device)
            fn = "pf_hmm_prior" if m.kind == "hmm" else "pf_lgm_prior"
            _lib.call(fn, self.params, self.code, _lib.ptr(self.x[0]), self.M, self.N,
                      _lib.ptr(self.keys), _lib.ptr(ztape), s)
        elif m.kind == "fhnnet":
            self.x[0].zero_()  # quiescent prior, no history (fhn.py:144-147)
            self.q[0].zero_()
        else:
            row = torch.from_numpy(m.initial_state()).to(self.device)
            _lib.call("pf_fill_rows", self.code, _lib.ptr(self.x[0]), self.MN, m.dim_x,
                      _lib.ptr(row), s)
            self._row_keepalive = row
        self.lnc.zero_()
        self.status.zero_()
        self.cur = 0
        self.steps_done = 0

    # -- one observation interval --------------------------------------------
    def _propagate(self, params, xin, anc, xout, y_ptr, logw, t, noise, qin=None, qout=None):
        s = _lib.stream_ptr()
        if self.model.kind == "fhnnet":
            stim, z = noise if noise is not None else (None, None)
            _lib.call("pf_fhnnet_step_ex", params, self.code, _lib.ptr(xin), _lib.ptr(qin),
                      _lib.ptr(anc), _lib.ptr(xout), _lib.ptr(qout), _lib.ptr(self.fmask),
                      y_ptr, _lib.ptr(self.obs_idx), _lib.ptr(logw), self.M, self.N,
                      _lib.ptr(self.keys), t, _lib.ptr(stim), _lib.ptr(z),
                      _lib.ptr(self.status), self.kernel_flags, s)
        elif self.model.kind in ("hmm", "lgm"):
            fn = "pf_hmm_propagate_weight" if self.model.kind == "hmm" else \
                "pf_lgm_propagate_weight"
            _lib.call(fn, params, self.code, _lib.ptr(xin), _lib.ptr(anc), _lib.ptr(xout), y_ptr,
                      _lib.ptr(logw), self.M, self.N, _lib.ptr(self.keys), t, _lib.ptr(noise),
                      _lib.ptr(self.status), s)
        elif self.model.kind == "lorenz":
            _lib.call("pf_lorenz_propagate_weight_ex", params, self.code, _lib.ptr(xin),
                      _lib.ptr(anc), _lib.ptr(xout), y_ptr, _lib.ptr(logw), self.M, self.N,
                      _lib.ptr(self.keys), t, _lib.ptr(noise), _lib.ptr(self.status),
                      self.kernel_flags, s)
        else:
            _lib.call("pf_fhn_interval_ex", params, self.code, _lib.ptr(xin), _lib.ptr(anc),
                      _lib.ptr(xout), y_ptr, _lib.ptr(self.obs_idx), _lib.ptr(logw),
                      self.M, self.N, _lib.ptr(self.keys), t, _lib.ptr(noise),
                      _lib.ptr(self.status), self.kernel_flags, s)

    def _resample(self, logw, uni, t, anc_out):
        _lib.call("pf_segmented_resample_ex", self.code, _lib.ptr(logw), self.M, self.N,
                  _lib.ptr(uni), _lib.ptr(self.keys), t, _lib.ptr(anc_out), _lib.ptr(self.lnc),
                  _lib.ptr(self.collapsed), _lib.ptr(self.status), _lib.ptr(self.ws),
                  self.ws_bytes, None, None, 0, self.rs_flags, _lib.stream_ptr())

    def _tape(self, lst, k):
        import torch

        a = np.ascontiguousarray(lst[k][self._rows()], dtype=np.float64)
        return torch.from_numpy(a).to(self.device)

    def _native_ok(self):
        return (self.tape is None and self.kernel_events is None
                and self.post_resample is None)

    def _bank_desc(self):
        import ctypes

        d = _lib.BankDesc()
        d.model = {"lorenz": _lib.PF_MODEL_LORENZ, "fhn": _lib.PF_MODEL_FHN,
                   "fhnnet": _lib.PF_MODEL_FHNNET, "hmm": _lib.PF_MODEL_HMM,
                   "lgm": _lib.PF_MODEL_LGM}[self.model.kind]
        d.dtype = self.code
        d.M, d.N = self.M, self.N
        if self.model.kind == "lorenz":
            d.lorenz = ctypes.pointer(self.params)
        elif self.model.kind == "hmm":
            d.hmm = ctypes.pointer(self.params)
        elif self.model.kind == "lgm":
            d.lgm = ctypes.pointer(self.params)
        elif self.model.kind == "fhnnet":
            d.fhnnet = ctypes.pointer(self.params)
            d.obs_idx = self.obs_idx.data_ptr()
            d.q[0], d.q[1] = self.q[0].data_ptr(), self.q[1].data_ptr()
            d.forcing_mask = self.fmask.data_ptr()
            d.est_bits = self.est_bits
        else:
            d.fhn = ctypes.pointer(self.params)
            d.obs_idx = self.obs_idx.data_ptr()
        d.x[0], d.x[1] = self.x[0].data_ptr(), self.x[1].data_ptr()
        d.logw, d.anc, d.lnc = self.logw.data_ptr(), self.anc.data_ptr(), self.lnc.data_ptr()
        d.collapsed, d.status = self.collapsed.data_ptr(), self.status.data_ptr()
        d.keys, d.ws, d.ws_bytes = self.keys.data_ptr(), self.ws.data_ptr(), self.ws_bytes
        d.obs, d.dim_y = self.obs.data_ptr(), self.model.dim_y
        d.est = self.est.data_ptr()
        d.est_step_stride = self.est.stride(0)
        d.est_offset = self.est_row * self.est_width
        d.est_stride_f = self.est_width
        d.est_stride_p, d.est_stride_d = self.est_strides
        d.est_dim = self.est_dim
        d.lnc_trace = self.lnc_tr.data_ptr()
        d.collapsed_trace = self.coll_tr.data_ptr()
        d.kernel_flags = self.kernel_flags
        d.use_graph = (self.graph_min_steps or 1) if self.use_graph else 0
        if self.island_desc is not None:
            d.islands = ctypes.pointer(self.island_desc)
        comm = getattr(self, "comm", None)
        if comm is not None:
            if self.est.shape[1] * self.est_width != self.exch_count or self.est_row < 0:
                raise ValueError("set_exchange: count must cover the whole (M_total, width) block")
            d.comm = comm.handle
            d.exch_count = self.exch_count
        if self.variant == "auxiliary":
            d.variant = 1
            d.params0 = ctypes.cast(ctypes.pointer(self.params0), ctypes.c_void_p)
            d.lam, d.anc1, d.anc_comp = (self.lam.data_ptr(), self.anc1.data_ptr(),
                                         self.anc_comp.data_ptr())
            d.x_tmp = self.x_tmp.data_ptr()
            d.q_tmp = self.q_tmp.data_ptr() if self.q_tmp is not None else None
            d.lnc_before, d.coll1 = self.lnc_before.data_ptr(), self.coll1.data_ptr()
        return d

    def set_exchange(self, comm, count: int):
        """Multi-GPU: after each observation the native driver all-reduces the
        `count` doubles of that observation's estimate block (est[k], the
        caller's disjoint-support (M_total, width) buffer) over `comm`
        (dist.NativeComm); None disables it."""
        self.comm = comm
        self.exch_count = int(count) if comm is not None else 0
        self._desc = None

    def run_native(self, k0: int, n_steps: int, time_propagate: bool = False,
                   time_steps: bool = False, slot: int | None = None):
        """Observations k0..k0+n_steps-1 in one native call (pf_bank_run).

        time_propagate=True returns the per-interval durations (ms) of the
        propagate kernel, measured with CUDA events on the launch stream;
        time_steps=True stores whole-interval durations in self.last_step_ms.
        slot=i (after prepare_timing(n)): record into intervals i.. of the
        prepared pool of n intervals without any host wait; read them later
        with pool_propagate_ms(n)."""
        import ctypes

        if self.obs is None:
            raise RuntimeError("load_observations() first")
        if not self._native_ok():
            raise RuntimeError("run_native: production banks only (no tape, no per-step hooks)")
        if self._desc is None:
            self._desc = self._bank_desc()
        timed = (time_propagate or time_steps) and n_steps > 0
        if slot is not None:  # slice of a larger prepared pool, nothing to wait for
            evs, handles = self._slot_pool
            if 4 * (slot + n_steps) > len(evs):
                raise ValueError("run_native: slot beyond the prepared timing pool")
            timed = False
        pool = self.__dict__.get("_event_pools", {}).get(4 * n_steps) if timed else None
        ms = sm = None
        if slot is not None:
            self._desc.events = ctypes.c_void_p(ctypes.addressof(handles) +
                                                4 * slot * ctypes.sizeof(ctypes.c_void_p))
        elif pool is not None:  # prepared events: recorded by the driver, no host wait
            evs, handles = pool
            self._desc.events = ctypes.cast(handles, ctypes.c_void_p)
        elif timed:  # the driver creates the events and waits for the last one
            if time_propagate:
                ms = (ctypes.c_float * n_steps)()
                self._desc.prop_ms = ctypes.cast(ms, ctypes.POINTER(ctypes.c_float))
            if time_steps:
                sm = (ctypes.c_float * n_steps)()
                self._desc.step_ms = ctypes.cast(sm, ctypes.POINTER(ctypes.c_float))
        try:
            _lib.call("pf_bank_run", self._desc, k0, n_steps, self.cur,
                      1 if self.steps_done > 0 else 0, _lib.stream_ptr())
        finally:
            self._desc.events = None
            self._desc.prop_ms = None
            self._desc.step_ms = None
        self.cur ^= n_steps & 1
        self.steps_done += n_steps
        self.last_step_ms = None
        if not timed:
            return None
        if pool is None:
            if sm is not None:
                self.last_step_ms = np.frombuffer(sm, dtype=np.float32).copy()
            return list(ms) if ms is not None else None
        evs[4 * n_steps - 1].synchronize()
        if time_steps:
            self.last_step_ms = np.array([evs[4 * i].elapsed_time(evs[4 * i + 3])
                                          for i in range(n_steps)], dtype=np.float32)
        return [evs[4 * i + 1].elapsed_time(evs[4 * i + 2]) for i in range(n_steps)] \
            if time_propagate else None

    def capture(self, k0: int, n_steps: int, slot: int | None = None) -> "BankGraph":
        """Capture observations k0..k0+n_steps-1 (the next ones this bank
        would run) into one instantiated CUDA graph (pf_bank_graph_create);
        BankGraph.launch() then enqueues them all.  slot=i records the
        prepare_timing pool's events i.. like run_native(..., slot=i)."""
        import ctypes

        if not self._native_ok():
            raise RuntimeError("capture: production banks only")
        if self._desc is None:
            self._desc = self._bank_desc()
        if slot is not None:
            evs, handles = self._slot_pool
            if 4 * (slot + n_steps) > len(evs):
                raise ValueError("capture: slot beyond the prepared timing pool")
            self._desc.events = ctypes.c_void_p(ctypes.addressof(handles) +
                                                4 * slot * ctypes.sizeof(ctypes.c_void_p))
        h = ctypes.c_void_p()
        try:
            _lib.call("pf_bank_graph_create", self._desc, k0, n_steps, self.cur,
                      1 if self.steps_done > 0 else 0, _lib.stream_ptr(), ctypes.byref(h))
        finally:
            self._desc.events = None
        return BankGraph(self, h, n_steps)

    def prepare_timing(self, n_steps: int):
        """Create the timing events of an n_steps run_native call ahead of time
        (keeps their creation out of a timed region); they also serve
        run_native(..., slot=i) calls of one interval each."""
        self._slot_pool = self._event_pool(4 * n_steps)

    def pool_propagate_ms(self, n_steps: int):
        """Propagate durations (ms) of intervals 0..n_steps-1 recorded through
        run_native(..., slot=i); waits for the last one."""
        evs, _ = self._slot_pool
        evs[4 * n_steps - 1].synchronize()
        return [evs[4 * i + 1].elapsed_time(evs[4 * i + 2]) for i in range(n_steps)]

    def _event_pool(self, n):
        """n timing events and their raw handles (ctypes array), created once
        per bank and size (each recorded once so the driver handle exists)."""
        import ctypes

        import torch

        pools = self.__dict__.setdefault("_event_pools", {})
        if n not in pools:
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
            for e in evs:
                e.record()
            pools[n] = (evs, (ctypes.c_void_p * n)(*[e.cuda_event for e in evs]))
        return pools[n]

    def step(self, k: int):
        if self.obs is None:
            raise RuntimeError("load_observations() first")
        if self._native_ok():
            self.run_native(k, 1)
            return
        t = k + 1
        s = _lib.stream_ptr()
        xin, xout = self.x[self.cur], self.x[1 - self.cur]
        anc = self.anc if self.steps_done > 0 else None
        y_ptr = _lib.c_vp(self.obs.data_ptr() + k * self.model.dim_y * 8)
        noise = uni = uni1 = None
        if self.tape is not None:
            noise = self._tape(self.tape.noise, k)
            if self.model.kind == "fhnnet":
                noise = (self._tape(self.tape.stim, k), noise)
            uni = self._tape(self.tape.uniforms, k)
            if self.variant == "auxiliary":
                uni1 = self._tape(self.tape.uniforms_first, k)
            self._tape_keepalive = (noise, uni, uni1)
        if self.variant == "auxiliary":
            self._apf_step(k, t, xin, xout, anc, y_ptr, noise, uni, uni1)
        else:
            if self.kernel_events is not None:
                self.kernel_events[0].record()
            self._propagate(self.params, xin, anc, xout, y_ptr, self.logw, t, noise,
                            self.q[self.cur], self.q[1 - self.cur])
            if self.kernel_events is not None:
                self.kernel_events[1].record()
            self._resample(self.logw, uni, t, self.anc)
        if self.post_resample is not None:
            self.post_resample(k, t)
        est_base = self.est[k].data_ptr() + self.est_row * self.est_width * 8
        sp, sd = self.est_strides
        _lib.call("pf_filter_estimate_ws", self.code, _lib.ptr(xout), sp, sd, self.est_dim,
                  _lib.ptr(self.anc), self.M, self.N, _lib.c_vp(est_base), self.est_width,
                  _lib.ptr(self.ws), self.ws_bytes, s)
        if self.est_bits:
            _lib.call("pf_bits_estimate", _lib.ptr(self.q[1 - self.cur]), self.model.nodes,
                      self.est_bits, _lib.ptr(self.anc), self.M, self.N,
                      _lib.c_vp(est_base + self.est_dim * 8), self.est_width, s)
        self.lnc_tr[k].copy_(self.lnc)
        self.coll_tr[k].copy_(self.collapsed)
        self.cur = 1 - self.cur
        self.steps_done += 1

    def _apf_step(self, k, t, xin, xout, anc_prev, y_ptr, noise, uni, uni1):
        """apf_step (filters.py:115-154) on the whole bank."""
        s = _lib.stream_ptr()
        # first stage: lambda = log p(y | noise-free prediction)
        self._propagate(self.params0, xin, anc_prev, self.x_tmp, y_ptr, self.lam, t, noise,
                        self.q[self.cur], self.q_tmp)
        _lib.call("pf_apf_first_stage_prepare", self.code, _lib.ptr(self.lam), self.M, self.N,
                  _lib.ptr(self.coll1), s)
        self.lnc_before.copy_(self.lnc)
        # first-stage uniforms use a distinct Philox time word in production
        self._resample(self.lam, uni1, t | 0x80000000, self.anc1)
        _lib.call("pf_compose_ancestors", _lib.ptr(self.anc1), _lib.ptr(anc_prev), self.MN,
                  _lib.ptr(self.anc_comp), s)
        # second stage: propagate the chosen ancestors, weights / lambda[anc1]
        if self.kernel_events is not None:
            self.kernel_events[0].record()
        self._propagate(self.params, xin, self.anc_comp, xout, y_ptr, self.logw, t, noise,
                        self.q[self.cur], self.q[1 - self.cur])
        if self.kernel_events is not None:
            self.kernel_events[1].record()
        _lib.call("pf_apf_second_stage_weights", self.code, _lib.ptr(self.logw),
                  _lib.ptr(self.lam), _lib.ptr(self.anc1), self.MN, s)
        self._resample(self.logw, uni, t, self.anc)
        _lib.call("pf_apf_finish", _lib.ptr(self.lnc), _lib.ptr(self.lnc_before),
                  _lib.ptr(self.collapsed), _lib.ptr(self.coll1), self.M, s)

    def run(self, on_step=None):
        if on_step is None and self._native_ok():
            self.run_native(0, self.T)
            return
        for k in range(self.T):
            self.step(k)
            if on_step is not None:
                on_step(k)

    # -- results ----------------------------------------------------------------
    def check_status(self):
        _lib.raise_status(self.status.cpu().numpy())

    def particles(self) -> np.ndarray:
        """Current (post-resampling) particle set, (M, N, dim_x) float64 host."""
        import torch

        x = self.x[self.cur]
        if self.model.kind == "fhnnet":
            anc = self.anc if self.steps_done > 0 else None
            return self.model.from_device(x, self.q[self.cur], anc).reshape(self.M, self.N, -1)
        anc = self.anc.long() if self.steps_done > 0 else torch.arange(self.MN, device=x.device)
        if self.model.kind in ("lorenz", "hmm", "lgm"):
            g = x[:, anc].t()
        else:
            g = x[anc]
        return g.to(torch.float64).reshape(self.M, self.N, -1).cpu().numpy()

    def collapse_steps(self) -> list[list[int]]:
        c = self.coll_tr.cpu().numpy()
        return [[int(k) + 1 for k in np.nonzero(c[:, f])[0]] for f in range(self.M)]


class BankGraph:
    """An instantiated CUDA graph of a bank's next n_steps intervals
    (FilterBank.capture); launch() once advances the bank like run_native."""

    def __init__(self, bank, handle, n_steps):
        self.bank, self.handle, self.n_steps, self.launched = bank, handle, n_steps, False

    def launch(self):
        if self.launched:
            raise RuntimeError("BankGraph: already launched (capture a new one)")
        _lib.call("pf_bank_graph_launch", self.handle, _lib.stream_ptr())
        self.launched = True
        self.bank.cur ^= self.n_steps & 1
        self.bank.steps_done += self.n_steps

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                import torch

                torch.cuda.synchronize()
                _lib.load().pf_bank_graph_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self.handle = None
