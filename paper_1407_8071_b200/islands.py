"""Double bootstrap (particle islands) on the GPU bank - drop-in for
run_double_bootstrap / dbf_init / dbf_step (filters.py:201-313).

The M islands are the bank's M filters (each a bootstrap filter with its
own Philox key from ``seed.spawn(M + 1)[m]``).  After every observation's
resampling the island log-weights accumulate the islands' lnc increments;
every ``island_period`` steps whole islands are resampled by those weights
with the island key (``spawn(M + 1)[M]``) through the same segmented
resampler (one segment of M "particles"), and island m takes over island
idx[m]'s ancestors, lnc and collapse flag - particle states are never
copied, the next propagate gathers them.  The pooled estimate and the
normalising-constant trace are computed on the device.

Single GPU: island selection is global, so sharding islands over ranks
would need a particle exchange every period; not done here.
"""

from __future__ import annotations

import numpy as np

from . import _lib, philox
from .bank import DrawTape, FilterBank
from .filters import FilterOutput, _bank_seconds


class IslandBank:
    def __init__(self, model, n_islands: int, n_particles: int, island_period: int, seed,
                 n_steps: int, *, dtype=None, tape: DrawTape | None = None):
        import torch

        if n_islands < 1:
            raise ValueError("n_islands must be >= 1")
        if island_period < 1:
            raise ValueError("island_period must be >= 1")
        if n_islands > 4096:
            raise ValueError("at most 4096 islands")
        ss = philox.as_seed_sequence(seed)
        children = ss.spawn(n_islands + 1)
        keys = np.stack([philox.seed_key(c) for c in children[:n_islands]]).astype(np.uint32)
        self.M, self.N, self.period, self.T = n_islands, n_particles, island_period, n_steps
        self.tape = tape
        self.bank = FilterBank(model, n_islands, n_particles, keys, n_steps, dtype=dtype,
                               tape=tape, estimate="full")
        dev = self.bank.device
        kw = dict(device=dev)
        ik = philox.seed_key(children[n_islands]).astype(np.uint32)[None, :]
        self.island_key = torch.from_numpy(ik.view(np.int32)).to(dev)
        self.lw = torch.zeros(n_islands, dtype=torch.float64, **kw)
        self.lnc_old = torch.empty(n_islands, dtype=torch.float64, **kw)
        self.idx = torch.empty(n_islands, dtype=torch.int32, **kw)
        self.anc_tmp = torch.empty_like(self.bank.anc)
        self.lnc_tmp = torch.empty_like(self.bank.lnc)
        self.coll_tmp = torch.empty_like(self.bank.collapsed)
        # scratch outputs of the island-level resample (1 segment of M)
        self.s_lnc = torch.zeros(1, dtype=torch.float64, **kw)
        self.s_coll = torch.zeros(1, dtype=torch.uint8, **kw)
        self.s_status = torch.zeros(1, dtype=torch.int32, **kw)
        wsb = int(_lib.load().pf_resample_workspace_bytes(1, n_islands))
        self.ws = torch.empty(max(wsb, 1), dtype=torch.uint8, **kw)
        self.ws_bytes = wsb
        self.est = torch.empty((n_steps, model.dim_x), dtype=torch.float64, **kw)
        self.trace = torch.empty(n_steps, dtype=torch.float64, **kw)
        self.bank.post_resample = self._islands
        self.island_steps = []

    def _islands(self, k, t):
        import torch

        b = self.bank
        s = _lib.stream_ptr()
        _lib.call("pf_island_accumulate", _lib.ptr(self.lw), _lib.ptr(b.lnc),
                  _lib.ptr(self.lnc_old), self.M, s)
        if t % self.period:
            return
        uni = None
        flags = 0
        if self.tape is not None:
            u = self.tape.islands.get(t)
            if u is None:
                raise ValueError(f"tape has no island uniforms for t={t}")
            uni = torch.from_numpy(np.ascontiguousarray(u, dtype=np.float64).reshape(1, -1)) \
                .to(b.device)
            self._keep = uni
            flags = _lib.PF_RS_REFERENCE_ORDER
        _lib.call("pf_segmented_resample_ex", _lib.PF_F64, _lib.ptr(self.lw), 1, self.M,
                  _lib.ptr(uni), _lib.ptr(self.island_key), t, _lib.ptr(self.idx),
                  _lib.ptr(self.s_lnc), _lib.ptr(self.s_coll), _lib.ptr(self.s_status),
                  _lib.ptr(self.ws), self.ws_bytes, None, None, 0, flags, s)
        _lib.call("pf_island_copy", _lib.ptr(self.idx), _lib.ptr(b.anc), _lib.ptr(b.lnc),
                  _lib.ptr(b.collapsed), _lib.ptr(self.lw), self.M, self.N,
                  _lib.ptr(self.anc_tmp), _lib.ptr(self.lnc_tmp), _lib.ptr(self.coll_tmp), s)
        self.island_steps.append(t)

    def run(self, observations):
        import torch

        b = self.bank
        b.load_observations(observations)
        b.init()
        self.lw.zero_()
        s = _lib.stream_ptr()
        events = [torch.cuda.Event(enable_timing=True) for _ in range(self.T + 1)]
        events[0].record()
        for k in range(self.T):
            self.lnc_old.copy_(b.lnc)
            b.step(k)
            _lib.call("pf_island_pool", _lib.ptr(b.est[k]), b.est_width, self.M,
                      self.bank.model.dim_x, _lib.ptr(self.lw),
                      _lib.c_vp(self.est.data_ptr() + k * self.est.stride(0) * 8), s)
            _lib.call("pf_island_trace", _lib.ptr(b.lnc), self.M,
                      _lib.c_vp(self.trace.data_ptr() + k * 8), s)
            events[k + 1].record()
        torch.cuda.synchronize()
        b.check_status()
        return _bank_seconds(events)

    def collapse_steps(self) -> list[int]:
        c = self.bank.coll_tr.cpu().numpy()
        return [int(k) + 1 for k in np.nonzero(c.any(axis=1))[0]]


def run_double_bootstrap(model, observations, n_islands: int, n_particles: int,
                         island_period: int, seed, *, dtype=None,
                         tape: DrawTape | None = None) -> FilterOutput:
    """filters.py:274-313 on the GPU bank; same seeding tree, estimates
    (pooled island posterior means) and diagnostic lnc trace."""
    obs = np.atleast_2d(np.asarray(observations, dtype=np.float64))
    if obs.shape[0] == 0:
        raise ValueError("observation sequence must be non-empty")
    if getattr(model, "dim_y", obs.shape[1]) == 1 and obs.shape[1] != 1:
        obs = obs.reshape(-1, 1)
    ib = IslandBank(model, n_islands, n_particles, island_period, seed, obs.shape[0],
                    dtype=dtype, tape=tape)
    secs = ib.run(obs)
    return FilterOutput("double-bf", n_islands * n_particles, seed, ib.est.cpu().numpy(),
                        ib.trace.cpu().numpy(), secs, ib.collapse_steps())
