"""Double bootstrap (particle islands) on the GPU bank - drop-in for
run_double_bootstrap / dbf_init / dbf_step (filters.py:201-313).

The M islands are the bank's M filters (each a bootstrap filter with its
own Philox key from ``seed.spawn(M + 1)[m]``).  After every observation's
resampling the island log-weights accumulate the islands' lnc increments;
every ``island_period`` steps whole islands are resampled by those weights
with the island key (``spawn(M + 1)[M]``) through the same segmented
resampler (one segment of M "particles"), and island m takes over island
idx[m]'s particles, lnc and collapse flag.  The pooled estimate and the
normalising-constant trace are computed on the device.

One GPU: island m simply takes island idx[m]'s *ancestors* (states are never
copied; the next propagate gathers them).  Several GPUs (one process per GPU,
islands block-sharded by id): the island log-weights, lnc and collapse flags
are combined with disjoint-support all-reduces, every rank draws the same
island selection, and islands that change rank move as particle blocks over
NCCL point-to-point (dist.exchange_islands); each rank then materialises its
new islands and continues with identity ancestors.  Results are identical
for any number of GPUs.
"""

from __future__ import annotations

import numpy as np

from . import _lib, dist, philox
from .bank import DrawTape, FilterBank
from .filters import FilterOutput


class IslandBank:
    def __init__(self, model, n_islands: int, n_particles: int, island_period: int, seed,
                 n_steps: int, *, dtype=None, tape: DrawTape | None = None, shard=None):
        import torch

        if n_islands < 1:
            raise ValueError("n_islands must be >= 1")
        if island_period < 1:
            raise ValueError("island_period must be >= 1")
        if n_islands > 4096:
            raise ValueError("at most 4096 islands")
        ss = philox.as_seed_sequence(seed)
        children = ss.spawn(n_islands + 1)
        keys = philox.seed_keys(children[:n_islands])
        self.M, self.N, self.period, self.T = n_islands, n_particles, island_period, n_steps
        self.tape = tape
        rank, world = dist.world()
        self.sharded = (world > 1 and shard is not False) or (shard is True and dist.initialized())
        if not self.sharded:
            rank, world = 0, 1
        if n_islands < world:
            # every rank takes this branch (same arguments), so all raise
            # together before any collective - none is left waiting
            raise ValueError(f"double bootstrap: {n_islands} islands cannot be sharded over "
                             f"{world} ranks (need n_islands >= world size)")
        self.lo, self.hi = dist.shard_range(n_islands, rank, world)
        dev = torch.device("cuda", torch.cuda.current_device())
        kw = dict(device=dev)
        # per-island estimates of every island (rows of other ranks arrive by all-reduce)
        self.est_isl = torch.zeros((n_steps, n_islands, model.dim_x), dtype=torch.float64, **kw)
        self.bank = FilterBank(model, self.hi - self.lo, n_particles, keys[self.lo:self.hi],
                               n_steps, dtype=dtype, tape=tape, estimate="full",
                               filter_offset=self.lo, est_buffer=self.est_isl,
                               est_row_offset=self.lo)
        ik = philox.seed_key(children[n_islands]).astype(np.uint32)[None, :]
        self.island_key = torch.from_numpy(ik.view(np.int32)).to(dev)
        Ml = self.hi - self.lo
        self.lw = torch.zeros(n_islands, dtype=torch.float64, **kw)  # full; local slice updated
        self.lnc_old = torch.empty(Ml, dtype=torch.float64, **kw)
        self.idx = torch.empty(n_islands, dtype=torch.int32, **kw)
        self.anc_tmp = torch.empty_like(self.bank.anc)
        self.lnc_tmp = torch.empty_like(self.bank.lnc)
        self.coll_tmp = torch.empty_like(self.bank.collapsed)
        self.lnc_all = torch.zeros(n_islands, dtype=torch.float64, **kw)
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

    # -- island selection -------------------------------------------------------
    def _select(self, t):
        import torch

        uni = None
        flags = 0
        if self.tape is not None:
            u = self.tape.islands.get(t)
            if u is None:
                raise ValueError(f"tape has no island uniforms for t={t}")
            uni = torch.from_numpy(np.ascontiguousarray(u, dtype=np.float64).reshape(1, -1)) \
                .to(self.bank.device)
            self._keep = uni
            flags = _lib.PF_RS_REFERENCE_ORDER
        _lib.call("pf_segmented_resample_ex", _lib.PF_F64, _lib.ptr(self.lw), 1, self.M,
                  _lib.ptr(uni), _lib.ptr(self.island_key), t, _lib.ptr(self.idx),
                  _lib.ptr(self.s_lnc), _lib.ptr(self.s_coll), _lib.ptr(self.s_status),
                  _lib.ptr(self.ws), self.ws_bytes, None, None, 0, flags, _lib.stream_ptr())

    def _islands(self, k, t):
        b = self.bank
        s = _lib.stream_ptr()
        Ml = self.hi - self.lo
        lw_local = self.lw[self.lo:self.hi]
        _lib.call("pf_island_accumulate", _lib.ptr(lw_local), _lib.ptr(b.lnc),
                  _lib.ptr(self.lnc_old), Ml, s)
        if t % self.period:
            return
        if not self.sharded:
            self._select(t)
            _lib.call("pf_island_copy", _lib.ptr(self.idx), _lib.ptr(b.anc), _lib.ptr(b.lnc),
                      _lib.ptr(b.collapsed), _lib.ptr(self.lw), self.M, self.N,
                      _lib.ptr(self.anc_tmp), _lib.ptr(self.lnc_tmp), _lib.ptr(self.coll_tmp), s)
        else:
            self._islands_sharded(t)
        self.island_steps.append(t)

    def _islands_sharded(self, t):
        """Cross-rank island resampling: full log-weights by a disjoint
        all-reduce, the same selection on every rank, particle blocks moved
        with NCCL point-to-point, new islands materialised locally."""
        import torch

        b = self.bank
        lo, hi, N = self.lo, self.hi, self.N
        others = torch.ones(self.M, dtype=torch.bool, device=self.lw.device)
        others[lo:hi] = False
        self.lw[others] = 0.0
        dist.allreduce_disjoint(self.lw)
        self._select(t)
        idx = self.idx.cpu().numpy()
        # every island's lnc and collapse flag (disjoint all-reduce)
        self.lnc_all.zero_()
        self.lnc_all[lo:hi] = b.lnc
        dist.allreduce_disjoint(self.lnc_all)
        coll_all = torch.zeros(self.M, dtype=torch.int32, device=self.lw.device)
        coll_all[lo:hi] = b.collapsed.to(torch.int32)
        dist.allreduce_disjoint(coll_all)
        # current particles of a local island: propagated rows through the ancestors
        xprop = b.x[1 - b.cur]  # the step's output buffer (cur flips after the step)
        planes = b.model.kind in ("lorenz", "hmm", "lgm")

        def get_island(src):
            rows = b.anc[(src - lo) * N:(src - lo + 1) * N].long()
            if planes:
                blk = xprop.index_select(1, rows)
            else:
                blk = xprop.index_select(0, rows)
            if b.q[0] is not None:
                return blk, b.q[1 - b.cur].index_select(0, rows)
            return blk

        template = get_island(lo) if hi > lo else None
        out = dist.exchange_islands(idx, self.M, get_island, template)
        new = torch.empty_like(xprop)
        newq = torch.empty_like(b.q[1 - b.cur]) if b.q[0] is not None else None
        for m, blk in out.items():
            j = m - lo
            if newq is not None:
                blk, qb = blk
                newq[j * N:(j + 1) * N] = qb
            if planes:
                new[:, j * N:(j + 1) * N] = blk
            else:
                new[j * N:(j + 1) * N] = blk
        xprop.copy_(new)
        if newq is not None:
            b.q[1 - b.cur].copy_(newq)
        torch.arange(0, (hi - lo) * N, dtype=torch.int32, out=b.anc)  # local rows
        sel = torch.from_numpy(idx[lo:hi].astype(np.int64)).to(self.lw.device)
        b.lnc.copy_(self.lnc_all[sel])
        b.collapsed.copy_(coll_all[sel].to(torch.uint8))
        self.lw.zero_()

    # -- driver ----------------------------------------------------------------------
    def start(self, observations):
        """dbf_init (filters.py:237-242) for every island."""
        b = self.bank
        b.load_observations(observations)
        b.init()
        self.lw.zero_()

    def step(self, k: int):
        """dbf_step (filters.py:245-265) for observation k, then the pooled
        estimate and the lnc trace of step k."""
        import torch

        b = self.bank
        s = _lib.stream_ptr()
        self.lnc_old.copy_(b.lnc)
        b.step(k)
        self.lnc_all.zero_()
        self.lnc_all[self.lo:self.hi] = b.lnc
        lw_full = self.lw
        if self.sharded:
            # rows / entries of other ranks' islands arrive by disjoint all-reduce
            dist.allreduce_disjoint(self.est_isl[k])
            dist.allreduce_disjoint(self.lnc_all)
            lw_full = self.lw.clone()
            mask = torch.ones(self.M, dtype=torch.bool, device=lw_full.device)
            mask[self.lo:self.hi] = False
            lw_full[mask] = 0.0
            dist.allreduce_disjoint(lw_full)
        _lib.call("pf_island_pool", _lib.ptr(self.est_isl[k]), self.est_isl.stride(1),
                  self.M, b.model.dim_x, _lib.ptr(lw_full),
                  _lib.c_vp(self.est.data_ptr() + k * self.est.stride(0) * 8), s)
        _lib.call("pf_island_trace", _lib.ptr(self.lnc_all), self.M,
                  _lib.c_vp(self.trace.data_ptr() + k * 8), s)

    def check_status(self):
        import torch

        b = self.bank
        st = torch.zeros(self.M, dtype=torch.int32, device=b.device)
        st[self.lo:self.hi] = b.status
        if self.sharded:
            dist.allreduce_disjoint(st)
        _lib.raise_status(st.cpu().numpy())

    def native_ok(self) -> bool:
        """The whole run can be one native call: single process, Philox
        draws (tape mode keeps the Python steps and their island tapes)."""
        return not self.sharded and self.tape is None

    def attach_native(self):
        """Hand the island step to the native bank driver (pf_island_desc):
        per interval, island weights, the island resampling every period,
        the pooled estimate and the trace - no Python between intervals."""
        b = self.bank
        d = _lib.IslandDesc()
        d.period = self.period
        d.key, d.lw, d.lnc_old = (self.island_key.data_ptr(), self.lw.data_ptr(),
                                  self.lnc_old.data_ptr())
        d.idx, d.anc_tmp = self.idx.data_ptr(), self.anc_tmp.data_ptr()
        d.lnc_tmp, d.coll_tmp = self.lnc_tmp.data_ptr(), self.coll_tmp.data_ptr()
        d.s_lnc, d.s_coll, d.s_status = (self.s_lnc.data_ptr(), self.s_coll.data_ptr(),
                                         self.s_status.data_ptr())
        d.ws, d.ws_bytes = self.ws.data_ptr(), self.ws_bytes
        d.pool, d.trace = self.est.data_ptr(), self.trace.data_ptr()
        d.pool_dim = self.est.shape[1]  # model.dim_x, as step() pools
        b.island_desc = d
        b.post_resample = None
        b._desc = None

    def run(self, observations):
        import torch

        self.start(observations)
        if self.native_ok():
            self.attach_native()
            self.bank.run_native(0, self.T, time_steps=True)
            steps = range(self.period, self.T + 1, self.period)
            self.island_steps.extend(steps)
            self.check_status()
            return self.bank.last_step_ms.astype(np.float64) / 1e3
        events = [torch.cuda.Event(enable_timing=True) for _ in range(self.T + 1)]
        events[0].record()
        for k in range(self.T):
            self.step(k)
            events[k + 1].record()
        torch.cuda.synchronize()
        self.check_status()
        return np.array([events[i].elapsed_time(events[i + 1]) / 1e3 for i in range(self.T)])

    def collapse_steps(self) -> list[int]:
        import torch

        c = torch.zeros((self.T, self.M), dtype=torch.int32, device=self.bank.device)
        c[:, self.lo:self.hi] = self.bank.coll_tr.to(torch.int32)
        if self.sharded:
            dist.allreduce_disjoint(c)
        c = c.cpu().numpy()
        return [int(k) + 1 for k in np.nonzero(c.any(axis=1))[0]]


def run_double_bootstrap(model, observations, n_islands: int, n_particles: int,
                         island_period: int, seed, *, dtype=None,
                         tape: DrawTape | None = None, shard=None) -> FilterOutput:
    """filters.py:274-313 on the GPU bank; same seeding tree, estimates
    (pooled island posterior means) and diagnostic lnc trace.  Under
    torch.distributed the islands are sharded over ranks (shard=None: when
    the world size is > 1); every rank returns the same FilterOutput."""
    obs = np.atleast_2d(np.asarray(observations, dtype=np.float64))
    if obs.shape[0] == 0:
        raise ValueError("observation sequence must be non-empty")
    if getattr(model, "dim_y", obs.shape[1]) == 1 and obs.shape[1] != 1:
        obs = obs.reshape(-1, 1)
    ib = IslandBank(model, n_islands, n_particles, island_period, seed, obs.shape[0],
                    dtype=dtype, tape=tape, shard=shard)
    secs = ib.run(obs)
    return FilterOutput("double-bf", n_islands * n_particles, seed, ib.est.cpu().numpy(),
                        ib.trace.cpu().numpy(), secs, ib.collapse_steps())


# ---------------------------------------------------------------------------
# Hook-level API (filters.py:201-271): IslandSystem, dbf_init, dbf_step
# ---------------------------------------------------------------------------


def _island_probs_device(log_weights):
    """softmax of the island log-weights in numpy's order (filters.py:225-227),
    through pf_island_pool with an identity estimate matrix."""
    import torch

    lw = torch.from_numpy(np.ascontiguousarray(log_weights, dtype=np.float64)).cuda()
    M = lw.shape[0]
    eye = torch.eye(M, dtype=torch.float64, device="cuda")
    out = torch.empty(M, dtype=torch.float64, device="cuda")
    _lib.call("pf_island_pool", _lib.ptr(eye), M, M, M, _lib.ptr(lw), _lib.ptr(out),
              _lib.stream_ptr())
    return out.cpu().numpy()


class IslandSystem:
    """M equally sized particle islands plus their accumulated log weights
    (filters.py:206-234)."""

    def __init__(self, islands, log_weights):
        sizes = {isl.n_particles for isl in islands}
        if len(sizes) != 1:
            raise ValueError("all islands must share the same particle count")
        self.islands = list(islands)
        self.log_weights = np.asarray(log_weights, dtype=np.float64)
        if self.log_weights.shape != (len(self.islands),):
            raise ValueError("one log weight per island required")

    @property
    def n_islands(self) -> int:
        return len(self.islands)

    def island_probs(self) -> np.ndarray:
        return _island_probs_device(self.log_weights)

    def pooled_estimate(self) -> np.ndarray:
        """sum_m p_m * posterior_mean(island m), islands in order (pf_island_pool)."""
        import torch

        from .core import posterior_mean

        est = torch.from_numpy(np.stack([np.asarray(posterior_mean(isl), dtype=np.float64)
                                         for isl in self.islands])).cuda()
        lw = torch.from_numpy(np.ascontiguousarray(self.log_weights)).cuda()
        out = torch.empty(est.shape[1], dtype=torch.float64, device="cuda")
        _lib.call("pf_island_pool", _lib.ptr(est), est.shape[1], self.n_islands, est.shape[1],
                  _lib.ptr(lw), _lib.ptr(out), _lib.stream_ptr())
        return out.cpu().numpy()


def _copy_island(isl):
    from .core import ParticleApproximation

    return ParticleApproximation(isl.particles.copy(), isl.weights.copy(), isl.log_norm_const,
                                 isl.t, collapsed=isl.collapsed)


def dbf_init(model, n_islands: int, n_particles: int, rngs) -> IslandSystem:
    """filters.py:237-242."""
    from .filters import bf_init

    if n_islands < 1:
        raise ValueError("n_islands must be >= 1")
    return IslandSystem([bf_init(model, n_particles, rngs[m]) for m in range(n_islands)],
                        np.zeros(n_islands))


def dbf_step(model, system: IslandSystem, y, t: int, island_period: int, rngs,
             island_rng) -> IslandSystem:
    """filters.py:245-271: one bootstrap step per island (island m on rngs[m]);
    every island_period steps whole islands are resampled by their
    accumulated weights with island_rng."""
    from .filters import bf_step
    from .resampling import multinomial_resample_indices

    if island_period < 1:
        raise ValueError("island_period must be >= 1")
    new_islands, log_weights = [], system.log_weights.copy()
    for m, isl in enumerate(system.islands):
        stepped = bf_step(model, isl, y, rngs[m])
        log_weights[m] += stepped.log_norm_const - isl.log_norm_const
        new_islands.append(stepped)
    if t % island_period == 0:
        idx = multinomial_resample_indices(_island_probs_device(log_weights), system.n_islands,
                                           island_rng)
        new_islands = [_copy_island(new_islands[i]) for i in idx]
        log_weights = np.zeros(system.n_islands)
    return IslandSystem(new_islands, log_weights)
