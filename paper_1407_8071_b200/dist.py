"""Multi-GPU plumbing: one process per GPU, filters block-sharded by global id.

The reference's only parallelism is a fork pool over filters with results
pickled back and averaged in the parent (ensemble.py:96-108); filters never
communicate.  Here each rank owns a contiguous block of global filter ids
(`shard_range`).  Per observation time the per-filter estimates are combined
with ONE all-reduce(sum) over a disjoint-support buffer of shape
(M_total, dim): every rank writes only its own rows and zeros elsewhere, and
x + 0 is exact, so every rank receives the exact per-filter estimates and can
average them in the reference's fixed left-to-right order
(ensemble.py:68-73).  The result is therefore bit-identical for any number of
GPUs.  Nothing downstream consumes the estimate until the end of the run, so
the all-reduce is issued on a side stream and overlaps the next interval.
"""

from __future__ import annotations

import os


def world():
    """(rank, world_size) of the initialised default process group, else (0, 1)."""
    try:
        import torch.distributed as dist
    except Exception:  # pragma: no cover
        return 0, 1
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def initialized() -> bool:
    try:
        import torch.distributed as dist
    except Exception:  # pragma: no cover
        return False
    return dist.is_available() and dist.is_initialized()


def shard_range(n_filters: int, rank: int, world_size: int) -> tuple[int, int]:
    """Contiguous block [start, stop) of global filter ids owned by `rank`."""
    if n_filters < 1 or world_size < 1 or not 0 <= rank < world_size:
        raise ValueError("bad shard request")
    base, rem = divmod(n_filters, world_size)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


class EstimateExchange:
    """Disjoint-support all-reduce of per-filter traces, one call per step."""

    def __init__(self, buffer, overlap: bool = True):
        import torch

        self.buffer = buffer  # (T, M_total, dim) zero-initialised
        self.works = []
        self.side = None
        if overlap and buffer.is_cuda:
            self.side = torch.cuda.Stream(device=buffer.device)

    def step_done(self, k: int):
        """Issue the all-reduce of step k's rows (after the producing kernels)."""
        import torch
        import torch.distributed as dist

        if self.side is not None:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(self.buffer.device))
            with torch.cuda.stream(self.side):
                self.side.wait_event(ev)
                self.works.append(dist.all_reduce(self.buffer[k], async_op=True))
        else:
            self.works.append(dist.all_reduce(self.buffer[k], async_op=True))

    def finish(self):
        import torch

        for w in self.works:
            w.wait()
        self.works.clear()
        if self.side is not None:
            torch.cuda.current_stream(self.buffer.device).wait_stream(self.side)


class NativeComm:
    """The NCCL communicator of libpfbank's native exchange (pf_comm_*),
    built over the default process group: rank 0 creates the NCCL id, the
    group broadcasts it, every rank joins.  The native bank driver issues
    each observation's estimate all-reduce itself (pf_bank_desc.comm), so a
    sharded record is one host call per rank with no Python per observation.
    """

    def __init__(self):
        import ctypes

        import torch
        import torch.distributed as dist

        from . import _lib

        rank, size = world()
        self.rank, self.size = rank, size
        buf = (ctypes.c_uint8 * _lib.PF_COMM_ID_BYTES)()
        if rank == 0:
            _lib.call("pf_comm_unique_id", ctypes.cast(buf, ctypes.c_void_p))
        if size > 1:
            dev = torch.device("cuda", torch.cuda.current_device()) \
                if dist.get_backend() == "nccl" else torch.device("cpu")
            t = torch.tensor(list(bytes(buf)), dtype=torch.uint8, device=dev)
            dist.broadcast(t, src=0)
            buf = (ctypes.c_uint8 * _lib.PF_COMM_ID_BYTES)(*t.cpu().tolist())
        self.handle = ctypes.c_void_p()
        _lib.call("pf_comm_init", ctypes.cast(buf, ctypes.c_void_p), size, rank,
                  ctypes.byref(self.handle))
        self.nccl_version = _lib.load().pf_comm_nccl_version()

    def join(self, stream=None):
        """The stream (default: current) waits for every exchange issued so far."""
        from . import _lib

        _lib.call("pf_comm_join", self.handle, _lib.stream_ptr(stream))

    def allreduce_f64(self, t):
        """In-place sum over ranks of a contiguous float64 CUDA tensor,
        ordered on the current stream."""
        from . import _lib

        assert t.dtype.itemsize == 8 and t.is_contiguous() and t.is_cuda
        _lib.call("pf_comm_allreduce_f64", self.handle, _lib.ptr(t), t.numel(),
                  _lib.stream_ptr())
        return t

    def exchange_steps(self, est, k0, n_steps):
        """The per-observation exchanges of est[k0:k0+n] (T, M, width) without a
        bank (a rank that owns no filters joins every collective)."""
        from . import _lib

        _lib.call("pf_comm_exchange_steps", self.handle, _lib.ptr(est), est.stride(0),
                  est[0].numel(), k0, n_steps, _lib.stream_ptr())

    def close(self):
        from . import _lib

        if self.handle:
            _lib.call("pf_comm_destroy", self.handle)
            self.handle = None


_NATIVE = {}


def native_comm():
    """The process's NativeComm for the default group (created on first use,
    collectively: every rank must call it), or None when the group is not
    NCCL or libpfbank cannot bind NCCL (then the torch EstimateExchange
    path is used)."""
    import torch.distributed as dist

    from . import _lib

    if not initialized() or dist.get_backend() != "nccl":
        return None
    if not _lib.load().pf_comm_available():
        return None
    key = (world(), id(dist.group.WORLD))
    if key not in _NATIVE:
        for stale in _NATIVE.values():  # a previous process group's communicator
            stale.close()
        _NATIVE.clear()
        _NATIVE[key] = NativeComm()
    return _NATIVE[key]


def allreduce_disjoint(t):
    """Blocking disjoint-support all-reduce (small end-of-run traces)."""
    import torch.distributed as dist

    if initialized():
        dist.all_reduce(t)
    return t


def local_rank() -> int:
    return int(os.environ.get("LOCAL_RANK", "0"))


def owner_of(i: int, n: int, world_size: int) -> int:
    """Rank owning global id i under shard_range's block partition."""
    base, rem = divmod(n, world_size)
    cut = rem * (base + 1)
    return i // (base + 1) if i < cut else rem + (i - cut) // max(base, 1)


def exchange_islands(idx, n_islands: int, get_island, template):
    """Whole-island resampling across ranks (double bootstrap, filters.py:258-263,
    SURVEY §8f #4).  Island m (owned by rank owner_of(m)) becomes a copy of
    island idx[m]; ``idx`` is the same on every rank (identical selection).

    get_island(src) returns the particle block (tensor or tuple of tensors)
    of a LOCAL island src; ``template`` gives the block shapes/dtypes for
    receive buffers.  Returns {m: block} for every local destination m.
    Sends and receives between any two ranks are issued in increasing m, so
    they match in order (NCCL groups them with batch_isend_irecv)."""
    import torch
    import torch.distributed as dist

    rank, world_size = world()
    lo, hi = shard_range(n_islands, rank, world_size)
    as_tuple = lambda b: b if isinstance(b, tuple) else (b,)  # noqa: E731
    ops, out, cache = [], {}, {}

    def local(src):
        if src not in cache:
            cache[src] = tuple(x.contiguous() for x in as_tuple(get_island(src)))
        return cache[src]

    for m in range(n_islands):
        src = int(idx[m])
        dst_rank, src_rank = owner_of(m, n_islands, world_size), owner_of(src, n_islands,
                                                                           world_size)
        if src_rank == rank and dst_rank != rank:
            for part in local(src):
                ops.append(("send", part, dst_rank))
        elif dst_rank == rank:
            if src_rank == rank:
                out[m] = local(src)
            else:
                bufs = tuple(torch.empty_like(t) for t in as_tuple(template))
                for part in bufs:
                    ops.append(("recv", part, src_rank))
                out[m] = bufs
    if ops:
        if dist.get_backend() == "nccl":
            p2p = [dist.P2POp(dist.isend if kind == "send" else dist.irecv, t, peer)
                   for kind, t, peer in ops]
            for w in dist.batch_isend_irecv(p2p):
                w.wait()
        else:
            works = [(dist.isend if kind == "send" else dist.irecv)(t, peer)
                     for kind, t, peer in ops]
            for w in works:
                w.wait()
    single = not isinstance(template, tuple)
    return {m: (b[0] if single else b) for m, b in out.items()}
