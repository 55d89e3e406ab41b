"""Multi-process (gloo, world size 2, CPU) tests of the sharding and the
disjoint-support estimate exchange used by run_ensemble on N GPUs."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1407_8071_b200 import dist as pdist


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_range_partitions_filters():
    for m in (1, 2, 7, 64, 4096):
        for w in (1, 2, 3, 8):
            # m < w: the high ranks own an empty block (they run no bank but
            # join every collective, ensemble.run_ensemble)
            spans = [pdist.shard_range(m, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        pdist.shard_range(4, 2, 2)


def _worker(rank, world, port, T, M, dim, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(0)
        full = rng.standard_normal((T, M, dim))  # every filter's estimate trace
        lo, hi = pdist.shard_range(M, rank, world)
        buf = torch.zeros((T, M, dim), dtype=torch.float64)
        ex = pdist.EstimateExchange(buf)
        for k in range(T):
            buf[k, lo:hi] = torch.from_numpy(full[k, lo:hi])  # this rank's kernel output
            ex.step_done(k)
        ex.finish()
        # every rank now holds every filter's exact estimate
        assert np.array_equal(buf.numpy(), full)
        # fixed left-to-right average == the reference's average_estimates order
        acc = buf[:, 0].clone()
        for m in range(1, M):
            acc += buf[:, m]
        mean = (acc / M).numpy()
        ref = full[:, 0].copy()
        for m in range(1, M):
            ref += full[:, m]
        ref /= float(M)
        assert mean.tobytes() == ref.tobytes()
        st = torch.zeros(M, dtype=torch.int32)
        st[lo:hi] = rank + 1
        pdist.allreduce_disjoint(st)
        hi0 = pdist.shard_range(M, 0, world)[1]
        assert st.tolist() == [1 if f < hi0 else 2 for f in range(M)]
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - surfaced through the queue
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("M", [7, 1])  # M=1 < world: rank 1 owns no filter
def test_disjoint_allreduce_two_ranks_bit_identical(M):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 5, M, 4, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def test_owner_of_matches_shard_range():
    for n in (1, 5, 7, 64):
        for w in (1, 2, 3, 4):
            if n < w:
                continue
            for r in range(w):
                lo, hi = pdist.shard_range(n, r, w)
                assert all(pdist.owner_of(i, n, w) == r for i in range(lo, hi))


def _island_worker(rank, world, port, M, idx, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = pdist.shard_range(M, rank, world)
        # island i's particle block: (3, 4) values 100*i + j, plus a tuple member
        blocks = {i: (torch.arange(12, dtype=torch.float32).reshape(3, 4) + 100 * i,
                      torch.full((4,), i, dtype=torch.int32)) for i in range(lo, hi)}
        tmpl = (torch.zeros(3, 4), torch.zeros(4, dtype=torch.int32))
        out = pdist.exchange_islands(idx, M, lambda s: blocks[s], tmpl)
        assert sorted(out) == list(range(lo, hi))
        for m, (a, b) in out.items():
            src = idx[m]
            assert torch.equal(a, torch.arange(12, dtype=torch.float32).reshape(3, 4) + 100 * src)
            assert torch.equal(b, torch.full((4,), src, dtype=torch.int32))
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_island_exchange_two_ranks():
    """Double-bootstrap island copies across ranks (gloo, world size 2)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    idx = [4, 4, 0, 2, 1]  # cross-rank copies in both directions, duplicates
    procs = [ctx.Process(target=_island_worker, args=(r, 2, port, 5, idx, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def test_bench_gpus_flag_fails_loudly_without_enough_gpus():
    """`bench.py --gpus 2` on a box with fewer GPUs exits non-zero with an
    error line instead of silently measuring one rank."""
    import json
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "1", "--warmup", "3"],
                       cwd=repo, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 2, (r.returncode, r.stderr[-2000:])
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert "error" in line and line["n_gpus"] == 2


def test_bench_launcher_spawns_one_rank_per_gpu(monkeypatch):
    """With N GPUs visible and no WORLD_SIZE, bench.py re-execs itself under
    torch.distributed.run with N ranks on 127.0.0.1 and NCCL init logging."""
    import importlib
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, repo)
    bench = importlib.import_module("bench")
    seen = {}
    monkeypatch.setattr(torch.cuda, "device_count", lambda: 8)
    monkeypatch.setattr(subprocess, "call", lambda cmd, env: seen.update(cmd=cmd, env=env) or 0)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "8", "--steps", "5"])
    assert bench.main() == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "8", "--steps", "5"]
    assert seen["env"]["NCCL_DEBUG"] == "INFO"
    # under torchrun the world size must match --gpus
    monkeypatch.setenv("WORLD_SIZE", "4")
    assert bench.main() == 2
