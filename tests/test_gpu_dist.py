"""The NCCL estimate-exchange path on one GPU (world size 1: no ranks wait
on one another) produces exactly the same bytes as the unsharded bank, and
a world-size-2 torchrun of bench.py is exercised when >= 2 GPUs exist."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.environ["REPO"])
from oracle import parpf_oracle as orc
import paper_1407_8071_b200 as pf
torch.cuda.set_device(0)
dist.init_process_group("nccl", init_method="tcp://127.0.0.1:%s" % os.environ["PORT"],
                        rank=0, world_size=1, device_id=torch.device("cuda", 0))
truth0, _, obs = orc.lorenz_truth(seed=5, n_obs=8)
m = pf.Lorenz63Model(substeps=40, obs_var=2.0, noise_scale=0.5, observe="x1x3",
                     prior_mean=tuple(truth0), prior_var=1.0)
a = pf.run_ensemble(m, obs, "bootstrap", 6, 256, 3, shard=True)
b = pf.run_ensemble(m, obs, "bootstrap", 6, 256, 3, shard=False)
assert a.same_result(b), "exchange path changed the result"
assert a.mean_estimates.tobytes() == b.mean_estimates.tobytes()
# the sharded record ran through the native driver's NCCL exchange (pf_comm)
from paper_1407_8071_b200 import dist as pdist
assert pdist._NATIVE, "native NCCL exchange not used"
fm, _, fobs = pf.simulate.fhn_truth(4, 3, pf.FhnLatticeModel())
fa = pf.run_ensemble(fm, fobs, "bootstrap", 3, 64, 3, dtype="float32", estimate="projection",
                     shard=True)
fb = pf.run_ensemble(fm, fobs, "bootstrap", 3, 64, 3, dtype="float32", estimate="projection",
                     shard=False)
assert fa.same_result(fb), "FH-N exchange path changed the result"
# double bootstrap: the sharded island path (disjoint all-reduces, island
# materialisation, point-to-point exchange) equals the single-GPU path
from paper_1407_8071_b200 import islands
for model, ob in ((m, obs), (pf.FhnNetworkModel(J=8, n_zones=2, zone_width=2, stim_prob=0.05),
                             pf.simulate.simulate(pf.FhnNetworkModel(J=8, n_zones=2,
                                                  zone_width=2, stim_prob=0.05), 12, 4)[1])):
    da = islands.run_double_bootstrap(model, ob, 5, 128, 3, 9, shard=True)
    db = islands.run_double_bootstrap(model, ob, 5, 128, 3, 9, shard=False)
    assert da.same_result(db), "sharded island path changed the result"
dist.destroy_process_group()
print("OK")
"""


def _port():
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_nccl_exchange_path_is_bit_identical():
    env = dict(os.environ, REPO=REPO, PORT=str(_port()))
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, r.stderr[-3000:]


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_bench_two_ranks():  # pragma: no cover - only on multi-GPU boxes
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus",
           "2", "--steps", "2", "--warmup", "1", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=REPO, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
