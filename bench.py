#!/usr/bin/env python3
"""Benchmark of the filter-bank hot path (BASELINE.json metric:
particle-steps/s = M x N x Euler steps per second, whole job).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4]
    python bench.py --impl reference ...      # the reference CPU path arm

A "step" is one observation interval of the whole bank: propagate (n_sub
Euler steps per particle, fused gather + log-likelihood) -> per-filter
logsumexp + multinomial resampling -> per-filter estimate (-> one
disjoint-support NCCL all-reduce of the estimate for N>1 GPUs).

Default workload: BASELINE cfg4 (FitzHugh-Nagumo 30x50 lattice, fp32,
M=64 filters x N=4096 particles, 50 Euler steps per observation), the
largest single-GPU config and the HBM showcase; filters are sharded
M/N_gpu per rank (strong scaling: the total bank is fixed).  cfg2 (Lorenz,
M x N = 2^22) is available via --config.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "particle-steps/s (M x N x Euler steps)"

CONFIGS = {
    # name: (kind, M, N, dtype, description)
    "cfg4": dict(kind="fhn", M=64, N=4096, dtype="float32",
                 desc="FitzHugh-Nagumo 30x50 lattice, M=64 x N=4096, 50 Euler steps/obs, fp32"),
    "cfg3": dict(kind="fhn", M=8, N=512, dtype="float32",
                 desc="FitzHugh-Nagumo 30x50 lattice, M=8 x N=512, 50 Euler steps/obs, fp32"),
    "cfg2": dict(kind="lorenz", M=4096, N=1024, dtype="float32",
                 desc="Lorenz-63, M=4096 x N=1024 (M*N=2^22), 40 Euler steps/obs, fp32"),
    "cfg2m256": dict(kind="lorenz", M=256, N=16384, dtype="float32",
                     desc="Lorenz-63, M=256 x N=16384 (M*N=2^22), 40 Euler steps/obs, fp32"),
    # the rest of BASELINE cfg2's M sweep: 16 filters of 2^18 and the
    # centralised filter of 2^22 particles (device-wide resampling; M=1 does
    # not shard - replicas only)
    "cfg2m16": dict(kind="lorenz", M=16, N=1 << 18, dtype="float32",
                    desc="Lorenz-63, M=16 x N=2^18 (M*N=2^22), 40 Euler steps/obs, fp32"),
    "cfg2m1": dict(kind="lorenz", M=1, N=1 << 22, dtype="float32",
                   desc="Lorenz-63, centralised M=1 x N=2^22, 40 Euler steps/obs, fp32"),
    "cfg1b": dict(kind="resample", M=1 << 16, N=1 << 10, dtype="float32",
                  desc="resampling microbench: bank M=2^16 x N=2^10, fp32 logw ~ N(0, sigma^2), "
                       "logsumexp + multinomial + 3-float ancestor gather"),
    "cfg1c": dict(kind="resample", M=1, N=1 << 26, dtype="float32",
                  desc="resampling microbench: centralised M=1 x N=2^26, fp32 logw ~ "
                       "N(0, sigma^2), logsumexp + multinomial + 3-float ancestor gather"),
    "cfg0": dict(kind="lorenz", M=4, N=1000, dtype="float64",
                 desc="Lorenz-63, M=4 x N=1000, 40 Euler steps/obs, fp64"),
    # one rank's share of cfg4 at 8 GPUs (8 of the 64 filters), on one GPU:
    # the measured input of the scaling model; not a BASELINE line
    "cfg4shard8": dict(kind="fhn", M=8, N=4096, dtype="float32",
                       desc="FH-N 30x50 lattice, M=8 x N=4096 (one rank's share of cfg4 at 8 "
                            "GPUs), 50 Euler steps/obs, fp32"),
    "cfg2shard8": dict(kind="lorenz", M=512, N=1024, dtype="float32",
                       desc="Lorenz-63, M=512 x N=1024 (one rank's share of cfg2 M=4096 at 8 "
                            "GPUs), 40 Euler steps/obs, fp32"),
    # the paper's own lattice (models/fhn.py:85-207): not a
    # BASELINE config; same metric, one Euler step per observation
    # SURVEY §8f rows on the same metric: the auxiliary filter (two-stage
    # resampling with a noise-free lookahead propagate; filter particle-steps
    # counted, the lookahead is extra work) and the double bootstrap (islands)
    "cfg4apf": dict(kind="fhn", variant="auxiliary", M=64, N=4096, dtype="float32",
                    desc="FH-N 30x50 lattice, auxiliary PF, M=64 x N=4096, 50 Euler steps/obs "
                         "(+50 lookahead steps not counted), fp32"),
    "cfg2apf": dict(kind="lorenz", variant="auxiliary", M=4096, N=1024, dtype="float32",
                    desc="Lorenz-63 auxiliary PF, M=4096 x N=1024, 40 Euler steps/obs "
                         "(+40 lookahead steps not counted), fp32"),
    "dbf": dict(kind="lorenz", variant="double-bf", M=64, N=65536, dtype="float32", period=5,
                desc="Lorenz-63 double bootstrap, 64 islands x 65536 particles, island "
                     "resampling every 5 observations, fp32"),
    "netapf": dict(kind="fhnnet", variant="auxiliary", M=64, N=4096, dtype="float32",
                   desc="paper FH-N network 32x32, auxiliary PF (the paper's experiment, "
                        "verify.py:356-414), M=64 x N=4096, 1 Euler step/obs (+1 noise-free "
                        "lookahead step not counted), fp32"),
    "net": dict(kind="fhnnet", M=64, N=4096, dtype="float32",
                desc="paper FH-N network 32x32 (stimuli, forcing, 25-step history), "
                     "M=64 x N=4096, 1 Euler step/obs, fp32"),
}

# Algorithmic work per particle-step
FHN_BYTES_PER_PS = 24000.0   # 16 B/node/Euler step (v,w read+write fp32) x 1500 nodes
NET_BYTES_PER_NODE = 24.0    # U,V fp32 + history bits, read + write, per node-step
LORENZ_FLOP_PER_PS = 20.0    # FMA = 2 (accel.py:73-75)
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # 74.4 nominal
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # 37.2 nominal


def fp32_peak():
    """Measured FP32 peak (TFLOP/s): the library's FFMA-chain probe
    (pf_probe_fp32_fma: SMs x 8 blocks x 256 threads x 8 independent chains),
    best of 3 timed launches after a warm-up, CUDA events; run outside any
    timed region.  Falls back to the nominal figure if the probe fails."""
    import torch

    from paper_1407_8071_b200 import _lib

    try:
        sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
        sink = torch.zeros(256, dtype=torch.float32, device="cuda")
        iters = 40000
        flop = sms * 8 * 256 * 256 * iters
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = None
        for rep in range(4):
            a.record()
            _lib.call("pf_probe_fp32_fma", _lib.ptr(sink), iters, _lib.stream_ptr())
            b.record()
            b.synchronize()
            if rep:
                t = a.elapsed_time(b) / 1e3
                best = t if best is None else min(best, t)
        return flop / best / 1e12, "measured: FFMA-chain probe (pf_probe_fp32_fma), best of 3"
    except Exception as exc:  # pragma: no cover - reported, not hidden
        return FP32_PEAK_TFLOPS, f"nominal 148 SM x 128 lanes x 2 x 1.965 GHz (probe failed: {exc})"


def _peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0}, "fallback"


class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: NVML
    (in-process, every 10 ms, plus one sample right at entry and one at exit,
    so even a sub-millisecond region has two readings); nvidia-smi if NVML is
    unavailable.  Reported: median SM MHz, max SM MHz, the throttle reasons
    seen (hw_slowdown, hw_thermal_slowdown, sw_thermal_slowdown,
    sw_power_cap) and the sample count."""

    PERIOD_S = 0.01
    REASONS = (("hw_slowdown", 0x8), ("sw_thermal_slowdown", 0x20),
               ("hw_thermal_slowdown", 0x40), ("sw_power_cap", 0x4))

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.samples = []  # (sm_mhz, max_mhz, reason bitmask)
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            ids = [v for v in vis.split(",") if v.strip() != ""]
            phys = int(ids[gpu_index]) if ids and ids[gpu_index].isdigit() else gpu_index
            self._h = pynvml.nvmlDeviceGetHandleByIndex(phys)
            self._nvml = pynvml
        except Exception:
            self._nvml = None

    def _sample(self):
        try:
            if self._nvml is not None:
                n = self._nvml
                sm = n.nvmlDeviceGetClockInfo(self._h, n.NVML_CLOCK_SM)
                mx = n.nvmlDeviceGetMaxClockInfo(self._h, n.NVML_CLOCK_SM)
                get = getattr(n, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    n.nvmlDeviceGetCurrentClocksThrottleReasons
                rs = get(self._h)
                self.samples.append((float(sm), float(mx), int(rs)))
                return
            out = subprocess.run(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.active", "--format=csv,noheader,nounits"],
                capture_output=True, text=True, timeout=5)
            if out.returncode == 0 and out.stdout.strip():
                sm, mx, rs = [v.strip() for v in out.stdout.strip().split(",")]
                self.samples.append((float(sm), float(mx), int(rs, 16)))
        except Exception:
            pass

    def _run(self):
        while not self._stop.wait(self.PERIOD_S):
            self._sample()

    def __enter__(self):
        self._sample()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._sample()
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock query unavailable"]}
        sm = [s[0] for s in self.samples]
        reasons = sorted({name for s in self.samples for name, bit in self.REASONS
                          if s[2] & bit})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(s[1] for s in self.samples),
                "sm_mhz_min": min(sm), "reasons": reasons, "samples": len(self.samples),
                "source": "nvml" if self._nvml is not None else "nvidia-smi"}


def _dist_setup():
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return rank, world, local


def _barrier(world):
    import torch
    import torch.distributed as dist

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()


def _max_over_ranks(x, world):
    import torch
    import torch.distributed as dist

    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _make_model_and_obs(cfg, n_obs, seed=2026):
    from paper_1407_8071_b200 import simulate
    from paper_1407_8071_b200.models import FhnLatticeModel, Lorenz63Model

    if cfg["kind"] == "fhn":
        model, _, obs = simulate.fhn_truth(seed, n_obs, FhnLatticeModel())
    elif cfg["kind"] == "fhnnet":
        from paper_1407_8071_b200.models import FhnNetworkModel

        model = FhnNetworkModel()
        _, obs = simulate.simulate(model, n_obs, seed)
    else:
        base = Lorenz63Model(substeps=40, obs_var=2.0, noise_scale=0.5, observe="x1x3")
        truth0, _, obs = simulate.lorenz_truth(seed, n_obs, base)
        model = Lorenz63Model(substeps=40, obs_var=2.0, noise_scale=0.5, observe="x1x3",
                              prior_mean=tuple(truth0), prior_var=1.0)
    return model, obs


# ----------------------------------------------------------------- CPU baseline

def cpu_baseline(cfg, budget_s=12.0, steps=1):
    """Reference CPU path (oracle port: numpy driver + C kernels, the role of
    the reference's numba twins) on a bounded sample of the workload, all
    host cores via a fork pool over filters (ensemble.py:100-105)."""
    from concurrent.futures import ProcessPoolExecutor
    from multiprocessing import get_context

    from oracle import ckernels
    from oracle import parpf_oracle as orc

    ckernels.install()
    cores = orc.cpu_cores()
    if cfg["kind"] == "fhn":
        model, _, obs = orc.fhn_truth(seed=2026, n_obs=max(steps, 1))
        n_part, per_ps = 16, None
        n_sub = model.substeps
    elif cfg["kind"] == "fhnnet":
        model = orc.FhnNetworkModel()
        _, obs = orc.simulate(model, max(steps, 1), 2026)
        n_part, n_sub = 64, 1
    else:
        truth0, _, obs = orc.lorenz_truth(seed=2026, n_obs=max(steps, 1))
        model = orc.LorenzConfigModel(prior_mean=tuple(truth0))
        n_part = 1024 if cfg["N"] >= 1024 else cfg["N"]
        n_sub = model.substeps
    variant = cfg.get("variant", "bootstrap")
    if variant == "double-bf":
        return _cpu_baseline_dbf(cfg, model, obs, n_sub, budget_s)
    # calibrate: one filter, one step
    t0 = time.perf_counter()
    orc.run_filter(model, obs[:1], n_part, 0, variant=variant)
    one = max(time.perf_counter() - t0, 1e-6)
    per_worker = max(1, int(budget_s / max(steps, 1) / one))
    # never more filters than the workload has (cfg0 has M=4): the reference
    # pool then runs min(M, cores) workers (ensemble.py:100-105)
    n_filters = min(cores * per_worker, cfg["M"]) if cfg["kind"] == "lorenz" else cores
    workers = min(cores, n_filters)
    if cfg["kind"] == "fhn":
        n_part = max(4, min(256, int(16 * budget_s / max(steps, 1) / one)))
        n_filters = cores
    elif cfg["kind"] == "fhnnet":
        n_part = max(16, min(cfg["N"], int(64 * budget_s / max(steps, 1) / one)))
        n_filters = cores
    t0 = time.perf_counter()
    with ProcessPoolExecutor(max_workers=workers, mp_context=get_context("fork")) as pool:
        list(pool.map(orc._filter_task,
                      [(model, obs[:steps], n_part, s, False, variant)
                       for s in orc.filter_seeds(1, n_filters)]))
    wall = time.perf_counter() - t0
    ps = n_filters * n_part * n_sub * steps
    return {"value": ps / wall, "unit": "particle-steps/s", "cores": workers, "kind": "port",
            "sample": (f"{n_filters} {variant} filters x {n_part} particles x {steps} obs x "
                       f"{n_sub} Euler steps of the {cfg['kind']} config model, fp64 numpy "
                       f"driver + C kernels (oracle/), fork pool of {workers} workers; "
                       f"{wall:.1f} s wall")}


def _cpu_baseline_dbf(cfg, model, obs, n_sub, budget_s):
    """The reference's double bootstrap runs its islands in one process
    (filters.py:274-313): one core, a bounded island count / size."""
    from oracle import parpf_oracle as orc

    M, period = min(cfg["M"], 16), cfg.get("period", 5)
    n_part, steps = 256, max(period, 1)
    obs_s = np.resize(obs, (steps, obs.shape[1]))
    t0 = time.perf_counter()
    orc.run_double_bootstrap(model, obs_s[:1], M, n_part, period, 0)
    one = max(time.perf_counter() - t0, 1e-6)
    n_part = max(64, min(cfg["N"], int(n_part * budget_s / (one * steps))))
    t0 = time.perf_counter()
    orc.run_double_bootstrap(model, obs_s, M, n_part, period, 1)
    wall = time.perf_counter() - t0
    ps = M * n_part * n_sub * steps
    return {"value": ps / wall, "unit": "particle-steps/s", "cores": 1, "kind": "port",
            "sample": (f"double bootstrap, {M} islands x {n_part} particles x {steps} obs "
                       f"(one island resampling) x {n_sub} Euler steps, fp64 numpy driver + C "
                       f"kernels, single process; {wall:.1f} s wall")}


def run_reference_arm(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    resample = cfg["kind"] == "resample"

    def sample(budget):
        if resample:
            return cpu_resample_baseline(cfg, args.sigma, budget_s=budget)
        return cpu_baseline(cfg, budget_s=budget, steps=1)

    for _ in range(args.warmup):
        sample(2.0)
    vals = []
    t0 = time.perf_counter()
    cb = None
    for _ in range(args.steps):
        cb = sample(max(3.0, 60.0 / max(args.steps, 1)))
        vals.append(cb["value"])
    wall = time.perf_counter() - t0
    value = float(np.median(vals))
    cb["value"] = value
    ref_config = {"workload": args.config, "desc": cfg["desc"]}
    if cfg.get("variant", "bootstrap") == "bootstrap" and cfg["kind"] in _KIND_SHAPE:
        ref_config = _bank_config(args, cfg, args.gpus, *_KIND_SHAPE[cfg["kind"]])
    unit = "particles/s" if resample else "particle-steps/s"
    metric = "particles/s (logsumexp + multinomial resampling + gather)" if resample else METRIC
    line = {"impl": "reference", "metric": metric, "value": value, "unit": unit,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * wall / max(args.steps, 1), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": ref_config,
            "cpu_baseline": cb,
            "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------- cfg1: resampling

RESAMPLE_BYTES_PER_PARTICLE = 32.0  # logw 4 + ancestor 4 + gather read 12 + write 12


def cpu_resample_baseline(cfg, sigma, budget_s=10.0):
    """Reference CPU path for cfg1 on one core (the reference has no
    intra-filter parallelism): normalize_log_weights + multinomial_resample
    (numpy cumsum + exponential spacings + C merge) + gather, fp64."""
    from oracle import ckernels
    from oracle import parpf_oracle as orc

    ckernels.install()
    rng = np.random.default_rng(0)
    n = min(cfg["N"], 1 << 22)
    m_per = max(1, (1 << 20) // n)
    lw = (rng.standard_normal((m_per, n)) * sigma).astype(np.float32)
    x = rng.standard_normal((m_per * n, 3)).astype(np.float32)
    done, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < budget_s:
        for f in range(m_per):
            w, _ = orc.normalize_log_weights(lw[f])
            idx = orc.multinomial_resample_indices(w, n, rng)
            _ = x[f * n + idx]
        done += m_per * n
    wall = time.perf_counter() - t0
    return {"value": done / wall, "unit": "particles/s", "cores": 1, "kind": "port",
            "sample": f"{m_per} filter(s) x N={n}, repeated for {wall:.1f} s on 1 core, fp64 "
                      f"(numpy + C merge)"}


E2E_REPS = 3


def _median_call_s(fn, world):
    """Median wall time (s) of E2E_REPS calls of fn, each bracketed by a
    barrier and a device synchronize: one slow call (a host hiccup, a
    collector pause) does not set the end-to-end figure."""
    import torch

    times = []
    for _ in range(E2E_REPS):
        _barrier(world)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
        del out
    return float(np.median(times))


def _wide_launches(N, flags):
    """Kernels of one wide (N > 8192) production resample (launch_resample):
    tile stats + filter totals (gamma + 3 chunk kernels when N > 2^21, else
    one) + tile CDF + partition + merge; the merge-path / separate-gather
    variants add the gather pass, the recomputing variant drops the tile CDF."""
    chunked = (N + 2047) // 2048 > 1024
    n = 8 if chunked else 5
    if flags & (2 | 4):
        n += 1
    if flags & 8:
        n -= 1
    return n


def run_resample(args, cfg):
    import torch

    from paper_1407_8071_b200 import _lib, philox

    rank, world, local = _dist_setup()
    M, N = cfg["M"], cfg["N"]
    lo, hi = (0, M)
    if world > 1:
        from paper_1407_8071_b200 import dist as pdist

        if M % world:
            raise SystemExit(f"M={M} does not shard over {world} GPUs (replicas only)")
        lo, hi = pdist.shard_range(M, rank, world)
    Ml = hi - lo
    MN = Ml * N
    g = torch.Generator(device="cuda").manual_seed(1234 + rank)
    logw = (torch.randn(MN, device="cuda", generator=g) * args.sigma).float()
    x_in = torch.randn((3, MN), device="cuda", generator=g)
    x_out = torch.empty_like(x_in)
    anc = torch.empty(MN, dtype=torch.int32, device="cuda")
    lnc = torch.zeros(Ml, dtype=torch.float64, device="cuda")
    coll = torch.zeros(Ml, dtype=torch.uint8, device="cuda")
    st = torch.zeros(Ml, dtype=torch.int32, device="cuda")
    keys = torch.from_numpy(philox.filter_keys(7, M)[lo:hi].view(np.int32)).cuda()
    wsb = _lib.load().pf_resample_workspace_bytes(Ml, N)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device="cuda")
    s = _lib.stream_ptr()

    def step(k):
        _lib.call("pf_segmented_resample_ex", _lib.PF_F32, _lib.ptr(logw), Ml, N, None,
                  _lib.ptr(keys), k + 1, _lib.ptr(anc), _lib.ptr(lnc), _lib.ptr(coll),
                  _lib.ptr(st), _lib.ptr(ws), wsb, _lib.ptr(x_in), _lib.ptr(x_out), 3,
                  args.kernel_flags, s)  # cfg1: --kernel-flags are PF_RS_* flags

    for k in range(args.warmup):
        step(k)
    _barrier(world)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        start.record()
        for i in range(args.steps):
            step(args.warmup + i)
        end.record()
        torch.cuda.synchronize()
    _barrier(world)
    local_s = start.elapsed_time(end) / 1e3
    elapsed = _max_over_ranks(local_s, world)
    value = M * N * args.steps / elapsed
    per = local_s / args.steps
    peaks, peak_src = _peaks()
    achieved = MN * RESAMPLE_BYTES_PER_PARTICLE / per / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": achieved / peaks["hbm_gbs"], "peak_source": peak_src,
            "kernel": ("pf_segmented_resample_ex (resample_bank_kernel with fused gather)"
                       if N <= 8192 else
                       "pf_segmented_resample_ex (wide pipeline: tile stats, filter totals, "
                       "tile CDF, partition, merge, fused gather)"),
            "algorithmic": f"{RESAMPLE_BYTES_PER_PARTICLE:.0f} B/particle x {MN} particles",
            "traffic": _ncu_traffic(args.config), "ncu_pipes": _ncu_pipes(args.config)}
    if N <= 8192:  # one resample launch per step: the step time is the kernel time
        roof["issue"] = _issue_roofline(roof["ncu_pipes"], per * 1e3)
    # e2e: host logw in (pinned), host ancestors out, through the C ABI.  A bank
    # of many filters is streamed in filter chunks on three streams (H2D of
    # chunk c+1 and D2H of chunk c-1 overlap the resample of chunk c; PCIe is
    # full duplex); one centralised filter needs all its weights first, so its
    # copies and kernels are serial.
    h_lw = logw.cpu().pin_memory()
    h_anc = torch.empty(MN, dtype=torch.int32).pin_memory()
    chunks = 8 if (N <= 8192 and Ml % 8 == 0) else 1
    cM, cMN = Ml // chunks, MN // chunks
    xs_in = [torch.randn((3, cMN), device="cuda", generator=g) for _ in range(chunks)]
    xs_out = [torch.empty_like(x) for x in xs_in]
    st_h2d, st_cmp, st_d2h = (torch.cuda.Stream() for _ in range(3))

    def e2e_step(k):
        # the previous step's copies and kernels are done before its buffers
        # are overwritten (overlap is across chunks within a step)
        st_h2d.wait_stream(st_d2h)
        for c in range(chunks):
            sl = slice(c * cMN, (c + 1) * cMN)
            with torch.cuda.stream(st_h2d):
                logw[sl].copy_(h_lw[sl], non_blocking=True)
            st_cmp.wait_stream(st_h2d)
            _lib.call("pf_segmented_resample_ex", _lib.PF_F32, _lib.c_vp(logw[sl].data_ptr()),
                      cM, N, None, _lib.c_vp(keys[c * cM:].data_ptr()), k + 1,
                      _lib.c_vp(anc[sl].data_ptr()), _lib.c_vp(lnc[c * cM:].data_ptr()),
                      _lib.c_vp(coll[c * cM:].data_ptr()), _lib.c_vp(st[c * cM:].data_ptr()),
                      _lib.ptr(ws), wsb, _lib.ptr(xs_in[c]), _lib.ptr(xs_out[c]), 3, 0,
                      _lib.c_vp(st_cmp.cuda_stream))
            st_d2h.wait_stream(st_cmp)
            with torch.cuda.stream(st_d2h):
                h_anc[sl].copy_(anc[sl], non_blocking=True)

    e2e_step(0)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(args.steps):
        e2e_step(i)
    torch.cuda.synchronize()
    e2e_s = _max_over_ranks(time.perf_counter() - t0, world)
    if rank == 0:
        cb = None if (world > 1 or args.no_cpu_baseline) else cpu_resample_baseline(cfg, args.sigma)
        line = {"metric": "particles/s (logsumexp + multinomial resampling + gather)",
                "value": value, "unit": "particles/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps,
                "higher_is_better": True, "scaling": "weak" if M > 1 else "replicas",
                "vs_baseline": None, "dtype": "f32 logw / f64 CDF", "data": "synthetic",
                "config": {"workload": args.config, "desc": cfg["desc"], "sigma": args.sigma,
                           "M": M, "N": N},
                "roofline": roof, "cpu_baseline": cb,
                "e2e": {"value": M * N * args.steps / e2e_s, "unit": "particles/s",
                        "h2d_bytes_per_step": MN * 4, "d2h_bytes_per_step": MN * 4,
                        "api": f"pf_segmented_resample_ex on pinned host log-weights -> host "
                               f"ancestors, {chunks} filter chunk(s) pipelined over H2D / "
                               f"compute / D2H streams"},
                "gpu_launches": (1 if N <= 8192 else _wide_launches(N, args.kernel_flags))
                * args.steps,
                "clocks": clocks.summary()}
        print(json.dumps(line))
    return 0


# ----------------------------------------------------------------- our arm

def run_ours(args, cfg):
    import torch

    import paper_1407_8071_b200 as pf
    from paper_1407_8071_b200 import _lib, dist as pdist, philox

    rank, world, local = _dist_setup()
    M, N = cfg["M"], cfg["N"]
    if M % world:
        raise SystemExit(f"M={M} not divisible by {world} GPUs")
    # W warm-up + K timed intervals, then K more with CUDA events around the
    # propagate kernel (its duration, for the roofline, without event nodes
    # inside the timed region)
    T = args.warmup + 2 * args.steps
    model, obs = _make_model_and_obs(cfg, T)
    n_sub = getattr(model, "substeps", 1)
    lo, hi = pdist.shard_range(M, rank, world)
    keys = philox.filter_keys(7, M)
    dev = torch.device("cuda", torch.cuda.current_device())
    est_dim = 3 if cfg["kind"] == "lorenz" else model.nodes
    est_full = torch.zeros((T, M, est_dim), dtype=torch.float64, device=dev)
    bank = pf.FilterBank(model, hi - lo, N, keys[lo:hi], T, dtype=cfg["dtype"],
                         filter_offset=lo, estimate="projection", est_buffer=est_full,
                         est_row_offset=lo, kernel_flags=args.kernel_flags)
    bank.load_observations(obs)
    bank.init()
    comm = None
    if world > 1:
        # the native driver all-reduces each observation's disjoint-support
        # estimate block over NCCL on a side stream (pf_comm, dist.NativeComm)
        comm = pdist.native_comm()
        if comm is None:
            raise SystemExit("multi-GPU bench needs the native NCCL exchange (pf_comm)")
        bank.set_exchange(comm, M * est_dim)
        sys.stderr.write(f"[bench] rank {rank}/{world} (GPU {local}): NCCL "
                         f"{comm.nccl_version} communicator of {comm.size} ranks, filters "
                         f"[{lo}, {hi}) of {M}\n")

    # warm-up, then K timed intervals in one native call (pf_bank_run)
    bank.run_native(0, args.warmup)
    if comm is not None:
        comm.join()
    # launch-bound banks: the K intervals as one prebuilt CUDA graph
    graph = bank.capture(args.warmup, args.steps) if bank.use_graph and comm is None else None
    _barrier(world)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        start.record()
        if graph is not None:
            graph.launch()
        else:
            bank.run_native(args.warmup, args.steps)
        if comm is not None:  # the last observation's exchange is part of the step
            comm.join()
        end.record()
        torch.cuda.synchronize()
    # the dominant kernel's duration: K more intervals, CUDA events around
    # each propagate launch on its stream (prepared pool, no host waits)
    bank.prepare_timing(args.steps)
    bank.run_native(args.warmup + args.steps, args.steps, slot=0)
    kern_list = bank.pool_propagate_ms(args.steps)
    if comm is not None:
        comm.join()
    _barrier(world)
    local_s = start.elapsed_time(end) / 1e3
    elapsed = _max_over_ranks(local_s, world)
    bank.check_status()
    ps_total = M * N * n_sub * args.steps
    value = ps_total / elapsed
    kern_ms = float(np.mean(kern_list))
    kern_share = kern_ms * args.steps / (local_s * 1e3)
    ps_per_launch = (hi - lo) * N * n_sub
    if args.profile:  # ncu runs: the timed launches only (no probes, no e2e)
        if rank == 0:
            print(json.dumps({"profile_run": args.config, "value": value, "kernel_ms": kern_ms}))
        return 0

    peaks, peak_src = _peaks()
    if cfg["kind"] == "fhnnet":
        per_ps = NET_BYTES_PER_NODE * model.nodes
        achieved = ps_per_launch * per_ps / (kern_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "peak_source": peak_src,
                "kernel": "fhnnet_fast_kernel (fp32, Philox)",
                "algorithmic": f"{per_ps:.0f} B/particle-step (24 B/node: U,V fp32 + history "
                               f"bits, read + write) x {ps_per_launch} particle-steps per launch"}
    elif cfg["kind"] == "fhn":
        # The kernel keeps each particle on chip for all n_sub Euler steps
        # (DESIGN §3), so HBM is not its bound: the headline is the issue
        # roofline (SURVEY §7 hard part 3).  Beside it: the physical HBM
        # fraction (bytes the launch must move / kernel time) and, labelled,
        # the SURVEY §8d per-step streaming model.
        pipes = _ncu_pipes(args.config)
        roof = _issue_roofline(pipes, kern_ms) or {"bound": "issue", "achieved": None,
                                                    "frac": None, "unit": "warp-inst/s"}
        roof["kernel"] = "fhn_cm_kernel<30,50,6> (fp32, Philox; column-major strip slots)"
        roof["algorithmic"] = (f"{pipes['warp_inst_per_launch']:.4g} warp instructions per "
                               f"launch (ncu smsp__inst_executed.sum, same launch) / live "
                               f"kernel time" if pipes else "no committed ncu count")
        phys = ps_per_launch / n_sub * (2 * 2 * model.nodes * 4 + 4 + 4)
        roof["hbm_physical"] = {
            "bytes_per_launch": phys, "achieved": phys / (kern_ms / 1e3) / 1e9,
            "peak": peaks["hbm_gbs"], "unit": "GB/s", "peak_source": peak_src,
            "frac": phys / (kern_ms / 1e3) / 1e9 / peaks["hbm_gbs"],
            "note": "gathered state read + state write (16 B/node) + logw + ancestor per "
                    "particle per launch"}
        model_gbs = ps_per_launch * FHN_BYTES_PER_PS / (kern_ms / 1e3) / 1e9
        roof["streaming_model"] = {
            "achieved": model_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": model_gbs / peaks["hbm_gbs"],
            "note": f"SURVEY §8d model {FHN_BYTES_PER_PS:.0f} B/particle-step (16 B/node per "
                    f"Euler step) x {ps_per_launch} particle-steps; NOT HBM traffic (the "
                    f"kernel does not stream every step)"}
    elif cfg["dtype"] == "float64":  # cfg0: the fp64 reference-precision bank
        achieved = ps_per_launch * LORENZ_FLOP_PER_PS / (kern_ms / 1e3) / 1e12
        roof = {"bound": "fp64", "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS,
                "peak_source": "nominal 148 SM x 64 FP64 lanes x 2 x 1.965 GHz",
                "kernel": "lorenz_small_kernel (fp64, Philox; one warp per particle)",
                "algorithmic": f"{LORENZ_FLOP_PER_PS:.0f} flop/particle-step x {ps_per_launch}",
                "note": f"latency-bound: {ps_per_launch // n_sub} particles occupy "
                        f"{ps_per_launch // n_sub * 32 / (148 * 2048):.1%} of the resident "
                        f"thread slots even at one warp per particle"}
    else:
        achieved = ps_per_launch * LORENZ_FLOP_PER_PS / (kern_ms / 1e3) / 1e12
        fpk, fsrc = fp32_peak()
        roof = {"bound": "fp32", "achieved": achieved, "peak": fpk,
                "unit": "TFLOP/s", "frac": achieved / fpk, "peak_source": fsrc,
                "peak_nominal": FP32_PEAK_TFLOPS,
                "kernel": "lorenz_fast_kernel (fp32, Philox)",
                "algorithmic": f"{LORENZ_FLOP_PER_PS:.0f} flop/particle-step x {ps_per_launch}"}
    roof["kernel_ms"] = kern_ms
    roof["kernel_share_of_step"] = kern_share
    roof["traffic"] = _ncu_traffic(args.config)
    roof["ncu_pipes"] = _ncu_pipes(args.config)
    if roof["bound"] != "issue":
        roof["issue"] = _issue_roofline(roof["ncu_pipes"], kern_ms)

    # e2e through the public API (host observations in, host results out)
    _barrier(world)
    e2e_obs = obs[: args.steps]
    # release the timed bank so the caching allocator can serve the e2e call
    used_graph = graph is not None
    comm_version = comm.nccl_version if comm is not None else None
    del graph, bank, est_full
    # one untimed call of the same shape (first-use costs: lazy module
    # loading of the e2e path, allocator growth), then the timed call
    warm = pf.run_ensemble(model, e2e_obs, "bootstrap", M, N, 7, dtype=cfg["dtype"],
                           estimate="projection")
    del warm
    torch.cuda.synchronize()
    e2e_local = _median_call_s(
        lambda: pf.run_ensemble(model, e2e_obs, "bootstrap", M, N, 7, dtype=cfg["dtype"],
                                estimate="projection"), world)
    e2e_s = _max_over_ranks(e2e_local, world)
    e2e = {"value": ps_total / e2e_s, "unit": "particle-steps/s",
           "h2d_bytes_per_step": int(model.dim_y * 8),
           "d2h_bytes_per_step": int(M * est_dim * 8 + M * 8 + M * 4),
           "api": "paper_1407_8071_b200.run_ensemble (host numpy observations -> "
                  "EnsembleOutput), includes bank allocation + prior init; median of "
                  f"{E2E_REPS} timed calls after one untimed warm-up call"}

    line = None
    if rank == 0:
        cb = None
        if world == 1 and not args.no_cpu_baseline:
            cb = cpu_baseline(cfg)
        line = {"metric": METRIC, "value": value, "unit": "particle-steps/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32" if cfg["dtype"] ==
                "float32" else "f64", "data": "synthetic",
                "config": _bank_config(args, cfg, world, n_sub, _state_bytes(model)),
                "roofline": roof, "cpu_baseline": cb, "e2e": e2e,
                "cuda_graph": used_graph,
                "nccl": {"ranks": world, "version": comm_version,
                         "exchange": "native pf_comm all-reduce per observation"}
                if world > 1 else None,
                # per step: propagate + resample (+ the estimate pass unless the
                # planar-state estimate is fused into the bank resampler)
                "gpu_launches": (2 if cfg["kind"] == "lorenz" and N <= 8192 else 3) *
                args.steps,
                "clocks": clocks.summary()}
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def run_variant(args, cfg):
    """Auxiliary PF / double bootstrap on one GPU: W untimed steps, K timed
    steps bracketed by CUDA events (synchronised), the propagate kernel
    timed with events around its launch."""
    import torch

    import paper_1407_8071_b200 as pf
    from paper_1407_8071_b200 import islands, philox

    rank, world, local = _dist_setup()
    if world > 1:
        raise SystemExit(f"{args.config}: single-GPU workload")
    M, N, variant = cfg["M"], cfg["N"], cfg["variant"]
    dbf = variant == "double-bf"
    # double bootstrap: the timed K intervals as one prebuilt CUDA graph of the
    # native island sequence (~16 short launches per interval), and K more
    # intervals with events around each propagate for the kernel time
    T = args.warmup + (2 if dbf else 1) * args.steps
    model, obs = _make_model_and_obs(cfg, T)
    n_sub = getattr(model, "substeps", 1)
    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    if dbf:  # the island step inside the native driver, as run_double_bootstrap
        runner = islands.IslandBank(model, M, N, cfg["period"], 7, T, dtype=cfg["dtype"])
        runner.start(obs)
        runner.attach_native()
        bank, step = runner.bank, runner.step
    else:
        bank = pf.FilterBank(model, M, N, philox.filter_keys(7, M), T, dtype=cfg["dtype"],
                             estimate="projection", variant=variant)
        bank.load_observations(obs)
        bank.init()
        step = bank.step
    # the whole apf_step / island sequence in pf_bank_run
    native = variant == "auxiliary" or dbf
    if native:
        bank.run_native(0, args.warmup)
        bank.prepare_timing(args.steps)
    else:
        bank.kernel_events = ev
        for k in range(args.warmup):
            step(k)
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    kern_list = []
    graph = bank.capture(args.warmup, args.steps) if dbf else None
    with ClockSampler(local) as clocks:
        start.record()
        if graph is not None:
            graph.launch()
        elif native:
            kern_list = bank.run_native(args.warmup, args.steps, time_propagate=True)
        else:
            for i in range(args.steps):
                bank.kernel_events = evs[i]  # events around this step's propagate launch
                step(args.warmup + i)
        end.record()
        torch.cuda.synchronize()
    elapsed = start.elapsed_time(end) / 1e3
    if graph is not None:
        bank.run_native(args.warmup + args.steps, args.steps, slot=0)
        kern_list = bank.pool_propagate_ms(args.steps)
        del graph
    bank.check_status()
    ps_total = M * N * n_sub * args.steps
    value = ps_total / elapsed
    kern_ms = float(np.mean(kern_list if native else [a.elapsed_time(b) for a, b in evs]))
    peaks, peak_src = _peaks()
    if args.profile:
        print(json.dumps({"profile_run": args.config, "value": value, "kernel_ms": kern_ms}))
        return 0
    if cfg["kind"] == "fhn":
        # the noisy second-stage propagate is the production lattice kernel
        # (cfg4's capture): issue roofline, as run_ours
        roof = _issue_roofline(_ncu_pipes("cfg4"), kern_ms) or {"bound": "issue", "frac": None}
        roof["kernel"] = "fhn_cm_kernel (second-stage propagate)"
        roof["algorithmic"] = "cfg4's ncu warp-instruction count per launch / live kernel time"
        ach = M * N * n_sub * FHN_BYTES_PER_PS / (kern_ms / 1e3) / 1e9
        roof["streaming_model"] = {"achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                                   "frac": ach / peaks["hbm_gbs"],
                                   "note": "SURVEY §8d per-step model; not HBM traffic"}
    elif cfg["kind"] == "fhnnet":
        per_ps = NET_BYTES_PER_NODE * model.nodes
        ach = M * N * per_ps / (kern_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": ach / peaks["hbm_gbs"], "peak_source": peak_src,
                "kernel": "fhnnet_fast_kernel (second-stage propagate)",
                "algorithmic": f"{per_ps:.0f} B/particle-step x {M * N}"}
    else:
        ach = M * N * n_sub * LORENZ_FLOP_PER_PS / (kern_ms / 1e3) / 1e12
        fpk, fsrc = fp32_peak()
        roof = {"bound": "fp32", "achieved": ach, "peak": fpk, "unit": "TFLOP/s",
                "frac": ach / fpk, "peak_source": fsrc, "peak_nominal": FP32_PEAK_TFLOPS,
                "kernel": "lorenz_fast_kernel (propagate)",
                "algorithmic": f"{LORENZ_FLOP_PER_PS:.0f} flop/particle-step x {M * N * n_sub}"}
    roof["kernel_ms"] = kern_ms
    roof["kernel_share_of_step"] = kern_ms * args.steps / (elapsed * 1e3)
    roof["traffic"] = None
    del bank, step
    if variant == "double-bf":
        del runner
    e2e_obs = obs[: args.steps]
    call = (lambda o: islands.run_double_bootstrap(model, o, M, N, cfg["period"], 7,
                                                   dtype=cfg["dtype"])) \
        if variant == "double-bf" else \
        (lambda o: pf.run_ensemble(model, o, variant, M, N, 7, dtype=cfg["dtype"],
                                   estimate="projection"))
    call(e2e_obs)  # untimed warm-up call (same shapes as the timed ones)
    torch.cuda.synchronize()
    e2e_s = _median_call_s(lambda: call(e2e_obs), 1)
    est_dim = model.dim_x if variant == "double-bf" else (3 if cfg["kind"] == "lorenz"
                                                          else model.nodes)
    e2e = {"value": ps_total / e2e_s, "unit": "particle-steps/s",
           "h2d_bytes_per_step": int(model.dim_y * 8),
           "d2h_bytes_per_step": int((1 if variant == "double-bf" else M) * est_dim * 8 + M * 9),
           "api": ("paper_1407_8071_b200.islands.run_double_bootstrap" if variant == "double-bf"
                   else "paper_1407_8071_b200.run_ensemble(variant='auxiliary')") +
                  f" (host numpy observations -> host outputs), median of {E2E_REPS} timed "
                  "calls after one untimed warm-up call"}
    cb = None if args.no_cpu_baseline else cpu_baseline(cfg)
    line = {"metric": METRIC, "value": value, "unit": "particle-steps/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": args.config, "desc": cfg["desc"], "M": M, "N": N,
                       "variant": variant, "euler_steps_per_obs": n_sub,
                       "parallelism": "single GPU"},
            "roofline": roof, "cpu_baseline": cb, "e2e": e2e,
            # APF: 2 propagates, 2 resamples, prepare, compose, weights, finish, estimate;
            # double bootstrap (N = 65536 per island): propagate, the wide resampler's 5
            # kernels, accumulate, the chunked estimate's 2, pool, trace (+ island select
            # and copy every period)
            "gpu_launches": args.steps * 9 if variant == "auxiliary" else
            args.steps * 11 + 2 * ((args.warmup + args.steps) // cfg["period"]
                                   - args.warmup // cfg["period"]),
            "native_driver": native, "cuda_graph": dbf,
            "clocks": clocks.summary()}
    print(json.dumps(line))
    return 0


def _bank_config(args, cfg, world, n_sub, state_bytes):
    """`config` of a bootstrap-bank line - the same dict on both arms."""
    M, N = cfg["M"], cfg["N"]
    return {"workload": args.config, "desc": cfg["desc"], "M": M, "N": N,
            "euler_steps_per_obs": n_sub, "parallelism": f"filters/{world}",
            "l2": "inputs larger than L2 (state "
                  f"{2 * M * N * state_bytes:.3g} B, double-buffered)"
            if cfg["kind"] in ("fhn", "fhnnet") else "state < L2; compute-bound kernel"}


# the reference arm names the same workload without building the GPU model:
# (Euler steps per observation, device bytes of one fp32 particle) by model kind
_KIND_SHAPE = {"fhn": (50, 2 * 30 * 50 * 4), "lorenz": (40, 3 * 4)}


def _state_bytes(model):
    """Device bytes of one fp32 particle."""
    if model.kind == "fhnnet":
        return model.nodes * 12  # U, V fp32 + 32-bit history field
    return model.dim_x * 4


def _ncu_traffic(config):
    try:
        with open(os.path.join(REPO, "profiles", "traffic.json")) as fh:
            return json.load(fh).get(config)
    except OSError:
        return None


DISPATCH_SLOTS = {"imad_wide": 3.2, "mufu": 1.5, "other": 1.0}


def _issue_roofline(pipes, kern_ms, sm_mhz=1965.0):
    """Second roofline for the issue-bound kernels: warp instructions per launch
    (committed ncu count of the same launch) / the live kernel time, against
    148 SMs x 4 schedulers x 1 instruction/clock at the max SM clock."""
    if not pipes or "warp_inst_per_launch" not in pipes or not kern_ms:
        return None
    achieved = pipes["warp_inst_per_launch"] / (kern_ms / 1e3)
    peak = 148 * 4 * sm_mhz * 1e6
    roof = {"bound": "issue", "achieved": achieved, "peak": peak, "unit": "warp-inst/s",
            "frac": achieved / peak, "peak_source": "148 SMs x 4 schedulers x 1 warp-inst/clk "
                                                   f"x {sm_mhz:.0f} MHz",
            "source": "smsp__inst_executed.sum (profiles/pipes.json) / live kernel time"}
    if "imad_wide_per_launch" in pipes:
        # Dispatch-slot model measured by tools/probes/pipe_probe.cu on this B200
        # (profiles/r02_pipe_probe.txt): in mixes of independent chains the time per
        # group is additive - IMAD.WIDE.U32 holds an SMSP's dispatch for ~3.2 clocks,
        # a MUFU for ~1.5, every other instruction for ~1 - so the Philox multiplies
        # cost issue slots no other warp can use.
        scale = pipes["warp_inst_per_launch"] / pipes.get("warp_inst_captured",
                                                          pipes["warp_inst_per_launch"])
        slots = (pipes["warp_inst_per_launch"]
                 + scale * (DISPATCH_SLOTS["imad_wide"] - 1.0) * pipes["imad_wide_per_launch"]
                 + scale * (DISPATCH_SLOTS["mufu"] - 1.0) * pipes["mufu_per_launch"])
        roof["dispatch_model"] = {
            "frac": slots / (kern_ms / 1e3) / peak, "slots_per_launch": slots,
            "slots": DISPATCH_SLOTS,
            "note": "secondary: dispatch slots (warp instructions weighted by the clocks each "
                    "opcode holds the SMSP dispatch port, pipe_probe mixes) / live kernel time "
                    "/ peak; the fraction of the kernel time the instruction mix itself needs"}
    return roof


def _ncu_pipes(config):
    """Pipe utilisation of the workload's dominant kernel from the committed
    ncu capture (profiles/pipes.json): the issue/FMA-pipe evidence behind a
    low algorithmic-flop fraction (cfg2: the Gaussian draws, not the 20
    flop/particle-step of the dynamics, fill the pipes)."""
    try:
        with open(os.path.join(REPO, "profiles", "pipes.json")) as fh:
            pipes = json.load(fh)
    except OSError:
        return None
    if config in pipes:
        return pipes[config]
    # the same kernel as a captured config at another bank size: its warp
    # instructions scale with the particle-steps per launch
    src = {"cfg3": "cfg4", "cfg4shard8": "cfg4", "cfg2m256": "cfg2", "cfg2m16": "cfg2",
           "cfg2m1": "cfg2", "cfg2shard8": "cfg2"}.get(config)
    if src is None or src not in pipes:
        return None
    scaled = dict(pipes[src])
    ratio = (CONFIGS[config]["M"] * CONFIGS[config]["N"]) / (CONFIGS[src]["M"] *
                                                             CONFIGS[src]["N"])
    scaled["warp_inst_captured"] = pipes[src]["warp_inst_per_launch"]
    scaled["warp_inst_per_launch"] = pipes[src]["warp_inst_per_launch"] * ratio
    scaled["source"] = f"{src} capture scaled by particle-steps per launch ({ratio:.4g})"
    return scaled


def _free_port():
    import socket

    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def launch_ranks(n):
    """`bench.py --gpus N` outside torchrun: re-exec this command under
    torch.distributed.run with N ranks (one per GPU, NCCL), after checking
    that N GPUs are visible - a box with fewer GPUs fails loudly instead of
    silently measuring one rank.  NCCL_DEBUG=INFO (init subsystem, written to
    stderr) logs the communicator lines with their rank counts."""
    import torch

    have = torch.cuda.device_count()
    if have < n:
        print(json.dumps({"error": f"--gpus {n} requested but {have} CUDA device(s) visible",
                          "n_gpus": n}))
        sys.stderr.write(f"bench.py: --gpus {n} needs {n} GPUs, found {have}\n")
        return 2
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    # NCCL logs to stdout by default; keep stdout for the JSON line
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sigma", type=float, default=1.0, help="cfg1 log-weight std")
    ap.add_argument("--kernel-flags", type=int, default=0,
                    help="PF_KERNEL_* for the propagate kernels (comparison runs only)")
    ap.add_argument("--profile", action="store_true",
                    help="timed steps only (no e2e / CPU baseline): for ncu captures")
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return launch_ranks(args.gpus)
    if world != args.gpus:
        sys.stderr.write(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}\n")
        return 2
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference_arm(args, cfg)
    if cfg["kind"] == "resample":
        return run_resample(args, cfg)
    if cfg.get("variant", "bootstrap") != "bootstrap":
        return run_variant(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
