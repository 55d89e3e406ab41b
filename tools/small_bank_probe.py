"""Per-step cost of a small bank (cfg0 shape) through pf_bank_run: device
time with and without per-step propagate events, and host enqueue time."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1407_8071_b200 as pf  # noqa: E402
from paper_1407_8071_b200 import philox, simulate  # noqa: E402

base = pf.Lorenz63Model(substeps=40, obs_var=2.0, noise_scale=0.5, observe="x1x3")
truth0, _, obs = simulate.lorenz_truth(2026, 400, base)
model = pf.Lorenz63Model(substeps=40, obs_var=2.0, noise_scale=0.5, observe="x1x3",
                         prior_mean=tuple(truth0), prior_var=1.0)
for timed in (False, True):
    bank = pf.FilterBank(model, 4, 1000, philox.filter_keys(7, 4), 400, dtype="float64")
    bank.load_observations(obs)
    bank.init()
    bank.run_native(0, 50)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    s.record()
    bank.run_native(50, 300, time_propagate=timed)
    t1 = time.perf_counter()
    e.record()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"time_propagate={timed}: device {s.elapsed_time(e) / 300 * 1e3:.1f} us/step, "
          f"host enqueue {(t1 - t0) / 300 * 1e6:.1f} us/step, wall {(t2 - t0) / 300 * 1e6:.1f}")
