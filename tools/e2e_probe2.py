import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1407_8071_b200 as pf  # noqa: E402
from paper_1407_8071_b200 import simulate  # noqa: E402

base = pf.Lorenz63Model(substeps=40, obs_var=2.0, noise_scale=0.5, observe="x1x3")
truth0, _, obs = simulate.lorenz_truth(2026, 13, base)
model = pf.Lorenz63Model(substeps=40, obs_var=2.0, noise_scale=0.5, observe="x1x3",
                         prior_mean=tuple(truth0), prior_var=1.0)
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = pf.run_ensemble(model, obs[:10], "bootstrap", 4096, 1024, 7, dtype="float32",
                          estimate="projection")
    torch.cuda.synchronize()
    print("e2e ms", 1e3 * (time.perf_counter() - t0), "device ms",
          1e3 * out.filter_outputs[0].total_seconds)
pr = cProfile.Profile()
pr.enable()
out = pf.run_ensemble(model, obs[:10], "bootstrap", 4096, 1024, 7, dtype="float32",
                      estimate="projection")
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
