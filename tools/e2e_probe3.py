"""Where the cfg2 end-to-end time goes (run_ensemble on host observations)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1407_8071_b200 as pf  # noqa: E402
from paper_1407_8071_b200 import simulate  # noqa: E402
from paper_1407_8071_b200.models import Lorenz63Model  # noqa: E402

base = Lorenz63Model(substeps=40, obs_var=2.0, noise_scale=0.5, observe="x1x3")
truth0, _, obs = simulate.lorenz_truth(2026, 13, base)
model = Lorenz63Model(substeps=40, obs_var=2.0, noise_scale=0.5, observe="x1x3",
                      prior_mean=tuple(truth0), prior_var=1.0)
o = obs[:10]
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = pf.run_ensemble(model, o, "bootstrap", 4096, 1024, 7, dtype="float32",
                          estimate="projection")
    torch.cuda.synchronize()
    print("cfg2 e2e ms", round(1e3 * (time.perf_counter() - t0), 3))
import cProfile  # noqa: E402
import pstats  # noqa: E402

pr = cProfile.Profile()
pr.enable()
out = pf.run_ensemble(model, o, "bootstrap", 4096, 1024, 7, dtype="float32", estimate="projection")
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
