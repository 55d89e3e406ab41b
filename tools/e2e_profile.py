"""Where the fixed cost of one small run_ensemble call goes (cfg0 shape,
K observations): cProfile of the call after a warm-up call."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1407_8071_b200 as pf  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg0"]
model, obs = bench._make_model_and_obs(cfg, 13)
o = obs[:10]
for _ in range(3):
    pf.run_ensemble(model, o, "bootstrap", cfg["M"], cfg["N"], 7, dtype=cfg["dtype"],
                    estimate="projection")
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    pf.run_ensemble(model, o, "bootstrap", cfg["M"], cfg["N"], 7, dtype=cfg["dtype"],
                    estimate="projection")
torch.cuda.synchronize()
print("mean call ms", (time.perf_counter() - t0) / 20 * 1e3)
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    pf.run_ensemble(model, o, "bootstrap", cfg["M"], cfg["N"], 7, dtype=cfg["dtype"],
                    estimate="projection")
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
