"""Where the time of one run_double_bootstrap call goes (bench dbf shape,
10 observations): wall time per call after warm-up, then a cProfile."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1407_8071_b200 import islands  # noqa: E402

cfg = bench.CONFIGS["dbf"]
model, obs = bench._make_model_and_obs(cfg, 13)
o = obs[:10]
call = lambda: islands.run_double_bootstrap(model, o, cfg["M"], cfg["N"], cfg["period"], 7,  # noqa: E731
                                            dtype=cfg["dtype"])
for _ in range(2):
    call()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    call()
torch.cuda.synchronize()
print("mean call ms", (time.perf_counter() - t0) / 5 * 1e3)
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    call()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
