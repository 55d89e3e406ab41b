import time, sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1407_8071_b200 as pf
from paper_1407_8071_b200 import simulate
from paper_1407_8071_b200.models import FhnLatticeModel, FhnNetworkModel
model, _, obs = simulate.fhn_truth(2026, 10, FhnLatticeModel())
for rep in range(5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    out = pf.run_ensemble(model, obs, "bootstrap", 8, 512, 7, dtype="float32", estimate="projection")
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print("cfg3 e2e ms", round(1e3*(t1-t0),2), "device ms", round(1e3*out.filter_outputs[0].total_seconds,2))
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
out = pf.run_ensemble(model, obs, "bootstrap", 8, 512, 7, dtype="float32", estimate="projection")
torch.cuda.synchronize()
pr.disable(); pstats.Stats(pr).sort_stats('cumulative').print_stats(18)
