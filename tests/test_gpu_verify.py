"""The reference's acceptance suite (verify.py, default = acceptance-level
parameters) run on the GPU bank, plus the sweep driver (bench.py:136-214)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1407_8071_b200 import verify  # noqa: E402
from paper_1407_8071_b200.config import ExperimentConfig  # noqa: E402
from paper_1407_8071_b200.harness import run_sweep  # noqa: E402
from paper_1407_8071_b200.io import read_metric_records, write_metric_records  # noqa: E402


@pytest.mark.parametrize("name", [n for n in verify.ALL_CHECKS if n != "fhn_tracking"])
def test_acceptance_check(name):
    res = verify.run_checks([name])[0]
    print(res.line())
    assert res.passed, res.line()


def test_sweep_all_variants(tmp_path):
    cfg = ExperimentConfig(model="lorenz63",
                           variants=["centralised-bf", "ensemble-bf", "ensemble-apf", "double-bf"],
                           n_filters_list=[2, 4], n_particles_list=[64], replicates=4,
                           n_observations=12, seed=11, proxy_particles=2000,
                           out_path=str(tmp_path / "m.csv"))
    recs = run_sweep(cfg)
    assert [(r.variant, r.n_filters) for r in recs] == [
        (v, m) for v in cfg.variants for m in (2, 4)]
    for r in recs:
        assert r.total_particles == r.n_filters * r.n_particles and r.replicates == 4
        assert np.isfinite(r.mse_mean) and r.mse_mean > 0 and np.isfinite(r.bias_sq)
    idx = {r.variant: r.time_error_index for r in recs if r.n_filters == 4}
    assert idx["centralised-bf"] == 1.0 and idx["ensemble-bf"] == 0.25 + 1 / 64
    assert np.isnan(idx["double-bf"])
    write_metric_records(cfg.out_path, recs)
    back = read_metric_records(cfg.out_path)
    from paper_1407_8071_b200.io import format_value

    assert [[format_value(v) for v in b.to_row()] for b in back] == \
        [[format_value(v) for v in r.to_row()] for r in recs]
    again = run_sweep(cfg)
    for a, b in zip(recs, again):
        assert (a.mse_mean, a.mse_var, a.bias_sq, a.collapse_count) == \
            (b.mse_mean, b.mse_var, b.bias_sq, b.collapse_count)


def test_sweep_fhn_network_truth_reference():
    cfg = ExperimentConfig(model="fhn", variants=["ensemble-apf", "centralised-bf"],
                           n_filters_list=[2], n_particles_list=[32], replicates=2,
                           n_observations=20, seed=3, fhn_grid=16)
    recs = run_sweep(cfg)
    assert cfg.reference == "truth"
    assert all(np.isfinite(r.mse_mean) for r in recs)
