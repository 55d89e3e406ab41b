"""ExperimentConfig (the sweep specification run_sweep consumes) and the
sweep statistics in metrics.py."""

import pytest

from paper_1407_8071_b200.config import ExperimentConfig
from paper_1407_8071_b200.exceptions import ConfigError
from paper_1407_8071_b200.metrics import MetricRecord, bias_variance, empirical_mse, loglog_slope


def test_defaults_and_cells():
    cfg = ExperimentConfig(model="fhn", variants=["ensemble-bf", "double-bf"],
                           n_filters_list=[1, 2], n_particles_list=[100])
    assert cfg.reference == "truth" and cfg.workers >= 1
    assert ExperimentConfig().reference == "proxy"
    assert cfg.cells == [("ensemble-bf", 1, 100), ("ensemble-bf", 2, 100),
                         ("double-bf", 1, 100), ("double-bf", 2, 100)]


@pytest.mark.parametrize("bad", [{"model": "x"}, {"variants": ["nope"]}, {"variants": []},
                                 {"n_filters_list": []}, {"n_particles_list": [0]},
                                 {"replicates": 0}, {"reference": "both"},
                                 {"island_period": 0}, {"workers": -1},
                                 {"n_observations": -1}])
def test_rejections(bad):
    with pytest.raises(ConfigError):
        ExperimentConfig(**bad)


def test_metrics():
    assert empirical_mse([[1.0, 2.0]], [[0.0, 0.0]]) == 2.5
    with pytest.raises(ValueError):
        empirical_mse([1.0, 2.0], [[1.0, 2.0]])
    b, v = bias_variance([1.0, 3.0], 1.0)
    assert b == 1.0 and v == 2.0
    assert abs(loglog_slope([1, 2, 4], [1.0, 0.5, 0.25]) + 1.0) < 1e-12
    assert abs(loglog_slope([1, 10, 100], [3.0, 0.3, 0.03]) + 1.0) < 1e-12
    with pytest.raises(ValueError):
        loglog_slope([1, 2], [1.0, -1.0])
    with pytest.raises(ValueError):
        MetricRecord("v", 2, 3, 5, 1, 0, 0, 0, 0, 0, 0, 0)
    r = MetricRecord("v", 2, 3, 6, 1, 0.5, 0.1, 0.01, 1e-3, 1e-2, 0.8, 0)
    assert MetricRecord.from_row([str(x) for x in r.to_row()]) == r
    assert MetricRecord.CSV_HEADER[:5] == ("variant", "M", "N", "K", "reps")
