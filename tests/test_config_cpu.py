"""ExperimentConfig / parse_config (drop-in for parpf/config.py)."""

import pytest

from paper_1407_8071_b200.config import ExperimentConfig, config_field_names, parse_config
from paper_1407_8071_b200.exceptions import ConfigError
from paper_1407_8071_b200.metrics import MetricRecord, bias_variance, empirical_mse, loglog_slope


def test_file_and_overrides(tmp_path):
    f = tmp_path / "c.cfg"
    f.write_text("# sweep\nmodel = fhn\nM = 1,2,4\nN=100\nvariants=ensemble-bf, double-bf\n"
                 "reps=3\nT=20\nfhn_grid=8\n")
    cfg = parse_config(str(f), {"reps": "5", "seed": None})
    assert cfg.model == "fhn" and cfg.n_filters_list == [1, 2, 4]
    assert cfg.variants == ["ensemble-bf", "double-bf"] and cfg.replicates == 5
    assert cfg.reference == "truth" and cfg.fhn_grid == 8
    assert parse_config(None, {"model": "lorenz63"}).reference == "proxy"
    assert "island_period" in config_field_names()


@pytest.mark.parametrize("bad", [{"model": "x"}, {"variants": "nope"}, {"M": "1,a"},
                                 {"reps": "0"}, {"bogus": "1"}, {"T": "x"},
                                 {"reference": "both"}, {"island_period": "0"}])
def test_rejections(bad):
    with pytest.raises(ConfigError):
        parse_config(None, bad)


def test_bad_line(tmp_path):
    f = tmp_path / "c.cfg"
    f.write_text("model lorenz63\n")
    with pytest.raises(ConfigError):
        parse_config(str(f))


def test_metrics():
    assert empirical_mse([[1.0, 2.0]], [[0.0, 0.0]]) == 2.5
    b, v = bias_variance([1.0, 3.0], 1.0)
    assert b == 1.0 and v == 2.0
    assert abs(loglog_slope([1, 2, 4], [1.0, 0.5, 0.25]) + 1.0) < 1e-12
    with pytest.raises(ValueError):
        MetricRecord("v", 2, 3, 5, 1, 0, 0, 0, 0, 0, 0, 0)
    r = MetricRecord("v", 2, 3, 6, 1, 0.5, 0.1, 0.01, 1e-3, 1e-2, 0.8, 0)
    assert MetricRecord.from_row([str(x) for x in r.to_row()]) == r
    with pytest.raises(ValueError):
        ExperimentConfig(n_filters_list=[])
