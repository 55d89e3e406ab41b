"""CSV persistence (drop-in for parpf/io.py) and the harness data helpers."""

import os

import numpy as np
import pytest

from paper_1407_8071_b200 import harness, io


def test_csv_bytes_identical_to_reference(golden, tmp_path):
    g = golden["lorenz"]
    path = tmp_path / "obs.csv"
    io.write_array_csv(path, "y", g["sim_obs"][:5])
    assert path.read_text() == str(g["csv_text"])


def test_array_csv_round_trip_is_exact(tmp_path):
    rng = np.random.default_rng(0)
    a = rng.standard_normal((7, 3)) * 10.0 ** rng.integers(-300, 300, size=(7, 3))
    a[0, 0] = np.nextafter(1.0, 2.0)
    io.write_array_csv(tmp_path / "a.csv", "x", a, first_step=0)
    steps, b = io.read_array_csv(tmp_path / "a.csv")
    assert steps.tolist() == list(range(7))
    assert b.tobytes() == a.tobytes()


def test_empty_and_bad_headers(tmp_path):
    io.write_array_csv(tmp_path / "e.csv", "y", np.zeros((0, 2)))
    steps, v = io.read_array_csv(tmp_path / "e.csv")
    assert steps.shape == (0,) and v.shape == (0, 2)
    io.write_csv(tmp_path / "bad.csv", ["s", "y0"], [[1, 0.5]])
    with pytest.raises(ValueError):
        io.read_array_csv(tmp_path / "bad.csv")
    assert io.format_value(0.1) == "0.10000000000000001" and io.format_value(3) == "3"


def test_seed_hierarchy_matches_reference_bench():
    """bench.py:37-52: spawn_child(parent, i) == parent.spawn(...)[i]."""
    root = np.random.SeedSequence(42)
    kids = root.spawn(4)
    for i in range(4):
        c = harness.spawn_child(np.random.SeedSequence(42), i)
        assert c.entropy == kids[i].entropy and c.spawn_key == kids[i].spawn_key
    sim, ref, sweep = harness.root_sequences(7)
    assert sim.spawn_key == (0,) and ref.spawn_key == (1,) and sweep.spawn_key == (2,)


def test_prepare_data_reads_existing_files(tmp_path):
    obs = np.arange(6.0).reshape(3, 2)
    states = np.arange(12.0).reshape(4, 3)
    io.write_array_csv(tmp_path / "y.csv", "y", obs)
    io.write_array_csv(tmp_path / "x.csv", "x", states, first_step=0)
    s, o = harness.prepare_data(None, 3, 1, str(tmp_path / "y.csv"), str(tmp_path / "x.csv"))
    assert np.array_equal(o, obs) and np.array_equal(s, states)
    with pytest.raises(OSError):
        harness.compute_reference(None, None, o, 1, reference="truth")
