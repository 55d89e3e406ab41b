"""Host-side checks of bench.py's roofline bookkeeping (no GPU)."""
import importlib
import json
import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    sys.path.insert(0, REPO)
    return importlib.import_module("bench")


def test_issue_roofline_and_dispatch_model(bench):
    """frac = warp instructions / kernel time / (148 x 4 x clock); the dispatch
    model adds (slots - 1) per IMAD.WIDE and MUFU and scales with the bank."""
    pipes = {"warp_inst_per_launch": 1.0e9, "imad_wide_per_launch": 2.0e8,
             "mufu_per_launch": 1.0e8}
    roof = bench._issue_roofline(pipes, 2.0)
    peak = 148 * 4 * 1965e6
    assert roof["bound"] == "issue" and roof["peak"] == peak
    assert roof["frac"] == pytest.approx(1.0e9 / 2.0e-3 / peak)
    slots = 1.0e9 + (bench.DISPATCH_SLOTS["imad_wide"] - 1) * 2.0e8 \
        + (bench.DISPATCH_SLOTS["mufu"] - 1) * 1.0e8
    assert roof["dispatch_model"]["slots_per_launch"] == pytest.approx(slots)
    assert roof["dispatch_model"]["frac"] == pytest.approx(slots / 2.0e-3 / peak)
    # a capture scaled to another bank size scales the opcode counts with it
    half = dict(pipes, warp_inst_captured=1.0e9, warp_inst_per_launch=0.5e9)
    assert bench._issue_roofline(half, 1.0)["dispatch_model"]["frac"] == pytest.approx(
        roof["dispatch_model"]["frac"])
    assert bench._issue_roofline(None, 1.0) is None
    assert "dispatch_model" not in bench._issue_roofline({"warp_inst_per_launch": 1e9}, 1.0)


def test_committed_pipe_tables_feed_the_model(bench):
    """profiles/pipes.json carries the opcode counts of the captured kernels and
    the scaled configs inherit them."""
    with open(os.path.join(REPO, "profiles", "pipes.json")) as fh:
        pipes = json.load(fh)
    for cfg in ("cfg4", "cfg2"):
        p = pipes[cfg]
        assert 0 < p["imad_wide_per_launch"] < p["warp_inst_per_launch"]
        assert 0 < p["mufu_per_launch"] < p["warp_inst_per_launch"]
    cfg3 = bench._ncu_pipes("cfg3")
    ratio = (8 * 512) / (64 * 4096)
    assert cfg3["warp_inst_per_launch"] == pytest.approx(
        pipes["cfg4"]["warp_inst_per_launch"] * ratio)
    assert cfg3["warp_inst_captured"] == pipes["cfg4"]["warp_inst_per_launch"]


def test_both_arms_name_the_same_config(bench):
    """The reference arm's `config` equals the GPU arm's for the bank workloads
    (the driver compares them)."""
    class A:
        config = "cfg4"
        gpus = 1
    cfg = bench.CONFIGS["cfg4"]
    ours = bench._bank_config(A, cfg, 1, 50, 2 * 30 * 50 * 4)
    ref = bench._bank_config(A, cfg, A.gpus, *bench._KIND_SHAPE["fhn"])
    assert ours == ref
    assert ours["M"] == 64 and ours["N"] == 4096 and ours["euler_steps_per_obs"] == 50
    assert bench._KIND_SHAPE["lorenz"] == (40, 12)
