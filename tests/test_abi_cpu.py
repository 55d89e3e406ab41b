"""CPU-side checks of the C-ABI boundary: libpfbank.so loads without a GPU
and exports every symbol include/pfbank.h declares, with matching ctypes
signatures; the Philox host mirror reproduces the published known answers."""

import os
import re

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(REPO, "include", "pfbank.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pf_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1407_8071_b200 import _build, _lib

    if not os.path.exists(_lib.LIB_PATH):
        _build.build(verbose=False)
    return _lib.load()


def test_header_declares_the_abi():
    fns = _header_functions()
    for name in ("pf_segmented_resample", "pf_lorenz_propagate_weight", "pf_fhn_interval",
                 "pf_filter_estimate", "pf_op_resample_indices", "pf_op_lorenz_euler_block",
                 "pf_op_fhn_euler_block", "pf_op_normalize_log_weights"):
        assert name in fns


def test_library_exports_every_header_symbol(lib):
    from paper_1407_8071_b200 import _lib

    for name in _header_functions():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"
    assert set(_lib.SIGNATURES) == set(_header_functions())


def test_library_basic_calls_without_gpu(lib):
    assert lib.pf_version() >= 10000
    # argument validation happens before any CUDA call
    from paper_1407_8071_b200 import _lib

    with pytest.raises(ValueError):
        _lib.call("pf_segmented_resample", _lib.PF_F32, None, 1, 16, None, None, 1, None, None,
                  None, None, None, 0, None)
    assert lib.pf_resample_workspace_bytes(4, 1024) == 0
    assert lib.pf_resample_workspace_bytes(1, 1 << 26) > 8 * (1 << 26)


def test_philox_known_answers():
    """Random123 philox4x32-10 known-answer vectors (kat_vectors)."""
    from paper_1407_8071_b200.philox import philox4x32_10

    ctr = np.array([[0, 0, 0, 0], [0xFFFFFFFF] * 4,
                    [0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344]], dtype=np.uint32)
    key = np.array([[0, 0], [0xFFFFFFFF, 0xFFFFFFFF], [0xA4093822, 0x299F31D0]], dtype=np.uint32)
    want = np.array([[0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8],
                     [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD],
                     [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]], dtype=np.uint32)
    assert np.array_equal(philox4x32_10(ctr, key), want)


def test_seed_keys_follow_the_reference_seed_tree():
    from paper_1407_8071_b200 import philox

    ks = philox.filter_keys(5, 3)
    kids = np.random.SeedSequence(5).spawn(3)
    for k, c in zip(ks, kids):
        assert np.array_equal(k, c.generate_state(2, dtype=np.uint32))
    assert np.array_equal(philox.seed_key(philox.filter_seeds(5, 1)[0]), ks[0])


@pytest.mark.parametrize("entropy", [0, 1, 5, 7107, 2**32, 2**40 + 3, 12345678901234567890,
                                     [3, 1, 4, 1, 5, 9, 2, 6]])
def test_vectorised_seed_keys_equal_numpy_seed_sequence(entropy):
    """philox.child_keys / seed_keys restate numpy's SeedSequence hashing;
    they must equal generate_state(2) of the objects numpy builds."""
    import copy

    from paper_1407_8071_b200 import philox

    root = np.random.SeedSequence(entropy)
    parents = [root, root.spawn(2)[1], root.spawn(3)[2].spawn(5)[4],
               np.random.SeedSequence(entropy, spawn_key=(2**33, 7))]
    for par in parents:
        for extra in (0, 3):
            p2 = copy.deepcopy(par)
            if extra:
                p2.spawn(extra)
            start = p2.n_children_spawned
            want = np.stack([c.generate_state(2, np.uint32) for c in p2.spawn(41)])
            assert np.array_equal(philox.child_keys(par, start, 41), want)
    seeds = [root] + parents[1:] + np.random.SeedSequence(entropy).spawn(5) + [9, 2**70]
    want = np.stack([philox.seed_key(s) for s in seeds])
    assert np.array_equal(philox.seed_keys(seeds), want)


def test_ensemble_seeds_advance_a_seed_sequence_master_like_the_reference():
    """ensemble.py:56-60: the filters of run_ensemble(master=ss) are
    ss.spawn(M), which advances ss; the filter outputs carry those children."""
    from paper_1407_8071_b200 import philox

    ss = np.random.SeedSequence(11)
    ss.spawn(2)
    keys, seeds = philox.filter_keys_and_seeds(ss, 4)
    assert ss.n_children_spawned == 6
    ref = np.random.SeedSequence(11).spawn(6)[2:]
    for f in range(4):
        assert seeds[f].spawn_key == ref[f].spawn_key
        assert np.array_equal(keys[f], ref[f].generate_state(2, np.uint32))
    # an int master is not advanced (there is no object) and starts at child 0
    k5, s5 = philox.filter_keys_and_seeds(5, 3)
    assert s5[2].spawn_key == (2,)
    assert np.array_equal(k5, philox.filter_keys(5, 3))


def test_product_fails_loudly_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1407_8071_b200 as pf

    with pytest.raises(RuntimeError, match="CUDA"):
        pf.normalize_log_weights(np.zeros(4))


def _header_prototypes():
    src = open(os.path.join(REPO, "include", "pfbank.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    out = {}
    for m in re.finditer(r"\b(pf_[a-z0-9_]+)\s*\(([^)]*)\)\s*;", src):
        args = m.group(2).strip()
        out[m.group(1)] = 0 if args in ("", "void") else len(args.split(","))
    return out


def test_ctypes_argument_counts_match_header():
    from paper_1407_8071_b200 import _lib

    protos = _header_prototypes()
    for name, (_, argtypes) in _lib.SIGNATURES.items():
        assert protos[name] == len(argtypes), name


def test_ctypes_struct_layouts_match_c(tmp_path):
    """sizeof/offsetof of every ABI struct as gcc lays it out == ctypes."""
    import ctypes
    import shutil
    import subprocess

    from paper_1407_8071_b200 import _lib

    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    structs = {"pf_lorenz_params": _lib.LorenzParams, "pf_fhn_params": _lib.FhnParams,
               "pf_fhnnet_params": _lib.FhnNetParams, "pf_hmm_params": _lib.HmmParams,
               "pf_lgm_params": _lib.LgmParams, "pf_bank_desc": _lib.BankDesc,
               "pf_island_desc": _lib.IslandDesc}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "pfbank.h"',
             "int main(void) {"]
    for cname, cls in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            lines.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0; }")
    c = tmp_path / "layout.c"
    c.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(REPO, "include"), str(c), "-o", str(exe)],
                   check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True,
                                                       text=True, check=True).stdout.splitlines())
    for cname, cls in structs.items():
        assert int(got[cname]) == ctypes.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(cls, fname).offset, (cname, fname)


def test_library_binds_every_symbol_now(lib):
    """RTLD_NOW load: every symbol the library references resolves (catches an
    internal C++ entry point declared but not linked in)."""
    import ctypes

    from paper_1407_8071_b200 import _lib

    ctypes.CDLL(_lib.LIB_PATH, mode=os.RTLD_NOW)


def test_nccl_bound_at_run_time(lib):
    """pf_comm_* binds the libnccl.so.2 torch already loaded (no link-time
    NCCL dependency; one NCCL per process)."""
    import torch  # noqa: F401  (loads libnccl.so.2)

    assert lib.pf_comm_available() == 1
    assert lib.pf_comm_nccl_version() >= 21800
    import subprocess

    out = subprocess.run(["readelf", "-d", str(lib._name)], capture_output=True, text=True).stdout
    assert "libnccl" not in out


def test_kernel_flags_are_per_call():
    """No process-wide kernel switches: the library's sources read no
    environment variables (the generic/fast choice is the *_ex calls' flags
    argument; the static CUDA runtime's own getenv use is not ours)."""
    import glob

    for path in glob.glob(os.path.join(REPO, "paper_1407_8071_b200", "csrc", "*.cu*")):
        assert "getenv" not in open(path).read(), path
