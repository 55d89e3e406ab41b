"""compute-sanitizer (memcheck, racecheck, synccheck) on small launches of
the shared-memory kernels: the warp-specialised and
per-particle FH-N lattice kernels, the bank and wide resamplers, the FH-N
network bulk-copy ring and the Lorenz bank.  Each must report 0 errors.
Where the GPU pool disables compute-sanitizer, tests/test_gpu_guard.py
covers the same kernels with canary-guarded buffers and repeat-launch
determinism.""" 

import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.skipif(not os.path.exists(SAN), reason="compute-sanitizer not installed")
@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
@pytest.mark.parametrize("what", ["fhn", "fhn_tape", "resample_bank", "wide", "fhnnet", "lorenz"])
def test_kernels_are_sanitizer_clean(tool, what):
    # only the library's kernels (namespace pf: mangled _ZN2pf...)
    cmd = [SAN, "--tool", tool, "--error-exitcode", "3", "--kernel-name", "regex:_ZN2pf",
           "--launch-timeout", "120", sys.executable,
           os.path.join(REPO, "tests", "sanitize_driver.py"), what]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=REPO)
    out = r.stdout + r.stderr
    if "closed on this pool" in out:  # the GPU pool disables the tool (tests/test_gpu_guard.py)
        pytest.skip("compute-sanitizer is disabled on this GPU pool")
    assert "driver ok" in out, out[-3000:]
    assert "ERROR SUMMARY: 0 errors" in out, out[-3000:]
    assert r.returncode == 0, out[-3000:]
