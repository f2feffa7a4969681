"""Hazard checks over every kernel family (tools/kernel_zoo.py: each kernel
on small shapes) -- the analogue of the reference's race detection
(race_check, R/src/interp.cpp:548-580, and the VDLA token check,
R/src/vdla.cpp:835-853):
  * results against the oracle (host path);
  * out-of-bounds writes: 1 MiB canary guards around every output (device
    path) must survive;
  * races: repeated launches, and launches on fewer persistent CTAs, must be
    bit-identical (every reduction order is fixed by construction);
  * compute-sanitizer memcheck / racecheck / synccheck when the GPU pool
    allows it (this pool refuses it: runs under it left GPUs needing a reset
    -- the tests then skip with the pool's message);
  * a mutation test of the pipeline's mbarrier watchdog: with one
    accumulator-free arrive dropped (TEC_SM100_FAULT=1) the kernel must TRAP
    within the watchdog window instead of hanging the GPU."""
import os
import shutil
import subprocess
import sys
import time

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ZOO = os.path.join(REPO, "tools", "kernel_zoo.py")
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


def test_kernel_zoo_plain():
    r = subprocess.run([sys.executable, ZOO], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.skipif(not os.path.exists(SAN), reason="compute-sanitizer not installed")
@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer(tool):
    r = subprocess.run([SAN, "--tool", tool, "--error-exitcode", "9", "--print-limit", "20",
                        sys.executable, ZOO], capture_output=True, text=True, timeout=1800)
    out = r.stdout + r.stderr
    if "closed on this pool" in out:
        pytest.skip(out.strip().splitlines()[0])
    assert "ERROR SUMMARY: 0 errors" in out, out[-4000:]
    assert r.returncode == 0, out[-4000:]


def test_dropped_arrive_traps_instead_of_hanging():
    t0 = time.time()
    r = subprocess.run([sys.executable, ZOO, "--fault"], capture_output=True, text=True,
                       timeout=300)
    dt = time.time() - t0
    out = r.stdout + r.stderr
    assert r.returncode != 0, out
    assert "returned without a trap" not in out
    assert "CudaError" in out or "CUDA" in out, out[-2000:]
    assert dt < 120, dt
