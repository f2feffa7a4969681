"""The reference-side C++ binding (integration/tec_sm100_shim.*) compiles
against the reference's own headers and links against the reference library
and libtec_sm100.so (CPU: build only; tests/test_integration_gpu.py runs it)."""
import os
import shutil
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/proj"


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "include")), reason="no reference tree")
def test_shim_builds_against_the_reference():
    if not shutil.which("make"):
        pytest.skip("no make")
    subprocess.run(["make", "-s", "-C", os.path.join(REPO, "oracle"), "shim"], check=True,
                   capture_output=True)
    exe = os.path.join(REPO, "oracle", "_ref", "shim_driver")
    assert os.path.exists(exe)
    out = subprocess.run([exe], capture_output=True, text=True)
    assert out.returncode == 2 and "usage" in out.stderr
