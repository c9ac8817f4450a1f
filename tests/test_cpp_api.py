"""Runs the C++ drop-in API suites (tests/cpp/*.cpp, linked against libssbh.so ->
libssbh_cuda.so) on the GPU. They mirror the reference's own doctest suites
(proj/tests/test_{prf,toeplitz,sampling}.cpp, test_pipeline.cpp:126-149)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "bin")


@pytest.mark.gpu
@pytest.mark.parametrize("suite", ["test_prf", "test_toeplitz", "test_sampling", "test_extract",
                                   "test_pipeline"])
def test_cpp_suite(suite):
    exe = os.path.join(BIN, suite)
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", ROOT, "cpptests"], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, cwd="/tmp", timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "0 failed cases" in r.stdout
