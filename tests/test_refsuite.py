"""The reference's OWN doctest suites (proj/tests/test_{bitstring,prf,toeplitz,sampling,
pipeline,bbm92}.cpp), compiled unmodified against the B200 drop-in (include/ssbh +
libssbh.so -> libssbh_cuda.so) by tests/refsuite/Makefile with a doctest-compatible shim.

test_pipeline runs twice: with the reference's own run_extraction (its per-block loop,
pipeline.cpp:129-136, calling the GPU toeplitz_hash / KeyedStream::bits / assign_subblocks /
sift_partition) and with the drop-in's fused GPU run_extraction (the reference's
pipeline.cpp kept only for scenario_compare / scenario_csv). The binaries are built in the
build container (they need /root/reference) and travel to the GPU box."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "refsuite", "bin")
SUITES = ["bitstring", "prf", "toeplitz", "sampling", "pipeline_loop", "pipeline_fused", "bbm92"]


def _exe(suite):
    exe = os.path.join(BIN, f"ref_test_{suite}")
    if not os.path.exists(exe):
        if os.path.isdir("/root/reference/proj"):
            subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "refsuite")], check=True)
        else:
            pytest.skip("reference suites not built (needs /root/reference at build time)")
    return exe


def test_refsuite_binaries_link_the_drop_in():
    """Every suite binary resolves ssbh:: data-path symbols from libssbh.so (no reference
    bitstring/prf/sampling/toeplitz objects are linked)."""
    for suite in SUITES:
        exe = _exe(suite)
        syms = subprocess.run(["nm", "-C", exe], capture_output=True, text=True).stdout
        for fn in ("ssbh::toeplitz_hash(", "ssbh::assign_subblocks(",
                   "ssbh::sift_partition(", "ssbh::KeyedStream::bits("):
            defined = [l for l in syms.splitlines()
                       if fn in l and len(l.split(None, 2)) == 3 and l.split(None, 2)[1] in "TtWw"]
            assert not defined, (suite, defined)
        libs = subprocess.run(["ldd", exe], capture_output=True, text=True).stdout
        assert "libssbh.so" in libs and "libssbh_cuda.so" in libs, libs


@pytest.mark.gpu
@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_on_drop_in(suite):
    exe = _exe(suite)
    r = subprocess.run([exe], capture_output=True, text=True, cwd="/tmp", timeout=1500)
    tail = r.stdout[-2000:] + r.stderr[-4000:]
    assert r.returncode == 0, tail
    assert " 0 failed cases" in r.stdout, tail
    print(r.stdout.strip().splitlines()[-1])
