"""CPU-only tests of the product's host side (no GPU needed):

* libssbh_cuda.so / libssbh.so load and export every symbol include/ssbh_cuda.h declares;
* host scalar numerics of the C-ABI (block_limit, tail bound, cycle model) == oracle/reference;
* without a GPU every compute entry point fails loudly with SSBH_NO_DEVICE (no CPU fallback);
* the C++ drop-in BitString suite (host container) passes;
* multi-GPU sharding + key gathering logic over a world-size-2 gloo group.
"""
import ctypes
import os
import re
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "ssbh_cuda.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ssbh_[a-z0-9_]+)\s*\(", text)))


def test_abi_exports_every_declared_symbol():
    import paper_2308_02856_b200 as P

    names = header_functions()
    assert len(names) >= 30
    L = ctypes.CDLL(P.LIB_PATH)
    for nm in names:
        assert hasattr(L, nm), f"{nm} declared in include/ssbh_cuda.h but not exported"
    assert set(P.ABI_SYMBOLS) == set(names)
    assert P.lib.ssbh_abi_version() == 1
    out = subprocess.run(["nm", "-D", "--defined-only", P.CXX_LIB_PATH], capture_output=True,
                         text=True).stdout
    for sym in ("toeplitz_hash", "assign_subblocks", "sift_partition", "KeyedStream",
                "BitString", "blocked_toeplitz_hash", "block_limit", "extract"):
        assert sym in out, f"libssbh.so lacks {sym}"


def test_host_scalars_match_oracle(oracle):
    import paper_2308_02856_b200 as P

    for args in [(1000, 0.5, 0.5, 1), (999, 0.5, 0.5, 1), (1000, 0.5, 1e-6, 1),
                 (30000, 0.98 * 0.98 / 17, 1e-8, 17), (1 << 30, 1 / 1024, 1e-8, 1024)]:
        want, err = oracle.block_limit(*args)
        assert err == 0
        assert P.block_limit(*args) == want
    with pytest.raises(P.Infeasible):
        P.block_limit(20, 0.99, 1e-15, 1)
    with pytest.raises(P.Infeasible):
        P.block_limit(1000, 0.5, 1e-290, 1 << 40)
    for bad in [(1000, 0.0, 0.5, 1), (1000, 0.5, 0.0, 1), (1000, 0.5, 0.5, 0), (0, 0.5, 0.5, 1)]:
        with pytest.raises(ValueError):
            P.block_limit(*bad)
    for n, L, p in [(1000, 600, 0.5), (377, 200, 0.3), (10, 9, 0.05)]:
        # host libm numerics: the C restatement agrees to ~1 ulp; the reference itself
        # (when built) must agree exactly (test_host_scalars_match_reference)
        assert P.binomial_tail_bound(n, L, p) == pytest.approx(
            oracle.binomial_tail_bound(n, L, p), rel=1e-12)
    assert P.relative_entropy(0.6, 0.5) == pytest.approx(oracle.relative_entropy(0.6, 0.5),
                                                         rel=1e-14)
    assert P.abort_check([10, 10, 10], 10) and not P.abort_check([10, 11, 10], 10)
    assert P.abort_check([], 0)
    assert P.cycle_estimate(96040000, 6054000, 2000) == 290821228000
    with pytest.raises(ValueError):
        P.cycle_estimate(10, 10, 0)
    with pytest.raises(OverflowError):
        P.cycle_estimate(2**64 - 1, 2**64 - 1, 1)
    assert P.tag("sampling") == oracle.tag("sampling")
    # scalar Threefry (same __host__ __device__ function the kernels use)
    assert int(P.prf_block([0] * 4, [0] * 4)[0]) == 0x09218EBDE6C85537


def test_host_scalars_match_reference(reference):
    import paper_2308_02856_b200 as P

    for n, L, p in [(1000, 600, 0.5), (377, 200, 0.3), (10, 9, 0.05), (1 << 20, 17000, 1 / 64)]:
        assert P.binomial_tail_bound(n, L, p) == reference.L.ref_binomial_tail_bound(n, L, p)
    for args in [(1 << 24, 1 / 256, 1e-8, 256), (1 << 34, 1 / 16384, 1e-8, 16384)]:
        assert P.block_limit(*args) == reference.block_limit(*args)[0]


def test_no_cpu_fallback_without_gpu():
    import paper_2308_02856_b200 as P

    if P.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(P.NoDeviceError):
        P.stream_bits(1, "x", 0, 100)
    with pytest.raises(P.NoDeviceError):
        P.toeplitz_hash(np.zeros(1, np.uint64), 2, 3, np.zeros(1, np.uint64))
    with pytest.raises(P.NoDeviceError):
        P.extract(np.zeros(16, np.uint64), 1024, 4, 64, 1, 2)
    with pytest.raises(P.NoDeviceError):
        P.assign_subblocks(100, 4, 0)
    # argument errors are still reported with the reference's semantics first
    with pytest.raises(ValueError):
        P.assign_subblocks(100, 0, 0)


def test_cpp_bitstring_suite():
    exe = os.path.join(ROOT, "tests", "cpp", "bin", "test_bitstring")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", ROOT, "cpptests"], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, cwd="/tmp")
    assert r.returncode == 0, r.stdout + r.stderr


def test_owned_ranges_partition_blocks():
    from paper_2308_02856_b200.multigpu import owned_range

    for s in (1, 7, 64, 1024, 16384, 32768):
        for world in (1, 2, 3, 4, 8):
            got = [owned_range(r, world, s) for r in range(world)]
            assert got[0][0] == 0
            assert sum(c for _, c in got) == s
            for (f0, c0), (f1, _) in zip(got, got[1:]):
                assert f0 + c0 == f1
            assert max(c for _, c in got) - min(c for _, c in got) <= 1


def test_concat_bits_matches_append(oracle):
    from paper_2308_02856_b200.multigpu import concat_bits

    rng = np.random.default_rng(3)
    parts, lens, allbits = [], [], []
    for _ in range(6):
        nb = int(rng.integers(0, 300))
        b = rng.integers(0, 2, nb).astype(np.uint8)
        allbits.append(b)
        lens.append(nb)
        w = np.packbits(np.concatenate([b, np.zeros((-nb) % 64, np.uint8)]),
                        bitorder="little").view(np.uint64)
        parts.append(w)
    got = concat_bits(parts, lens)
    want_bits = np.concatenate(allbits)
    got_bits = np.unpackbits(got.view(np.uint8), bitorder="little")
    assert (got_bits[: len(want_bits)] == want_bits).all()
    assert not got_bits[len(want_bits):].any()


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.pyoracle import Oracle
    from paper_2308_02856_b200.multigpu import gather_key, owned_range

    o = Oracle()
    res = []
    for (n, s, k) in ((200000, 10, 640), (150000, 7, 77)):
        x = o.make_input(5, 0.5, n)
        first, count = owned_range(rank, world, s)
        # stand-in for the rank's GPU: the oracle computes this rank's owned blocks
        keys, _ = o.extract_selected(x, n, s, 6, 7, 0, k, list(range(first, first + count)),
                                     nthreads=2)
        bits = np.unpackbits(keys.view(np.uint8), bitorder="little").reshape(count, -1)[:, :k]
        local = np.packbits(np.concatenate([bits.reshape(-1),
                                            np.zeros((-count * k) % 64, np.uint8)]),
                            bitorder="little").view(np.uint64)
        full = gather_key(torch.from_numpy(local.view(np.int64).copy()), s, k)
        want, _ = o.extract(x, n, s, 6, 7, 0, k, nthreads=2)
        res.append(bool((full == want).all()))
    dist.destroy_process_group()
    q.put((rank, res))


def test_gloo_world2_shard_and_gather():
    import multiprocessing as mp
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, res in out:
        assert all(res), (rank, res)
