"""GPU parity of both hash engines.

Plans hash on the tcgen05 tensor cores by default (csrc/toeplitz_mma.cu, SSBH_ENGINE_TENSOR):
shared seeds as one u8 GEMM mod 2 over all blocks, per-block seeds as matrix-vector products
tiled into 128 x 128 Hankel blocks; SSBH_ENGINE_LOP3 keeps a plan on the integer ALUs
(csrc/toeplitz.cu). The keys must be bit-identical to the reference's toeplitz_hash
(proj/src/toeplitz.cpp:34-52) — checked here against the oracle restatement, the golden
digests made by the compiled reference, and each other. Every call runs sm_100a kernels
through the C-ABI. (The rest of the GPU suite runs shared-seed plans on the default engine.)
"""
import os

import numpy as np
import pytest

from test_gpu_parity import SURVEY_C3, _stream_run

pytestmark = pytest.mark.gpu
U64 = np.uint64


def _run_plan(dev, x, n, s, k, samp, hsh, engine, **kw):
    plan = dev.Plan(n, s, k, samp, hsh, engine=engine, **kw)
    assert plan.engine == engine
    key, nj, st = plan.run_host(x)
    plan.close()
    return key, nj, st


ENGINES = pytest.mark.parametrize("engine", [1, 2], ids=["lop3", "tensor"])


@pytest.fixture(autouse=True)
def _tensor_engine_suite(request):
    """This file pins engines per plan; a session that forces the LOP3 engine for every plan
    (--ssbh-override engine=1) runs the engine-agnostic suites instead."""
    if any(kv.replace(" ", "") == "engine=1" for kv in request.config.getoption("--ssbh-override")):
        pytest.skip("the session forces the LOP3 engine")


def test_default_engine_is_tensor(dev):
    plan = dev.Plan(100000, 8, 64, 2, 3)
    assert plan.engine == dev.ENGINE_TENSOR
    plan.set_engine(dev.ENGINE_LOP3)
    assert plan.engine == dev.ENGINE_LOP3
    plan.set_engine(dev.ENGINE_AUTO)
    assert plan.engine == dev.ENGINE_TENSOR
    plan.close()
    plan = dev.Plan(100000, 8, 64, 2, 3, per_block=True)
    assert plan.engine == dev.ENGINE_TENSOR
    plan.set_engine(dev.ENGINE_LOP3)
    assert plan.engine == dev.ENGINE_LOP3
    plan.close()


@ENGINES
def test_engine_random_shapes_vs_oracle(dev, oracle, engine):
    rng = np.random.default_rng(2308)
    shapes = [(1000, 1, 1), (5000, 3, 31), (70000, 8, 256), (300000, 64, 1024),
              (200000, 100, 33), (250000, 130, 512), (400000, 200, 96), (123457, 7, 3000),
              (1 << 20, 64, 8192), (90000, 129, 64), (60000, 2, 257), (500000, 256, 160)]
    for (n, s, k) in shapes:
        x = oracle.make_input(int(rng.integers(1000)), float(rng.choice([0.5, 0.2, 0.9])), n)
        want, wnj = oracle.extract(x, n, s, 41, 42, 0, k)
        got, nj, st = _run_plan(dev, x, n, s, k, 41, 42, engine)
        assert (nj == wnj).all()
        assert (got == want).all(), (n, s, k)
        assert int(st.hash_word_ops) == n * k // 32


def test_tensor_engine_all_ones_input(dev, oracle):
    # every operand byte saturated (0xff >> kc): the s32 sums wrap many times; the parity
    # must still be exact
    for (n, s, k) in ((1 << 18, 4, 4096), (1 << 20, 16, 2048)):
        x = np.full((n + 63) // 64, np.iinfo(np.uint64).max, dtype=U64)
        want, _ = oracle.extract(x, n, s, 5, 6, 0, k)
        got, _, _ = _run_plan(dev, x, n, s, k, 5, 6, dev.ENGINE_TENSOR)
        assert (got == want).all(), (n, s, k)


def test_shared_seed_long_blocks_use_the_tiled_kernel(dev, oracle):
    """Shared seeds with long blocks (mean n_j >= 620 K bits) run the tiled matrix-vector kernel
    (y chunks reused for 256 D steps) instead of the all-blocks GEMM; same key."""
    n, s, k = 1 << 22, 4, 4096
    x = oracle.make_input(13, 0.5, n)
    want, _ = oracle.extract(x, n, s, 9, 10, 0, k)
    plan = dev.Plan(n, s, k, 9, 10)
    assert plan.hash_kernel.startswith("k_toeplitz_mma_pb")
    got, _, _ = plan.run_host(x)
    plan.close()
    assert (got == want).all()
    if dev.get_overrides()["shared_tiled"] < 0:  # the heuristic, unless forced
        plan = dev.Plan(1 << 20, 64, 8192, 2, 3)  # config 1: short blocks keep the GEMM kernel
        assert plan.hash_kernel in ("k_toeplitz_f4", "k_toeplitz_mma")
        plan.close()


@pytest.mark.parametrize("s,k", [(64, 1024), (4096, 256)], ids=["single-level", "two-level"])
def test_host_run_overlaps_input_copy(dev, oracle, s, k):
    """Host runs of >= 2^24 rounds copy the input on a second stream while the count pass runs
    (it needs only the round indices); the scatter / bucket split take the data bits from the
    input. Same key and lengths as the oracle, and as the device-resident run."""
    import torch

    n = (1 << 26) + 12345
    x = oracle.make_input(17, 0.5, n)
    want, wnj = oracle.extract(x, n, s, 3, 4, 0, k)
    plan = dev.Plan(n, s, k, 3, 4)
    for _ in range(2):  # plan reuse: the second copy waits for the first run
        got, nj, _ = plan.run_host(x)
        assert (nj == wnj).all()
        assert (got == want).all()
    d_in = torch.from_numpy(x.view(np.int32).copy()).cuda()
    d_key = torch.zeros(((s * k + 63) // 64) * 2, dtype=torch.int32, device="cuda")
    plan.run_device(d_in.data_ptr(), d_key.data_ptr())
    plan.check()
    assert (d_key.cpu().numpy().view(U64)[: len(want)] == want).all()
    plan.close()


def _split_possible():
    """The split runs on the tensor engine unless the session forces the LOP3 engine or the
    GEMM kernel for shared seeds (--ssbh-override)."""
    import paper_2308_02856_b200 as P

    o = P.get_overrides()
    return o["engine"] != P.ENGINE_LOP3 and o["shared_tiled"] != 0


@pytest.mark.parametrize("levels,budget_mb", [(1, None), (1, 1), (2, 1), (3, None), (4, 1),
                                              (None, None)],
                         ids=["L1", "L1-batched", "L2-batched", "L3", "L4-batched", "auto"])
def test_split_hash_vs_oracle_and_lop3(dev, oracle, levels, budget_mb, ovr):
    """3-for-4 split (toeplitz_split.cu): many small squares vs the oracle (leaf buffers in
    batches of blocks when the budget is small, the last batch partial), and BASELINE-sized
    squares with a remainder vs the LOP3 engine on the same input."""
    import torch

    # levels None: the cost model; budget None: the default leaf budget
    ovr(split_levels=-1 if levels is None else levels, split_budget_mb=budget_mb or 0)
    n, s, k = (1 << 22) + 4321, 5, 4096  # T = 204 squares of 4096 per block + remainder
    x = oracle.make_input(21, 0.5, n)
    want, wnj = oracle.extract(x, n, s, 5, 6, 0, k)
    plan = dev.Plan(n, s, k, 5, 6)
    # the cost model splits only squares of >= ~2^18 (window ramp vs saved MACs)
    if _split_possible() and _split_possible():
        assert plan.hash_kernel.endswith("+split") == (levels is not None)
    got, nj, _ = plan.run_host(x)
    plan.close()
    assert (nj == wnj).all()
    assert (got == want).all()
    n, s, k = (1 << 24) + 777, 16, 1 << 19  # T = 2 squares of 2^19 per block + remainder
    x = oracle.make_input(22, 0.5, n)
    d_in = torch.from_numpy(x.view(np.int32).copy()).cuda()
    keys = []
    for engine in (dev.ENGINE_TENSOR, dev.ENGINE_LOP3):
        plan = dev.Plan(n, s, k, 7, 8, engine=engine)
        if engine == dev.ENGINE_TENSOR and _split_possible():
            assert plan.hash_kernel.endswith("+split")
        d_key = torch.zeros(s * k // 32, dtype=torch.int32, device="cuda")
        plan.run_device(d_in.data_ptr(), d_key.data_ptr())
        plan.check()
        keys.append(d_key.cpu().numpy())
        plan.close()
    assert (keys[0] == keys[1]).all()


@pytest.mark.parametrize("levels,leaf", [(5, "gemm"), (6, "gemm"), (2, "pb")])
def test_split_deep_levels_and_leaf_kernels(dev, oracle, levels, leaf, ovr):
    """Shared-seed leaves run as one GEMM per leaf matrix (k_toeplitz_f4, 128-block groups,
    512-bit padded leaf inputs) by default, or on the tiled kernel (split_tiled_leaves=1):
    deep splits and both leaf kernels vs the LOP3 engine on T = 2 squares of 2^19 + remainder."""
    import torch

    ovr(split_levels=levels, split_tiled_leaves=int(leaf == "pb"))
    n, s, k = (1 << 24) + 4097, 16, 1 << 19
    x = oracle.make_input(25, 0.5, n)
    d_in = torch.from_numpy(x.view(np.int32).copy()).cuda()
    keys = []
    for engine in (dev.ENGINE_TENSOR, dev.ENGINE_LOP3):
        plan = dev.Plan(n, s, k, 13, 14, engine=engine)
        if engine == dev.ENGINE_TENSOR and _split_possible():
            want = "k_leaf_gemm+split" if leaf == "gemm" else "k_toeplitz_mma_pb+split"
            assert plan.hash_kernel == want
            assert plan.split_geometry[:2] == (levels, 2)
        d_key = torch.zeros(s * k // 32, dtype=torch.int32, device="cuda")
        plan.run_device(d_in.data_ptr(), d_key.data_ptr())
        plan.check()
        keys.append(d_key.cpu().numpy())
        plan.close()
    assert (keys[0] == keys[1]).all()


@pytest.mark.parametrize("levels", [8, 9, None], ids=["L8-leaf-256-pieces", "L9-parent", "auto"])
def test_split_config5_block_shape(dev, oracle, levels, ovr):
    """Config 5's block shape (k = 2^21, m = 2^22) on two blocks: L = 8 runs the leaf GEMM's leaf
    mode with up to 256 input pieces per leaf (more than the 4 A warps x 32 lanes that compute
    the piece offsets in one pass), L = 9 its parent mode with 8-level combines; the cost model
    picks 9. Keys against the LOP3 engine."""
    import torch

    ovr(split_levels=-1 if levels is None else levels)
    n, s, k = (1 << 23) + 12345, 2, 1 << 21
    x = oracle.make_input(31, 0.5, n)
    d_in = torch.from_numpy(x.view(np.int32).copy()).cuda()
    keys = []
    for engine in (dev.ENGINE_TENSOR, dev.ENGINE_LOP3):
        plan = dev.Plan(n, s, k, 15, 16, engine=engine)
        if engine == dev.ENGINE_TENSOR and _split_possible():
            assert plan.hash_kernel == "k_leaf_gemm+split"
            assert plan.split_geometry[:2] == (9 if levels is None else levels, 2)
        d_key = torch.zeros(s * k // 32, dtype=torch.int32, device="cuda")
        plan.run_device(d_in.data_ptr(), d_key.data_ptr())
        plan.check()
        keys.append(d_key.cpu().numpy())
        plan.close()
    assert (keys[0] == keys[1]).all()


@pytest.mark.parametrize("levels,budget_mb", [(1, None), (3, 2), (4, None), (None, None)],
                         ids=["L1", "L3-batched", "L4", "auto"])
def test_split_per_block_seeds(dev, oracle, levels, budget_mb, ovr):
    """The split with per-block seeds (config-4 style): leaf seeds are XORs of windows of each
    block's own seed region, made per leaf batch. Small squares vs the oracle; a config-4-like
    shape (k = 3 * 2^17, T = 2 squares + a remainder) vs the LOP3 engine."""
    import torch

    ovr(split_levels=-1 if levels is None else levels, split_budget_mb=budget_mb or 0)
    if levels is not None:
        n, s, k = (1 << 21) + 999, 7, 4096
        x = oracle.make_input(23, 0.5, n)
        want, wnj = oracle.extract(x, n, s, 9, 10, 1, k)
        plan = dev.Plan(n, s, k, 9, 10, per_block=True)
        if _split_possible() and _split_possible():
            assert plan.hash_kernel.endswith("+split")
            assert plan.split_geometry[0] == levels
        got, nj, _ = plan.run_host(x)
        plan.close()
        assert (nj == wnj).all()
        assert (got == want).all()
    n, s, k = (1 << 24) + 777, 16, 3 << 17
    x = oracle.make_input(24, 0.5, n)
    d_in = torch.from_numpy(x.view(np.int32).copy()).cuda()
    keys = []
    for engine in (dev.ENGINE_TENSOR, dev.ENGINE_LOP3):
        plan = dev.Plan(n, s, k, 11, 12, per_block=True, engine=engine)
        if engine == dev.ENGINE_TENSOR:
            assert plan.hash_kernel.endswith("+split")
        d_key = torch.zeros(s * k // 32, dtype=torch.int32, device="cuda")
        plan.run_device(d_in.data_ptr(), d_key.data_ptr())
        plan.check()
        keys.append(d_key.cpu().numpy())
        plan.close()
    assert (keys[0] == keys[1]).all()


@pytest.mark.parametrize("name,levels", [("split_smoke", None), ("split_t2", None),
                                         ("split_deep", 7), ("split_deep", 3),
                                         ("split_perblock", None), ("split_perblock", 2)])
def test_split_reference_digests(dev, oracle, golden, name, levels, ovr):
    """The headline path — the 3-for-4 split (csrc/toeplitz_split.cu: leaf GEMMs / tiled
    leaves, remainder, level combine) — against digests made by running the compiled
    reference (toeplitz.cpp:34-52 hashing every block directly; gen_golden.py --split)."""
    ovr(split_levels=-1 if levels is None else levels)
    c = golden["extract"][name]
    n, s, k = c["n"], c["s"], c["k"]
    x = oracle.make_input(c["seed_in"], c["p"], n)
    plan = dev.Plan(n, s, k, c["seed_samp"], c["seed_hash"], per_block=bool(c["per_block"]))
    if _split_possible() and _split_possible():
        assert plan.hash_kernel.endswith("+split"), plan.hash_kernel
        if levels is not None:
            assert plan.split_geometry[0] == levels
    key, nj, _ = plan.run_host(x)
    plan.close()
    assert f"{oracle.fnv(nj):016x}" == c["nj_fnv"]
    assert int(np.unpackbits(key.view(np.uint8)).sum()) == c["key_popcount"]
    assert f"{oracle.fnv(key):016x}" == c["key_fnv"]


def test_split_budget_few_long_blocks(dev, ovr):
    """Few very long shared-seed blocks: GEMM leaf groups are padded to 128 blocks, so the
    leaf budget (split_budget_mb, default 8 GB) is charged for the padded batch and the plan
    falls back to tiled leaves / fewer levels instead of allocating ~390 GB (s = 4,
    n = 2^32, k = 2^19: T = 2048 squares per block)."""
    ovr(split_levels=-1, split_budget_mb=0)
    n = 1 << 32
    plan = dev.Plan(n, 4, 1 << 19, 2, 3)
    kernel, geom, nbytes = plan.hash_kernel, plan.split_geometry, plan.device_bytes
    plan.close()
    # payload (2 B/round) + reversed blocks + seed + key + the leaf budget
    assert nbytes < 2 * n + n // 8 * 2 + (8 << 30) + (1 << 30), (kernel, geom, nbytes)
    assert kernel.endswith("+split"), kernel


def test_split_host_run_key_slices(dev, oracle):
    """Host runs of >= 2^24 rounds (late input copy) on a single-batch GEMM-split plan combine
    the key in block slices and send each slice to the host behind its combine
    (abi.cu seg_hash): the host key = the device-run key = the LOP3 engine's key, on repeated
    runs through the same plan (block ranges too)."""
    import torch

    n, s, k = 1 << 26, 64, 1 << 19
    x = oracle.make_input(5, 0.5, n)
    d_in = torch.from_numpy(x.view(np.int32).copy()).cuda()
    keys = {}
    for engine in (dev.ENGINE_TENSOR, dev.ENGINE_LOP3):
        plan = dev.Plan(n, s, k, 7, 8, engine=engine)
        d_key = torch.zeros(s * k // 32, dtype=torch.int32, device="cuda")
        d_len = torch.zeros(s, dtype=torch.int64, device="cuda")
        plan.run_device(d_in.data_ptr(), d_key.data_ptr(), d_len.data_ptr())
        plan.check()
        keys[engine] = d_key.cpu().numpy().view(np.uint64)
        if engine == dev.ENGINE_TENSOR:
            assert plan.hash_kernel == "k_leaf_gemm+split"
            for _ in range(2):
                hk, hl, _ = plan.run_host(x)
                assert (hk == keys[engine]).all()
                assert (hl == d_len.cpu().numpy().view(np.uint64)).all()
        plan.close()
    assert (keys[dev.ENGINE_TENSOR] == keys[dev.ENGINE_LOP3]).all()
    plan = dev.Plan(n, s, k, 7, 8, block_first=16, block_count=40)
    hk, _, _ = plan.run_host(x)
    plan.close()
    assert (hk == keys[dev.ENGINE_TENSOR][16 * k // 64: 56 * k // 64]).all()


def test_split_disabled_by_override(dev, ovr):
    """split_levels = 0 keeps long shared blocks on the direct tiled kernel."""
    ovr(split_levels=0)
    plan = dev.Plan((1 << 22) + 4321, 5, 4096, 5, 6)
    assert not plan.hash_kernel.endswith("+split")
    plan.close()


def test_tensor_engine_block_longer_than_2p24(dev, oracle):
    """A shared-seed block of more than 2^24 input bits: the FP4 variant's f32 accumulator
    counts exactly only below 2^24, so such items accumulate in rounds whose parities XOR."""
    n, s, k = (1 << 25) + 12345, 1, 96
    x = oracle.make_input(6, 0.5, n)
    want, _ = oracle.extract(x, n, s, 7, 8, 0, k)
    got, nj, _ = _run_plan(dev, x, n, s, k, 7, 8, dev.ENGINE_TENSOR)
    assert int(nj[0]) == n
    assert (got == want).all()


@ENGINES
@pytest.mark.parametrize("name", ["1", "2", "small_k_odd", "small_k_32"])
def test_engine_golden(dev, oracle, golden, name, engine):
    c = golden["extract"][name]
    assert not c["per_block"]
    x = oracle.make_input(c["seed_in"], c["p"], c["n"])
    key, nj, _ = _run_plan(dev, x, c["n"], c["s"], c["k"], c["seed_samp"], c["seed_hash"],
                           engine)
    assert f"{oracle.fnv(nj):016x}" == c["nj_fnv"]
    assert f"{oracle.fnv(key):016x}" == c["key_fnv"]


def test_tensor_engine_switch_graph_and_ranges(dev, oracle):
    import torch

    n, s, k = 600000, 200, 2048
    x = oracle.make_input(4, 0.5, n)
    want, wnj = oracle.extract(x, n, s, 7, 8, 0, k)
    plan = dev.Plan(n, s, k, 7, 8)
    d_in = torch.from_numpy(x.view(np.int32).copy()).cuda()
    d_key = torch.zeros(s * k // 32, dtype=torch.int32, device="cuda")
    stream = torch.cuda.Stream()
    for engine in (dev.ENGINE_LOP3, dev.ENGINE_TENSOR, dev.ENGINE_TENSOR, dev.ENGINE_LOP3):
        plan.set_engine(engine)
        d_key.zero_()
        torch.cuda.synchronize()
        plan.run_device(d_in.data_ptr(), d_key.data_ptr(), 0, stream.cuda_stream)  # graph path
        plan.check()
        assert (d_key.cpu().numpy().view(U64) == want).all(), engine
    plan.close()
    # owned block ranges (multi-GPU shards) on the tensor engine
    kw = k // 64
    for first, cnt in ((0, 77), (77, 123), (190, 10)):
        got, nj, _ = _run_plan(dev, x, n, s, k, 7, 8, dev.ENGINE_TENSOR, block_first=first,
                               block_count=cnt)
        assert (got == want[first * kw:(first + cnt) * kw]).all(), (first, cnt)
        assert (nj == wnj[first:first + cnt]).all()


@ENGINES
def test_engine_streaming(dev, oracle, engine):
    n, s, k, cb = 700000, 40, 1536, 1 << 16
    x = oracle.make_input(12, 0.5, n)
    want, _ = oracle.extract(x, n, s, 31, 32, 0, k)
    import paper_2308_02856_b200 as P

    orig = P.Plan.__init__

    def init(self, *a, **kw):
        orig(self, *a, **kw)
        self.set_engine(engine)

    P.Plan.__init__ = init
    try:
        got, _, _ = _stream_run(dev, x, n, s, k, 31, 32, cb)
    finally:
        P.Plan.__init__ = orig
    assert (got[: len(want)] == want).all()


@ENGINES
def test_per_block_seeds_random_shapes_vs_oracle(dev, oracle, engine):
    """Per-block seeds (KeyedStream(hash, "hash-seed", j), pipeline.cpp:132): on the tensor
    engine every block is a matrix-vector product tiled into 128 x 128 Hankel blocks (row
    windows of 256 tiles; k = 70000 spans three windows)."""
    rng = np.random.default_rng(4)
    shapes = [(1000, 1, 1), (5000, 3, 31), (70000, 8, 256), (300000, 16, 1024),
              (200000, 10, 33), (123457, 7, 3000), (90000, 3, 70000), (400000, 40, 4096),
              (60000, 2, 257), (250000, 5, 32896)]
    for (n, s, k) in shapes:
        x = oracle.make_input(int(rng.integers(1000)), 0.5, n)
        want, wnj = oracle.extract(x, n, s, 51, 52, 1, k)
        got, nj, st = _run_plan(dev, x, n, s, k, 51, 52, engine, per_block=True)
        assert (nj == wnj).all()
        assert (got == want).all(), (n, s, k)


@ENGINES
def test_per_block_golden_and_ranges(dev, oracle, golden, engine):
    c = golden["extract"]["small_perblock"]
    x = oracle.make_input(c["seed_in"], c["p"], c["n"])
    key, nj, _ = _run_plan(dev, x, c["n"], c["s"], c["k"], c["seed_samp"], c["seed_hash"],
                           engine, per_block=True)
    assert f"{oracle.fnv(key):016x}" == c["key_fnv"]
    # owned block ranges: block j keeps its own seed stream sub = j
    n, s, k = 300000, 12, 1536
    x = oracle.make_input(8, 0.4, n)
    want, _ = oracle.extract(x, n, s, 3, 4, 1, k)
    kw = k // 64
    for first, cnt in ((0, 5), (5, 7)):
        got, _, _ = _run_plan(dev, x, n, s, k, 3, 4, engine, per_block=True, block_first=first,
                              block_count=cnt)
        assert (got == want[first * kw:(first + cnt) * kw]).all()


def test_tensor_engine_empty_block_semantics(dev, oracle):
    x = oracle.make_input(1, 0.5, 64)
    plan = dev.Plan(64, 1000, 8, 2, 3, engine=dev.ENGINE_TENSOR)
    with pytest.raises(ValueError):  # ToeplitzSeed throws for n_j = 0 (toeplitz.cpp:11-12)
        plan.run_host(x)
    plan.close()


@pytest.mark.slow
def test_lop3_engine_config3_full_key_digest(dev, oracle, golden):
    """The integer-ALU engine (north_star's kernel) on BASELINE config 3; the default-engine
    run is test_gpu_parity.py::test_config3_full_key_digest."""
    import torch

    c = dev.CONFIGS[3]
    want = golden["extract"].get("3", SURVEY_C3)
    n, s, k = c["n"], c["s"], c["k"]
    plan = dev.Plan(n, s, k, c["seed_samp"], c["seed_hash"], engine=dev.ENGINE_LOP3)
    d_in = torch.zeros((n + 63) // 64 * 2, dtype=torch.int32, device="cuda")
    dev.make_input_device(c["seed_in"], c["p"], n, d_in.data_ptr())
    d_key = torch.zeros(s * k // 32, dtype=torch.int32, device="cuda")
    d_len = torch.zeros(s, dtype=torch.int64, device="cuda")
    plan.run_device(d_in.data_ptr(), d_key.data_ptr(), d_len.data_ptr())
    plan.check()
    key = d_key.cpu().numpy().view(U64)
    assert int(np.unpackbits(key.view(np.uint8)).sum()) == want["key_popcount"]
    assert f"{oracle.fnv(key):016x}" == want["key_fnv"]
    plan.close()
