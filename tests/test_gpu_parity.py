"""GPU parity: the B200 path (through the C-ABI) vs the CPU oracle / golden vectors.

Bit-exact for everything (integer/bit work). Mirrors the reference's own tests
(proj/tests/test_{prf,toeplitz,sampling,bitstring,pipeline}.cpp) and extends them to the
BASELINE configs. Every call below runs sm_100a kernels; there is no CPU fallback.
"""
import os

import numpy as np
import pytest

from conftest import words

pytestmark = pytest.mark.gpu
U64 = np.uint64


def bits_to_words(bits):
    n = len(bits)
    w = np.zeros(max((n + 63) // 64, 1), dtype=U64)
    for i, b in enumerate(bits):
        if b:
            w[i // 64] |= U64(1) << U64(i % 64)
    return w[: (n + 63) // 64]


def get_bit(w, i):
    return (int(w[i // 64]) >> (i % 64)) & 1


# ---------------------------------------------------------------------------------- PRF
def test_prf_block_and_kat(dev, golden):
    for c in golden["prf_block"]:
        assert (dev.prf_block(words(c["key"]), words(c["ctr"])) == words(c["out"])).all()
    w = dev.stream_words([0, 0, 0, 0], "kat", 0, 0, 2)  # test_prf.cpp:88-94
    assert int(w[0]) == 0xCAEE3B9563A0641A and int(w[1]) == 0x33477B8A6E8573EE
    for t, h in golden["tags"].items():
        assert dev.tag(t) == int(h, 16)


def test_stream_bits_golden(dev, golden, oracle):
    for c in golden["stream_bits"]:
        got = dev.stream_bits(words(c["key"]), c["purpose"], c["sub"], c["nbits"])
        assert (got == words(c["words"])).all()
    for nb in (1, 31, 32, 33, 255, 256, 257, 100003):
        assert (dev.stream_bits(3, "hash-seed", 5, nb) == oracle.bits(3, "hash-seed", 5, nb)).all()


def test_stream_uniform_bernoulli(dev, golden, oracle):
    for c in golden["uniform_below"]:
        got = dev.stream_uniform_below(words(c["key"]), c["purpose"], c["sub"], c["bound"], 0,
                                       len(c["values"]))
        assert [int(v) for v in got] == c["values"]
    got = dev.stream_uniform_below(9, "u", 2, 1000003, 1 << 40, 4096)
    want = [oracle.uniform_below(9, "u", 2, 1000003, (1 << 40) + i) for i in range(4096)]
    assert [int(v) for v in got] == want
    for c in golden["bernoulli"]:
        got = dev.stream_bernoulli(words(c["key"]), c["purpose"], 0, c["p"], 0, 256)
        assert "".join(str(get_bit(got, i)) for i in range(256)) == c["bits"]
    with pytest.raises(ValueError):
        dev.stream_uniform_below(0, "u", 0, 0, 0, 4)
    with pytest.raises(ValueError):
        dev.stream_bernoulli(0, "b", 0, 1.5, 0, 4)


def test_make_input_device(dev, oracle, golden):
    import torch

    for c in golden["extract"].values():
        if c["n"] > (1 << 24):
            continue
        buf = torch.zeros(((c["n"] + 63) // 64) * 2, dtype=torch.int32, device="cuda")
        dev.make_input_device(c["seed_in"], c["p"], c["n"], buf.data_ptr())
        torch.cuda.synchronize()
        x = buf.cpu().numpy().view(np.uint64)
        assert f"{oracle.fnv(x):016x}" == c["input_fnv"]


# ----------------------------------------------------------------------------- Toeplitz
def test_toeplitz_worked_example(dev):
    seed, x = bits_to_words([1, 0, 1, 1]), bits_to_words([1, 1, 0])
    out = dev.toeplitz_hash(seed, 2, 3, x)
    assert int(out[0]) == 1  # (1, 0), zero tail


def test_toeplitz_identity_and_zero(dev, oracle):
    assert int(dev.toeplitz_hash(bits_to_words([1]), 1, 1, bits_to_words([1]))[0]) == 1
    rng = np.random.default_rng(3)
    for m, n in ((1, 1), (5, 9), (64, 33)):
        x = oracle.bits(int(rng.integers(1 << 60)), "x", 0, n)
        out = dev.toeplitz_hash(np.zeros((m + n - 1 + 63) // 64, dtype=U64), m, n, x)
        assert int(np.unpackbits(out.view(np.uint8)).sum()) == 0


def test_toeplitz_golden(dev, golden):
    for c in golden["toeplitz"]:
        got = dev.toeplitz_hash(words(c["seed"]), c["m"], c["n"], words(c["x"]))
        assert (got == words(c["out"])).all(), (c["m"], c["n"])


def _batch_check(dev, oracle, m, cases):
    """cases: list of (seed_words, n, x_words); one GPU batch vs oracle per case."""
    ns, ins, ioff, sds, soff = [], [], [], [], []
    pos_i = pos_s = 0
    for seed, n, x in cases:
        ns.append(n)
        ioff.append(pos_i)
        soff.append(pos_s)
        ins.append(x)
        sds.append(seed)
        pos_i += len(x)
        pos_s += len(seed)
    got = dev.toeplitz_hash_batch(m, ns, np.concatenate(ins), ioff, np.concatenate(sds), soff)
    bits = np.unpackbits(got.view(np.uint8), bitorder="little")
    for q, (seed, n, x) in enumerate(cases):
        want = np.unpackbits(oracle.dense_toeplitz(seed, m, n, x).view(np.uint8),
                             bitorder="little")[:m] if m * n <= 4096 else np.unpackbits(
            oracle.toeplitz_hash(seed, m, n, x).view(np.uint8), bitorder="little")[:m]
        assert (bits[q * m:(q + 1) * m] == want).all(), (m, n, q)


def test_toeplitz_exhaustive_m_n_le_6(dev, oracle):
    # SPEC.md:524 acceptance bar (exhaustive m, n <= 6), beyond test_toeplitz.cpp:51-73
    for m in range(1, 7):
        for n in range(1, 7):
            cases = []
            for sv in range(1 << (m + n - 1)):
                for xv in range(1 << n):
                    cases.append((np.array([sv], dtype=U64), n, np.array([xv], dtype=U64)))
            _batch_check(dev, oracle, m, cases)


def test_toeplitz_randomized_1000(dev, oracle):
    # 1000 randomized cases, m <= 64, n <= 128 (test_toeplitz.cpp:75-87)
    rng = np.random.default_rng(17)
    by_m = {}
    for _ in range(1000):
        m, n = int(rng.integers(1, 65)), int(rng.integers(1, 129))
        seed = oracle.bits(int(rng.integers(1 << 62)), "s", 0, m + n - 1)
        x = oracle.bits(int(rng.integers(1 << 62)), "x", 0, n)
        by_m.setdefault(m, []).append((seed, n, x))
    for m, cases in by_m.items():
        _batch_check(dev, oracle, m, cases)


def test_toeplitz_large_shapes(dev, oracle):
    rng = np.random.default_rng(23)
    shapes = [(6300, 100000), (8192, 16384), (32768, 65536), (4097, 3), (3, 70001),
              (100, 200000), (65536, 4096), (12345, 54321)]
    for m, n in shapes:
        seed = oracle.bits(int(rng.integers(1 << 62)), "s", 0, m + n - 1)
        x = oracle.bits(int(rng.integers(1 << 62)), "x", 0, n)
        want = oracle.toeplitz_hash(seed, m, n, x)
        assert (dev.toeplitz_hash(seed, m, n, x) == want).all(), (m, n)
        # production blocking (test_toeplitz.cpp:97-103): bit-identical
        assert (dev.blocked_toeplitz_hash(seed, m, n, x, 2000, 1) == want).all()


def test_toeplitz_linearity_and_columns(dev, oracle):
    rng = np.random.default_rng(29)
    for _ in range(10):
        m, n = int(rng.integers(1, 5000)), int(rng.integers(1, 9000))
        seed = oracle.bits(int(rng.integers(1 << 62)), "s", 0, m + n - 1)
        x = oracle.bits(int(rng.integers(1 << 62)), "x", 0, n)
        y = oracle.bits(int(rng.integers(1 << 62)), "y", 0, n)
        hx, hy = dev.toeplitz_hash(seed, m, n, x), dev.toeplitz_hash(seed, m, n, y)
        assert (dev.toeplitz_hash(seed, m, n, x ^ y) == (hx ^ hy)).all()
    m, n = 9, 13  # unit vectors read out columns (test_toeplitz.cpp:121-132)
    seed = oracle.bits(31, "s", 0, m + n - 1)
    for j in range(n):
        e = np.zeros(1, dtype=U64)
        e[0] = U64(1) << U64(j)
        col = dev.toeplitz_hash(seed, m, n, e)
        for i in range(m):
            assert get_bit(col, i) == get_bit(seed, n - 1 + i - j)


def test_toeplitz_dimension_errors(dev):
    # test_toeplitz.cpp:134-140
    with pytest.raises(ValueError):
        dev.toeplitz_hash(np.zeros(1, dtype=U64), 3, 3, np.zeros(1, dtype=U64), input_bits=4)
    with pytest.raises(ValueError):
        dev.blocked_toeplitz_hash(np.zeros(1, dtype=U64), 3, 3, np.zeros(1, dtype=U64), 0, 1)
    with pytest.raises(ValueError):
        dev.toeplitz_hash(np.zeros(1, dtype=U64), 0, 3, np.zeros(1, dtype=U64))


# ------------------------------------------------------------------------------ sampler
def test_assign_subblocks(dev, oracle, golden):
    for c in golden["assign_subblocks"]:
        a, cnt = dev.assign_subblocks(c["n"], c["s"], c["seed"])
        assert [int(v) for v in a[:32]] == c["assign_head"]
        assert f"{oracle.fnv(a.astype(U64)):016x}" == c["assign_fnv"]
        assert f"{oracle.fnv(cnt):016x}" == c["raw_counts_fnv"]
    for n, s in ((1 << 20, 1024), (123457, 17), (1, 1), (33, 3), (5000, 7)):
        a, cnt = dev.assign_subblocks(n, s, 2)
        ea, ec = oracle.assign_subblocks(n, s, 2)
        assert (a == ea).all() and (cnt == ec).all()
    with pytest.raises(ValueError):
        dev.assign_subblocks(10, 0, 0)


def test_sift_partition(dev, oracle):
    rng = np.random.default_rng(5)
    for n, s in ((10000, 4), (64, 4), (1 << 18, 1000), (77777, 33), (100, 1)):
        a, _ = oracle.assign_subblocks(n, s, 0)
        for keep in (np.ones(n, np.uint8), np.zeros(n, np.uint8),
                     rng.integers(0, 2, n).astype(np.uint8)):
            off, idx, ml = dev.sift_partition(keep, a, s)
            eoff, eidx = oracle.sift_partition(keep, a, s)
            assert (off == eoff).all() and (idx == eidx).all()
            assert ml == (int(np.diff(eoff).max()) if s else 0)
    a, _ = oracle.assign_subblocks(8, 2, 0)
    with pytest.raises(ValueError):
        dev.sift_partition(np.ones(7, np.uint8), a, 2)


# ---------------------------------------------------------------------------- fused path
@pytest.mark.parametrize("name", ["1", "2", "small_perblock", "small_k_odd", "small_k_32"])
def test_extract_golden(dev, oracle, golden, name):
    c = golden["extract"][name]
    x = oracle.make_input(c["seed_in"], c["p"], c["n"])
    key, nj, st = dev.extract(x, c["n"], c["s"], c["k"], c["seed_samp"], c["seed_hash"],
                              per_block=bool(c["per_block"]))
    assert f"{oracle.fnv(nj):016x}" == c["nj_fnv"]
    assert f"{oracle.fnv(key):016x}" == c["key_fnv"]
    assert int(st.max_len) == c["nj_max"] and int(st.min_len) == c["nj_min"]
    assert int(st.hash_word_ops) == c["n"] * c["k"] // 32


def test_extract_random_vs_oracle(dev, oracle):
    rng = np.random.default_rng(11)
    for _ in range(12):
        n = int(rng.integers(1000, 300000))
        s = int(rng.choice([1, 2, 3, 8, 16, 50, 64, 100]))
        k = int(rng.choice([1, 31, 32, 33, 64, 100, 512, 1024, 3000]))
        pb = bool(rng.integers(0, 2))
        x = oracle.make_input(int(rng.integers(100)), float(rng.choice([0.5, 0.1, 0.9])), n)
        key, nj = oracle.extract(x, n, s, 21, 22, pb, k)
        gkey, gnj, _ = dev.extract(x, n, s, k, 21, 22, per_block=pb)
        assert (gnj == nj).all()
        assert (gkey == key).all(), (n, s, k, pb)


def test_extract_block_ranges_concatenate(dev, oracle):
    # multi-GPU sharding: owned block ranges concatenate to the full key (k % 64 == 0)
    n, s, k = 400000, 64, 1024
    x = oracle.make_input(3, 0.5, n)
    full, nj, _ = dev.extract(x, n, s, k, 2, 3)
    parts, lens = [], []
    for first, cnt in ((0, 16), (16, 16), (32, 20), (52, 12)):
        kk, ll, _ = dev.extract(x, n, s, k, 2, 3, block_first=first, block_count=cnt)
        parts.append(kk)
        lens.append(ll)
    assert (np.concatenate(parts) == full).all()
    assert (np.concatenate(lens) == nj).all()


def test_extract_empty_block_and_abort(dev, oracle):
    x = oracle.make_input(1, 0.5, 64)
    # 64 rounds into 1000 blocks: empty sub-blocks -> ToeplitzSeed throws (toeplitz.cpp:11-12)
    with pytest.raises(ValueError):
        dev.extract(x, 64, 1000, 8, 2, 3)
    # strict abort (sampling.cpp:92-96): limit below max n_j -> oversize abort
    x = oracle.make_input(1, 0.5, 100000)
    _, nj, _ = dev.extract(x, 100000, 8, 64, 2, 3)
    with pytest.raises(dev.AbortOversize):
        dev.extract(x, 100000, 8, 64, 2, 3, limit=int(nj.max()) - 1)
    key, _, _ = dev.extract(x, 100000, 8, 64, 2, 3, limit=int(nj.max()))
    assert len(key) == 8


def test_plan_reuse_and_device_path(dev, oracle, golden):
    import torch

    c = golden["extract"]["1"]
    n, s, k = c["n"], c["s"], c["k"]
    plan = dev.Plan(n, s, k, c["seed_samp"], c["seed_hash"])
    d_in = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
    dev.make_input_device(c["seed_in"], c["p"], n, d_in.data_ptr())
    d_key = torch.zeros(s * k // 32, dtype=torch.int32, device="cuda")
    d_len = torch.zeros(s, dtype=torch.int64, device="cuda")
    for _ in range(3):
        plan.run_device(d_in.data_ptr(), d_key.data_ptr(), d_len.data_ptr())
        plan.check()
        key = d_key.cpu().numpy().view(np.uint64)
        assert f"{oracle.fnv(key):016x}" == c["key_fnv"]
    # other seeds through the same plan
    plan.run_device(d_in.data_ptr(), d_key.data_ptr(), d_len.data_ptr(), samp=5, hsh=6)
    plan.check()
    x = d_in.cpu().numpy().view(np.uint64)
    ekey, enj = oracle.extract(x, n, s, 5, 6, 0, k)
    assert (d_key.cpu().numpy().view(np.uint64) == ekey).all()
    assert (d_len.cpu().numpy().view(np.uint64) == enj).all()
    # CUDA-graph path (capturable stream, timing off): captured once, replayed, re-captured
    # when the seeds change
    stream = torch.cuda.Stream()
    for seeds in ((c["seed_samp"], c["seed_hash"]), (c["seed_samp"], c["seed_hash"]), (5, 6)):
        d_key.zero_()
        torch.cuda.synchronize()
        plan.run_device(d_in.data_ptr(), d_key.data_ptr(), d_len.data_ptr(), stream.cuda_stream,
                        samp=seeds[0], hsh=seeds[1])
        plan.check()
        want = ekey if seeds == (5, 6) else None
        got = d_key.cpu().numpy().view(np.uint64)
        if want is None:
            assert f"{oracle.fnv(got):016x}" == c["key_fnv"]
        else:
            assert (got == want).all()
    plan.close()


@pytest.mark.parametrize("window", [-1, 0, 1, 2, 64])
def test_ranked_scatter_windows(dev, oracle, ovr, window):
    """Pass 3 of in-memory single-level plans (sampler.cu): per-bit global atomics (-1), the
    shared-memory cell window from the model (0) and forced windows — 1 and 2 words push most
    cells past the window onto the per-bit tail, 64 words hold any cell. Host runs take the
    data bit from the input (late), device runs from the payload; owned block ranges shift
    j_lo; ragged n leaves a partial last chunk."""
    import torch

    ovr(scatter_window=window)
    cases = [(300001, 3, 64, False), (200000, 64, 128, False), (1 << 20, 64, 256, False),
             (777777, 100, 96, True), (50000, 1, 32, False), (1 << 21, 1024, 32, False)]
    for n, s, k, pb in cases:
        x = oracle.make_input(n % 97, 0.5 if s != 100 else 0.2, n)
        want, wnj = oracle.extract(x, n, s, 31, 32, pb, k)
        got, nj, _ = dev.extract(x, n, s, k, 31, 32, per_block=pb)
        assert (nj == wnj).all(), (n, s, k, pb)
        assert (got == want).all(), (n, s, k, pb)
        plan = dev.Plan(n, s, k, 31, 32, per_block=pb)
        d_in = torch.from_numpy(x.view(np.int32).copy()).cuda()
        d_key = torch.zeros((s * k + 31) // 32 + 1, dtype=torch.int32, device="cuda")
        d_len = torch.zeros(s, dtype=torch.int64, device="cuda")
        plan.run_device(d_in.data_ptr(), d_key.data_ptr(), d_len.data_ptr())
        plan.check()
        assert (d_len.cpu().numpy().view(np.uint64) == wnj).all()
        if (s * k) % 64 == 0:
            assert (d_key.cpu().numpy()[: s * k // 32].view(np.uint64) == want).all(), (n, s, k)
        plan.close()
    n, s, k = 400000, 64, 1024
    x = oracle.make_input(3, 0.5, n)
    want, wnj = oracle.extract(x, n, s, 2, 3, False, k)
    parts = [dev.extract(x, n, s, k, 2, 3, block_first=f, block_count=c)[0]
             for f, c in ((0, 20), (20, 33), (53, 11))]
    assert (np.concatenate(parts) == want).all()


@pytest.mark.slow
@pytest.mark.parametrize("s", [1, 2])
def test_ranked_long_cells(dev, oracle, s):
    """Ranked passes at their largest cells: 2^29 rounds give chunks of 2^15 rounds, and with
    one or two sub-blocks a (chunk, block) cell holds up to all of them — ranks up to 2^15 in
    the payload's 16 rank bits, windows of hundreds of words in the scatter."""
    n, k = (1 << 29) + 12345, 64
    x = oracle.make_input(9, 0.5, n)
    want, wnj = oracle.extract(x, n, s, 41, 42, False, k)
    got, nj, _ = dev.extract(x, n, s, k, 41, 42)
    assert (nj == wnj).all()
    assert (got == want).all()


# ----------------------------------------------------------------- BASELINE full sizes
# SURVEY §8a anchors (computed with the compiled reference); tests/golden/gen_golden.py
# --config3 re-derives config 3 from the reference into golden.json.
SURVEY_C3 = {"key_fnv": "ea34efc57d4887a3", "nj_min": 1045673, "nj_max": 1052053,
             "nj_0": 1047749, "key_popcount": 268442266}


@pytest.mark.slow
def test_config3_full_key_digest(dev, oracle, golden):
    import torch

    c = dev.CONFIGS[3]
    want = golden["extract"].get("3", SURVEY_C3)
    n, s, k = c["n"], c["s"], c["k"]
    plan = dev.Plan(n, s, k, c["seed_samp"], c["seed_hash"])
    d_in = torch.zeros((n + 63) // 64 * 2, dtype=torch.int32, device="cuda")
    dev.make_input_device(c["seed_in"], c["p"], n, d_in.data_ptr())
    d_key = torch.zeros(s * k // 32, dtype=torch.int32, device="cuda")
    d_len = torch.zeros(s, dtype=torch.int64, device="cuda")
    plan.run_device(d_in.data_ptr(), d_key.data_ptr(), d_len.data_ptr())
    st = plan.check()
    key = d_key.cpu().numpy().view(np.uint64)
    nj = d_len.cpu().numpy().view(np.uint64)
    assert int(nj.min()) == want["nj_min"] and int(nj.max()) == want["nj_max"]
    assert int(nj[0]) == want["nj_0"] and int(nj.sum()) == n
    assert int(np.unpackbits(key.view(np.uint8)).sum()) == want["key_popcount"]
    assert f"{oracle.fnv(key):016x}" == want["key_fnv"]
    assert int(st.hash_word_ops) == n * k // 32
    plan.close()


@pytest.mark.slow
def test_config3_host_run_digest(dev, oracle, golden):
    """BASELINE configs[2] through the host entry point (ssbh_plan_run_host: input copy behind
    the count pass, key read back in slices behind the combine), twice through one plan: the
    reference's whole-key digest and block lengths."""
    import torch

    c = dev.CONFIGS[3]
    want = golden["extract"].get("3", SURVEY_C3)
    n, s, k = c["n"], c["s"], c["k"]
    d_in = torch.zeros((n + 63) // 64 * 2, dtype=torch.int32, device="cuda")
    dev.make_input_device(c["seed_in"], c["p"], n, d_in.data_ptr())
    x = d_in.cpu().numpy().view(np.uint64)
    del d_in
    plan = dev.Plan(n, s, k, c["seed_samp"], c["seed_hash"])
    for _ in range(2):
        key, nj, _ = plan.run_host(x)
        assert int(nj.sum()) == n and int(nj.max()) == want["nj_max"]
        assert f"{oracle.fnv(key):016x}" == want["key_fnv"]
    plan.close()


@pytest.mark.slow
def test_config3_block_ranges_concatenate(dev, oracle, golden):
    """Multi-GPU sharding at BASELINE configs[2]: the sub-block ranges the ranks of an N = 4 run
    own (uneven on purpose), each extracted by its own plan from the whole input, concatenate to
    the reference's whole-key digest."""
    import torch

    c = dev.CONFIGS[3]
    want = golden["extract"].get("3", SURVEY_C3)
    n, s, k = c["n"], c["s"], c["k"]
    d_in = torch.zeros((n + 63) // 64 * 2, dtype=torch.int32, device="cuda")
    dev.make_input_device(c["seed_in"], c["p"], n, d_in.data_ptr())
    d_key = torch.zeros(s * k // 32, dtype=torch.int32, device="cuda")
    d_len = torch.zeros(s, dtype=torch.int64, device="cuda")
    for first, cnt in ((0, 256), (256, 300), (556, 212), (768, 256)):
        plan = dev.Plan(n, s, k, c["seed_samp"], c["seed_hash"], block_first=first,
                        block_count=cnt)
        plan.run_device(d_in.data_ptr(), d_key[first * (k // 32):].data_ptr(),
                        d_len[first:].data_ptr())
        plan.check()
        plan.close()
    key = d_key.cpu().numpy().view(np.uint64)
    nj = d_len.cpu().numpy().view(np.uint64)
    assert int(nj.sum()) == n and int(nj.min()) == want["nj_min"]
    assert f"{oracle.fnv(key):016x}" == want["key_fnv"]


@pytest.mark.slow
@pytest.mark.parametrize("cfg", [3, 4])
def test_full_size_linearity(dev, cfg):
    """Size-independent property at BASELINE's full sizes (configs[2] and configs[3]): with the
    sampling and hash seeds fixed the extractor is GF(2)-linear in the raw string — the sampler
    moves bit i of every input to the same place and the Toeplitz product is linear — so
    key(x ^ y) = key(x) ^ key(y) and the block lengths do not depend on the data."""
    import torch

    c = dev.CONFIGS[cfg]
    n, s, k = c["n"], c["s"], c["k"]
    plan = dev.Plan(n, s, k, c["seed_samp"], c["seed_hash"], per_block=c["per_block"])
    words = (n + 63) // 64 * 2
    xs = [torch.zeros(words, dtype=torch.int32, device="cuda") for _ in range(2)]
    dev.make_input_device(c["seed_in"], c["p"], n, xs[0].data_ptr())
    dev.make_input_device(c["seed_in"] + 1000, 0.5, n, xs[1].data_ptr())
    keys, lens = [], []
    for x in (xs[0], xs[1], xs[0] ^ xs[1]):
        d_key = torch.zeros(s * k // 32, dtype=torch.int32, device="cuda")
        d_len = torch.zeros(s, dtype=torch.int64, device="cuda")
        plan.run_device(x.data_ptr(), d_key.data_ptr(), d_len.data_ptr())
        plan.check()
        keys.append(d_key)
        lens.append(d_len)
    assert bool((keys[2] == (keys[0] ^ keys[1])).all())
    assert bool((lens[0] == lens[1]).all()) and bool((lens[0] == lens[2]).all())
    assert int(keys[0].ne(0).sum()) > 0 and not bool((keys[0] == keys[1]).all())
    plan.close()


# ------------------------------------------------------------------- streaming plans
def _stream_run(dev, x_words, n, s, k, samp, hsh, chunk_bits, per_block=False, order=None,
                block_first=0, block_count=0):
    import torch

    plan = dev.Plan(n, s, k, samp, hsh, per_block=per_block, block_first=block_first,
                    block_count=block_count, chunk_bits=chunk_bits)
    owned = block_count or s
    x32 = torch.from_numpy(np.ascontiguousarray(x_words).view(np.int32).copy())
    nchunks = (n + chunk_bits - 1) // chunk_bits
    d_key = torch.zeros(((owned * k + 63) // 64) * 2, dtype=torch.int32, device="cuda")
    d_len = torch.zeros(owned, dtype=torch.int64, device="cuda")
    plan.stream_begin()
    for c in (order if order is not None else range(nchunks)):
        lo = c * chunk_bits // 32
        hi = min((c + 1) * chunk_bits, n)
        chunk = x32[lo:(hi + 31) // 32].cuda()
        plan.stream_chunk(c, chunk.data_ptr())
        torch.cuda.synchronize()
    plan.stream_finish(d_key.data_ptr(), d_len.data_ptr())
    st = plan.check()
    plan.close()
    return d_key.cpu().numpy().view(np.uint64), d_len.cpu().numpy().view(np.uint64), st


def test_streaming_plan_matches_oracle(dev, oracle):
    rng = np.random.default_rng(77)
    for (n, s, k, cb, pb) in ((300000, 16, 1024, 1 << 16, False), (250001, 50, 77, 1 << 15, True),
                              (1 << 20, 64, 8192, 1 << 17, False), (70000, 3, 96, 1 << 10, False)):
        x = oracle.make_input(int(rng.integers(1000)), 0.5, n)
        want, wnj = oracle.extract(x, n, s, 31, 32, pb, k)
        nch = (n + cb - 1) // cb
        order = list(rng.permutation(nch))  # chunks may arrive in any order
        got, nj, _ = _stream_run(dev, x, n, s, k, 31, 32, cb, per_block=pb, order=order)
        assert (nj == wnj).all()
        assert (got[: len(want)] == want).all(), (n, s, k, cb, pb)
    # owned block range in streaming mode
    n, s, k = 200000, 16, 640
    x = oracle.make_input(9, 0.5, n)
    want, _ = oracle.extract(x, n, s, 31, 32, 0, k)
    got, _, _ = _stream_run(dev, x, n, s, k, 31, 32, 1 << 14, block_first=4, block_count=8)
    kw = k // 64
    assert (got == want[4 * kw:12 * kw]).all()


@pytest.mark.slow
def test_config3_streaming_8_chunks_digest(dev, oracle, golden):
    c = dev.CONFIGS[3]
    want = golden["extract"].get("3", SURVEY_C3)
    x = oracle.make_input(c["seed_in"], c["p"], c["n"])
    got, nj, st = _stream_run(dev, x, c["n"], c["s"], c["k"], c["seed_samp"], c["seed_hash"],
                              c["n"] // 8)
    assert int(nj.min()) == want["nj_min"] and int(nj.max()) == want["nj_max"]
    assert f"{oracle.fnv(got):016x}" == want["key_fnv"]


# ------------------------------------------------ config 4 (per-block seeds, 2^34 rounds)
@pytest.mark.slow
def test_config4_full_blocks_vs_reference(dev, oracle, golden):
    """BASELINE configs[3] on one GPU: all 16384 n_j and four sub-block keys against the
    reference's own streaming computation (gen_golden.py --config4, ref_extract_selected)."""
    import torch

    want = golden["extract"].get("4")
    if want is None:
        pytest.skip("golden config-4 anchors not generated")
    c = dev.CONFIGS[4]
    n, s, k = c["n"], c["s"], c["k"]
    plan = dev.Plan(n, s, k, c["seed_samp"], c["seed_hash"], per_block=True)
    d_in = torch.zeros((n + 63) // 64 * 2, dtype=torch.int32, device="cuda")
    dev.make_input_device(c["seed_in"], c["p"], n, d_in.data_ptr())
    d_key = torch.zeros(s * k // 32, dtype=torch.int32, device="cuda")
    d_len = torch.zeros(s, dtype=torch.int64, device="cuda")
    plan.run_device(d_in.data_ptr(), d_key.data_ptr(), d_len.data_ptr())
    st = plan.check()
    nj = d_len.cpu().numpy().view(np.uint64)
    assert f"{oracle.fnv(nj):016x}" == want["nj_fnv"]
    assert int(nj.min()) == want["nj_min"] and int(nj.max()) == want["nj_max"]
    kw = k // 64
    key64 = d_key.view(torch.int64)
    for q, j in enumerate(want["which"]):
        blk = key64[j * kw:(j + 1) * kw].cpu().numpy().view(np.uint64)
        assert f"{oracle.fnv(blk):016x}" == want["block_fnv"][q], j
    assert int(st.hash_word_ops) == n * k // 32
    plan.close()
    _every_block_spot_check(oracle, want, d_in, d_key, n, s, k, c)


def _every_block_spot_check(oracle, want, d_in, d_key, n, s, k, c, rows=64):
    """EVERY block checked, not only the reference-pinned ones. The oracle
    rebuilds the whole partition from the seeds (assign_subblocks + sift + gather,
    sampling.cpp:10-39, without the 12 B/round Partition) from the input — whose digest must be
    the reference's — and recomputes `rows` output bits of each block (0, k-1 and seeded rows)
    from the definition (toeplitz.cpp:34-52, seeds of pipeline.cpp:132)."""
    x = d_in.cpu().numpy().view(np.uint64)[: (n + 63) // 64]
    assert f"{oracle.fnv(x):016x}" == want["input_fnv"]
    nj, yoff, y = oracle.partition_reversed(x, n, s, c["seed_samp"])
    assert f"{oracle.fnv(nj):016x}" == want["nj_fnv"]
    del x
    key = d_key.cpu().numpy().view(np.uint64)
    bad, first = oracle.spot_check(y, yoff, nj, c["seed_hash"], c["per_block"], k, key, rows)
    assert bad == 0, f"{bad} mismatching rows, first in block {first}"
    print(f"every-block spot check: {s} blocks x {rows} rows from the definition, 0 mismatches")


# ------------------------------------- config 5 (2^37 rounds streamed in 8 chunks, k = 2^21)
@pytest.mark.slow
def test_config5_streamed_vs_reference(dev, oracle, golden):
    """BASELINE configs[4] on one GPU through the streaming plan (8 input chunks of 2^34
    rounds): all 32768 n_j and sub-blocks 0 and 32767 against the reference's own streaming
    computation (gen_golden.py --config5, 1728 s of reference CPU time), then 64 rows of every
    block from the definition (~200 s on a 16-core host, 40 GB of host memory)."""
    import torch

    want = golden["extract"].get("5")
    if want is None:
        pytest.skip("golden config-5 anchors not generated")
    c = dev.CONFIGS[5]
    n, s, k = c["n"], c["s"], c["k"]
    chunk = n // 8
    plan = dev.Plan(n, s, k, c["seed_samp"], c["seed_hash"], per_block=False, chunk_bits=chunk)
    d_in = torch.zeros(n // 32, dtype=torch.int32, device="cuda")
    dev.make_input_device(c["seed_in"], c["p"], n, d_in.data_ptr())
    d_key = torch.zeros(s * k // 32, dtype=torch.int32, device="cuda")
    d_len = torch.zeros(s, dtype=torch.int64, device="cuda")
    plan.stream_begin()
    for ci in range(8):
        plan.stream_chunk(ci, d_in.data_ptr() + ci * (chunk // 8))
    plan.stream_finish(d_key.data_ptr(), d_len.data_ptr())
    st = plan.check()
    nj = d_len.cpu().numpy().view(np.uint64)
    assert f"{oracle.fnv(nj):016x}" == want["nj_fnv"]
    assert int(nj.min()) == want["nj_min"] and int(nj.max()) == want["nj_max"]
    assert int(nj[0]) == want["nj_0"] and int(nj[-1]) == want["nj_last"]
    kw = k // 64
    key64 = d_key.view(torch.int64)
    for q, j in enumerate(want["which"]):
        blk = key64[j * kw:(j + 1) * kw].cpu().numpy().view(np.uint64)
        assert f"{oracle.fnv(blk):016x}" == want["block_fnv"][q], j
    assert int(st.hash_word_ops) == n * k // 32
    plan.close()
    _every_block_spot_check(oracle, want, d_in, d_key, n, s, k, c)


# ------------------------------------------------------- sifted runs (keep flags)
def test_extract_sifted_matches_oracle(dev, oracle):
    rng = np.random.default_rng(21)
    for n, s, k, pb, pk in ((300000, 16, 512, False, 0.5), (200000, 33, 96, True, 0.9),
                            (150000, 5, 77, False, 0.2), (1 << 20, 32768, 64, False, 0.99)):
        x = oracle.make_input(int(rng.integers(1000)), 0.5, n)
        keep = (rng.random(n) < pk).astype(np.uint8)
        keep_words = np.packbits(np.concatenate([keep, np.zeros((-n) % 64, np.uint8)]),
                                 bitorder="little").view(np.uint64)
        try:
            want, wnj = oracle.extract_sifted(x, keep, n, s, 41, 42, pb, k)
        except ValueError:
            with pytest.raises(ValueError):  # an empty sifted sub-block, like ToeplitzSeed
                dev.extract(x, n, s, k, 41, 42, per_block=pb, keep=keep_words)
            continue
        got, nj, _ = dev.extract(x, n, s, k, 41, 42, per_block=pb, keep=keep_words)
        assert (nj == wnj).all()
        assert (got == want).all(), (n, s, k, pb, pk)


# --------------------------------------- protocol rounds + run_extraction (pipeline.cpp)
def _rounds_fnv(oracle, rounds):
    pad = np.zeros((len(rounds) + 7) // 8 * 8, dtype=np.uint8)
    pad[: len(rounds)] = rounds
    return f"{oracle.fnv(pad.view(np.uint64)):016x}"


def test_simulate_rounds_gpu(dev, oracle, golden):
    """GPU simulate_rounds vs the reference's rounds (golden) and the oracle, host and
    device entry points, aligned and unaligned device buffers, ragged lengths."""
    import torch

    for name, c in golden["pipeline"].items():
        sp = c["sim"]
        r = dev.simulate_rounds(sp["n_rounds"], sp["p_x"], sp["e_ph"], sp["e_bit"], sp["p_det"],
                                words(c["seed"]))
        assert _rounds_fnv(oracle, r) == c["rounds_fnv"], name
    rng = np.random.default_rng(71)
    for n in (1, 3, 4, 31, 33, 1000, 65537):
        args = (n, float(rng.uniform(0.01, 0.9)), float(rng.uniform(0, 0.3)),
                float(rng.uniform(0, 0.5)), float(rng.uniform(0, 1)))
        seed = [int(v) for v in rng.integers(0, 1 << 62, 4)]
        want = oracle.simulate_rounds(*args, seed)
        assert (dev.simulate_rounds(*args, seed) == want).all(), n
        buf = torch.zeros(n + 16, dtype=torch.uint8, device="cuda")
        for off in (0, 1, 3):
            buf.zero_()
            dev.simulate_rounds_device(*args, seed, buf.data_ptr() + off)
            torch.cuda.synchronize()
            got = buf.cpu().numpy()
            assert (got[off:off + n] == want).all() and not got[:off].any(), (n, off)
            assert not got[off + n:].any(), (n, off)
    with pytest.raises(ValueError):
        dev.simulate_rounds(10, 1.5, 0.0, 0.0, 1.0, 0)


def _extraction_params(dev, c):
    hp = c["params"]
    return dev.extraction_params(c["ns"], c["block_limit"], words(c["seed"]), c["key_length"],
                                 hp["eps_sec"], hp["p_x"], hp["q_tol"], hp["eta_tol"],
                                 hp["eps_abort"])


def test_run_extraction_gpu_golden(dev, oracle, golden):
    """ssbh_run_extraction vs the reference's ExtractionReport (run_extraction,
    pipeline.cpp:75-138): abort kind, bits_per_block, block lengths, key digest, epsilon."""
    for name, c in golden["pipeline"].items():
        sp = c["sim"]
        rounds = oracle.simulate_rounds(sp["n_rounds"], sp["p_x"], sp["e_ph"], sp["e_bit"],
                                        sp["p_det"], words(c["seed"]))
        key, lens, res = dev.run_extraction(rounds, _extraction_params(dev, c))
        assert res.abort == c["abort"], name
        assert res.bits_per_block == c["bits_per_block"], name
        assert res.total_epsilon == c["total_epsilon"], name
        if c["abort"] != 2:
            assert res.lengths_valid and [int(v) for v in lens] == c["block_lengths"], name
        assert res.key_bits == c["key_bits"], name
        assert f"{oracle.fnv(key):016x}" == c["key_fnv"], name


def test_run_extraction_gpu_device_rounds(dev, oracle, golden):
    """Device-resident rounds (simulate_rounds_device -> run_extraction_device), including an
    unaligned rounds pointer (byte-wise split path), vs the oracle's restatement."""
    import torch

    c = golden["pipeline"]["deterministic_ns4"]
    sp = c["sim"]
    n = sp["n_rounds"]
    want = oracle.simulate_rounds(n, sp["p_x"], sp["e_ph"], sp["e_bit"], sp["p_det"],
                                  words(c["seed"]))
    for off in (0, 5):
        buf = torch.zeros(n + 16, dtype=torch.uint8, device="cuda")
        dev.simulate_rounds_device(n, sp["p_x"], sp["e_ph"], sp["e_bit"], sp["p_det"],
                                   words(c["seed"]), buf.data_ptr() + off)
        torch.cuda.synchronize()
        key, lens, res = dev.run_extraction(None, _extraction_params(dev, c),
                                            d_rounds_ptr=buf.data_ptr() + off, n=n)
        assert f"{oracle.fnv(key):016x}" == c["key_fnv"], off
        assert [int(v) for v in lens] == c["block_lengths"]
        _, _, counts = oracle.rounds_split(want)
        assert [res.test_rounds, res.phase_errors, res.no_detections, res.key_rounds] == counts
        assert res.hash_seconds > 0


def test_run_extraction_gpu_random_vs_oracle(dev, oracle):
    """Random shapes (non-power-of-two s, p_det < 1, eta_tol < 1, odd bit counts) vs the
    oracle's restatement of the hash stage."""
    rng = np.random.default_rng(73)
    for trial in range(6):
        n = int(rng.integers(20000, 400000))
        ns = int(rng.choice([1, 2, 3, 5, 8, 13]))
        p_x, p_det = float(rng.uniform(0.02, 0.2)), float(rng.uniform(0.6, 1.0))
        eta = float(rng.uniform(0.3, 1.0)) if trial % 2 else 1.0
        seed = [int(v) for v in rng.integers(0, 1 << 62, 4)]
        rounds = oracle.simulate_rounds(n, p_x, 0.01, 0.02, p_det, seed)
        kl = int(rng.integers(0, 4000))
        lim = n  # generous cap
        args = (ns, lim, seed, kl, 1e-6, p_x, 0.05, eta, 1e-8)
        want_abort, want_key, want_lens, want_bpb = oracle.run_extraction(rounds, *args)
        key, lens, res = dev.run_extraction(rounds, dev.extraction_params(*args))
        assert res.abort == want_abort, trial
        assert res.bits_per_block == want_bpb, trial
        if want_abort != 2:
            assert (lens == want_lens).all(), trial
        assert (key == want_key).all(), trial


# ------------------------------------------- two-level split (large key spaces, BucketGeom)
# Plans with >= 4096 owned blocks split rounds by bucket (>= 128 blocks, <= 64 buckets) into staging regions
# first; the plan override buckets=1 forces that path at small sizes so every case is checked against the
# oracle: several buckets and a partial last one, non-power-of-two s, per-block seeds,
# k % 32 != 0, owned block ranges, keep masks, streaming chunks in any order, graph replay.
@pytest.fixture
def two_level(ovr):
    ovr(buckets=1)


def test_two_level_extract_vs_oracle(dev, oracle, two_level):
    rng = np.random.default_rng(91)
    cases = [(300000, 1000, 64, False), (500000, 4096, 32, True), (250000, 333, 77, True),
             (2000000, 20000, 32, False),
             (400000, 129, 1024, False), (100000, 7, 96, False)]
    for n, s, k, pb in cases:
        x = oracle.make_input(int(rng.integers(100)), float(rng.choice([0.5, 0.3])), n)
        want, wnj = oracle.extract(x, n, s, 21, 22, pb, k)
        got, nj, _ = dev.extract(x, n, s, k, 21, 22, per_block=pb)
        assert (nj == wnj).all(), (n, s, k, pb)
        assert (got == want).all(), (n, s, k, pb)
    for name in ("1", "2"):
        c = __import__("json").load(open(os.path.join(os.path.dirname(__file__), "golden",
                                                      "golden.json")))["extract"][name]
        x = oracle.make_input(c["seed_in"], c["p"], c["n"])
        key, nj, _ = dev.extract(x, c["n"], c["s"], c["k"], c["seed_samp"], c["seed_hash"])
        assert f"{oracle.fnv(key):016x}" == c["key_fnv"]


def test_two_level_ranges_keep_and_graph(dev, oracle, two_level):
    import torch

    n, s, k = 600000, 1000, 64
    x = oracle.make_input(4, 0.5, n)
    full, nj, _ = dev.extract(x, n, s, k, 2, 3)
    kk, ll, _ = dev.extract(x, n, s, k, 2, 3, block_first=300, block_count=500)
    assert (ll == nj[300:800]).all()
    assert (kk == full[300 * k // 64:800 * k // 64]).all()
    rng = np.random.default_rng(5)
    keep = (rng.random(n) < 0.7).astype(np.uint8)
    kw = np.packbits(np.concatenate([keep, np.zeros((-n) % 64, np.uint8)]),
                     bitorder="little").view(np.uint64)
    want, wnj = oracle.extract_sifted(x, keep, n, s, 2, 3, True, k)
    got, gnj, _ = dev.extract(x, n, s, k, 2, 3, per_block=True, keep=kw)
    assert (gnj == wnj).all() and (got == want).all()
    # device plan: graph capture / replay with changing seeds
    plan = dev.Plan(n, s, k, 2, 3)
    d_in = torch.from_numpy(x.view(np.int32).copy()).cuda()
    d_key = torch.zeros(s * k // 32, dtype=torch.int32, device="cuda")
    stream = torch.cuda.Stream()
    for seeds in ((2, 3), (2, 3), (8, 9)):
        plan.run_device(d_in.data_ptr(), d_key.data_ptr(), 0, stream.cuda_stream, samp=seeds[0],
                        hsh=seeds[1])
        plan.check()
        ref = full if seeds == (2, 3) else oracle.extract(x, n, s, 8, 9, 0, k)[0]
        assert (d_key.cpu().numpy().view(np.uint64) == ref).all(), seeds
    plan.close()


def test_two_level_streaming(dev, oracle, two_level):
    rng = np.random.default_rng(93)
    for (n, s, k, cb, pb) in ((600000, 1000, 64, 1 << 16, False), (300001, 257, 96, 1 << 15, True)):
        x = oracle.make_input(int(rng.integers(1000)), 0.5, n)
        want, wnj = oracle.extract(x, n, s, 31, 32, pb, k)
        # two-level streaming plans keep the blocks' running ranks from chunk to chunk (no count
        # pass over the whole input): chunks in order; any other order is refused
        got, nj, _ = _stream_run(dev, x, n, s, k, 31, 32, cb, per_block=pb)
        assert (nj == wnj).all()
        assert (got[: len(want)] == want).all(), (n, s, k, cb, pb)
        order = list(range((n + cb - 1) // cb))[::-1]
        with pytest.raises(ValueError):
            _stream_run(dev, x, n, s, k, 31, 32, cb, per_block=pb, order=order)
    n, s, k = 400000, 600, 64
    x = oracle.make_input(9, 0.5, n)
    want, _ = oracle.extract(x, n, s, 31, 32, 0, k)
    got, _, _ = _stream_run(dev, x, n, s, k, 31, 32, 1 << 14, block_first=100, block_count=300)
    assert (got == want[100:400]).all()


# ------------------------------------------------ one process over several GPUs (C-ABI)
@pytest.mark.parametrize("ndev", [2, 3])
def test_extract_multi_vs_oracle(dev, oracle, ndev):
    """ssbh_extract_multi with ranks on repeated device ids (1-GPU box): same key and n_j as
    the oracle, including bit-offset concatenation (k % 64 != 0) and per-block seeds."""
    rng = np.random.default_rng(101 + ndev)
    for n, s, k, pb in ((300000, 16, 512, False), (250001, 33, 77, True), (1 << 20, 64, 8192, False)):
        x = oracle.make_input(int(rng.integers(1000)), 0.5, n)
        want, wnj = oracle.extract(x, n, s, 2, 3, pb, k)
        got, nj, st = dev.extract_multi(x, n, s, k, 2, 3, [0] * ndev, per_block=pb)
        assert (nj == wnj).all(), (n, s, k, ndev)
        assert (got == want).all(), (n, s, k, ndev)
        assert int(st.hash_word_ops) > 0
    with pytest.raises(ValueError):
        dev.extract_multi(x, n, s, k, 2, 3, [0, 99])


def test_extract_multi_two_level_owners(dev, oracle, two_level):
    n, s, k = 600000, 900, 64
    x = oracle.make_input(12, 0.5, n)
    want, wnj = oracle.extract(x, n, s, 2, 3, True, k)
    got, nj, _ = dev.extract_multi(x, n, s, k, 2, 3, [0, 0], per_block=True)
    assert (nj == wnj).all() and (got == want).all()
