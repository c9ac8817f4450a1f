"""CPU tests: pin the C restatement (oracle/oracle.c) against the reference itself.

(1) the reference's own known-answer tests (proj/tests/test_prf.cpp:88-94,
    test_toeplitz.cpp:39-49, test_bitstring.cpp:29-46), (2) golden vectors produced by
running the compiled reference (tests/golden/golden.json, gen_golden.py), and (3) live
cross-checks against oracle/_ref when it is present.
"""
import numpy as np
import pytest

from conftest import words

U64 = np.uint64


def bits_to_words(bits):
    n = len(bits)
    w = np.zeros(max((n + 63) // 64, 1), dtype=U64)
    for i, b in enumerate(bits):
        if b:
            w[i // 64] |= U64(1) << U64(i % 64)
    return w[: (n + 63) // 64]


def test_threefry_kat(oracle, golden):
    # proj/tests/test_prf.cpp:88-94
    assert oracle.word([0, 0, 0, 0], "kat", 0, 0) == 0xCAEE3B9563A0641A
    assert oracle.word([0, 0, 0, 0], "kat", 0, 1) == 0x33477B8A6E8573EE
    for case in golden["prf_block"]:
        assert (oracle.threefry(words(case["key"]), words(case["ctr"])) == words(case["out"])).all()


def test_tags(oracle, golden):
    for t, h in golden["tags"].items():
        assert oracle.tag(t) == int(h, 16)


def test_stream_bits(oracle, golden):
    for c in golden["stream_bits"]:
        got = oracle.bits(words(c["key"]), c["purpose"], c["sub"], c["nbits"])
        assert (got == words(c["words"])).all()
    # prefix stability (prf.cpp:104-115): bits(1000) is a prefix of bits(5000)
    a = oracle.bits(3, "hash-seed", 0, 1000)
    b = oracle.bits(3, "hash-seed", 0, 5000)
    assert (a[:-1] == b[: len(a) - 1]).all()
    assert a[-1] == b[len(a) - 1] & U64((1 << (1000 % 64)) - 1)


def test_uniform_and_bernoulli(oracle, golden):
    for c in golden["uniform_below"]:
        got = [oracle.uniform_below(words(c["key"]), c["purpose"], c["sub"], c["bound"], i)
               for i in range(len(c["values"]))]
        assert got == c["values"]
    for c in golden["bernoulli"]:
        got = "".join(str(oracle.bernoulli(words(c["key"]), c["purpose"], 0, c["p"], i))
                      for i in range(256))
        assert got == c["bits"]


def test_toeplitz_worked_example(oracle):
    # proj/tests/test_toeplitz.cpp:39-49: seed (1,0,1,1), x = (1,1,0) -> (1,0)
    seed, x = bits_to_words([1, 0, 1, 1]), bits_to_words([1, 1, 0])
    out = oracle.toeplitz_hash(seed, 2, 3, x)
    assert int(out[0]) & 3 == 1
    assert (oracle.dense_toeplitz(seed, 2, 3, x) == out).all()


def test_toeplitz_golden(oracle, golden):
    for c in golden["toeplitz"]:
        seed, x = words(c["seed"]), words(c["x"])
        assert (oracle.toeplitz_hash(seed, c["m"], c["n"], x) == words(c["out"])).all()


def test_toeplitz_exhaustive_small(oracle):
    # proj/tests/test_toeplitz.cpp:51-73 (m, n <= 4, every seed and input) + blockings
    for m in range(1, 5):
        for n in range(1, 5):
            for sv in range(1 << (m + n - 1)):
                seed = np.array([sv], dtype=U64)
                for xv in range(1 << n):
                    x = np.array([xv], dtype=U64)
                    want = oracle.dense_toeplitz(seed, m, n, x)
                    assert (oracle.toeplitz_hash(seed, m, n, x) == want).all()
                    for mp, np_ in ((1, 1), (2, 3), (3, 2), (64, 64)):
                        assert (oracle.blocked_toeplitz_hash(seed, m, n, x, mp, np_) == want).all()


def test_toeplitz_vs_reference_random(oracle, reference):
    rng = np.random.default_rng(17)
    for _ in range(200):
        m, n = int(rng.integers(1, 300)), int(rng.integers(1, 600))
        seed = oracle.bits(int(rng.integers(1 << 62)), "s", 0, m + n - 1)
        x = oracle.bits(int(rng.integers(1 << 62)), "x", 0, n)
        want = reference.toeplitz_hash(seed, m, n, x)
        assert (oracle.toeplitz_hash(seed, m, n, x) == want).all()
        mp, np_ = int(rng.integers(1, m + 4)), int(rng.integers(1, n + 4))
        assert (reference.blocked_toeplitz_hash(seed, m, n, x, mp, np_) == want).all()
        assert (oracle.blocked_toeplitz_hash(seed, m, n, x, mp, np_) == want).all()


def test_toeplitz_rows_definition(oracle):
    rng = np.random.default_rng(5)
    for _ in range(30):
        m, n = int(rng.integers(1, 400)), int(rng.integers(1, 900))
        seed = oracle.bits(int(rng.integers(1 << 62)), "s", 0, m + n - 1)
        x = oracle.bits(int(rng.integers(1 << 62)), "x", 0, n)
        out = oracle.toeplitz_hash(seed, m, n, x)
        padded = np.zeros(len(seed) + (n + 63) // 64 + 4, dtype=U64)
        padded[: len(seed)] = seed
        rows = np.arange(m, dtype=U64)
        got = oracle.toeplitz_rows(padded, n, oracle.reverse_bits(x, n), rows)
        want = np.array([(int(out[i // 64]) >> (i % 64)) & 1 for i in range(m)], dtype=np.uint8)
        assert (got == want).all()


def test_partition_golden(oracle, golden):
    for c in golden["assign_subblocks"]:
        a, cnt = oracle.assign_subblocks(c["n"], c["s"], c["seed"])
        assert [int(v) for v in a[:32]] == c["assign_head"]
        assert f"{oracle.fnv(a.astype(U64)):016x}" == c["assign_fnv"]
        assert f"{oracle.fnv(cnt):016x}" == c["raw_counts_fnv"]


def test_sift_vs_reference(oracle, reference):
    rng = np.random.default_rng(5)
    n = 10000
    a, _ = oracle.assign_subblocks(n, 4, [0, 0, 0, 0])
    keep = (rng.integers(0, 2, n)).astype(np.uint8)
    off, idx = oracle.sift_partition(keep, a, 4)
    roff, ridx, ml = reference.sift_partition(keep, a, 4)
    assert (off == roff).all() and (idx == ridx).all()
    assert ml == int(np.diff(off).max())


def test_block_limit_vs_reference(oracle, reference):
    for args in [(1000, 0.5, 0.5, 1), (999, 0.5, 0.5, 1), (1000, 0.5, 1e-6, 1),
                 (30000, 0.98 * 0.98 / 17, 1e-8, 17), (1 << 20, 1 / 64, 1e-8, 64),
                 (20, 0.99, 1e-15, 1), (1000, 0.5, 1e-290, 1 << 40)]:
        got, err = oracle.block_limit(*args)
        want, rerr = reference.block_limit(*args)
        assert got == want and bool(err) == bool(rerr)
    assert reference.block_limit(1000, 0.5, 0.5, 1)[0] == 500  # test_sampling.cpp:133-137


def test_extract_golden_small(oracle, golden):
    for name, c in golden["extract"].items():
        if c["n"] > (1 << 24):
            continue
        x = oracle.make_input(c["seed_in"], c["p"], c["n"])
        assert f"{oracle.fnv(x):016x}" == c["input_fnv"]
        key, nj = oracle.extract(x, c["n"], c["s"], c["seed_samp"], c["seed_hash"],
                                 c["per_block"], c["k"])
        assert f"{oracle.fnv(key):016x}" == c["key_fnv"], name
        assert int(nj.min()) == c["nj_min"] and int(nj.max()) == c["nj_max"]
        assert f"{oracle.fnv(nj):016x}" == c["nj_fnv"]


def test_extract_selected_matches_full(oracle):
    n, s, k = 200000, 16, 640
    x = oracle.make_input(4, 0.5, n)
    for pb in (0, 1):
        key, nj = oracle.extract(x, n, s, 5, 6, pb, k)
        which = [0, 7, 15]
        keys, nj2 = oracle.extract_selected(x, n, s, 5, 6, pb, k, which)
        assert (nj == nj2).all()
        kw = k // 64
        for q, j in enumerate(which):
            assert (keys[q] == key[j * kw:(j + 1) * kw]).all()


def test_extract_sifted_vs_reference_loop(oracle, reference):
    # run_extraction's sift + per-block hash (pipeline.cpp:109-136) composed from the
    # reference's own assign_subblocks / sift_partition / bits / toeplitz_hash
    rng = np.random.default_rng(8)
    for n, s, k, pb in ((30000, 4, 256, 1), (20000, 7, 100, 0)):
        x = oracle.make_input(3, 0.5, n)
        keep = rng.integers(0, 2, n).astype(np.uint8)
        key, nj = oracle.extract_sifted(x, keep, n, s, 5, 6, pb, k)
        a, _ = reference.assign_subblocks(n, s, 5)
        off, idx, _ = reference.sift_partition(keep, a, s)
        xbits = np.unpackbits(x.view(np.uint8), bitorder="little")
        outbits = []
        for j in range(s):
            blk = idx[int(off[j]):int(off[j + 1])]
            nb = len(blk)
            assert nj[j] == nb
            xb = np.packbits(np.concatenate([xbits[blk], np.zeros((-nb) % 64, np.uint8)]),
                             bitorder="little").view(np.uint64)
            seed = reference.bits(6, "hash-seed", j if pb else 0, k + nb - 1)
            h = reference.toeplitz_hash(seed, k, nb, xb)
            outbits.append(np.unpackbits(h.view(np.uint8), bitorder="little")[:k])
        allb = np.concatenate(outbits)
        got = np.unpackbits(key.view(np.uint8), bitorder="little")[: s * k]
        assert (got == allb).all()


def test_cycle_estimate(oracle, reference):
    assert oracle.cycle_estimate(123, 0, 2000) == (123, 0)
    assert oracle.cycle_estimate(2000, 2000, 2000) == (8000, 0)
    # proj/tests/reference_values.hpp:84
    assert oracle.cycle_estimate(96040000, 6054000, 2000)[0] == 290821228000
    assert reference.cycle_estimate(96040000, 6054000, 2000)[0] == 290821228000


# ------------------------------------------------- protocol rounds / run_extraction (pipeline)
def _rounds_fnv(oracle, rounds):
    pad = np.zeros((len(rounds) + 7) // 8 * 8, dtype=np.uint8)
    pad[: len(rounds)] = rounds
    return f"{oracle.fnv(pad.view(np.uint64)):016x}"


def test_simulate_rounds_golden(oracle, golden):
    """oracle.c simulate_rounds vs rounds frozen from the reference (gen_golden --pipeline)."""
    for name, c in golden["pipeline"].items():
        sp = c["sim"]
        r = oracle.simulate_rounds(sp["n_rounds"], sp["p_x"], sp["e_ph"], sp["e_bit"],
                                   sp["p_det"], words(c["seed"]))
        assert _rounds_fnv(oracle, r) == c["rounds_fnv"], name


def test_simulate_rounds_vs_reference(oracle, reference):
    from oracle.pyoracle import bbm92

    rng = np.random.default_rng(5)
    for _ in range(6):
        n = int(rng.integers(1, 70000))
        p = bbm92(n, p_x=float(rng.uniform(0.01, 0.9)), e_ph=float(rng.uniform(0, 0.3)),
                  e_bit=float(rng.uniform(0, 0.5)), q_tol=0.45,
                  p_det=float(rng.uniform(0, 1)))
        seed = [int(v) for v in rng.integers(0, 1 << 62, 4)]
        want = reference.simulate_rounds(p, seed)
        got = oracle.simulate_rounds(n, p.p_x, p.e_ph, p.e_bit, p.p_det, seed)
        assert (want == got).all()


def test_run_extraction_golden(oracle, golden):
    """run_extraction's hash stage restated (pyoracle Oracle.run_extraction) vs the
    reference's ExtractionReport frozen by gen_golden --pipeline."""
    for name, c in golden["pipeline"].items():
        sp, hp = c["sim"], c["params"]
        r = oracle.simulate_rounds(sp["n_rounds"], sp["p_x"], sp["e_ph"], sp["e_bit"],
                                   sp["p_det"], words(c["seed"]))
        abort, key, lens, bpb = oracle.run_extraction(
            r, c["ns"], c["block_limit"], words(c["seed"]), c["key_length"], hp["eps_sec"],
            hp["p_x"], hp["q_tol"], hp["eta_tol"], hp["eps_abort"])
        assert abort == c["abort"], name
        assert bpb == c["bits_per_block"], name
        if abort != 2:
            assert [int(v) for v in lens] == c["block_lengths"], name
        assert f"{oracle.fnv(key):016x}" == c["key_fnv"], name


def test_partition_reversed_and_spot_check(oracle):
    """The configs-4/5 checker (or_partition_reversed + or_spot_check) against the oracle's
    full extraction at small sizes; a single flipped key bit is found in its block."""
    for (n, s, k, pb) in [(100000, 16, 1000, 1), (200000, 7, 640, 0), (1 << 20, 64, 8192, 0),
                          (300000, 32, 96, 1), (70001, 1, 64, 0)]:
        x = oracle.make_input(5, 0.5, n)
        key, nj_want = oracle.extract(x, n, s, 2, 3, pb, k)
        nj, yoff, y = oracle.partition_reversed(x, n, s, 2)
        assert (nj == nj_want).all()
        for j in (0, s - 1):
            blk = y[int(yoff[j]):int(yoff[j + 1])]
            assert (blk == oracle.reverse_bits(_gather(oracle, x, n, s, j), int(nj[j]))).all()
        assert oracle.spot_check(y, yoff, nj, 3, pb, k, key, rows=64) == (0, None)
        j = s // 2
        bad_key = key.copy()
        bad_key[(j * k) // 64] ^= np.uint64(1) << np.uint64((j * k) % 64)  # block j, row 0
        assert oracle.spot_check(y, yoff, nj, 3, pb, k, bad_key, rows=2) == (1, j)


def _gather(oracle, x, n, s, j):
    a, _ = oracle.assign_subblocks(n, s, 2)
    idx = np.nonzero(a == j + 1)[0]
    bits = (x[idx // 64] >> (idx % 64).astype(np.uint64)) & np.uint64(1)
    out = np.zeros((len(idx) + 63) // 64, dtype=np.uint64)
    for q in range(len(idx)):
        out[q // 64] |= bits[q] << np.uint64(q % 64)
    return out
