#!/usr/bin/env python3
"""Generate tests/golden/golden.json by running the REFERENCE implementation itself.

The reference C++ sources (/root/reference/proj/src) are compiled unmodified by
oracle/Makefile into oracle/_ref/libssbh_ref.so; this script calls them through the
extern "C" shim (oracle/ref_shim.cpp) and freezes their outputs as small fixtures.
Runs only in the build container (the reference tree does not exist on the GPU box).

    python tests/golden/gen_golden.py            # configs 1-2 + unit vectors (~1 min)
    python tests/golden/gen_golden.py --config3  # + full config-3 key digest (~30 min, 8 cores)
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.pyoracle import Oracle, Reference, bbm92, key_of, nwords  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")


def hexw(a):
    return [f"{int(v):016x}" for v in np.asarray(a, dtype=np.uint64)]


def fnv(o, a):
    return f"{o.fnv(np.asarray(a, dtype=np.uint64)):016x}"


def sim_params(n, **kw):
    """test_pipeline.cpp:14-25 desk-scale simulation point."""
    d = dict(p_x=0.05, e_ph=0.0082, e_bit=0.02, q_tol=0.02, eps_sec=1e-5, eps_abort=1e-8)
    d.update(kw)
    return bbm92(n, **d)


def pipeline_cases(ref, o):
    """run_extraction cases of test_pipeline.cpp (deterministic, sized by the reference's own
    key-length solver, oversize and statistics aborts) plus two infeasible/large-ns points."""
    aa, bb = [0xAAAAAAAAAAAAAAAA] * 4, [0xBBBBBBBBBBBBBBBB] * 4
    cases = [  # name, sim params, extraction params, ns, seed, block_limit override
        ("deterministic_ns4", sim_params(1000000), None, 4, aa, 0),
        ("single_block", sim_params(300000), None, 1, bb, 0),
        ("oversize", sim_params(50000), None, 4, 0, 10),
        ("statistics", sim_params(200000, e_ph=0.4, q_tol=0.4), sim_params(200000), 4, 0, 0),
        ("infeasible_ns16", sim_params(1000000), None, 16, aa, 0),
        ("ns64", sim_params(8000000, p_x=0.03), None, 64, 5, 0),
        ("p_det_eta", sim_params(1000000, p_det=0.7, eta_tol=0.6), None, 2, 6, 0),
        ("ns3_nonpow2", sim_params(1500000), None, 3, 9, 0),
    ]
    out = {}
    for name, sim, hon, ns, seed, lim_over in cases:
        hon = hon or sim
        t = time.time()
        rounds = ref.simulate_rounds(sim, seed)
        lim = lim_over or ref.plan_block_limit(hon, ns)
        kl, feas = ref.key_length(hon, ns)
        rep = ref.run_extraction(rounds, hon, ns, lim, seed)
        pad = np.zeros(nwords(len(rounds) * 8) * 8, dtype=np.uint8)
        pad[: len(rounds)] = rounds
        out[name] = {
            "sim": {f: getattr(sim, f) for f, _ in sim._fields_},
            "params": {f: getattr(hon, f) for f, _ in hon._fields_},
            "ns": ns, "seed": hexw(key_of(seed)), "block_limit": lim,
            "key_length": kl if feas else 0, "feasible": feas,
            "rounds_fnv": fnv(o, pad.view(np.uint64)),
            "abort": rep["abort"], "bits_per_block": rep["bits_per_block"],
            "key_bits": rep["key_bits"], "key_fnv": fnv(o, rep["key"]),
            "cycle_count": rep["cycle_count"], "total_epsilon": rep["total_epsilon"],
            "block_lengths": [int(v) for v in rep["block_lengths"]],
            "ref_seconds": round(time.time() - t, 2)}
        print(name, {k: v for k, v in out[name].items() if k != "block_lengths"}, flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config3", action="store_true")
    ap.add_argument("--config4", action="store_true")
    ap.add_argument("--config5", action="store_true")
    ap.add_argument("--pipeline", action="store_true",
                    help="run_extraction / simulate_rounds cases (pipeline.cpp)")
    ap.add_argument("--split", action="store_true",
                    help="shapes that take the 3-for-4 split path (k >= 2^18, T >= 1 squares)")
    ap.add_argument("--only-large", action="store_true", help="skip the small vectors")
    args = ap.parse_args()
    ref, o = Reference(), Oracle()
    g = json.load(open(OUT)) if os.path.exists(OUT) else {}
    g["_meta"] = {
        "generator": "tests/golden/gen_golden.py",
        "source": "reference compiled from /root/reference/proj/src by oracle/Makefile",
        "digest": "FNV-1a-64 over little-endian bytes of the uint64 words",
    }

    # ---- PRF ------------------------------------------------------------------------
    rng = np.random.default_rng(1234)
    prf = []
    for _ in range(16):
        key = rng.integers(0, 2**63, 4, dtype=np.uint64) * 2 + rng.integers(0, 2, 4, dtype=np.uint64)
        ctr = rng.integers(0, 2**63, 4, dtype=np.uint64) * 2 + rng.integers(0, 2, 4, dtype=np.uint64)
        prf.append({"key": hexw(key), "ctr": hexw(ctr), "out": hexw(ref.prf_block(key, ctr))})
    prf.append({"key": hexw([0] * 4), "ctr": hexw([0] * 4), "out": hexw(ref.prf_block([0] * 4, [0] * 4))})
    g["prf_block"] = prf
    g["tags"] = {t: f"{ref.L.ref_tag(t.encode()):016x}" for t in
                 ("sampling", "hash-seed", "input", "kat", "bench-input")}
    g["kat_words"] = [f"{ref.word([0] * 4, 'kat', 0, i):016x}" for i in range(4)]
    k7 = [0x7777777777777777] * 4
    g["stream_bits"] = [
        {"key": hexw(k7), "purpose": "bits", "sub": 3, "nbits": nb,
         "words": hexw(ref.bits(k7, "bits", 3, nb))} for nb in (1, 63, 64, 131, 1000, 4099)]
    g["uniform_below"] = [
        {"key": hexw(key_of(5)), "purpose": "sampling", "sub": 0, "bound": b, "first": 0,
         "values": [ref.uniform_below(5, "sampling", 0, b, i) for i in range(96)]}
        for b in (1, 7, 17, 64, 1000, 32768)]
    g["bernoulli"] = [
        {"key": hexw([0] * 4), "purpose": "bern", "sub": 0, "p": p,
         "bits": "".join(str(ref.bernoulli([0] * 4, "bern", 0, p, i)) for i in range(256))}
        for p in (0.0, 0.02, 0.3, 0.5, 0.4, 1.0)]

    # ---- Toeplitz -------------------------------------------------------------------
    cases = []
    for (m, n) in [(2, 3), (1, 1), (5, 9), (64, 33), (33, 64), (100, 200), (6300, 10000),
                   (8192, 16384), (1000, 1), (1, 1000), (777, 1501)]:
        seed = o.bits(99, "golden-seed", m * 100003 + n, m + n - 1)
        x = o.bits(98, "golden-x", m * 100003 + n, n)
        cases.append({"m": m, "n": n, "seed": hexw(seed), "x": hexw(x),
                      "out": hexw(ref.toeplitz_hash(seed, m, n, x))})
    g["toeplitz"] = cases

    # ---- partition ------------------------------------------------------------------
    parts = []
    for (n, s, sd) in [(5000, 7, 5), (1000, 1, 0), (65536, 64, 2), (100000, 1000, 2),
                       (1 << 17, 32768, 2), (10000, 4, 0)]:
        a, c = ref.assign_subblocks(n, s, sd)
        parts.append({"n": n, "s": s, "seed": sd, "assign_fnv": fnv(o, a.astype(np.uint64)),
                      "assign_head": [int(v) for v in a[:32]], "raw_counts_fnv": fnv(o, c)})
    g["assign_subblocks"] = parts

    # ---- whole path: BASELINE configs 1-2 (full keys) -------------------------------
    cfgs = {1: (1 << 20, 64, 8192, 0.5, 1, 2, 3, 0), 2: (1 << 24, 256, 32768, 0.3, 11, 2, 3, 0)}
    # small extra shapes: per-block seeds, k % 64 != 0, k % 32 != 0
    cfgs["small_perblock"] = (100000, 16, 1000, 0.5, 7, 8, 9, 1)
    cfgs["small_k_odd"] = (50000, 8, 77, 0.5, 7, 8, 9, 0)
    cfgs["small_k_32"] = (70000, 32, 96, 0.3, 7, 8, 9, 0)
    # 3-for-4 split shapes (csrc/toeplitz_split.cu runs them; the reference hashes them directly)
    split = {"split_smoke": (1 << 20, 2, 1 << 18, 0.5, 31, 32, 33, 0),
             "split_t2": ((1 << 24) + 777, 16, 1 << 19, 0.5, 22, 7, 8, 0),
             "split_deep": ((1 << 24) + 4097, 16, 1 << 19, 0.5, 25, 13, 14, 0),
             "split_perblock": ((1 << 24) + 777, 16, 3 << 17, 0.5, 24, 11, 12, 1)}
    todo = {} if args.only_large else dict(cfgs)
    if args.split:
        todo = dict(split) if args.only_large else {**todo, **split}
    ext = g.get("extract", {})
    for name, (n, s, k, p, si, ss, sh, pb) in todo.items():
        x = o.make_input(si, p, n)
        t = time.time()
        key, nj = ref.extract(x, n, s, ss, sh, pb, k)
        ext[str(name)] = {
            "n": n, "s": s, "k": k, "p": p, "seed_in": si, "seed_samp": ss, "seed_hash": sh,
            "per_block": pb, "input_popcount": int(np.unpackbits(x.view(np.uint8)).sum()),
            "input_fnv": fnv(o, x), "nj_min": int(nj.min()), "nj_max": int(nj.max()),
            "nj_0": int(nj[0]), "nj_fnv": fnv(o, nj), "key_fnv": fnv(o, key),
            "key_word0": f"{int(key[0]):016x}",
            "key_popcount": int(np.unpackbits(key.view(np.uint8)).sum()),
            "ref_seconds": round(time.time() - t, 3)}
        print(name, ext[str(name)], flush=True)
    if args.config3:
        n, s, k = 1 << 30, 1024, 1 << 19
        x = o.make_input(1, 0.5, n)
        t = time.time()
        key, nj = ref.extract(x, n, s, 2, 3, 0, k)
        kw = k // 64
        ext["3"] = {
            "n": n, "s": s, "k": k, "p": 0.5, "seed_in": 1, "seed_samp": 2, "seed_hash": 3,
            "per_block": 0, "input_fnv": fnv(o, x), "nj_min": int(nj.min()),
            "nj_max": int(nj.max()), "nj_0": int(nj[0]), "nj_fnv": fnv(o, nj),
            "key_fnv": fnv(o, key), "key_word0": f"{int(key[0]):016x}",
            "key_popcount": int(np.unpackbits(key.view(np.uint8)).sum()),
            "block0_fnv": fnv(o, key[:kw]), "block1023_fnv": fnv(o, key[1023 * kw:]),
            "ref_seconds": round(time.time() - t, 1)}
        print(3, ext["3"], flush=True)
    if args.config4:
        # configs 4: the reference API cannot hold its Partition (192 GiB): stream with the
        # reference's own KeyedStream / toeplitz_hash (ref_extract_selected)
        n, s, k = 1 << 34, 16384, 3 << 18
        which = [0, 1, 8191, 16383]
        x = o.make_input(1, 0.4, n)
        t = time.time()
        keys, nj = ref.extract_selected(x, n, s, 2, 3, 1, k, which)
        ext["4"] = {
            "n": n, "s": s, "k": k, "p": 0.4, "seed_in": 1, "seed_samp": 2, "seed_hash": 3,
            "per_block": 1, "input_fnv": fnv(o, x), "nj_min": int(nj.min()),
            "nj_max": int(nj.max()), "nj_0": int(nj[0]), "nj_last": int(nj[-1]),
            "nj_fnv": fnv(o, nj), "which": which,
            "block_fnv": [fnv(o, keys[q]) for q in range(len(which))],
            "block_word0": [f"{int(keys[q][0]):016x}" for q in range(len(which))],
            "block_popcount": [int(np.unpackbits(keys[q].view(np.uint8)).sum())
                               for q in range(len(which))],
            "ref_seconds": round(time.time() - t, 1)}
        print(4, ext["4"], flush=True)
    if args.config5:
        # config 5: 2^37 rounds (16 GiB input), s = 32768, shared seed, k = 2^21 —
        # streaming with the reference's own KeyedStream / toeplitz_hash
        n, s, k = 1 << 37, 32768, 1 << 21
        which = [0, 32767]
        x = o.make_input(1, 0.5, n)
        t = time.time()
        keys, nj = ref.extract_selected(x, n, s, 2, 3, 0, k, which)
        ext["5"] = {
            "n": n, "s": s, "k": k, "p": 0.5, "seed_in": 1, "seed_samp": 2, "seed_hash": 3,
            "per_block": 0, "input_fnv": fnv(o, x), "nj_min": int(nj.min()),
            "nj_max": int(nj.max()), "nj_0": int(nj[0]), "nj_last": int(nj[-1]),
            "nj_fnv": fnv(o, nj), "which": which,
            "block_fnv": [fnv(o, keys[q]) for q in range(len(which))],
            "block_word0": [f"{int(keys[q][0]):016x}" for q in range(len(which))],
            "block_popcount": [int(np.unpackbits(keys[q].view(np.uint8)).sum())
                               for q in range(len(which))],
            "ref_seconds": round(time.time() - t, 1)}
        print(5, ext["5"], flush=True)
    g["extract"] = ext
    if args.pipeline:
        g["pipeline"] = pipeline_cases(ref, o)
    json.dump(g, open(OUT, "w"), indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
