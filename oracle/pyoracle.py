"""ctypes bindings for the CPU checker (TEST / BASELINE INFRASTRUCTURE ONLY).

* ``Oracle`` wraps ``oracle/liboracle.so`` — the C restatement in ``oracle.c``.
* ``Reference`` wraps ``oracle/_ref/libssbh_ref.so`` — the unmodified reference
  sources (``/root/reference/proj/src``) compiled by ``oracle/Makefile`` behind an
  ``extern "C"`` shim (``oracle/ref_shim.cpp``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg import this module. The product package never does.
Words are numpy ``uint64`` arrays, bit k = bit k%64 of word k/64 (LSB first).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
U64P = C.POINTER(C.c_uint64)
U32P = C.POINTER(C.c_uint32)
U8P = C.POINTER(C.c_uint8)


def _p64(a):
    return a.ctypes.data_as(U64P)


def _p32(a):
    return a.ctypes.data_as(U32P)


def _p8(a):
    return a.ctypes.data_as(U8P)


def key_of(seed) -> np.ndarray:
    """BASELINE integer seed N -> MasterSeed::from_hex('%064x' % N) = {0,0,0,N}."""
    if isinstance(seed, np.ndarray):
        return seed.astype(np.uint64)
    if isinstance(seed, (list, tuple)):
        return np.array(seed, dtype=np.uint64)
    return np.array([0, 0, 0, int(seed)], dtype=np.uint64)


def nwords(nbits: int) -> int:
    return (int(nbits) + 63) // 64


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class Oracle:
    def __init__(self, path: str | None = None):
        path = path or os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        self.L = L
        L.or_tag.restype = C.c_uint64
        L.or_tag.argtypes = [C.c_char_p]
        L.or_threefry.argtypes = [U64P, U64P, U64P]
        L.or_stream_word.restype = C.c_uint64
        L.or_stream_word.argtypes = [U64P, C.c_uint64, C.c_uint64, C.c_uint64]
        L.or_uniform_below.restype = C.c_uint64
        L.or_uniform_below.argtypes = [U64P, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64]
        L.or_bernoulli.restype = C.c_int
        L.or_bernoulli.argtypes = [U64P, C.c_uint64, C.c_uint64, C.c_double, C.c_uint64]
        L.or_stream_bits.argtypes = [U64P, C.c_uint64, C.c_uint64, C.c_uint64, U64P]
        L.or_make_input.argtypes = [U64P, C.c_double, C.c_uint64, U64P, C.c_int]
        L.or_assign_subblocks.restype = C.c_int
        L.or_assign_subblocks.argtypes = [C.c_uint64, C.c_uint32, U64P, U32P, U64P, C.c_int]
        L.or_sift_partition.argtypes = [U8P, C.c_uint64, U32P, C.c_uint32, U64P, U64P]
        L.or_xor_bit_range.argtypes = [U64P, C.c_uint64, C.c_uint64, U64P, C.c_uint64,
                                       C.c_uint64, C.c_uint64]
        for f in ("or_toeplitz_hash", "or_dense_toeplitz"):
            getattr(L, f).argtypes = [U64P, C.c_uint64, C.c_uint64, U64P, U64P]
        L.or_blocked_toeplitz_hash.argtypes = [U64P, C.c_uint64, C.c_uint64, U64P, C.c_uint64,
                                               C.c_uint64, U64P]
        L.or_reverse_bits.argtypes = [U64P, C.c_uint64, U64P]
        L.or_toeplitz_rows.argtypes = [U64P, C.c_uint64, U64P, U64P, C.c_uint64, U8P]
        L.or_relative_entropy.restype = C.c_double
        L.or_relative_entropy.argtypes = [C.c_double, C.c_double]
        L.or_binomial_tail_bound.restype = C.c_double
        L.or_binomial_tail_bound.argtypes = [C.c_uint64, C.c_uint64, C.c_double]
        L.or_block_limit.restype = C.c_uint64
        L.or_block_limit.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_uint64,
                                     C.POINTER(C.c_int)]
        L.or_cycle_estimate.restype = C.c_uint64
        L.or_cycle_estimate.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(C.c_int)]
        L.or_extract.restype = C.c_int
        L.or_extract.argtypes = [U64P, C.c_uint64, C.c_uint32, U64P, U64P, C.c_int, C.c_uint64,
                                 U64P, U64P, C.c_int]
        L.or_extract_selected.restype = C.c_int
        L.or_extract_selected.argtypes = [U64P, C.c_uint64, C.c_uint32, U64P, U64P, C.c_int,
                                          C.c_uint64, U32P, C.c_uint32, U64P, U64P, C.c_int]
        L.or_fnv_words.restype = C.c_uint64
        L.or_fnv_words.argtypes = [U64P, C.c_uint64]

    # -- PRF --------------------------------------------------------------------
    def tag(self, name: str) -> int:
        return int(self.L.or_tag(name.encode()))

    def threefry(self, key, ctr) -> np.ndarray:
        k, c = key_of(key), np.array(ctr, dtype=np.uint64)
        out = np.zeros(4, dtype=np.uint64)
        self.L.or_threefry(_p64(k), _p64(c), _p64(out))
        return out

    def word(self, key, purpose, sub, index) -> int:
        return int(self.L.or_stream_word(_p64(key_of(key)), self.tag(purpose), sub, index))

    def uniform_below(self, key, purpose, sub, bound, index) -> int:
        return int(self.L.or_uniform_below(_p64(key_of(key)), self.tag(purpose), sub, bound,
                                           index))

    def bernoulli(self, key, purpose, sub, p, index) -> int:
        return int(self.L.or_bernoulli(_p64(key_of(key)), self.tag(purpose), sub, p, index))

    def bits(self, key, purpose, sub, nbits) -> np.ndarray:
        out = np.zeros(max(nwords(nbits), 1), dtype=np.uint64)
        self.L.or_stream_bits(_p64(key_of(key)), self.tag(purpose), sub, nbits, _p64(out))
        return out[: nwords(nbits)]

    def make_input(self, key, p, nbits, nthreads=0) -> np.ndarray:
        out = np.zeros(max(nwords(nbits), 1), dtype=np.uint64)
        self.L.or_make_input(_p64(key_of(key)), float(p), nbits, _p64(out), nthreads)
        return out[: nwords(nbits)]

    # -- sampler ----------------------------------------------------------------
    def assign_subblocks(self, n, s, key, nthreads=0):
        a = np.zeros(max(n, 1), dtype=np.uint32)
        c = np.zeros(max(s, 1), dtype=np.uint64)
        rc = self.L.or_assign_subblocks(n, s, _p64(key_of(key)), _p32(a), _p64(c), nthreads)
        if rc:
            raise ValueError("assign_subblocks: n_subblocks must be positive")
        return a[:n], c[:s]

    def sift_partition(self, keep, assignment, s):
        keep = np.ascontiguousarray(keep, dtype=np.uint8)
        assignment = np.ascontiguousarray(assignment, dtype=np.uint32)
        n = len(keep)
        off = np.zeros(s + 1, dtype=np.uint64)
        idx = np.zeros(max(int(keep.sum()), 1), dtype=np.uint64)
        self.L.or_sift_partition(_p8(keep), n, _p32(assignment), s, _p64(off), _p64(idx))
        return off, idx[: int(off[-1])]

    # -- toeplitz ---------------------------------------------------------------
    def toeplitz_hash(self, seed, m, n, x) -> np.ndarray:
        seed = np.ascontiguousarray(seed, dtype=np.uint64)
        x = np.ascontiguousarray(x, dtype=np.uint64)
        out = np.zeros(max(nwords(m), 1), dtype=np.uint64)
        self.L.or_toeplitz_hash(_p64(seed), m, n, _p64(x), _p64(out))
        return out[: nwords(m)]

    def dense_toeplitz(self, seed, m, n, x) -> np.ndarray:
        seed = np.ascontiguousarray(seed, dtype=np.uint64)
        x = np.ascontiguousarray(x, dtype=np.uint64)
        out = np.zeros(max(nwords(m), 1), dtype=np.uint64)
        self.L.or_dense_toeplitz(_p64(seed), m, n, _p64(x), _p64(out))
        return out[: nwords(m)]

    def blocked_toeplitz_hash(self, seed, m, n, x, mp, np_) -> np.ndarray:
        seed = np.ascontiguousarray(seed, dtype=np.uint64)
        x = np.ascontiguousarray(x, dtype=np.uint64)
        out = np.zeros(max(nwords(m), 1), dtype=np.uint64)
        self.L.or_blocked_toeplitz_hash(_p64(seed), m, n, _p64(x), mp, np_, _p64(out))
        return out[: nwords(m)]

    def reverse_bits(self, x, n) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.uint64)
        y = np.zeros(max(nwords(n), 1), dtype=np.uint64)
        self.L.or_reverse_bits(_p64(x), n, _p64(y))
        return y

    def toeplitz_rows(self, seed, n, y_rev, rows) -> np.ndarray:
        """K[i] for each i in rows; seed must be padded to cover max(rows)+64*ceil(n/64)+64."""
        seed = np.ascontiguousarray(seed, dtype=np.uint64)
        y_rev = np.ascontiguousarray(y_rev, dtype=np.uint64)
        rows = np.ascontiguousarray(rows, dtype=np.uint64)
        out = np.zeros(max(len(rows), 1), dtype=np.uint8)
        self.L.or_toeplitz_rows(_p64(seed), n, _p64(y_rev), _p64(rows), len(rows), _p8(out))
        return out[: len(rows)]

    # -- abort threshold --------------------------------------------------------
    def block_limit(self, n, p, eps, m):
        err = C.c_int(0)
        v = self.L.or_block_limit(n, p, eps, m, C.byref(err))
        return int(v), err.value

    def binomial_tail_bound(self, n, L, p):
        return float(self.L.or_binomial_tail_bound(n, L, p))

    def relative_entropy(self, x, p):
        return float(self.L.or_relative_entropy(x, p))

    def cycle_estimate(self, i, o, mp):
        err = C.c_int(0)
        v = self.L.or_cycle_estimate(i, o, mp, C.byref(err))
        return int(v), err.value

    # -- whole path -------------------------------------------------------------
    def extract(self, x, n, s, samp, hsh, per_block, k, nthreads=0):
        x = np.ascontiguousarray(x, dtype=np.uint64)
        key = np.zeros(max(nwords(s * k), 1), dtype=np.uint64)
        nj = np.zeros(s, dtype=np.uint64)
        rc = self.L.or_extract(_p64(x), n, s, _p64(key_of(samp)), _p64(key_of(hsh)),
                               int(per_block), k, _p64(key), _p64(nj), nthreads)
        if rc:
            raise ValueError("toeplitz: m and n must be positive (empty sub-block)")
        return key[: nwords(s * k)], nj

    def extract_sifted(self, x, keep_u8, n, s, samp, hsh, per_block, k, nthreads=0):
        x = np.ascontiguousarray(x, dtype=np.uint64)
        kp = np.ascontiguousarray(keep_u8, dtype=np.uint8)
        key = np.zeros(max(nwords(s * k), 1), dtype=np.uint64)
        nj = np.zeros(s, dtype=np.uint64)
        self.L.or_extract_sifted.restype = C.c_int
        self.L.or_extract_sifted.argtypes = [U64P, U8P, C.c_uint64, C.c_uint32, U64P, U64P,
                                             C.c_int, C.c_uint64, U64P, U64P, C.c_int]
        rc = self.L.or_extract_sifted(_p64(x), _p8(kp), n, s, _p64(key_of(samp)),
                                      _p64(key_of(hsh)), int(per_block), k, _p64(key), _p64(nj),
                                      nthreads)
        if rc:
            raise ValueError("toeplitz: m and n must be positive (empty sub-block)")
        return key[: nwords(s * k)], nj

    def extract_selected(self, x, n, s, samp, hsh, per_block, k, which, nthreads=0):
        x = np.ascontiguousarray(x, dtype=np.uint64)
        which = np.ascontiguousarray(which, dtype=np.uint32)
        kw = nwords(k)
        keys = np.zeros(max(len(which) * kw, 1), dtype=np.uint64)
        nj = np.zeros(s, dtype=np.uint64)
        rc = self.L.or_extract_selected(_p64(x), n, s, _p64(key_of(samp)), _p64(key_of(hsh)),
                                        int(per_block), k, _p32(which), len(which),
                                        _p64(keys), _p64(nj), nthreads)
        if rc:
            raise ValueError("toeplitz: m and n must be positive (empty sub-block)")
        return keys[: len(which) * kw].reshape(len(which), kw), nj

    def partition_reversed(self, x, n, s, samp, nthreads=0):
        """Every block's input, reversed (bit c = x_j[n_j-1-c]), at u64 word yoff[j] of y —
        the whole partition in 1/8 B per round (configs 4-5; no 12 B/round Partition)."""
        x = np.ascontiguousarray(x, dtype=np.uint64)
        nj = np.zeros(s, dtype=np.uint64)
        yoff = np.zeros(s + 1, dtype=np.uint64)
        y = np.zeros(n // 64 + s + 1, dtype=np.uint64)
        f = self.L.or_partition_reversed
        f.restype = C.c_int
        f.argtypes = [U64P, C.c_uint64, C.c_uint32, U64P, C.c_int, U64P, U64P, U64P]
        rc = f(_p64(x), n, s, _p64(key_of(samp)), nthreads, _p64(nj), _p64(yoff), _p64(y))
        if rc:
            raise ValueError("partition_reversed: n_subblocks must be positive")
        return nj, yoff, y

    def spot_check(self, y, yoff, nj, hsh, per_block, k, key, rows=64, row_seed=2308,
                   nthreads=0):
        """(mismatching rows, first bad block or None): `rows` output bits of every block
        (rows 0, k-1 and seeded ones) recomputed from the definition against the key."""
        f = self.L.or_spot_check
        f.restype = C.c_uint64
        f.argtypes = [U64P, U64P, U64P, C.c_uint32, U64P, C.c_int, C.c_uint64, U64P,
                      C.c_uint32, C.c_uint64, C.c_int, U64P]
        key = np.ascontiguousarray(key, dtype=np.uint64)
        first = np.zeros(1, dtype=np.uint64)
        bad = f(_p64(y), _p64(yoff), _p64(nj), len(nj), _p64(key_of(hsh)), int(per_block), k,
                _p64(key), rows, row_seed, nthreads, _p64(first))
        return int(bad), (None if int(first[0]) == 2**64 - 1 else int(first[0]))

    def fnv(self, words) -> int:
        w = np.ascontiguousarray(words, dtype=np.uint64)
        return int(self.L.or_fnv_words(_p64(w), len(w)))


class Reference:
    """The reference's own implementation (compiled from /root/reference by oracle/Makefile)."""

    def __init__(self, path: str | None = None):
        path = path or os.path.join(HERE, "_ref", "libssbh_ref.so")
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        self.L = L
        L.ref_prf_block.argtypes = [U64P, U64P, U64P]
        L.ref_tag.restype = C.c_uint64
        L.ref_tag.argtypes = [C.c_char_p]
        L.ref_stream_word.restype = C.c_uint64
        L.ref_stream_word.argtypes = [U64P, C.c_char_p, C.c_uint64, C.c_uint64]
        L.ref_uniform_below.restype = C.c_int
        L.ref_uniform_below.argtypes = [U64P, C.c_char_p, C.c_uint64, C.c_uint64, C.c_uint64,
                                        U64P]
        L.ref_bernoulli.restype = C.c_int
        L.ref_bernoulli.argtypes = [U64P, C.c_char_p, C.c_uint64, C.c_double, C.c_uint64]
        L.ref_stream_bits.argtypes = [U64P, C.c_char_p, C.c_uint64, C.c_uint64, U64P]
        L.ref_assign_subblocks.restype = C.c_int
        L.ref_assign_subblocks.argtypes = [C.c_uint64, C.c_uint32, U64P, U32P, U64P]
        L.ref_sift_partition.restype = C.c_int
        L.ref_sift_partition.argtypes = [U8P, C.c_uint64, U32P, C.c_uint32, U64P, U64P, U64P]
        L.ref_toeplitz_hash.restype = C.c_int
        L.ref_toeplitz_hash.argtypes = [U64P, C.c_uint64, C.c_uint64, U64P, C.c_uint64, U64P]
        L.ref_blocked_toeplitz_hash.restype = C.c_int
        L.ref_blocked_toeplitz_hash.argtypes = [U64P, C.c_uint64, C.c_uint64, U64P, C.c_uint64,
                                                C.c_uint64, C.c_uint64, U64P]
        L.ref_block_limit.restype = C.c_uint64
        L.ref_block_limit.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_uint64,
                                      C.POINTER(C.c_int)]
        L.ref_binomial_tail_bound.restype = C.c_double
        L.ref_binomial_tail_bound.argtypes = [C.c_uint64, C.c_uint64, C.c_double]
        L.ref_cycle_estimate.restype = C.c_uint64
        L.ref_cycle_estimate.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(C.c_int)]
        L.ref_extract.restype = C.c_int
        L.ref_extract.argtypes = [U64P, C.c_uint64, C.c_uint32, U64P, U64P, C.c_int,
                                  C.c_uint64, U64P, U64P]
        L.ref_time_sample.restype = C.c_double
        L.ref_time_sample.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_double, U64P, U64P,
                                      U64P, C.c_uint32, U64P, U64P]

    def prf_block(self, key, ctr):
        out = np.zeros(4, dtype=np.uint64)
        self.L.ref_prf_block(_p64(key_of(key)), _p64(np.array(ctr, dtype=np.uint64)), _p64(out))
        return out

    def word(self, key, purpose, sub, i):
        return int(self.L.ref_stream_word(_p64(key_of(key)), purpose.encode(), sub, i))

    def uniform_below(self, key, purpose, sub, bound, i):
        out = np.zeros(1, dtype=np.uint64)
        rc = self.L.ref_uniform_below(_p64(key_of(key)), purpose.encode(), sub, bound, i,
                                      _p64(out))
        if rc:
            raise ValueError("uniform_below: bound must be positive")
        return int(out[0])

    def bernoulli(self, key, purpose, sub, p, i):
        return int(self.L.ref_bernoulli(_p64(key_of(key)), purpose.encode(), sub, p, i))

    def bits(self, key, purpose, sub, nbits):
        out = np.zeros(max(nwords(nbits), 1), dtype=np.uint64)
        self.L.ref_stream_bits(_p64(key_of(key)), purpose.encode(), sub, nbits, _p64(out))
        return out[: nwords(nbits)]

    def assign_subblocks(self, n, s, key):
        a = np.zeros(max(n, 1), dtype=np.uint32)
        c = np.zeros(max(s, 1), dtype=np.uint64)
        rc = self.L.ref_assign_subblocks(n, s, _p64(key_of(key)), _p32(a), _p64(c))
        if rc:
            raise ValueError("assign_subblocks: n_subblocks must be positive")
        return a[:n], c[:s]

    def sift_partition(self, keep, assignment, s):
        keep = np.ascontiguousarray(keep, dtype=np.uint8)
        assignment = np.ascontiguousarray(assignment, dtype=np.uint32)
        off = np.zeros(s + 1, dtype=np.uint64)
        idx = np.zeros(max(int(keep.sum()), 1), dtype=np.uint64)
        ml = np.zeros(1, dtype=np.uint64)
        rc = self.L.ref_sift_partition(_p8(keep), len(keep), _p32(assignment), s, _p64(off),
                                       _p64(idx), _p64(ml))
        if rc:
            raise ValueError("sift_partition: flag count does not match partition")
        return off, idx[: int(off[-1])], int(ml[0])

    def toeplitz_hash(self, seed, m, n, x, nin=None):
        seed = np.ascontiguousarray(seed, dtype=np.uint64)
        x = np.ascontiguousarray(x, dtype=np.uint64)
        out = np.zeros(max(nwords(m), 1), dtype=np.uint64)
        rc = self.L.ref_toeplitz_hash(_p64(seed), m, n, _p64(x), n if nin is None else nin,
                                      _p64(out))
        if rc:
            raise ValueError(f"toeplitz: invalid argument (code {rc})")
        return out[: nwords(m)]

    def blocked_toeplitz_hash(self, seed, m, n, x, mp, np_):
        seed = np.ascontiguousarray(seed, dtype=np.uint64)
        x = np.ascontiguousarray(x, dtype=np.uint64)
        out = np.zeros(max(nwords(m), 1), dtype=np.uint64)
        rc = self.L.ref_blocked_toeplitz_hash(_p64(seed), m, n, _p64(x), n, mp, np_, _p64(out))
        if rc:
            raise ValueError(f"toeplitz: invalid argument (code {rc})")
        return out[: nwords(m)]

    def block_limit(self, n, p, eps, m):
        err = C.c_int(0)
        v = self.L.ref_block_limit(n, p, eps, m, C.byref(err))
        return int(v), err.value

    def cycle_estimate(self, i, o, mp):
        err = C.c_int(0)
        v = self.L.ref_cycle_estimate(i, o, mp, C.byref(err))
        return int(v), err.value

    def extract(self, x, n, s, samp, hsh, per_block, k):
        x = np.ascontiguousarray(x, dtype=np.uint64)
        key = np.zeros(max(nwords(s * k), 1), dtype=np.uint64)
        nj = np.zeros(s, dtype=np.uint64)
        rc = self.L.ref_extract(_p64(x), n, s, _p64(key_of(samp)), _p64(key_of(hsh)),
                                int(per_block), k, _p64(key), _p64(nj))
        if rc:
            raise ValueError(f"extract failed (code {rc})")
        return key[: nwords(s * k)], nj

    def time_sample(self, n_sample, s_sample, k, p, in_seed, samp, hsh, nblocks):
        bits = np.zeros(1, dtype=np.uint64)
        dig = np.zeros(1, dtype=np.uint64)
        secs = self.L.ref_time_sample(n_sample, s_sample, k, p, _p64(key_of(in_seed)),
                                      _p64(key_of(samp)), _p64(key_of(hsh)), nblocks,
                                      _p64(bits), _p64(dig))
        return float(secs), int(bits[0]), int(dig[0])


def _ref_extract_selected(self, x, n, s, samp, hsh, per_block, k, which):
    """Reference-code streaming extraction of selected blocks (ref_shim.cpp)."""
    x = np.ascontiguousarray(x, dtype=np.uint64)
    which = np.ascontiguousarray(which, dtype=np.uint32)
    kw = nwords(k)
    keys = np.zeros(max(len(which) * kw, 1), dtype=np.uint64)
    nj = np.zeros(s, dtype=np.uint64)
    L = self.L
    L.ref_extract_selected.restype = C.c_int
    L.ref_extract_selected.argtypes = [U64P, C.c_uint64, C.c_uint32, U64P, U64P, C.c_int,
                                       C.c_uint64, U32P, C.c_uint32, U64P, U64P]
    rc = L.ref_extract_selected(_p64(x), n, s, _p64(key_of(samp)), _p64(key_of(hsh)),
                                int(per_block), k, _p32(which), len(which), _p64(keys), _p64(nj))
    if rc:
        raise ValueError(f"extract_selected failed (code {rc})")
    return keys[: len(which) * kw].reshape(len(which), kw), nj


Reference.extract_selected = _ref_extract_selected


# ------------------------------------------------------------------ protocol rounds
def _or_simulate_rounds(self, n, p_x, e_ph, e_bit, p_det, seed, nthreads=0):
    """oracle.c restatement of simulate_rounds (pipeline.cpp:20-55)."""
    L = self.L
    L.or_simulate_rounds.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_double, C.c_double,
                                     U64P, U8P, C.c_int]
    out = np.zeros(max(n, 1), dtype=np.uint8)
    L.or_simulate_rounds(n, p_x, e_ph, e_bit, p_det, _p64(key_of(seed)), _p8(out), nthreads)
    return out[:n]


def _or_rounds_split(self, rounds):
    """(bit_a words, is_key_round bytes, counts {test, c1, c2, key})."""
    L = self.L
    L.or_rounds_split.argtypes = [U8P, C.c_uint64, U64P, U8P, U64P]
    r = np.ascontiguousarray(rounds, dtype=np.uint8)
    n = len(r)
    bits = np.zeros(max(nwords(n), 1), dtype=np.uint64)
    keep = np.zeros(max(n, 1), dtype=np.uint8)
    counts = np.zeros(4, dtype=np.uint64)
    L.or_rounds_split(_p8(r), n, _p64(bits), _p8(keep), _p64(counts))
    return bits[: nwords(n)], keep[:n], [int(c) for c in counts]


def _or_run_extraction(self, rounds, ns, block_limit, seed, key_length, eps_sec, p_x, q_tol,
                       eta_tol=1.0, eps_abort=1e-8):
    """run_extraction's hash stage restated from the oracle's pieces (pipeline.cpp:84-136):
    returns (abort, key words, block lengths, bits_per_block). abort: 0/1 oversize/2 stats."""
    bits, keep, (_, c1, c2, _) = self.rounds_split(rounds)
    n = len(rounds)
    px2 = p_x * p_x
    if c1 / n > px2 * eta_tol * q_tol or c2 / n > px2 * (1.0 - eta_tol):
        return 2, np.zeros(0, np.uint64), None, 0
    bpb = key_length // ns
    a, _ = self.assign_subblocks(n, ns, seed)
    offsets, _ = self.sift_partition(keep, a, ns)
    lens = np.diff(offsets).astype(np.uint64)
    if (lens > block_limit).any():
        return 1, np.zeros(0, np.uint64), lens, bpb
    if bpb == 0:
        return 0, np.zeros(0, np.uint64), lens, 0
    key, nj = self.extract_sifted(bits, keep, n, ns, seed, seed, True, bpb)
    assert (nj == lens).all()
    return 0, key, lens, bpb


Oracle.simulate_rounds = _or_simulate_rounds
Oracle.rounds_split = _or_rounds_split
Oracle.run_extraction = _or_run_extraction


class RefBbm92(C.Structure):
    """ref_shim.cpp ref_bbm92: the Bbm92Params fields the tests vary (others default)."""
    _fields_ = [("n_rounds", C.c_uint64), ("p_x", C.c_double), ("e_ph", C.c_double),
                ("e_bit", C.c_double), ("q_tol", C.c_double), ("eta_tol", C.c_double),
                ("f_ec", C.c_double), ("p_det", C.c_double), ("eps_sec", C.c_double),
                ("eps_abort", C.c_double)]


def bbm92(n_rounds, p_x=0.02, e_ph=0.0082, e_bit=0.058, q_tol=0.0082, eta_tol=1.0, f_ec=1.16,
          p_det=1.0, eps_sec=1e-6, eps_abort=1e-8) -> RefBbm92:
    """Bbm92Params with the reference defaults (bbm92.hpp:14-26)."""
    return RefBbm92(n_rounds, p_x, e_ph, e_bit, q_tol, eta_tol, f_ec, p_det, eps_sec, eps_abort)


def _ref_simulate_rounds(self, params: RefBbm92, seed):
    L = self.L
    L.ref_simulate_rounds.restype = C.c_int
    L.ref_simulate_rounds.argtypes = [C.POINTER(RefBbm92), U64P, U8P]
    out = np.zeros(max(params.n_rounds, 1), dtype=np.uint8)
    rc = L.ref_simulate_rounds(C.byref(params), _p64(key_of(seed)), _p8(out))
    if rc:
        raise ValueError(f"simulate_rounds failed (code {rc})")
    return out[: params.n_rounds]


def _ref_key_length(self, params: RefBbm92, ns):
    L = self.L
    L.ref_key_length.restype = C.c_int
    L.ref_key_length.argtypes = [C.POINTER(RefBbm92), C.c_uint32, U64P, C.POINTER(C.c_int)]
    out = np.zeros(1, dtype=np.uint64)
    feas = C.c_int(0)
    rc = L.ref_key_length(C.byref(params), ns, _p64(out), C.byref(feas))
    if rc:
        raise ValueError(f"key_length failed (code {rc})")
    return int(out[0]), bool(feas.value)


def _ref_plan_block_limit(self, params: RefBbm92, ns):
    L = self.L
    L.ref_plan_block_limit.restype = C.c_int
    L.ref_plan_block_limit.argtypes = [C.POINTER(RefBbm92), C.c_uint32, U64P]
    out = np.zeros(1, dtype=np.uint64)
    rc = L.ref_plan_block_limit(C.byref(params), ns, _p64(out))
    if rc:
        raise ValueError(f"block_limit failed (code {rc})")
    return int(out[0])


def _ref_run_extraction(self, rounds, params: RefBbm92, ns, block_limit, seed, m_prime=2000):
    """The reference's run_extraction (pipeline.cpp:75-138). Returns a dict of the
    ExtractionReport fields (key as uint64 words)."""
    L = self.L
    L.ref_run_extraction.restype = C.c_int
    L.ref_run_extraction.argtypes = [U8P, C.POINTER(RefBbm92), C.c_uint32, C.c_uint64, U64P,
                                     C.c_uint64, U64P, C.c_uint64, U64P, U64P,
                                     C.POINTER(C.c_double)]
    r = np.ascontiguousarray(rounds, dtype=np.uint8)
    cap = nwords(len(r)) + 2
    key = np.zeros(cap, dtype=np.uint64)
    lens = np.zeros(max(ns, 1), dtype=np.uint64)
    meta = np.zeros(5, dtype=np.uint64)
    dmeta = (C.c_double * 2)()
    rc = L.ref_run_extraction(_p8(r), C.byref(params), ns, block_limit, _p64(key_of(seed)),
                              m_prime, _p64(key), cap, _p64(lens), _p64(meta), dmeta)
    if rc:
        raise ValueError(f"run_extraction failed (code {rc})")
    nlen = int(meta[4])
    return {"abort": int(meta[0]), "bits_per_block": int(meta[1]), "key_bits": int(meta[2]),
            "cycle_count": int(meta[3]), "block_lengths": lens[:nlen].copy(),
            "key": key[: nwords(int(meta[2]))].copy(), "total_epsilon": dmeta[0],
            "wall_seconds": dmeta[1]}


def _ref_timing_model(self, input_len, output_len, kind, ns=1, m_prime=2000, eps_abort=1e-8,
                      limit_override=0, pad=True):
    L = self.L
    L.ref_timing_model.restype = C.c_int
    L.ref_timing_model.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_uint32, C.c_uint64,
                                   C.c_double, C.c_uint64, C.c_int, U64P]
    out = np.zeros(1, dtype=np.uint64)
    rc = L.ref_timing_model(input_len, output_len, kind, ns, m_prime, eps_abort, limit_override,
                            int(pad), _p64(out))
    if rc:
        raise ValueError(f"timing_model failed (code {rc})")
    return int(out[0])


Reference.simulate_rounds = _ref_simulate_rounds
Reference.key_length = _ref_key_length
Reference.plan_block_limit = _ref_plan_block_limit
Reference.run_extraction = _ref_run_extraction
Reference.timing_model = _ref_timing_model
