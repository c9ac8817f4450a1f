"""paper_2308_02856_b200 — B200-native sampled sub-block Toeplitz extractor.

The product is two in-tree native libraries:

* ``libssbh_cuda.so`` — hand-written sm_100a kernels behind the C-ABI declared in
  ``include/ssbh_cuda.h`` (Threefry sampler, stable bit partition, GF(2) Toeplitz
  hash, concatenation).
* ``libssbh.so`` — the reference's C++ API (``include/ssbh/*.hpp``: ``BitString``,
  ``KeyedStream``, ``assign_subblocks``, ``sift_partition``, ``toeplitz_hash`` …) as a
  drop-in over that C-ABI.

This module is a thin ``ctypes`` view of the C-ABI for the Python test-suite and
``bench.py``. It never falls back to a CPU implementation: loading fails loudly when
the CUDA library is missing, and compute calls raise ``NoDeviceError`` without a GPU.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# SSBH_CUDA_LIB: dev A/B of an alternative build of the same library (tools/); default in-tree
LIB_PATH = os.environ.get("SSBH_CUDA_LIB") or os.path.join(HERE, "libssbh_cuda.so")
CXX_LIB_PATH = os.path.join(HERE, "libssbh.so")

U64P = C.POINTER(C.c_uint64)
U32P = C.POINTER(C.c_uint32)
U8P = C.POINTER(C.c_uint8)

# status codes (include/ssbh_cuda.h)
OK, INVALID_ARGUMENT, INFEASIBLE, OVERFLOW, IO, CUDA, NO_DEVICE, ABORT_OVERSIZE = range(8)

# every exported symbol of include/ssbh_cuda.h
ABI_SYMBOLS = (
    "ssbh_abi_version", "ssbh_last_error", "ssbh_device_count", "ssbh_set_device",
    "ssbh_prf_block", "ssbh_prf_tag", "ssbh_stream_bits", "ssbh_stream_words",
    "ssbh_stream_uniform_below", "ssbh_stream_bernoulli", "ssbh_assign_subblocks",
    "ssbh_sift_partition", "ssbh_block_limit", "ssbh_binomial_tail_bound",
    "ssbh_relative_entropy", "ssbh_abort_check", "ssbh_toeplitz_hash",
    "ssbh_blocked_toeplitz_hash", "ssbh_cycle_estimate", "ssbh_toeplitz_hash_batch",
    "ssbh_plan_create", "ssbh_plan_destroy", "ssbh_plan_device_bytes", "ssbh_plan_run_device",
    "ssbh_plan_check", "ssbh_plan_set_timing", "ssbh_extract", "ssbh_plan_run_host",
    "ssbh_make_input_device", "ssbh_measure_lop3_peak", "ssbh_plan_create_streaming",
    "ssbh_plan_stream_begin", "ssbh_plan_stream_chunk", "ssbh_plan_stream_finish",
    "ssbh_plan_run_device_sifted", "ssbh_plan_run_host_sifted", "ssbh_extract_sifted",
    "ssbh_shard_create", "ssbh_shard_destroy", "ssbh_shard_info", "ssbh_shard_ipc_handle",
    "ssbh_shard_open_peers", "ssbh_shard_sample", "ssbh_shard_exchange", "ssbh_shard_finish",
    "ssbh_shard_check", "ssbh_shard_set_timing", "ssbh_simulate_rounds_device",
    "ssbh_simulate_rounds", "ssbh_run_extraction", "ssbh_run_extraction_device",
    "ssbh_extract_multi", "ssbh_plan_set_engine", "ssbh_plan_engine", "ssbh_measure_mma_f4_peak",
    "ssbh_probe_mma_f4", "ssbh_plan_hash_kernel", "ssbh_shard_hash_kernel",
    "ssbh_plan_split_geometry", "ssbh_shard_split_geometry", "ssbh_fnv1a64",
    "ssbh_toeplitz_hash_batch_ptrs", "ssbh_release_thread_cache", "ssbh_set_plan_overrides",
    "ssbh_get_plan_overrides", "ssbh_hash_batch_create", "ssbh_hash_batch_run",
    "ssbh_hash_batch_destroy",
)

ENGINE_AUTO, ENGINE_LOP3, ENGINE_TENSOR = 0, 1, 2


class SsbhError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[{status}] {msg}")
        self.status = status
        self.msg = msg


class InvalidArgument(SsbhError, ValueError):
    pass


class Infeasible(SsbhError):
    pass


class OverflowErr(SsbhError, OverflowError):
    pass


class NoDeviceError(SsbhError):
    pass


class AbortOversize(SsbhError):
    pass


_EXC = {INVALID_ARGUMENT: InvalidArgument, INFEASIBLE: Infeasible, OVERFLOW: OverflowErr,
        NO_DEVICE: NoDeviceError, ABORT_OVERSIZE: AbortOversize}


class ExtractParams(C.Structure):
    _fields_ = [("n_rounds", C.c_uint64), ("n_subblocks", C.c_uint32),
                ("per_block_seed", C.c_uint32), ("out_bits", C.c_uint64),
                ("samp_key", C.c_uint64 * 4), ("hash_key", C.c_uint64 * 4),
                ("block_first", C.c_uint32), ("block_count", C.c_uint32),
                ("block_limit", C.c_uint64)]


class ExtractStats(C.Structure):
    _fields_ = [("ms_sample", C.c_double), ("ms_scatter", C.c_double), ("ms_seed", C.c_double),
                ("ms_hash", C.c_double), ("ms_total", C.c_double),
                ("hash_word_ops", C.c_uint64), ("max_len", C.c_uint64),
                ("min_len", C.c_uint64), ("hash_launches", C.c_uint32),
                ("launches", C.c_uint32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class PlanOverrides(C.Structure):
    """ssbh_plan_overrides (include/ssbh_cuda.h): explicit testing / A-B hooks for which code
    path a plan takes; never read from the environment."""
    _fields_ = [("engine", C.c_int32), ("split_levels", C.c_int32),
                ("split_tiled_leaves", C.c_int32), ("shared_tiled", C.c_int32),
                ("buckets", C.c_int32), ("split_budget_mb", C.c_uint32),
                ("scatter_window", C.c_int32)]


DEFAULT_OVERRIDES = dict(engine=0, split_levels=-1, split_tiled_leaves=0, shared_tiled=-1,
                         buckets=-1, split_budget_mb=0, scatter_window=0)


class RoundParams(C.Structure):
    _fields_ = [("n_rounds", C.c_uint64), ("p_x", C.c_double), ("e_ph", C.c_double),
                ("e_bit", C.c_double), ("p_det", C.c_double)]


class ExtractionParams(C.Structure):
    _fields_ = [("n_subblocks", C.c_uint32), ("pad", C.c_uint32), ("block_limit", C.c_uint64),
                ("seed", C.c_uint64 * 4), ("eps_abort", C.c_double), ("eps_sec", C.c_double),
                ("p_x", C.c_double), ("eta_tol", C.c_double), ("q_tol", C.c_double),
                ("key_length", C.c_uint64)]


class ExtractionResult(C.Structure):
    _fields_ = [("abort", C.c_int32), ("pad", C.c_uint32), ("bits_per_block", C.c_uint64),
                ("key_bits", C.c_uint64), ("total_epsilon", C.c_double),
                ("hash_seconds", C.c_double), ("test_rounds", C.c_uint64),
                ("phase_errors", C.c_uint64), ("no_detections", C.c_uint64),
                ("key_rounds", C.c_uint64), ("lengths_valid", C.c_int32), ("pad2", C.c_uint32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_ if not f.startswith("pad")}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() (make) first — "
                          "the B200 path has no CPU fallback")
    L = C.CDLL(LIB_PATH)
    st = C.c_int
    L.ssbh_abi_version.restype = C.c_int
    L.ssbh_last_error.restype = C.c_char_p
    L.ssbh_device_count.restype = C.c_int
    L.ssbh_set_device.restype = st
    L.ssbh_set_device.argtypes = [C.c_int]
    L.ssbh_fnv1a64.restype = C.c_uint64
    L.ssbh_fnv1a64.argtypes = [U64P, C.c_uint64]
    L.ssbh_prf_block.restype = st
    L.ssbh_prf_block.argtypes = [U64P, U64P, U64P]
    L.ssbh_plan_set_engine.restype = st
    L.ssbh_plan_set_engine.argtypes = [C.c_void_p, C.c_int]
    L.ssbh_plan_engine.restype = C.c_int
    L.ssbh_plan_engine.argtypes = [C.c_void_p]
    L.ssbh_measure_mma_f4_peak.restype = st
    L.ssbh_measure_mma_f4_peak.argtypes = [C.c_uint32, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.ssbh_plan_hash_kernel.restype = C.c_char_p
    L.ssbh_plan_hash_kernel.argtypes = [C.c_void_p]
    L.ssbh_plan_split_geometry.restype = st
    L.ssbh_plan_split_geometry.argtypes = [C.c_void_p] + [C.POINTER(C.c_uint32)] * 3
    L.ssbh_shard_split_geometry.restype = st
    L.ssbh_shard_split_geometry.argtypes = [C.c_void_p] + [C.POINTER(C.c_uint32)] * 3
    L.ssbh_shard_hash_kernel.restype = C.c_char_p
    L.ssbh_shard_hash_kernel.argtypes = [C.c_void_p]
    L.ssbh_prf_tag.restype = C.c_uint64
    L.ssbh_prf_tag.argtypes = [C.c_char_p, C.c_size_t]
    L.ssbh_stream_bits.restype = st
    L.ssbh_stream_bits.argtypes = [U64P, C.c_uint64, C.c_uint64, C.c_uint64, U64P]
    L.ssbh_stream_words.restype = st
    L.ssbh_stream_words.argtypes = [U64P, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, U64P]
    L.ssbh_stream_uniform_below.restype = st
    L.ssbh_stream_uniform_below.argtypes = [U64P, C.c_uint64, C.c_uint64, C.c_uint64,
                                            C.c_uint64, C.c_uint64, U64P]
    L.ssbh_stream_bernoulli.restype = st
    L.ssbh_stream_bernoulli.argtypes = [U64P, C.c_uint64, C.c_uint64, C.c_double, C.c_uint64,
                                        C.c_uint64, U64P]
    L.ssbh_assign_subblocks.restype = st
    L.ssbh_assign_subblocks.argtypes = [C.c_uint64, C.c_uint32, U64P, U32P, U64P]
    L.ssbh_sift_partition.restype = st
    L.ssbh_sift_partition.argtypes = [U8P, C.c_uint64, U32P, C.c_uint32, U64P, U64P, U64P]
    L.ssbh_block_limit.restype = st
    L.ssbh_block_limit.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_uint64, U64P]
    L.ssbh_binomial_tail_bound.restype = st
    L.ssbh_binomial_tail_bound.argtypes = [C.c_uint64, C.c_uint64, C.c_double,
                                           C.POINTER(C.c_double)]
    L.ssbh_relative_entropy.restype = st
    L.ssbh_relative_entropy.argtypes = [C.c_double, C.c_double, C.POINTER(C.c_double)]
    L.ssbh_abort_check.restype = C.c_int
    L.ssbh_abort_check.argtypes = [U64P, C.c_uint64, C.c_uint64]
    L.ssbh_toeplitz_hash.restype = st
    L.ssbh_toeplitz_hash.argtypes = [U64P, C.c_uint64, C.c_uint64, U64P, C.c_uint64, U64P]
    L.ssbh_blocked_toeplitz_hash.restype = st
    L.ssbh_blocked_toeplitz_hash.argtypes = [U64P, C.c_uint64, C.c_uint64, U64P, C.c_uint64,
                                             C.c_uint64, C.c_uint64, U64P]
    L.ssbh_cycle_estimate.restype = st
    L.ssbh_cycle_estimate.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, U64P]
    L.ssbh_toeplitz_hash_batch.restype = st
    L.ssbh_toeplitz_hash_batch.argtypes = [C.c_uint64, C.c_uint64, U64P, U64P, U64P, U64P,
                                           U64P, U64P]
    L.ssbh_plan_create.restype = st
    L.ssbh_plan_create.argtypes = [C.POINTER(ExtractParams), C.POINTER(C.c_void_p)]
    L.ssbh_plan_destroy.restype = st
    L.ssbh_plan_destroy.argtypes = [C.c_void_p]
    L.ssbh_plan_device_bytes.restype = C.c_uint64
    L.ssbh_plan_device_bytes.argtypes = [C.c_void_p]
    L.ssbh_plan_run_device.restype = st
    L.ssbh_plan_run_device.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, U64P,
                                       U64P, C.c_void_p]
    L.ssbh_plan_check.restype = st
    L.ssbh_plan_check.argtypes = [C.c_void_p, C.POINTER(ExtractStats)]
    L.ssbh_plan_set_timing.restype = st
    L.ssbh_plan_set_timing.argtypes = [C.c_void_p, C.c_int]
    L.ssbh_extract.restype = st
    L.ssbh_extract.argtypes = [C.POINTER(ExtractParams), U64P, U64P, U64P,
                               C.POINTER(ExtractStats)]
    L.ssbh_plan_run_host.restype = st
    L.ssbh_plan_run_host.argtypes = [C.c_void_p, U64P, U64P, U64P, C.POINTER(ExtractStats)]
    L.ssbh_make_input_device.restype = st
    L.ssbh_make_input_device.argtypes = [U64P, C.c_double, C.c_uint64, C.c_void_p, C.c_void_p]
    vp = C.c_void_p
    L.ssbh_shard_create.restype = st
    L.ssbh_shard_create.argtypes = [C.POINTER(ExtractParams), C.c_uint32, C.c_uint32,
                                    C.POINTER(vp)]
    L.ssbh_shard_destroy.restype = st
    L.ssbh_shard_destroy.argtypes = [vp]
    L.ssbh_shard_info.restype = st
    L.ssbh_shard_info.argtypes = [vp, U64P, U64P, U32P, U32P]
    L.ssbh_shard_ipc_handle.restype = st
    L.ssbh_shard_ipc_handle.argtypes = [vp, vp]
    L.ssbh_shard_open_peers.restype = st
    L.ssbh_shard_open_peers.argtypes = [vp, vp]
    L.ssbh_shard_sample.restype = st
    L.ssbh_shard_sample.argtypes = [vp, vp, U64P, U64P, vp]
    L.ssbh_shard_exchange.restype = st
    L.ssbh_shard_exchange.argtypes = [vp, U64P, vp]
    L.ssbh_shard_finish.restype = st
    L.ssbh_shard_finish.argtypes = [vp, vp, vp, U64P, vp]
    L.ssbh_shard_check.restype = st
    L.ssbh_shard_check.argtypes = [vp, C.POINTER(ExtractStats)]
    L.ssbh_shard_set_timing.restype = st
    L.ssbh_shard_set_timing.argtypes = [vp, C.c_int]
    L.ssbh_plan_run_device_sifted.restype = st
    L.ssbh_plan_run_device_sifted.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                              C.c_void_p, U64P, U64P, C.c_void_p]
    L.ssbh_plan_run_host_sifted.restype = st
    L.ssbh_plan_run_host_sifted.argtypes = [C.c_void_p, U64P, U64P, U64P, U64P,
                                            C.POINTER(ExtractStats)]
    L.ssbh_extract_sifted.restype = st
    L.ssbh_extract_sifted.argtypes = [C.POINTER(ExtractParams), U64P, U64P, U64P, U64P,
                                      C.POINTER(ExtractStats)]
    L.ssbh_plan_create_streaming.restype = st
    L.ssbh_plan_create_streaming.argtypes = [C.POINTER(ExtractParams), C.c_uint64,
                                             C.POINTER(C.c_void_p)]
    L.ssbh_plan_stream_begin.restype = st
    L.ssbh_plan_stream_begin.argtypes = [C.c_void_p, U64P, U64P, C.c_void_p]
    L.ssbh_plan_stream_chunk.restype = st
    L.ssbh_plan_stream_chunk.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]
    L.ssbh_plan_stream_finish.restype = st
    L.ssbh_plan_stream_finish.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    L.ssbh_measure_lop3_peak.restype = st
    L.ssbh_measure_lop3_peak.argtypes = [C.c_uint32, C.POINTER(C.c_double),
                                         C.POINTER(C.c_double)]
    L.ssbh_simulate_rounds_device.restype = st
    L.ssbh_simulate_rounds_device.argtypes = [C.POINTER(RoundParams), U64P, C.c_void_p,
                                              C.c_void_p]
    L.ssbh_simulate_rounds.restype = st
    L.ssbh_simulate_rounds.argtypes = [C.POINTER(RoundParams), U64P, U8P]
    L.ssbh_run_extraction.restype = st
    L.ssbh_run_extraction.argtypes = [U8P, C.c_uint64, C.POINTER(ExtractionParams), U64P, U64P,
                                      C.POINTER(ExtractionResult)]
    L.ssbh_run_extraction_device.restype = st
    L.ssbh_run_extraction_device.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(ExtractionParams),
                                             U64P, U64P, C.POINTER(ExtractionResult)]
    L.ssbh_extract_multi.restype = st
    L.ssbh_extract_multi.argtypes = [C.POINTER(ExtractParams), U64P, C.POINTER(C.c_int), C.c_uint32,
                                     U64P, U64P, C.POINTER(ExtractStats)]
    return L


lib = _load()


def _check(status: int):
    if status != OK:
        msg = lib.ssbh_last_error().decode(errors="replace")
        raise _EXC.get(status, SsbhError)(status, msg)


def _p64(a):
    return a.ctypes.data_as(U64P)


def _p32(a):
    return a.ctypes.data_as(U32P)


def _p8(a):
    return a.ctypes.data_as(U8P)


def key_of(seed) -> np.ndarray:
    """BASELINE integer seed N -> MasterSeed::from_hex('%064x' % N) = words {0,0,0,N}."""
    if isinstance(seed, (list, tuple, np.ndarray)):
        return np.ascontiguousarray(seed, dtype=np.uint64)
    return np.array([0, 0, 0, int(seed)], dtype=np.uint64)


def nwords(nbits: int) -> int:
    return (int(nbits) + 63) // 64


def device_count() -> int:
    return int(lib.ssbh_device_count())


def tag(purpose: str) -> int:
    b = purpose.encode()
    return int(lib.ssbh_prf_tag(b, len(b)))


def prf_block(key, ctr) -> np.ndarray:
    out = np.zeros(4, dtype=np.uint64)
    _check(lib.ssbh_prf_block(_p64(key_of(key)), _p64(np.asarray(ctr, dtype=np.uint64)),
                              _p64(out)))
    return out


def stream_bits(key, purpose: str, sub: int, nbits: int) -> np.ndarray:
    out = np.zeros(max(nwords(nbits), 1), dtype=np.uint64)
    _check(lib.ssbh_stream_bits(_p64(key_of(key)), tag(purpose), sub, nbits, _p64(out)))
    return out[: nwords(nbits)]


def stream_words(key, purpose, sub, first, count) -> np.ndarray:
    out = np.zeros(max(count, 1), dtype=np.uint64)
    _check(lib.ssbh_stream_words(_p64(key_of(key)), tag(purpose), sub, first, count, _p64(out)))
    return out[:count]


def stream_uniform_below(key, purpose, sub, bound, first, count) -> np.ndarray:
    out = np.zeros(max(count, 1), dtype=np.uint64)
    _check(lib.ssbh_stream_uniform_below(_p64(key_of(key)), tag(purpose), sub, bound, first,
                                         count, _p64(out)))
    return out[:count]


def stream_bernoulli(key, purpose, sub, p, first, count) -> np.ndarray:
    out = np.zeros(max(nwords(count), 1), dtype=np.uint64)
    _check(lib.ssbh_stream_bernoulli(_p64(key_of(key)), tag(purpose), sub, p, first, count,
                                     _p64(out)))
    return out[: nwords(count)]


def assign_subblocks(n: int, s: int, key):
    a = np.zeros(max(n, 1), dtype=np.uint32)
    c = np.zeros(max(s, 1), dtype=np.uint64)
    _check(lib.ssbh_assign_subblocks(n, s, _p64(key_of(key)), _p32(a), _p64(c)))
    return a[:n], c[:s]


def sift_partition(keep, assignment, s: int):
    assignment = np.ascontiguousarray(assignment, dtype=np.uint32)
    n = len(assignment)
    kp = None if keep is None else np.ascontiguousarray(keep, dtype=np.uint8)
    if kp is not None and len(kp) != n:
        raise InvalidArgument(INVALID_ARGUMENT,
                              "sift_partition: flag count does not match partition")
    off = np.zeros(s + 1, dtype=np.uint64)
    idx = np.zeros(max(n, 1), dtype=np.uint64)
    ml = np.zeros(1, dtype=np.uint64)
    _check(lib.ssbh_sift_partition(None if kp is None else _p8(kp), n, _p32(assignment), s,
                                   _p64(off), _p64(idx), _p64(ml)))
    return off, idx[: int(off[-1])], int(ml[0])


def toeplitz_hash(seed, m: int, n: int, x, input_bits: int | None = None) -> np.ndarray:
    seed = np.ascontiguousarray(seed, dtype=np.uint64)
    x = np.ascontiguousarray(x, dtype=np.uint64)
    out = np.zeros(max(nwords(m), 1), dtype=np.uint64)
    _check(lib.ssbh_toeplitz_hash(_p64(seed), m, n, _p64(x), n if input_bits is None else
                                  input_bits, _p64(out)))
    return out[: nwords(m)]


def blocked_toeplitz_hash(seed, m, n, x, mp, np_) -> np.ndarray:
    seed = np.ascontiguousarray(seed, dtype=np.uint64)
    x = np.ascontiguousarray(x, dtype=np.uint64)
    out = np.zeros(max(nwords(m), 1), dtype=np.uint64)
    _check(lib.ssbh_blocked_toeplitz_hash(_p64(seed), m, n, _p64(x), n, mp, np_, _p64(out)))
    return out[: nwords(m)]


def toeplitz_hash_batch(m: int, ns, inputs, in_off, seeds, seed_off) -> np.ndarray:
    """Hash len(ns) blocks (each its own n and seed, common m); returns the concatenation."""
    ns = np.ascontiguousarray(ns, dtype=np.uint64)
    inputs = np.ascontiguousarray(inputs, dtype=np.uint64)
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    in_off = np.ascontiguousarray(in_off, dtype=np.uint64)
    seed_off = np.ascontiguousarray(seed_off, dtype=np.uint64)
    cnt = len(ns)
    out = np.zeros(max(nwords(cnt * m), 1), dtype=np.uint64)
    _check(lib.ssbh_toeplitz_hash_batch(cnt, m, _p64(ns), _p64(inputs), _p64(in_off),
                                        _p64(seeds), _p64(seed_off), _p64(out)))
    return out[: nwords(cnt * m)]


def block_limit(n, p, eps, m) -> int:
    out = np.zeros(1, dtype=np.uint64)
    _check(lib.ssbh_block_limit(n, p, eps, m, _p64(out)))
    return int(out[0])


def binomial_tail_bound(n, L, p) -> float:
    out = C.c_double(0)
    _check(lib.ssbh_binomial_tail_bound(n, L, p, C.byref(out)))
    return out.value


def relative_entropy(x, p) -> float:
    out = C.c_double(0)
    _check(lib.ssbh_relative_entropy(x, p, C.byref(out)))
    return out.value


def abort_check(lengths, limit) -> bool:
    a = np.ascontiguousarray(lengths, dtype=np.uint64)
    return bool(lib.ssbh_abort_check(_p64(a) if len(a) else None, len(a), limit))


def cycle_estimate(i, o, mp) -> int:
    out = np.zeros(1, dtype=np.uint64)
    _check(lib.ssbh_cycle_estimate(i, o, mp, _p64(out)))
    return int(out[0])


def make_params(n, s, k, samp, hsh, per_block=False, block_first=0, block_count=0,
                limit=0) -> ExtractParams:
    p = ExtractParams()
    p.n_rounds = n
    p.n_subblocks = s
    p.per_block_seed = 1 if per_block else 0
    p.out_bits = k
    p.samp_key[:] = [int(v) for v in key_of(samp)]
    p.hash_key[:] = [int(v) for v in key_of(hsh)]
    p.block_first = block_first
    p.block_count = block_count
    p.block_limit = limit
    return p


def extract(x, n, s, k, samp, hsh, per_block=False, block_first=0, block_count=0, limit=0,
            keep=None):
    """Host-buffer fused extraction (ssbh_extract / ssbh_extract_sifted when `keep` — bit-packed
    uint64 words, bit i = keep round i — is given). Returns (key words, n_j, stats)."""
    params = make_params(n, s, k, samp, hsh, per_block, block_first, block_count, limit)
    owned = block_count or s
    x = np.ascontiguousarray(x, dtype=np.uint64)
    key = np.zeros(max(nwords(owned * k), 1), dtype=np.uint64)
    lens = np.zeros(owned, dtype=np.uint64)
    st = ExtractStats()
    if keep is None:
        _check(lib.ssbh_extract(C.byref(params), _p64(x), _p64(key), _p64(lens), C.byref(st)))
    else:
        kp = np.ascontiguousarray(keep, dtype=np.uint64)
        _check(lib.ssbh_extract_sifted(C.byref(params), _p64(x), _p64(kp), _p64(key),
                                       _p64(lens), C.byref(st)))
    return key[: nwords(owned * k)], lens, st


def extract_multi(x, n, s, k, samp, hsh, devices, per_block=False, limit=0):
    """One process over several GPUs (ssbh_extract_multi: sharded sampling, owner split through
    peer memory, one host thread per device). Returns (key words, n_j, stats)."""
    params = make_params(n, s, k, samp, hsh, per_block, 0, 0, limit)
    x = np.ascontiguousarray(x, dtype=np.uint64)
    key = np.zeros(max(nwords(s * k), 1), dtype=np.uint64)
    lens = np.zeros(s, dtype=np.uint64)
    st = ExtractStats()
    devs = (C.c_int * len(devices))(*devices)
    _check(lib.ssbh_extract_multi(C.byref(params), _p64(x), devs, len(devices), _p64(key),
                                  _p64(lens), C.byref(st)))
    return key[: nwords(s * k)], lens, st


# ------------------------------------------------------------ protocol rounds (pipeline.hpp)
def round_params(n, p_x, e_ph, e_bit, p_det=1.0) -> RoundParams:
    rp = RoundParams()
    rp.n_rounds, rp.p_x, rp.e_ph, rp.e_bit, rp.p_det = n, p_x, e_ph, e_bit, p_det
    return rp


def simulate_rounds(n, p_x, e_ph, e_bit, p_det, seed) -> np.ndarray:
    """simulate_rounds (pipeline.cpp:20-55) on the GPU: one RoundRecord byte per round."""
    out = np.zeros(max(int(n), 1), dtype=np.uint8)
    k = key_of(seed)
    _check(lib.ssbh_simulate_rounds(C.byref(round_params(n, p_x, e_ph, e_bit, p_det)), _p64(k),
                                    _p8(out)))
    return out[:n]


def simulate_rounds_device(n, p_x, e_ph, e_bit, p_det, seed, d_rounds_ptr, stream=0):
    k = key_of(seed)
    _check(lib.ssbh_simulate_rounds_device(C.byref(round_params(n, p_x, e_ph, e_bit, p_det)),
                                           _p64(k), C.c_void_p(d_rounds_ptr),
                                           C.c_void_p(stream)))


def extraction_params(ns, block_limit, seed, key_length, eps_sec, p_x, q_tol, eta_tol=1.0,
                      eps_abort=1e-8) -> ExtractionParams:
    ep = ExtractionParams()
    ep.n_subblocks, ep.block_limit, ep.key_length = ns, block_limit, key_length
    ep.seed[:] = [int(v) for v in key_of(seed)]
    ep.eps_abort, ep.eps_sec, ep.p_x, ep.eta_tol, ep.q_tol = eps_abort, eps_sec, p_x, eta_tol, q_tol
    return ep


def run_extraction(rounds, params: ExtractionParams, d_rounds_ptr: int | None = None,
                   n: int | None = None):
    """run_extraction's statistics check + sift + sample + per-block hash on the GPU
    (ssbh_run_extraction). Returns (key words, block lengths, result)."""
    ns = params.n_subblocks
    key_bits = ns * (params.key_length // ns) if ns else 0
    key = np.zeros(max(nwords(key_bits), 1), dtype=np.uint64)
    lens = np.zeros(max(ns, 1), dtype=np.uint64)
    res = ExtractionResult()
    if d_rounds_ptr is None:
        r = np.ascontiguousarray(rounds, dtype=np.uint8)
        _check(lib.ssbh_run_extraction(_p8(r) if len(r) else None, len(r), C.byref(params),
                                       _p64(key), _p64(lens), C.byref(res)))
    else:
        _check(lib.ssbh_run_extraction_device(C.c_void_p(d_rounds_ptr), n, C.byref(params),
                                              _p64(key), _p64(lens), C.byref(res)))
    return key[: nwords(res.key_bits)], lens[:ns], res


class Plan:
    """Device plan (ssbh_plan_*): buffers sized once, reused across runs.
    chunk_bits > 0 creates a streaming plan (stream_begin / stream_chunk / stream_finish)."""

    def __init__(self, n, s, k, samp, hsh, per_block=False, block_first=0, block_count=0,
                 limit=0, chunk_bits=0, engine=ENGINE_AUTO):
        self.params = make_params(n, s, k, samp, hsh, per_block, block_first, block_count,
                                  limit)
        self.owned = block_count or s
        self.n, self.s, self.k = n, s, k
        self.chunk_bits = chunk_bits
        h = C.c_void_p()
        if chunk_bits:
            _check(lib.ssbh_plan_create_streaming(C.byref(self.params), chunk_bits, C.byref(h)))
        else:
            _check(lib.ssbh_plan_create(C.byref(self.params), C.byref(h)))
        self.h = h
        if engine != ENGINE_AUTO:
            self.set_engine(engine)

    def set_engine(self, engine: int):
        """ENGINE_LOP3 (integer ALUs) or ENGINE_TENSOR (tcgen05 u8 GEMM mod 2, shared seed)."""
        _check(lib.ssbh_plan_set_engine(self.h, engine))

    @property
    def engine(self) -> int:
        return int(lib.ssbh_plan_engine(self.h))

    @property
    def hash_kernel(self) -> str:
        """Name of the hash kernel this plan launches (k_toeplitz_f4 / _mma / _mma_pb / _hash)."""
        return lib.ssbh_plan_hash_kernel(self.h).decode()

    @property
    def split_geometry(self):
        """(levels, squares per block, blocks per leaf batch) of the 3-for-4 split; levels 0 =
        direct tiled product."""
        v = [C.c_uint32() for _ in range(3)]
        _check(lib.ssbh_plan_split_geometry(self.h, *[C.byref(x) for x in v]))
        return tuple(x.value for x in v)

    def stream_begin(self, stream: int = 0, samp=None, hsh=None):
        sk = None if samp is None else _p64(key_of(samp))
        hk = None if hsh is None else _p64(key_of(hsh))
        _check(lib.ssbh_plan_stream_begin(self.h, sk, hk, C.c_void_p(stream or None)))

    def stream_chunk(self, index: int, d_chunk_ptr: int, stream: int = 0):
        _check(lib.ssbh_plan_stream_chunk(self.h, index, C.c_void_p(d_chunk_ptr),
                                          C.c_void_p(stream or None)))

    def stream_finish(self, d_key_ptr: int, d_len_ptr: int = 0, stream: int = 0):
        _check(lib.ssbh_plan_stream_finish(self.h, C.c_void_p(d_key_ptr),
                                           C.c_void_p(d_len_ptr or None),
                                           C.c_void_p(stream or None)))

    @property
    def device_bytes(self) -> int:
        return int(lib.ssbh_plan_device_bytes(self.h))

    def set_timing(self, on=True):
        _check(lib.ssbh_plan_set_timing(self.h, 1 if on else 0))

    def run_device(self, d_input_ptr: int, d_key_ptr: int, d_len_ptr: int = 0, stream: int = 0,
                   samp=None, hsh=None):
        sk = None if samp is None else _p64(key_of(samp))
        hk = None if hsh is None else _p64(key_of(hsh))
        _check(lib.ssbh_plan_run_device(self.h, C.c_void_p(d_input_ptr), C.c_void_p(d_key_ptr),
                                        C.c_void_p(d_len_ptr or None), sk, hk,
                                        C.c_void_p(stream or None)))

    def check(self) -> ExtractStats:
        st = ExtractStats()
        _check(lib.ssbh_plan_check(self.h, C.byref(st)))
        return st

    def run_host(self, x_words, key_out=None, len_out=None):
        x = np.ascontiguousarray(x_words, dtype=np.uint64)
        key = key_out if key_out is not None else np.zeros(max(nwords(self.owned * self.k), 1),
                                                           dtype=np.uint64)
        lens = len_out if len_out is not None else np.zeros(self.owned, dtype=np.uint64)
        st = ExtractStats()
        _check(lib.ssbh_plan_run_host(self.h, _p64(x), _p64(key), _p64(lens), C.byref(st)))
        return key, lens, st

    def run_host_ptrs(self, x_ptr: int, key_ptr: int, len_ptr: int):
        st = ExtractStats()
        _check(lib.ssbh_plan_run_host(self.h, C.cast(x_ptr, U64P), C.cast(key_ptr, U64P),
                                      C.cast(len_ptr, U64P) if len_ptr else None, C.byref(st)))
        return st

    def close(self):
        if getattr(self, "h", None):
            lib.ssbh_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Shard:
    """One rank of a sharded multi-GPU extraction (ssbh_shard_*). The host protocol (handle
    exchange, count all-gather, barrier) lives in multigpu.ShardedExtractor."""

    IPC_BYTES = 64

    def __init__(self, n, s, k, samp, hsh, rank, world, per_block=False):
        self.params = make_params(n, s, k, samp, hsh, per_block)
        self.n, self.s, self.k, self.rank, self.world = n, s, k, rank, world
        h = C.c_void_p()
        _check(lib.ssbh_shard_create(C.byref(self.params), rank, world, C.byref(h)))
        self.h = h
        sf, sn = np.zeros(1, np.uint64), np.zeros(1, np.uint64)
        bf, bc = np.zeros(1, np.uint32), np.zeros(1, np.uint32)
        _check(lib.ssbh_shard_info(self.h, _p64(sf), _p64(sn), _p32(bf), _p32(bc)))
        self.slice_first, self.slice_rounds = int(sf[0]), int(sn[0])
        self.block_first, self.block_count = int(bf[0]), int(bc[0])

    @property
    def hash_kernel(self) -> str:
        return lib.ssbh_shard_hash_kernel(self.h).decode()

    @property
    def split_geometry(self):
        v = [C.c_uint32() for _ in range(3)]
        _check(lib.ssbh_shard_split_geometry(self.h, *[C.byref(x) for x in v]))
        return tuple(x.value for x in v)

    def ipc_handle(self) -> bytes:
        buf = C.create_string_buffer(self.IPC_BYTES)
        _check(lib.ssbh_shard_ipc_handle(self.h, buf))
        return buf.raw

    def open_peers(self, handles):
        blob = C.create_string_buffer(b"".join(handles), self.IPC_BYTES * self.world)
        _check(lib.ssbh_shard_open_peers(self.h, blob))

    def set_timing(self, on=True):
        _check(lib.ssbh_shard_set_timing(self.h, 1 if on else 0))

    def sample(self, d_slice_ptr: int, stream: int = 0, samp=None) -> np.ndarray:
        out = np.zeros(self.world, np.uint64)
        sk = None if samp is None else _p64(key_of(samp))
        _check(lib.ssbh_shard_sample(self.h, C.c_void_p(d_slice_ptr), sk, _p64(out),
                                     C.c_void_p(stream or None)))
        return out

    def exchange(self, counts_matrix, stream: int = 0):
        m = np.ascontiguousarray(counts_matrix, dtype=np.uint64).reshape(-1)
        _check(lib.ssbh_shard_exchange(self.h, _p64(m), C.c_void_p(stream or None)))

    def finish(self, d_key_ptr: int, d_len_ptr: int = 0, stream: int = 0, hsh=None):
        hk = None if hsh is None else _p64(key_of(hsh))
        _check(lib.ssbh_shard_finish(self.h, C.c_void_p(d_key_ptr), C.c_void_p(d_len_ptr or None),
                                     hk, C.c_void_p(stream or None)))

    def check(self) -> ExtractStats:
        st = ExtractStats()
        _check(lib.ssbh_shard_check(self.h, C.byref(st)))
        return st

    def close(self):
        if getattr(self, "h", None):
            lib.ssbh_shard_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def make_input_device(seed, p, nbits, d_out_ptr: int, stream: int = 0):
    _check(lib.ssbh_make_input_device(_p64(key_of(seed)), float(p), nbits,
                                      C.c_void_p(d_out_ptr), C.c_void_p(stream or None)))


def measure_lop3_peak(iters: int = 20000):
    """Measured LOP3 lane-ops/s of the current device (int-ALU roofline denominator)."""
    r, ms = C.c_double(0), C.c_double(0)
    _check(lib.ssbh_measure_lop3_peak(iters, C.byref(r), C.byref(ms)))
    return r.value, ms.value


def get_overrides() -> dict:
    o = PlanOverrides()
    _check(lib.ssbh_get_plan_overrides(C.byref(o)))
    return {f: getattr(o, f) for f, _ in PlanOverrides._fields_}


def set_overrides(**kw) -> dict:
    """Set plan-construction overrides (process-wide, read when a plan is created); fields not
    given keep their defaults (DEFAULT_OVERRIDES). Returns the previous values."""
    prev = get_overrides()
    vals = dict(DEFAULT_OVERRIDES)
    for key, v in kw.items():
        if key not in vals:
            raise TypeError(f"unknown override {key}")
        vals[key] = v
    _check(lib.ssbh_set_plan_overrides(C.byref(PlanOverrides(**vals))))
    return prev


class overrides:
    """Context manager: `with overrides(split_levels=3): plan = Plan(...)`; the previous
    overrides are restored on exit. Fields not given are merged over the current ones."""

    def __init__(self, **kw):
        self.kw = kw

    def __enter__(self):
        cur = get_overrides()
        cur.update(self.kw)
        self.prev = set_overrides(**cur)
        return self

    def __exit__(self, *exc):
        set_overrides(**self.prev)
        return False


def fnv1a64(words) -> int:
    """FNV-1a-64 key digest (ssbh_fnv1a64; host computation over u64 words)."""
    w = np.ascontiguousarray(words, dtype=np.uint64)
    return int(lib.ssbh_fnv1a64(w.ctypes.data_as(U64P), w.size))


def measure_mma_f4_peak(iters: int = 200000):
    """Measured tcgen05 kind::mxf4 MAC/s with the FP4 hash kernel's operand layouts."""
    r, ms = C.c_double(0), C.c_double(0)
    _check(lib.ssbh_measure_mma_f4_peak(iters, C.byref(r), C.byref(ms)))
    return r.value, ms.value


# BASELINE.json configs: one table in workloads.py at the repo root (plain data, so that
# bench.py's reference arm reads it without loading this package's CUDA library)
def _load_configs():
    import importlib.util

    spec = importlib.util.spec_from_file_location(
        "_ssbh_workloads", os.path.join(os.path.dirname(HERE), "workloads.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.CONFIGS


CONFIGS = _load_configs()
