#!/usr/bin/env python3
"""bench.py — throughput of the sampled sub-block Toeplitz extractor on B200.

Metric (BASELINE.json): input Gbit/s hashed (sample + Toeplitz), whole job, and the hash
kernel's fraction of the integer-ALU roofline. One step = one full extraction of the
workload: Threefry sampling of every round, stable partition into reversed packed
sub-blocks, Toeplitz seed generation, GF(2) hash of every owned sub-block,
concatenation — from a device-resident input to a device-resident key.

Default workload: BASELINE configs[2] ("single-GPU roofline case"): n = 2^30 rounds,
s = 1024 sub-blocks, k = 2^19 output bits per sub-block, p = 0.5, seeds 1/2/3.
``--config N`` selects another BASELINE config (1-4 fit one GPU).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config 3]
    python -m torch.distributed.run --nproc-per-node N bench.py --gpus N ...

Multi-GPU (default ``--multi sharded``): each rank owns a contiguous range of sub-blocks,
samples only its n/N slice of rounds and stores each round's payload straight into the
owning rank's receive buffer through NVLink peer memory; owners then hash their blocks.
``--multi replicated`` re-samples all rounds on every rank instead. Timing is the max
over ranks of the per-rank device time.
``--impl reference`` times the reference's own CPU implementation (oracle/_ref: the
unmodified reference sources compiled by oracle/Makefile) on a bounded sample of the
same workload on the host cores; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "input Gbit/s hashed (sample+Toeplitz)"
UNIT = "Gbit/s"


def _hbm_peak():
    """MEASURED_PEAKS.json hbm_gbs (driver-written copy bandwidth on this pool's B200s), else
    the profiling recipe's fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, KeyError, ValueError):
        return 6531.6, "fallback (no MEASURED_PEAKS.json)"


HBM_PEAK_GBS, HBM_PEAK_SRC = _hbm_peak()
GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.json")


def cfg_desc(cid, c):
    return {1: "BASELINE configs[0]: small CPU-runnable case",
            2: "BASELINE configs[1]: weak source",
            3: "BASELINE configs[2]: single-GPU roofline case",
            4: "BASELINE configs[3]: multi-GPU scaling case",
            5: "BASELINE configs[4]: DI-scale large-block case"}[cid]


def log2s(v):
    return f"2^{v.bit_length() - 1}" if v & (v - 1) == 0 else str(v)


def config_dict(cid, c, n_gpus):
    return {
        "workload": f"config{cid}: n={log2s(c['n'])} rounds, s={c['s']} sub-blocks, "
                    f"k={c['k']} out bits/sub-block, p={c['p']} ({cfg_desc(cid, c)})"
                    + (" [n/k OVERRIDDEN by --rounds/--out-bits: not a BASELINE shape]"
                       if c.get("rounds_override") else ""),
        "n_bits": c["n"], "n_subblocks": c["s"], "out_bits_per_block": c["k"], "p": c["p"],
        "seed_mode": "per-block (hash-seed sub=j)" if c["per_block"] else "shared (hash-seed sub=0)",
        "seeds": {"input": c["seed_in"], "sampling": c["seed_samp"], "hash": c["seed_hash"]},
        "parallelism": f"sub-blocks sharded over {n_gpus} GPU(s)",
        "l2": "L2 (126 MB) flushed between steps by a 256 MiB write outside the step events"
              + ("; input and payload exceed L2" if c["n"] >= (1 << 30) else ""),
        **({"overrides": c["overrides"]} if c.get("overrides") else {}),
    }


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def mark(self):
        """Start of the timed region: the sampler is started before the warm-up (nvidia-smi
        takes ~0.1 s to come up, longer than a short timed region) and only the samples from
        here on are reported."""
        self.first = len(self.lines)

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        self.lines = self.lines[getattr(self, "first", 0):]
        if not self.lines:  # timed region shorter than the poll period: one direct query
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=10).stdout
                self.lines = [ln.strip() for ln in out.splitlines() if ln.strip()]
            except (OSError, subprocess.TimeoutExpired):
                pass
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
                power.append(float(f[3]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        loaded = [v for v in sm if v > 500] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(power) if power else None}


def cpu_sample_shape(cid, c, threads):
    """Bounded CPU sample of the workload: T sub-blocks of the config's shape drawn by the
    reference sampler from a T*m-round prefix, hashed on T threads. The reference's hash costs
    ~k/128 u64 XORs per input bit whatever n_j is, so the per-bit rate is kept while m is cut
    to ~20 s of work per thread for large k (m = n/s up to config 3; 2^19 for config 4, 2^18
    for config 5)."""
    m = c["n"] // c["s"]
    while m > 1024 and m * (c["k"] / 128) / 3e8 > 20:
        m //= 2
    t = max(1, min(threads, 64, c["s"]))
    return t * m, t, t  # n_sample, s_sample, nblocks


def run_reference(args, cid, c):
    from oracle.pyoracle import Oracle, Reference

    threads = os.cpu_count() or 1
    try:
        ref, kind = Reference(), "reference"
    except FileNotFoundError:
        ref, kind = None, "port"
    n_s, s_s, nb = cpu_sample_shape(cid, c, threads)
    sample = (f"{nb} sub-blocks (n_j~{n_s // s_s}, k={c['k']}: config{cid}'s k) sampled "
              f"by assign_subblocks from a {n_s}-round prefix; assign_subblocks + sift_partition "
              f"+ gather + toeplitz_hash on {min(nb, threads)} threads")

    def one(n_sample, s_sample, k, nblocks):
        if ref is not None:
            secs, bits, _ = ref.time_sample(n_sample, s_sample, k, c["p"], c["seed_in"],
                                            c["seed_samp"], c["seed_hash"], nblocks)
            return secs, bits
        o = Oracle()
        x = o.make_input(c["seed_in"], c["p"], n_sample)
        t0 = time.perf_counter()
        o.extract(x, n_sample, s_sample, c["seed_samp"], c["seed_hash"], c["per_block"], k)
        return time.perf_counter() - t0, n_sample

    for _ in range(args.warmup):  # warm the code path on a small shape
        one(1 << 16, 4, 256, 4)
    tot_s, tot_bits = 0.0, 0
    for _ in range(args.steps):
        secs, bits = one(n_s, s_s, c["k"], nb)
        tot_s += secs
        tot_bits += bits
    val = tot_bits / tot_s / 1e9
    line = {
        "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot_s / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64 (GF(2) bit-packed)",
        "data": "synthetic (KeyedStream input, seeds per BASELINE)",
        "config": config_dict(cid, c, args.gpus), "impl": "reference",
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": min(nb, threads), "kind": kind,
                         "sample": sample},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_leg(cid, c):
    """Reference CPU path timed on this host (rank 0, N=1): one bounded sample."""
    from oracle.pyoracle import Reference

    threads = os.cpu_count() or 1
    n_s, s_s, nb = cpu_sample_shape(cid, c, threads)
    try:
        ref = Reference()
        secs, bits, _ = ref.time_sample(n_s, s_s, c["k"], c["p"], c["seed_in"], c["seed_samp"],
                                        c["seed_hash"], nb)
        kind = "reference"
    except FileNotFoundError:
        from oracle.pyoracle import Oracle

        o = Oracle()
        x = o.make_input(c["seed_in"], c["p"], n_s)
        t0 = time.perf_counter()
        o.extract(x, n_s, s_s, c["seed_samp"], c["seed_hash"], c["per_block"], c["k"])
        secs, bits, kind = time.perf_counter() - t0, n_s, "port"
    return {"value": bits / secs / 1e9, "unit": UNIT, "cores": min(nb, threads), "kind": kind,
            "sample": f"{nb} sub-blocks (n_j~{n_s // s_s}, k={c['k']}: config{cid}'s k) "
                      f"from a {n_s}-round prefix: assign_subblocks + sift_partition + gather + "
                      f"toeplitz_hash, {secs:.1f} s on {min(nb, threads)} threads"}


def sampler_line(n, world, stats, sharded):
    """Sampler phases (Threefry count pass + scans + layout, then the scatter) as achieved HBM
    GB/s over their algorithmic bytes per rank: input bits read (n/8), the 2 B/round payload
    written and read back, the reversed sub-block words written (n/8). The count pass is
    Threefry-bound on the integer ALU (~208 ALU instr/round, profiles/*ncu_sampler*)."""
    rounds = n // world if sharded else n
    ms = stats.ms_sample + stats.ms_scatter
    bytes_ = rounds / 8 + 2 * rounds + 2 * rounds + rounds / 8
    gbs = bytes_ / (ms * 1e-3) / 1e9 if ms > 0 else None
    return {"ms": ms, "rounds": rounds, "rounds_per_s": rounds / (ms * 1e-3) if ms else None,
            "hbm_bytes_algorithmic": int(bytes_), "achieved_gbs": gbs,
            "hbm_frac": gbs / HBM_PEAK_GBS if gbs else None, "peak_gbs": HBM_PEAK_GBS,
            "peak_source": HBM_PEAK_SRC,
            "bound": "int-alu (Threefry4x64-20 per round), not HBM"}


def spawn_ranks(n):
    """Re-launch this command as n ranks (torch.distributed.run on 127.0.0.1); rank 0 prints
    the JSON line. Returns the launcher's exit code."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def reference_digest(cid, c, key_u64, nj, fnv):
    """The whole key (configs 1-3) or the reference-pinned blocks (configs 4-5) against the
    digests tests/golden/gen_golden.py made by running the compiled reference
    (golden.json["extract"][cid]); n_j digest too when the lengths are at hand."""
    if c.get("rounds_override"):
        return {"match": None, "why": "n/k overridden: no reference digest for this shape"}
    try:
        with open(GOLDEN) as f:
            g = json.load(f)["extract"][str(cid)]
    except (OSError, KeyError):
        return {"match": None, "why": "no golden entry"}
    out = {"source": "tests/golden/golden.json (compiled reference, gen_golden.py)"}
    if "key_fnv" in g:
        got = f"{fnv(key_u64):016x}"
        out.update(scope="whole key", want=g["key_fnv"], got=got, match=got == g["key_fnv"])
    else:
        kw = c["k"] // 64
        got = [f"{fnv(key_u64[j * kw:(j + 1) * kw]):016x}" for j in g["which"]]
        out.update(scope=f"blocks {g['which']} (reference-pinned; every block is spot-checked "
                         "in tests/test_gpu_parity.py)", want=g["block_fnv"], got=got,
                   match=got == g["block_fnv"])
    if nj is not None:
        got = f"{fnv(nj):016x}"
        out["nj_match"] = got == g["nj_fnv"]
        out["match"] = out["match"] and out["nj_match"]
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--multi", default="sharded", choices=["sharded", "replicated"],
                    help="N>1: sharded sampling + peer-memory owner exchange, or every rank "
                         "re-sampling all rounds")
    ap.add_argument("--engine", default="auto", choices=["auto", "lop3", "tensor"],
                    help="hash engine (auto = tensor: tcgen05 kind::mxf4 counts mod 2; lop3 = the "
                         "integer-ALU kernel)")
    ap.add_argument("--no-lop3-compare", action="store_true",
                    help="skip the extra LOP3-engine step reported beside a tensor-engine line")
    ap.add_argument("--override", action="append", default=[], metavar="KEY=VALUE",
                    help="dev A/B: plan-construction override (ssbh_set_plan_overrides), e.g. "
                         "split_levels=0; the line then records it under config.overrides")
    ap.add_argument("--rounds", type=int, default=0,
                    help="testing aid: override n (the line's config then names the override)")
    ap.add_argument("--out-bits", type=int, default=0,
                    help="testing aid: override k (the line's config then names the override)")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N` without a launcher: one rank per GPU via torchrun
        sys.exit(spawn_ranks(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")

    from workloads import CONFIGS  # plain data: the reference arm loads no product code

    cid = args.config
    c = dict(CONFIGS[cid])
    if args.rounds:
        c["n"] = args.rounds
        c["rounds_override"] = True
    if args.out_bits:
        c["k"] = args.out_bits
        c["rounds_override"] = True
    if args.impl == "reference":
        if rank == 0:
            run_reference(args, cid, c)
        return

    import paper_2308_02856_b200 as P

    ovr = {kv.split("=", 1)[0]: int(kv.split("=", 1)[1]) for kv in args.override}
    if args.engine == "lop3":  # every plan this process creates (shard owners too)
        ovr["engine"] = P.ENGINE_LOP3
    if ovr:
        P.set_overrides(**ovr)
        c["overrides"] = ovr
    import torch
    import torch.distributed as dist

    dev_index = local % max(1, torch.cuda.device_count())  # identity on a full box
    torch.cuda.set_device(dev_index)
    P.lib.ssbh_set_device(dev_index)
    backend = os.environ.get("SSBH_DIST_BACKEND", "nccl")  # gloo: multi-rank test on 1 GPU
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator ranks in the log
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group(backend)
    coll_dev = "cuda" if backend == "nccl" else "cpu"

    from paper_2308_02856_b200.multigpu import ShardedExtractor, owned_range

    n, s, k = c["n"], c["s"], c["k"]
    first, count = owned_range(rank, world, s)
    # config 5 (2^37 rounds, "~2 GiB of input per GPU" on 8 GPUs): with >= 8 ranks each rank
    # samples its own 2^34-round input chunk and ships payloads to the owners (sharded, ~100 GB
    # per rank); with fewer ranks a rank cannot hold its 1/N slice's payloads, so every rank
    # runs a streaming plan over the 8 input chunks and keeps only its own blocks
    streaming = cid == 5 and not (world >= 8 and args.multi == "sharded")
    sharded = world > 1 and not streaming and args.multi == "sharded"
    chunk_bits = n // 8 if streaming else 0
    stream = torch.cuda.Stream()  # capturable: untimed runs replay one CUDA graph
    d_in = torch.zeros((n + 63) // 64 * 2, dtype=torch.int32, device="cuda")
    P.make_input_device(c["seed_in"], c["p"], n, d_in.data_ptr(), stream.cuda_stream)
    key_words64 = (count * k + 63) // 64
    d_key = torch.zeros(key_words64 * 2, dtype=torch.int32, device="cuda")
    d_len = torch.zeros(max(count, 1), dtype=torch.int64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    if sharded:
        # each rank samples only its slice; payloads reach their owners by peer stores
        ex = ShardedExtractor(n, s, k, c["seed_samp"], c["seed_hash"], per_block=c["per_block"])
        ex.shard.set_timing(True)
        slice_lo, slice_n = ex.slice
        slice_ptr = d_in.data_ptr() + (slice_lo // 32) * 4
        check, close = ex.check, ex.close
    else:
        plan = P.Plan(n, s, k, c["seed_samp"], c["seed_hash"], per_block=c["per_block"],
                      block_first=first, block_count=count, chunk_bits=chunk_bits)
        if args.engine == "tensor":
            plan.set_engine(P.ENGINE_TENSOR)
        plan.set_timing(True)
        check, close = plan.check, plan.close
    tensor = args.engine != "lop3"
    hash_kernel = ex.shard.hash_kernel if sharded else plan.hash_kernel

    # roofline denominators, measured live on this GPU: LOP3 issue rate (int-ALU engine) and
    # the tcgen05 MAC rate (kind::mxf4 or kind::i8) with the hash kernel's operand layouts
    peak, _ = P.measure_lop3_peak(20000)
    tc_peak = None
    if tensor:  # ~120-140 ms probes: the sustained rate
        tc_peak = P.measure_mma_f4_peak(200000)[0]

    def step():
        if sharded:
            ex.run(slice_ptr, d_key.data_ptr(), d_len.data_ptr(), stream.cuda_stream, coll_dev)
        elif not streaming:
            plan.run_device(d_in.data_ptr(), d_key.data_ptr(), d_len.data_ptr(),
                            stream.cuda_stream)
        else:
            plan.stream_begin(stream.cuda_stream)
            for ci in range(8):
                plan.stream_chunk(ci, d_in.data_ptr() + ci * (chunk_bits // 8), stream.cuda_stream)
            plan.stream_finish(d_key.data_ptr(), d_len.data_ptr(), stream.cuda_stream)

    clocks = ClockSampler(dev_index)
    clocks.start()
    for _ in range(max(3, args.warmup)):
        step()
        check()

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    hash_ms, hash_ops, stats = [], 0, None
    for i in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(i & 0xFF)  # evict L2 between steps (outside the step events)
        ev[i][0].record(stream)
        step()  # sharded: includes the host all-gather of counts and the barrier
        ev[i][1].record(stream)
        stats = check()
        hash_ms.append(stats.ms_hash)
        hash_ops = stats.hash_word_ops
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [a_.elapsed_time(b_) for a_, b_ in ev]
    total_ms = sum(step_ms)
    clk = clocks.stop()

    # ---- the north_star LOP3 kernel on the same workload, beside a tensor-engine line ------
    lop3_cmp = None
    if tensor and world == 1 and not streaming and not sharded and not args.no_lop3_compare:
        import hashlib as _h

        ref_key = _h.sha256(d_key.cpu().numpy().tobytes()).hexdigest()
        plan.set_engine(P.ENGINE_LOP3)
        step()
        check()  # warm (captures the LOP3 graph)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        st3 = check()
        torch.cuda.synchronize()
        ms3 = e0.elapsed_time(e1)
        lop3_cmp = {
            "engine": "lop3 (k_toeplitz_hash, integer ALU; north_star's kernel)", "steps": 1,
            "ms_per_step": ms3, "value": n / (ms3 * 1e-3) / 1e9, "unit": UNIT,
            "hash_ms": st3.ms_hash,
            "roofline": {"bound": "int-alu (LOP3)", "achieved": st3.hash_word_ops / (st3.ms_hash * 1e-3) / 1e12,
                         "peak": peak / 1e12, "unit": "T LOP3 word-ops/s",
                         "frac": st3.hash_word_ops / (st3.ms_hash * 1e-3) / peak},
            "key_matches_tensor_engine":
                _h.sha256(d_key.cpu().numpy().tobytes()).hexdigest() == ref_key,
        }
        plan.set_engine(P.ENGINE_TENSOR)
        step()
        check()

    # ---- e2e through the public host API (pinned H2D of the input, D2H of the key) ------
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else args.steps
    e2e = None
    same = None
    if sharded:
        x_host = d_in.view(torch.int64)[(slice_lo // 64):(slice_lo + slice_n + 63) // 64].cpu()
        x_host = x_host.pin_memory()
        key_host = torch.empty(key_words64, dtype=torch.int64).pin_memory()
        d_slice = torch.empty_like(x_host, device="cuda")
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            with torch.cuda.stream(stream):
                d_slice.copy_(x_host, non_blocking=True)
            ex.run(d_slice.data_ptr(), d_key.data_ptr(), d_len.data_ptr(), stream.cuda_stream,
                   coll_dev)
            with torch.cuda.stream(stream):
                key_host.copy_(d_key.view(torch.int64)[:key_words64], non_blocking=True)
            stream.synchronize()
        e2e_s = time.perf_counter() - t0
        same = True
        e2e = {"h2d": int(x_host.numel() * 8), "d2h": int(key_words64 * 8),
               "api": "ssbh_shard_sample/exchange/finish (C-ABI) via multigpu.ShardedExtractor"}
    elif not streaming:
        x_host = d_in.cpu().view(torch.int64).pin_memory()
        key_host = torch.empty(key_words64, dtype=torch.int64).pin_memory()
        len_host = torch.empty(count, dtype=torch.int64).pin_memory()
        plan.run_host_ptrs(x_host.data_ptr(), key_host.data_ptr(), len_host.data_ptr())  # warm
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            plan.run_host_ptrs(x_host.data_ptr(), key_host.data_ptr(), len_host.data_ptr())
        e2e_s = time.perf_counter() - t0
        same = bool(torch.equal(key_host.cuda().view(torch.int32), d_key))
        e2e = {"h2d": int(x_host.numel() * 8), "d2h": int(key_words64 * 8 + count * 8),
               "api": "ssbh_plan_run_host (C-ABI)"}
    else:
        # streaming (config 5): the 16 GiB input stays in host memory; each step stages every
        # chunk through one pinned buffer (host copy + H2D inside the region) and reads the key
        # back, so the host<->device traffic of the whole job is timed
        cw = chunk_bits // 32
        x_host = d_in.cpu()
        pinned = torch.empty(cw, dtype=torch.int32).pin_memory()
        d_chunk = torch.empty(cw, dtype=torch.int32, device="cuda")
        key_host = torch.empty(key_words64, dtype=torch.int64).pin_memory()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            plan.stream_begin(stream.cuda_stream)
            for ci in range(8):
                pinned.copy_(x_host[ci * cw:(ci + 1) * cw])
                with torch.cuda.stream(stream):
                    d_chunk.copy_(pinned, non_blocking=True)
                plan.stream_chunk(ci, d_chunk.data_ptr(), stream.cuda_stream)
                stream.synchronize()  # pinned buffer reused by the next chunk
            plan.stream_finish(d_key.data_ptr(), d_len.data_ptr(), stream.cuda_stream)
            with torch.cuda.stream(stream):
                key_host.copy_(d_key.view(torch.int64)[:key_words64])
            stream.synchronize()
        e2e_s = time.perf_counter() - t0
        check()
        same = bool(torch.equal(key_host.cuda().view(torch.int32), d_key))
        e2e = {"h2d": int(n // 8), "d2h": int(key_words64 * 8),
               "api": "ssbh_plan_stream_begin/chunk/finish (C-ABI), chunks staged through "
                      "pinned memory"}
        del x_host

    # ---- gather the owned key slices in block order (the only inter-GPU exchange) --------
    import hashlib

    if world > 1:
        from paper_2308_02856_b200.multigpu import gather_key

        full = gather_key(d_key.view(torch.int64)[:key_words64].to(coll_dev), s, k)
    else:
        full = d_key.view(torch.int64)[:key_words64].cpu().numpy().view("uint64")
    key_sha = hashlib.sha256(full.tobytes()).hexdigest()[:16]
    digest = None
    if rank == 0:
        nj_host = d_len[:count].cpu().numpy().view("uint64") if world == 1 else None
        digest = reference_digest(cid, c, full, nj_host, P.fnv1a64)

    vals = torch.tensor([total_ms, e2e_s, max(hash_ms)], dtype=torch.float64, device=coll_dev)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    total_ms, e2e_s = vals[0].item(), vals[1].item()

    if rank == 0:
        value = n * args.steps / (total_ms * 1e-3) / 1e9
        avg_hash_ms = sum(hash_ms) / len(hash_ms)
        achieved = hash_ops / (avg_hash_ms * 1e-3)  # rank-0 owned blocks, rank-0 launches
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "hash_traffic.json")
        if os.path.exists(tpath):
            traffic = json.load(open(tpath)).get(
                f"config{cid}_n{world}" + ("_tensor" if tensor else ""))
        hbm_ms = (n / 8 + count * k / 8) / (HBM_PEAK_GBS * 1e9) * 1e3
        split = (ex.shard if sharded else plan).split_geometry if tensor else (0, 0, 0)
        if tensor:
            macs = hash_ops * 32  # sum_j n_j * k bit products = tensor MACs doing useful work
            direct_macs = macs
            split_info = None
            if split[0]:
                # 3-for-4 split: T*3^L leaf products of (k/2^L)^2 per block + the remainder
                lv, sq, batch = split
                nj = d_len[:count].cpu()
                rem = int(torch.clamp(nj - sq * k, min=0).sum().item()) * k
                macs = count * sq * 3 ** lv * (k >> lv) ** 2 + rem
                split_info = {
                    "levels": lv, "squares_per_block": sq, "blocks_per_leaf_batch": batch,
                    "leaf_macs": macs - rem, "remainder_macs": rem,
                    "direct_bit_products": direct_macs,
                    "direct_equivalent_rate": direct_macs / (avg_hash_ms * 1e-3) / 1e12,
                    "note": "the hash computes the same key with (3/4)^L of the bit products "
                            "(csrc/toeplitz_split.cu); achieved/frac count the MACs it executes, "
                            "direct_equivalent_rate the sum_j n_j*k products of the direct form "
                            "per second (can exceed the MMA peak)"}
            roof = {
                "bound": "tensor (tcgen05 kind::mxf4)",
                "kernel": hash_kernel,
                "achieved": macs / (avg_hash_ms * 1e-3) / 1e12, "peak": tc_peak / 1e12,
                "unit": ("T MAC/s (E2M1 0/1.0 x 0/1.0 -> f32 exact integer counts; one MAC = "
                         "one GF(2) bit product)"),
                "frac": macs / (avg_hash_ms * 1e-3) / tc_peak,
                "traffic": traffic,
                "traffic_unit": "bytes per launch (dram read+write, ncu --set full, profiles/)",
                "algorithmic_per_launch": (
                    f"sum_j n_j*k = {macs} bit products (owned blocks; the LOP3 engine's "
                    f"{hash_ops} word-ops x 32)" if not split[0] else
                    f"{macs} MACs of the split (leaves + remainder) over the whole hash phase "
                    f"(leaf prep, leaf and remainder launches, combine)"),
                "split": split_info,
                "peak_source": ("measured live in this run: k_f4_probe mode 2 (csrc/diag.cu), "
                                "one CTA per SM issuing back-to-back 128x256x64 kind::mxf4 "
                                "MMAs with the hash kernel's operand layouts"),
                "int_alu_equivalent": {"achieved": achieved / 1e12, "peak": peak / 1e12,
                                       "unit": "T LOP3 word-ops/s",
                                       "times_lop3_peak": achieved / peak,
                                       "note": "not a roofline fraction: the direct-form work "
                                               "counted in north_star's LOP3 unit, divided by "
                                               "the live LOP3 peak (how many LOP3-peak GPUs "
                                               "this hash equals)"},
                "hbm_term_ms": hbm_ms,
            }
        else:
            roof = {
                "bound": "int-alu (LOP3)", "kernel": "k_toeplitz_hash",
                "achieved": achieved / 1e12, "peak": peak / 1e12,
                "unit": "T LOP3 word-ops/s", "frac": achieved / peak,
                "traffic": traffic,
                "traffic_unit": "bytes per launch (dram read+write, ncu --set full, profiles/)",
                "algorithmic_per_launch": f"sum_j n_j*k/32 = {hash_ops} word-ops (owned blocks)",
                "peak_source": "measured live in this run: k_lop3_peak (csrc/diag.cu), "
                               "148 SMs x 64 LOP3 lanes/clk at the running SM clock",
                "hbm_term_ms": hbm_ms,
            }
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup),
            "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": ("e2m1 (one GF(2) bit per element as 0 / 1.0) on tcgen05 kind::mxf4, "
                      "f32 accumulate of exact integer counts, parity = count mod 2; bit-exact"
                      if tensor else "u32 (GF(2) bit-packed; LOP3/SHF/POPC, no FP)"),
            "hash_engine": "tensor" if tensor else "lop3",
            "data": "synthetic (KeyedStream input on device, seeds per BASELINE/SURVEY §8a)",
            "config": config_dict(cid, c, world),
            "multi_gpu": (
                "sharded sampling: each rank samples n/N rounds, payloads stored into the "
                "owning rank by NVLink peer stores (IPC), owners hash their blocks"
                if sharded else ("streaming plan, 8 input chunks" if streaming else
                                 "single plan" if world == 1 else
                                 "replicated sampling, owned blocks hashed per rank")),
            "roofline": roof,
            "phases_ms_last_step": {"sample_count_scan_layout": stats.ms_sample,
                                    "scatter": stats.ms_scatter, "seeds": stats.ms_seed,
                                    "hash": stats.ms_hash, "total": stats.ms_total},
            "hash_share_of_step": avg_hash_ms / (total_ms / args.steps),
            "sampler": sampler_line(n, world, stats, sharded),
            "gpu_launches": int(stats.launches) * args.steps,
            "key_sha256_16": key_sha,
            "key_matches_reference_digest": digest["match"],
            "reference_digest": digest,
            "clocks": clk,
        }
        if lop3_cmp is not None:
            line["lop3_engine"] = lop3_cmp
        if e2e is not None:
            line["e2e"] = {"value": n * e2e_steps / e2e_s / 1e9, "unit": UNIT,
                           "h2d_bytes_per_step": e2e["h2d"], "d2h_bytes_per_step": e2e["d2h"],
                           "steps": e2e_steps, "api": e2e["api"],
                           "key_matches_device_run": same}
        if world == 1 and not args.no_cpu_baseline:
            try:
                line["cpu_baseline"] = cpu_baseline_leg(cid, c)
            except Exception as e:  # baseline failure must not hide the GPU number
                line["cpu_baseline"] = {"value": None, "error": str(e)}
        print(json.dumps(line), flush=True)
    close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
