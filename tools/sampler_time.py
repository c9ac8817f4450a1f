"""Per-phase timing of the sampler at BASELINE shapes with a tiny k (development aid, not
the bench): the count / scan / scatter passes depend on n and s only, so k = 64 isolates them
from the hash. Prints one JSON line per repetition; the SSBH_* env knobs of sampler.cu select
the variant under test."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2308_02856_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2n", type=int, default=34)
    ap.add_argument("--s", type=int, default=16384)
    ap.add_argument("--k", type=int, default=64)
    ap.add_argument("--chunks", type=int, default=0, help="streaming plan with this many chunks")
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    n, s, k = 1 << args.log2n, args.s, args.k
    tag = {e: os.environ[e] for e in os.environ if e.startswith("SSBH_")}
    cb = n // args.chunks if args.chunks else 0
    plan = P.Plan(n, s, k, 2, 3, per_block=True, chunk_bits=cb)
    plan.set_timing(True)
    d_in = torch.zeros(n // 32, dtype=torch.int32, device="cuda")
    P.make_input_device(1, 0.5, n, d_in.data_ptr())
    d_key = torch.zeros((s * k + 63) // 64 * 2, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    stream = torch.cuda.Stream()
    for r in range(args.reps + 1):
        if cb:
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.chunks + 2)]
            plan.stream_begin(stream.cuda_stream)
            ev[0].record(stream)
            for ci in range(args.chunks):
                plan.stream_chunk(ci, d_in.data_ptr() + ci * (cb // 8), stream.cuda_stream)
                ev[ci + 1].record(stream)
            plan.stream_finish(d_key.data_ptr(), 0, stream.cuda_stream)
            st = plan.check()
            chunk_ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.chunks)]
        else:
            plan.run_device(d_in.data_ptr(), d_key.data_ptr(), 0, stream.cuda_stream)
            st = plan.check()
            chunk_ms = None
        if r == 0:
            continue
        print(json.dumps({"env": tag, "n": f"2^{args.log2n}", "s": s, "k": k,
                          "ms_sample": round(st.ms_sample, 3), "ms_scatter": round(st.ms_scatter, 3),
                          "ms_hash": round(st.ms_hash, 3), "ms_total": round(st.ms_total, 3),
                          "chunk_scatter_ms": [round(x, 2) for x in chunk_ms] if chunk_ms else None,
                          "bytes": plan.device_bytes}), flush=True)
    plan.close()


if __name__ == "__main__":
    main()
