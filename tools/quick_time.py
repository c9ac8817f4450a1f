"""Quick per-phase timing of the fused path on one GPU (development aid, not the bench).
Prints one compact JSON line per (config, rep)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2308_02856_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--engine", default="auto", choices=["auto", "lop3", "tensor"])
    ap.add_argument("--per-block", action="store_true", help="force per-block seeds")
    ap.add_argument("--override", action="append", default=[], metavar="KEY=VALUE",
                    help="plan-construction override (ssbh_set_plan_overrides)")
    ap.add_argument("--f4-peak", action="store_true", help="also run the kind::mxf4 probe")
    args = ap.parse_args()
    tag = os.environ.get("SSBH_CUDA_LIB", "in-tree") + "".join(" " + o for o in args.override)
    if args.override:
        P.set_overrides(**{kv.split("=")[0]: int(kv.split("=")[1]) for kv in args.override})
    peak, _ = P.measure_lop3_peak(20000)
    print(json.dumps({"win": tag, "lop3_peak_T": round(peak / 1e12, 3)}), flush=True)
    if args.f4_peak:
        r, ms = P.measure_mma_f4_peak()
        print(json.dumps({"win": tag, "f4_peak_P": round(r / 1e15, 4), "ms": round(ms, 2)}),
              flush=True)
    for cid in [int(c) for c in args.configs.split(",")]:
        c = dict(P.CONFIGS[cid])

        if args.per_block:
            c["per_block"] = True
        n, s, k = c["n"], c["s"], c["k"]
        plan = P.Plan(n, s, k, c["seed_samp"], c["seed_hash"], per_block=c["per_block"])
        if args.engine != "auto":
            plan.set_engine(P.ENGINE_LOP3 if args.engine == "lop3" else P.ENGINE_TENSOR)
        plan.set_timing(True)
        d_in = torch.zeros((n + 63) // 64 * 2, dtype=torch.int32, device="cuda")
        P.make_input_device(c["seed_in"], c["p"], n, d_in.data_ptr())
        d_key = torch.zeros((s * k + 63) // 64 * 2, dtype=torch.int32, device="cuda")
        torch.cuda.synchronize()
        stream = torch.cuda.Stream()
        for r in range(args.reps + 1):
            plan.run_device(d_in.data_ptr(), d_key.data_ptr(), 0, stream.cuda_stream)
            st = plan.check()
            if r == 0:
                continue  # warm-up
            print(json.dumps({
                "win": tag, "config": cid, "ms_total": round(st.ms_total, 4),
                "ms_sample": round(st.ms_sample, 4), "ms_scatter": round(st.ms_scatter, 4),
                "ms_seed": round(st.ms_seed, 4), "ms_hash": round(st.ms_hash, 4),
                "frac": round(st.hash_word_ops / (st.ms_hash * 1e-3) / peak, 4),
                "gbit_s": round(n / (st.ms_total * 1e-3) / 1e9, 4)}), flush=True)
        sample = d_key[:8].cpu().tolist()
        import hashlib
        dig = hashlib.sha256(d_key.cpu().numpy().tobytes()).hexdigest()[:16]
        print(json.dumps({"win": tag, "engine": plan.engine, "config": cid, "key_head": sample,
                          "key_sha": dig}), flush=True)
        plan.close()
        del d_in, d_key
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
