"""Quick per-phase timing of the fused path on one GPU (development aid, not the bench)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2308_02856_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    peak, pms = P.measure_lop3_peak(20000)
    print(json.dumps({"lop3_peak_Tops": peak / 1e12, "ms": pms}), flush=True)
    for cid in [int(c) for c in args.configs.split(",")]:
        c = P.CONFIGS[cid]
        n, s, k = c["n"], c["s"], c["k"]
        t0 = time.time()
        plan = P.Plan(n, s, k, c["seed_samp"], c["seed_hash"], per_block=c["per_block"])
        plan.set_timing(True)
        d_in = torch.zeros((n + 63) // 64 * 2, dtype=torch.int32, device="cuda")
        P.make_input_device(c["seed_in"], c["p"], n, d_in.data_ptr())
        d_key = torch.zeros((s * k + 63) // 64 * 2, dtype=torch.int32, device="cuda")
        torch.cuda.synchronize()
        for r in range(args.reps):
            plan.run_device(d_in.data_ptr(), d_key.data_ptr())
            st = plan.check()
            d = st.as_dict()
            d.update(config=cid, rep=r, plan_gb=plan.device_bytes / 1e9,
                     hash_Tops=st.hash_word_ops / (st.ms_hash * 1e-3) / 1e12,
                     frac=st.hash_word_ops / (st.ms_hash * 1e-3) / peak,
                     gbit_s=n / (st.ms_total * 1e-3) / 1e9)
            print(json.dumps(d), flush=True)
        key = d_key.cpu().numpy().view(np.uint64)
        h = 0xCBF29CE484222325
        kb = key.tobytes() if key.nbytes <= (4 << 20) else b""
        for b in kb:
            h = ((h ^ b) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
        print(json.dumps({"config": cid, "key_fnv": f"{h:016x}", "setup_s": time.time() - t0}),
              flush=True)
        plan.close()
        del d_in, d_key
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
