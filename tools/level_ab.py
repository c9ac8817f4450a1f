"""Split-level A/B on a config-5-shaped plan with fewer blocks (development aid): n = s * 2^22
rounds, k = 2^21, shared seed; per level: hash ms and the key digest (must not change)."""
import argparse
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2308_02856_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--s", type=int, default=1024)
ap.add_argument("--k", type=int, default=1 << 21)
ap.add_argument("--m", type=int, default=1 << 22)
ap.add_argument("--levels", default="7,8,9")
ap.add_argument("--budget-mb", type=int, default=0)
args = ap.parse_args()
n, s, k = args.s * args.m, args.s, args.k
d_in = torch.zeros((n + 63) // 64 * 2, dtype=torch.int32, device="cuda")
P.make_input_device(1, 0.5, n, d_in.data_ptr())
d_key = torch.zeros((s * k + 63) // 64 * 2, dtype=torch.int32, device="cuda")
stream = torch.cuda.Stream()
for L in [int(x) for x in args.levels.split(",")]:
    P.set_overrides(split_levels=L, split_budget_mb=args.budget_mb)
    plan = P.Plan(n, s, k, 2, 3)
    plan.set_timing(True)
    for r in range(2):
        plan.run_device(d_in.data_ptr(), d_key.data_ptr(), 0, stream.cuda_stream)
        st = plan.check()
    dig = hashlib.sha256(d_key.cpu().numpy().tobytes()).hexdigest()[:16]
    print(json.dumps({"L": L, "kernel": plan.hash_kernel, "geom": plan.split_geometry,
                      "ms_hash": round(st.ms_hash, 2), "ms_total": round(st.ms_total, 2),
                      "bytes_GB": round(plan.device_bytes / 1e9, 2), "key_sha": dig}), flush=True)
    plan.close()
