"""Two config-3 plans on two streams, back to back without host synchronisation between them:
steady-state extractions per second (development probe for a pipelined mode)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2308_02856_b200 as P  # noqa: E402

c = P.CONFIGS[3]
n, s, k = c["n"], c["s"], c["k"]
plans = [P.Plan(n, s, k, c["seed_samp"], c["seed_hash"]) for _ in range(2)]
d_in = torch.zeros((n + 63) // 64 * 2, dtype=torch.int32, device="cuda")
P.make_input_device(c["seed_in"], c["p"], n, d_in.data_ptr())
keys = [torch.zeros((s * k + 63) // 64 * 2, dtype=torch.int32, device="cuda") for _ in range(2)]
streams = [torch.cuda.Stream(priority=0), torch.cuda.Stream(priority=-1)]
for mode in ("serial", "two-streams"):
    torch.cuda.synchronize()
    reps = 10
    t0 = time.perf_counter()
    for i in range(2 * reps):
        j = i % 2 if mode == "two-streams" else 0
        plans[j].run_device(d_in.data_ptr(), keys[j].data_ptr(), 0, streams[j].cuda_stream)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    for p in plans:
        p.check()
    print(json.dumps({"mode": mode, "ms_per_extraction": round(dt / (2 * reps) * 1e3, 3),
                      "gbit_s": round(n * 2 * reps / dt / 1e9, 2)}), flush=True)
import hashlib
print([hashlib.sha256(kk.cpu().numpy().tobytes()).hexdigest()[:16] for kk in keys])
