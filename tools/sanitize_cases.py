"""Small extractions through every hash kernel and the sampler, for compute-sanitizer runs
(tools/sanitize.sh): the all-blocks FP4 GEMM (k_toeplitz_f4), the tiled kernel with per-block
seeds and D-step parts (k_toeplitz_mma_pb), the 3-for-4 split (GEMM and tiled leaves), the
LOP3 kernel, the single- and two-level scatter. Each case is checked against the oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2308_02856_b200 as P  # noqa: E402
from oracle.pyoracle import Oracle  # noqa: E402

o = Oracle()
cases = [  # name, (n, s, k, per_block), overrides
    ("gemm", (300000, 64, 1024, False), {}),
    ("tiled-per-block", (200000, 3, 4096, True), {}),
    ("tiled-shared", (400000, 2, 2048, False), dict(shared_tiled=1)),
    ("split-gemm", (1 << 20, 2, 1 << 18, False), dict(split_levels=2)),
    ("split-tiled", (1 << 20, 2, 1 << 18, True), dict(split_levels=1)),
    ("lop3", (200000, 16, 512, False), dict(engine=P.ENGINE_LOP3)),
    ("two-level-scatter", (300000, 600, 64, False), dict(buckets=1)),
]
only = sys.argv[1:]
for name, (n, s, k, pb), ov in cases:
    if only and name not in only:
        continue
    P.set_overrides(**ov)
    x = o.make_input(3, 0.5, n)
    plan = P.Plan(n, s, k, 5, 6, per_block=pb)
    got, nj, _ = plan.run_host(x)
    kern = plan.hash_kernel
    plan.close()
    want, wnj = o.extract(x, n, s, 5, 6, int(pb), k)
    ok = bool((got == want).all() and (nj == wnj).all())
    print(f"{name}: {kern} {'ok' if ok else 'MISMATCH'}", flush=True)
    assert ok
P.set_overrides()
