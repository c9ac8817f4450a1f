"""Probe: CTA-pair (cta_group::2) kind::mxf4 with A from TMEM — layout (mode 1: one-hot rows,
D read back from both CTAs) and rate (mode 2). Development aid (csrc/diag.cu k_f4_pair_probe)."""
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2308_02856_b200 as P  # noqa: E402

f = P.lib.ssbh_probe_mma_f4_pair
f.restype = C.c_int
f.argtypes = [C.c_uint32, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
              C.POINTER(C.c_uint32), C.c_void_p]
for mode, iters in ((1, 1), (2, 200000)):
    r, ms, bad = C.c_double(), C.c_double(), C.c_uint32()
    d = np.zeros((256, 256), dtype=np.float32)
    st = f(iters, mode, C.byref(r), C.byref(ms), C.byref(bad), d.ctypes.data)
    out = {"mode": mode, "iters": iters, "status": st, "ms": round(ms.value, 3),
           "T_mac_s": round(r.value / 1e12, 1), "mismatches": bad.value}
    if mode == 1:
        out["hits"] = {int(rr): [int(n) for n in np.nonzero(d[rr])[0]][:6] for rr in (0, 1, 63, 64, 127, 128, 129, 200, 255)}
        out["sum"] = float(d.sum())
    print(json.dumps(out), flush=True)
peak, _ = P.measure_mma_f4_peak(200000)
print(json.dumps({"single_cta_hash_layout_T_mac_s": round(peak / 1e12, 1)}))
