"""Probe: can kind::mxf4 read its A operand from TMEM (tcgen05.mma [d], [a_tmem], b_desc)?
mode 0 exactness, mode 1 K-element layout of A in TMEM (one-hot rows vs one-hot B rows),
mode 2 rate. Development aid (csrc/diag.cu k_f4_tmem_a_probe)."""
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2308_02856_b200 as P  # noqa: E402

f = P.lib.ssbh_probe_mma_f4_tmem_a
f.restype = C.c_int
f.argtypes = [C.c_uint32, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
              C.POINTER(C.c_uint32), C.c_void_p]
for mode, iters in ((0, 1000), (0, (1 << 20) + 3), (1, 1), (2, 200000), (3, 400000)):
    r, ms, bad = C.c_double(), C.c_double(), C.c_uint32()
    d = np.zeros((128, 256), dtype=np.float32)
    st = f(iters, mode, C.byref(r), C.byref(ms), C.byref(bad), d.ctypes.data)
    out = {"mode": mode, "iters": iters, "status": st, "ms": round(ms.value, 3),
           "T_mac_s": round(r.value / 1e12, 1), "mismatches": bad.value}
    if mode == 1:
        # for each A row r: which B rows n (mod 64) got a 1
        hits = {int(rr): [int(n) for n in np.nonzero(d[rr, :64])[0]] for rr in range(0, 128, 9)}
        out["hits"] = hits
        out["sum"] = float(d.sum())
    print(json.dumps(out), flush=True)
peak, _ = P.measure_mma_f4_peak(200000)
print(json.dumps({"smem_a_hash_layout_T_mac_s": round(peak / 1e12, 1)}))
