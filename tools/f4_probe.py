"""FP4 (kind::mxf4, all scales 1.0) tensor-core probe: MAC rate and exactness of the f32
accumulation of integer sums — decides whether a GF(2) engine on FP4 operands is possible."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2308_02856_b200 as P  # noqa: E402

f = P.lib.ssbh_probe_mma_f4
f.restype = C.c_int
f.argtypes = [C.c_uint32, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
              C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
for mode, iters in ((0, 20000), (0, 200000), (2, 200000), (3, 200000), (1, 1000),
                    (1, (1 << 20) + 3), (1, (1 << 24) + 5)):
    r, ms, bad, smp = C.c_double(), C.c_double(), C.c_uint32(), C.c_uint32()
    st = f(iters, mode, C.byref(r), C.byref(ms), C.byref(bad), C.byref(smp))
    val = C.c_float.from_buffer(C.c_uint32(smp.value)).value
    print(json.dumps({"mode": mode, "iters": iters, "status": st, "ms": round(ms.value, 2),
                      "T_mac_s": round(r.value / 1e12, 1), "mismatches": bad.value,
                      "acc_sample": val}), flush=True)
