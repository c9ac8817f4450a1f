"""Measured tensor-core (tcgen05 kind::i8) and LOP3 peaks of this GPU, with the SM clock
sampled during each probe (development aid for the roofline denominators)."""
import json
import os
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2308_02856_b200 as P  # noqa: E402


def sampled(fn):
    clocks, stop = [], threading.Event()

    def poll():
        while not stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw",
                                      "--format=csv,noheader,nounits", "-i", "0"],
                                     capture_output=True, text=True, timeout=5).stdout
                c, p = out.strip().split(",")[:2]
                clocks.append((float(c), float(p)))
            except Exception:
                pass
            time.sleep(0.05)

    t = threading.Thread(target=poll, daemon=True)
    t.start()
    r = fn()
    stop.set()
    t.join()
    return r, clocks


for pairs in (False, True):
  for layout in (0, 1):
    for iters in (20000, 200000):
        (rate, ms), clk = sampled(lambda: P.measure_mma_i8_peak(iters, layout, pairs))
        print(json.dumps({"probe": "i8", "pairs": pairs, "layout": layout, "iters": iters,
                          "ms": round(ms, 2),
                          "T_mac_s": round(rate / 1e12, 1), "T_ops": round(2 * rate / 1e12, 1),
                          "sm_mhz": sorted(c for c, _ in clk)[len(clk) // 2] if clk else None,
                          "power_w_max": max((p for _, p in clk), default=None)}), flush=True)
(rate, ms), clk = sampled(lambda: P.measure_lop3_peak(200000))
print(json.dumps({"probe": "lop3", "T_s": round(rate / 1e12, 3), "ms": round(ms, 1),
                  "sm_mhz": sorted(c for c, _ in clk)[len(clk) // 2] if clk else None}), flush=True)
