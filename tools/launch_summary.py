"""Summarise ncu --csv launch lists: total ms per kernel name (one line per file)."""
import csv
import sys
from collections import defaultdict

for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    if not rows:
        print(f, "empty")
        continue
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("(anonymous namespace)::", "").replace("unnamed>::", "")
        tot[name] += float(r[vi].replace(",", "")) / 1e6
        cnt[name] += 1
    print("==", f)
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:12]:
        print(f"  {v:10.3f} ms  x{cnt[k]:<4d} {k}")
