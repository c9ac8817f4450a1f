"""Markdown table of the committed bench lines (profiles/r01_bench_config*.json)."""
import json
import os

ROOT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")
print("| config | value (input Gbit/s) | ms / step | hash kernel | frac of its live peak | e2e "
      "Gbit/s | LOP3 engine same run (Gbit/s, frac) | clocks | file |")
print("|---|---|---|---|---|---|---|---|---|")
for cid in (3, 1, 2, 4, 5):
    f = f"r01_bench_config{cid}.json"
    d = json.loads(open(os.path.join(ROOT, f)).read().strip().splitlines()[-1])
    r = d["roofline"]
    l3 = d.get("lop3_engine")
    l3s = f"{l3['value']:.3f}, {l3['roofline']['frac']:.3f}" if l3 else "—"
    clk = d.get("clocks", {})
    cs = f"{clk.get('sm_mhz')} MHz" + (f" ({', '.join(clk['reasons'])})" if clk.get("reasons") else "")
    e2e = d.get("e2e", {}).get("value")
    print(f"| {cid} | {d['value']:.3f} | {d['ms_per_step']:.3f} | `{r['kernel']}` | {r['frac']:.3f} "
          f"| {e2e:.3f} | {l3s} | {cs} | `{f}` |")
