"""Stall samples and executed instructions per CUDA source line from an ncu report
(ncu -i X.ncu-rep --page source --csv --print-source sass,cuda > mix.csv).
Usage: python tools/ncu_lines.py mix.csv [N]"""
import collections
import csv
import os
import sys


def f(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
agg = collections.OrderedDict()
cur, hdr = "?", None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = os.path.basename(r[1])
        continue
    if r[0] == "Line No":
        hdr = r
        S = hdr.index("Warp Stall Sampling (All Samples)")
        I = hdr.index("Instructions Executed")
        stalls = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_")]
        continue
    if hdr is None or not r[0] or not r[0].isdigit():
        continue
    agg[(cur, int(r[0]))] = (r[1], f(r[S]), f(r[I]), {h: f(r[i]) for i, h in stalls})
tot = sum(v[1] for v in agg.values())
itot = sum(v[2] for v in agg.values())
print(f"total stall samples {tot:.0f}, warp instructions {itot:.0f}")
for (fn, line), (src, s, ins, st) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:n]:
    top = sorted(((v, k) for k, v in st.items()), reverse=True)[:3]
    print(f"{fn[:14]:14s}:{line:<4d} {s:6.0f} {100 * s / tot:5.1f}% ins={ins:9.0f} {src.strip()[:60]:60s} "
          + " ".join(f"{k[6:]}={v:.0f}" for v, k in top if v))
