"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per kernel launches,
mean device time, share of the profiled total.  Usage: python tools/ncu_launches.py launches.csv"""
import collections
import csv
import io
import sys

text = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(text) if l.startswith('"ID"'))
rows = list(csv.DictReader(io.StringIO("\n".join(text[start:]))))
agg = collections.OrderedDict()
scale = {"ns": 1.0, "nsecond": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"]
    short = name.split("(")[0].replace("void ", "")
    v = float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1.0)
    agg.setdefault(short, []).append((v, r["Grid Size"], r["Block Size"]))
tot = sum(v for l in agg.values() for v, _, _ in l)
print(f"| kernel | launches | mean µs | share | grid x block |")
print("|---|---|---|---|---|")
for k, l in sorted(agg.items(), key=lambda kv: -sum(v for v, _, _ in kv[1])):
    s = sum(v for v, _, _ in l)
    print(f"| `{k}` | {len(l)} | {s / len(l) / 1e3:.1f} | {s / tot:.3f} | {l[0][1]} x {l[0][2]} |")
print(f"\ntotal profiled device time {tot / 1e3:.1f} µs over {sum(len(l) for l in agg.values())} launches")
