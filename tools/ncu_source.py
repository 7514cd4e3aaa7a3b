"""Top SASS instructions of an ncu --page source --csv export by stall samples and by excessive
shared-memory wavefronts.  Usage: python tools/ncu_source.py src.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = rows[2:]


def num(r, k):
    try:
        return float(r[idx[k]].replace(",", "")) if r[idx[k]] else 0.0
    except (KeyError, ValueError, IndexError):
        return 0.0


tot = sum(num(r, "Warp Stall Sampling (All Samples)") for r in data)
print(f"total stall samples {tot:.0f}")
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
for key in ("Warp Stall Sampling (All Samples)", "L1 Wavefronts Shared Excessive"):
    print(f"\n== top by {key}")
    for r in sorted(data, key=lambda r: -num(r, key))[:n]:
        top = sorted(((num(r, s), s) for s in stalls), reverse=True)[:2]
        print(f"{r[idx['Address']]:>6} {num(r, key):8.0f}  {r[idx['Source']][:60]:60s} "
              + " ".join(f"{s[6:]}={v:.0f}" for v, s in top if v))
