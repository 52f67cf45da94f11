"""Summarise an ncu source-page CSV (--page source --csv --print-source sass)
by SASS line ranges: samples and stall reasons per region.
usage: python tools/ncu_regions.py src.csv name:lo-hi [name:lo-hi ...]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[i_s] or 0) for r in data)
def f(x):
    try: return float(x)
    except ValueError: return 0.0
for spec in sys.argv[2:]:
    name, rng = spec.split(":")
    lo, hi = map(int, rng.split("-"))
    sub = data[lo:hi + 1]
    s = sum(f(r[i_s]) for r in sub)
    st = {h: sum(f(r[hdr.index(h)]) for r in sub) for h in stalls}
    top = sorted(st.items(), key=lambda kv: -kv[1])[:6]
    print(f"{name:12s} {s / tot * 100:5.1f}%  " + "  ".join(f"{k[6:]}={v / max(s, 1) * 100:.0f}%" for k, v in top))
