"""Per-instruction stall breakdown from an ncu source-page CSV (sass):  python tools/stalls.py file.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
h = rows[1]
reasons = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
si = h.index("Warp Stall Sampling (All Samples)")
tot = {r: 0 for r in reasons}
data = []
for r in rows[2:]:
    if len(r) < len(h) or not (r[si] or "0").isdigit():
        continue
    s = int(r[si] or 0)
    rs = {x: int(r[h.index(x)] or 0) for x in reasons}
    for x in reasons:
        tot[x] += rs[x]
    data.append((s, r[h.index("Address")][-5:], r[h.index("Source")][:70], rs))
T = sum(tot.values())
print("reason totals:", ", ".join(f"{k[6:]}={100*v/T:.1f}%" for k, v in sorted(tot.items(), key=lambda kv: -kv[1]) if v))
for s, a, src, rs in sorted(data, key=lambda d: -d[0])[:n]:
    top = sorted(rs.items(), key=lambda kv: -kv[1])[:2]
    print(f"{s:7d} {a} {src:70s} " + " ".join(f"{k[6:]}:{v}" for k, v in top if v))
