"""Per-source-line executed instructions / hop (ncu --page source --csv --print-source sass,cuda):
python tools/ncu_lines.py src.csv [hops] [min_per_hop]"""
import collections
import csv
import sys

HOPS = float(sys.argv[2]) if len(sys.argv) > 2 else 1.61e6
MIN = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
rows = list(csv.reader(open(sys.argv[1])))
cur = None
hdr = None
agg = collections.defaultdict(int)
src = {}
for x in rows:
    if not x:
        continue
    if x[0] == "File Path":
        cur = x[1].split("/")[-1]
        continue
    if x[0] == "Line No":
        hdr = x
        continue
    if hdr is None or not x[0]:
        continue
    try:
        ln = int(x[0])
    except ValueError:
        continue
    v = x[hdr.index("Instructions Executed")]
    agg[(cur, ln)] += int(v) if v.isdigit() else 0
    src[(cur, ln)] = x[1].strip()[:100]
tot = sum(agg.values())
for k in sorted(agg):
    if agg[k] / HOPS >= MIN:
        print(f"{k[0][:18]:18s} {k[1]:4d} {agg[k] / HOPS:6.1f}  {src[k]}")
print(f"total {tot / HOPS:.1f} /hop")
