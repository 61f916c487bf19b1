"""Executed-instruction mix by SASS opcode (ncu --page source --csv --print-source sass,cuda): python tools/ncu_opmix.py src.csv [hops]"""
import collections
import csv
import sys

HOPS = float(sys.argv[2]) if len(sys.argv) > 2 else 1.371e6
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
seen = set()
agg = collections.Counter()
for x in rows:
    if not x:
        continue
    if x[0] == "Line No":
        hdr = x
        continue
    if hdr is None or x[0] or len(x) < 8:
        continue
    addr, sass = x[2], x[3].strip()
    if addr in seen:
        continue
    seen.add(addr)
    v = x[hdr.index("Instructions Executed")]
    n = int(v) if v.isdigit() else 0
    toks = sass.split()
    op = toks[0]
    if op.startswith("@"):
        op = toks[1]
    agg[op.split(".")[0]] += n
tot = sum(agg.values())
for op, n in agg.most_common(40):
    print(f"{op:10s} {n / HOPS:7.1f} /hop  {100 * n / tot:5.1f}%")
print(f"total {tot / HOPS:.1f} /hop")
