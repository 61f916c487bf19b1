"""Aggregate ncu source-page samples / instructions of search.cu by line range (region map)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
regions = [tuple(x.split(":")) for x in sys.argv[2:]]  # name:lo:hi  (search.cu lines)
cur = None
hdr = None
agg = collections.defaultdict(lambda: [0, 0])
for x in rows:
    if not x:
        continue
    if x[0] == "File Path":
        cur = x[1].split("/")[-1]
        continue
    if x[0] == "Line No":
        hdr = x
        continue
    if hdr is None:
        continue
    try:
        ln = int(x[0])
    except ValueError:
        continue
    f = lambda v: int(v) if v.isdigit() else 0  # noqa: E731
    s = f(x[hdr.index("# Samples")])
    i = f(x[hdr.index("Instructions Executed")])
    name = f"other:{cur}"
    if cur == "search.cu":
        for nm, lo, hi in regions:
            if int(lo) <= ln <= int(hi):
                name = nm
                break
    agg[name][0] += s
    agg[name][1] += i
ts = sum(v[0] for v in agg.values())
ti = sum(v[1] for v in agg.values())
for k, (s, i) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:28s} samples {100*s/ts:5.1f}%  instr {100*i/ti:5.1f}%  ({i/1e6:.1f} M)")
