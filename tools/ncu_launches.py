"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv --log-file): per-kernel count, mean, share."""
import collections
import csv
import sys

lines = [ln for ln in open(sys.argv[1]) if not ln.startswith("==")]
r = list(csv.reader(lines))
h = r[0]
agg = collections.defaultdict(list)
for x in r[1:]:
    if len(x) < len(h):
        continue
    n = x[h.index("Kernel Name")].split("(")[0].replace("vsag::<unnamed>::", "").replace("unnamed>::", "")
    n = n.replace("void ", "")
    agg[n].append(float(x[h.index("Metric Value")]))
tot = sum(sum(v) for v in agg.values())
for n, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{n[:60]:60s} launches {len(v):3d}  mean {sum(v) / len(v) / 1e3:9.1f} us  share {100 * sum(v) / tot:5.1f}%")
