"""Per-hop instruction breakdown of search_kernel by code region (ncu source page csv, sass+cuda)."""
import collections
import csv
import os
import sys

HOPS = float(sys.argv[2]) if len(sys.argv) > 2 else 1.61e6
rows = list(csv.reader(open(sys.argv[1])))
cur = None
hdr = None
agg = collections.defaultdict(int)
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
root = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2503_17911_b200", "csrc")


def lines(f):
    return open(os.path.join(root, f)).read().split("\n")


def find(src, t):
    for i, l in enumerate(src):
        if t in l:
            return i + 1
    raise KeyError(t)


def rng(f, a, b):
    return sum(v for (ff, l), v in agg.items() if ff == f and a <= l <= b) / HOPS


k = lines("search_kernel.cuh")
c = lines("search_common.cuh")
regions = [
    ("merge", "search_kernel.cuh", find(k, "template <int E, bool DEDUP>"), find(k, "// VAR 0: generic")),
    ("preamble/init", "search_kernel.cuh", find(k, "// VAR 0: generic"), find(k, "const int lim = min(ef, psz);") - 1),
    ("select", "search_kernel.cuh", find(k, "const int lim = min(ef, psz);"), find(k, "// neighbour ids (lines 7-10")),
    ("ids+filter", "search_kernel.cuh", find(k, "// neighbour ids (lines 7-10"), find(k, "// lines 13-17")),
    ("gather", "search_kernel.cuh", find(k, "// lines 13-17"), find(k, "// The next expansion is the smaller")),
    ("predict", "search_kernel.cuh", find(k, "// The next expansion is the smaller"), find(k, "if (ns > 0) {")),
    ("lower_bound", "search_common.cuh", find(c, "__device__ __forceinline__ int pool_lower_bound"),
     find(c, "// Visited-set test-and-insert, u32")),
    ("visit16", "search_common.cuh", find(c, "__device__ __forceinline__ bool any_half_eq"), find(c, "// Trace outputs")),
    ("finish", "search_common.cuh", find(c, "// Trace outputs"), 100000),
]
tot = sum(agg.values()) / HOPS
acc = 0
for name, f, a, b in regions:
    v = rng(f, a, b)
    acc += v
    print(f"{name:16s} {v:7.1f} /hop")
for f in sorted(set(k2[0] for k2 in agg)):
    if f not in ("search_kernel.cuh", "search_common.cuh"):
        v = sum(x for (ff, _), x in agg.items() if ff == f) / HOPS
        acc += v
        print(f"{'  ' + f:16s} {v:7.1f} /hop")
print(f"{'total':16s} {tot:7.1f} /hop")
