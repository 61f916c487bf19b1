import csv, sys, collections
path = sys.argv[1]
rows = list(csv.reader(open(path)))
cur_file = None; hdr = None
agg = collections.defaultdict(lambda: [0, 0, ""])
for x in rows:
    if not x: continue
    if x[0] == "File Path": cur_file = x[1].split("/")[-1]; continue
    if x[0] == "Function Name": continue
    if x[0] == "Line No": hdr = x; continue
    if hdr is None: continue
    try:
        ln = int(x[0])
    except ValueError:
        continue
    ni = hdr.index("# Samples"); ii = hdr.index("Instructions Executed")
    s = int(x[ni]) if x[ni].isdigit() else 0; ins = int(x[ii]) if x[ii].isdigit() else 0
    a = agg[(cur_file, ln)]
    a[0] += s; a[1] += ins; a[2] = x[1][:100]
tot = sum(v[0] for v in agg.values()); toti = sum(v[1] for v in agg.values())
print("samples", tot, "instr", toti)
for (f, ln), (s, i, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 50]:
    print(f"{s / tot * 100:5.1f}% {i / toti * 100:5.1f}%  {f}:{ln:<4} {src.strip()}")
