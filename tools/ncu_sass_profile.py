"""Dynamic SASS listing from `ncu --page source --csv --print-source sass,cuda`: every
instruction in address order with its source line, executions per hop and stall samples.
python tools/ncu_sass_profile.py src.csv hops > out.txt"""
import csv
import sys

hops = float(sys.argv[2])
rows = list(csv.reader(open(sys.argv[1])))
cur = None
hdr = None
line = None
ins = {}
for x in rows:
    if not x:
        continue
    if x[0] == "File Path":
        cur = x[1].split("/")[-1]
        continue
    if x[0] == "Line No":
        hdr = x
        ie = hdr.index("Instructions Executed")
        ia = hdr.index("Address")
        ist = hdr.index("# Samples")
        continue
    if hdr is None:
        continue
    if x[0]:
        line = f"{cur[:16]}:{x[0]}"
        continue
    if x[ia].startswith("0x"):
        a = int(x[ia], 16)
        ins[a] = (line, x[ia + 1].strip(), int(x[ie]) if x[ie].isdigit() else 0, int(x[ist]) if x[ist].isdigit() else 0)
base = min(ins)
tot = 0
tots = sum(v[3] for v in ins.values())
for a in sorted(ins):
    l, sass, n, st = ins[a]
    tot += n
    print(f"{a - base:05x} {l:24s} {n / hops:7.3f} {100.0 * st / max(tots, 1):5.2f}%  {sass}")
print(f"total {tot / hops:.1f} per hop")
