"""Print SASS with execution counts for a source line range of one file (ncu --page source --print-source sass,cuda csv)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
fname, lo, hi = sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
cur = None
hdr = None
ln = None
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
    if x[0]:
        try:
            ln = int(x[0])
        except ValueError:
            continue
        if cur == fname and lo <= ln <= hi:
            print(f"--- {ln}: {x[1][:110]}")
        continue
    if cur == fname and ln is not None and lo <= ln <= hi:
        print(f"    {x[2][-5:]} {x[3][:70]:70s} ex={x[7]:>9} smp={x[6]}")
