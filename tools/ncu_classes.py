"""Per-byte-class memory evidence of search_kernel from one `ncu --set full --import-source on`
capture (north_star: HBM/L2 traffic on gathered codes, adjacency and re-rank rows, sector
efficiency, stall reasons).

    ncu -i prof.ncu-rep --page source --csv --print-source sass,cuda > src.csv
    ncu -i prof.ncu-rep --page raw --csv > raw.csv
    python tools/ncu_classes.py src.csv raw.csv [queries] [hops_per_query]

Every global load instruction of the kernel is attributed to the CUDA source line it comes
from, and the line to a class by its text: id rows (adjacency), codes (the gathered SQ
codes), re-rank rows (fp32 base rows), query (fp32 query for the re-rank + the SQ operand),
pool init (the seed pool from seed_select).  Per class: executed load instructions, L1 tag
requests, L2 sectors requested (ncu's "L2 Theoretical Sectors Global"), the ideal sector
count for the bytes requested, bytes per sector used, and stall samples on the class's loads
and on the instructions that first consume them are NOT separated (ncu attributes a stall to
the waiting instruction); the stall table below is per source line.
"""
import collections
import csv
import sys

CLASSES = [
    # (the predicted next row is copied to shared memory by cp.async = LDGSTS; a mispredicted
    # hop loads its row with LDG)
    ("id rows (adjacency)", ("__ldg(ids + t)", "__ldg(ids2 + t)", "cp.async.ca.shared.global")),
    ("codes (SQ gather)", ("ldg16(cp",)),
    ("re-rank rows (fp32 base)", ("ldg16_stream(row(u)",)),
    ("query (fp32 / SQ operand)", ("reinterpret_cast<const float4 *>(qv)", "opq + c * QW")),
    ("pool init (seed select)", ("p.init_keys", "p.init_psz")),
]


def cls_of(src):
    for name, pats in CLASSES:
        if any(p in src for p in pats):
            return name
    return "other"


def main():
    src_csv, raw_csv = sys.argv[1], sys.argv[2]
    nq = float(sys.argv[3]) if len(sys.argv) > 3 else 10000
    rows = list(csv.reader(open(src_csv)))
    # ncu lists an inlined instruction once per source file it maps to (the call site and the
    # inlined helper); keep one attribution per SASS address, preferring the kernel's own files
    own = ("search_kernel.cuh", "search_common.cuh", "dist.cuh")
    hdr, cur_src, cur_file, cur_line = None, "", "", 0
    by_addr = {}
    in_kernel = False
    for x in rows:
        if not x:
            continue
        if x[0] == "File Path":
            cur_file = x[1].split("/")[-1]
            continue
        if x[0] == "Function Name":
            in_kernel = "search_kernel" in x[1]
            continue
        if x[0] == "Line No":
            hdr = {h: i for i, h in enumerate(x)}
            continue
        if hdr is None or not in_kernel:
            continue
        if x[0]:  # a source line
            cur_line, cur_src = x[0], x[1]
            continue
        addr = x[2]
        if addr in by_addr and by_addr[addr][0][0] in own and cur_file not in own:
            continue
        by_addr[addr] = ((cur_file, cur_line), cur_src, x)
    agg = collections.defaultdict(lambda: collections.Counter())
    line_stall = collections.Counter()
    line_text = {}
    for key, src, x in by_addr.values():
        sass = x[3]
        line_text[key] = src.strip()[:90]

        def num(col):
            v = x[hdr[col]] if col in hdr else ""
            try:
                return float(v)
            except ValueError:
                return 0.0
        line_stall[key] += num("Warp Stall Sampling (All Samples)")
        if "LDG" in sass and "LDGDEPBAR" not in sass:
            c = agg[cls_of(src)]
            c["inst"] += num("Instructions Executed")
            c["req"] += num("L1 Tag Requests Global")
            c["sect"] += num("L2 Theoretical Sectors Global")
            c["ideal"] += num("L2 Theoretical Sectors Global Ideal")
            c["exc"] += num("L2 Theoretical Sectors Global Excessive")
            c["stall"] += num("Warp Stall Sampling (All Samples)")
    raw = list(csv.reader(open(raw_csv)))
    rh, rv = raw[0], raw[2]
    d = dict(zip(rh, rv))

    def g(k):
        try:
            return float(d.get(k, "nan"))
        except ValueError:
            return float("nan")
    print("## per-class global loads (one launch, %d queries)\n" % nq)
    print("| class | load inst / query | L1 requests / query | L2 sectors / query | ideal sectors | "
          "bytes / sector used | MB requested / launch |")
    print("|---|---|---|---|---|---|---|")
    tot = collections.Counter()
    for name, _ in CLASSES + [("other", ())]:
        c = agg.get(name)
        if not c or not c["inst"]:
            continue
        tot.update(c)
        eff = 32.0 * c["ideal"] / c["sect"] if c["sect"] else float("nan")
        print(f"| {name} | {c['inst'] / nq:.1f} | {c['req'] / nq:.1f} | {c['sect'] / nq:.1f} | "
              f"{c['ideal'] / nq:.1f} | {eff:.1f} | {c['sect'] * 32 / 1e6:.1f} |")
    print(f"| total | {tot['inst'] / nq:.1f} | {tot['req'] / nq:.1f} | {tot['sect'] / nq:.1f} | "
          f"{tot['ideal'] / nq:.1f} | {32.0 * tot['ideal'] / max(tot['sect'], 1):.1f} | {tot['sect'] * 32 / 1e6:.1f} |")
    print("\n## kernel-wide memory counters\n")
    keys = [
        "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_bytes.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread"]
    for k in keys:
        if k in d:
            print(f"- `{k}` = {d[k]}")
    s, r = g("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"), g("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum")
    if s == s and r == r and r:
        print(f"- sector efficiency (global loads): {s / r:.2f} sectors per request")
    print("\n## warp stall reasons (kernel, pc sampling)\n")
    st = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v)) for k, v in d.items()
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and v not in ("", "0")]
    tot_s = sum(v for _, v in st) or 1
    for k, v in sorted(st, key=lambda kv: -kv[1])[:12]:
        print(f"- {k}: {v:.0f} ({100 * v / tot_s:.1f}%)")
    print("\n## source lines with the most stall samples\n")
    tot_l = sum(line_stall.values()) or 1
    for key, v in line_stall.most_common(15):
        print(f"- {key[0]}:{key[1]} {100 * v / tot_l:.1f}%  `{line_text.get(key, '')}`")


if __name__ == "__main__":
    main()
