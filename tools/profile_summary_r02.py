"""Write profiles/<tag>_ncu_summary.md and profiles/ncu_summary.json from tools/profile_r02.sh outputs.

python tools/profile_summary_r02.py r02_v2 <gpurun_out dir> "<one-line description>"
"""
import csv
import io
import json
import os
import subprocess
import sys

tag, d, desc = sys.argv[1], sys.argv[2], sys.argv[3]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def raw(rep, kname):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    for row in r[2:]:
        dd = dict(zip(r[0], row))
        if kname in dd["Kernel Name"]:
            return dd
    return {}


plain = json.load(open(os.path.join(d, "plain.json")))
ef = plain["config"]["ef"]
ctr = plain["roofline"]["counters"]
hops_total = ctr["hops"] * 10000
launches = subprocess.run([sys.executable, os.path.join(root, "tools", "ncu_launches.py"), os.path.join(d, "launches.csv")],
                          capture_output=True, text=True).stdout.splitlines()
ours = [ln for ln in launches if any(k in ln for k in ("search_kernel", "seed_", "query_prep"))]
# shares among the search path's own kernels (the list also holds the bench's ground-truth GEMMs)
vals = []
for ln in ours:
    parts = ln.split()
    i = parts.index("launches")
    vals.append((" ".join(parts[:i]), int(parts[i + 1]), float(parts[i + 3])))
tot = sum(n * m for _, n, m in vals)
src_csv = "/tmp/_r02_src.csv"
open(src_csv, "w").write(subprocess.run(["ncu", "-i", os.path.join(d, "prof_search.ncu-rep"), "--page", "source", "--csv",
                                         "--print-source", "sass,cuda"], capture_output=True, text=True).stdout)
raw_csv = "/tmp/_r02_raw.csv"
open(raw_csv, "w").write(subprocess.run(["ncu", "-i", os.path.join(d, "prof_search.ncu-rep"), "--page", "raw", "--csv"],
                                        capture_output=True, text=True).stdout)
classes = subprocess.run([sys.executable, os.path.join(root, "tools", "ncu_classes.py"), src_csv, raw_csv, "10000"],
                         capture_output=True, text=True).stdout
opmix = subprocess.run([sys.executable, os.path.join(root, "tools", "ncu_opmix.py"), src_csv, str(hops_total)],
                       capture_output=True, text=True).stdout
s = raw(os.path.join(d, "prof_search.ncu-rep"), "search_kernel")
dram = (float(s["dram__bytes_read.sum"]) + float(s["dram__bytes_write.sum"])) * 1e6  # ncu reports MB
seed_rows = []
for kn in ("seed_tau_umma_kernel", "seed_select_reg_kernel"):
    k = raw(os.path.join(d, "prof_seed.ncu-rep"), kn)
    if k:
        seed_rows.append((kn, k))
with open(os.path.join(root, "profiles", f"{tag}_ncu_summary.md"), "w") as f:
    f.write(f"# {tag} ncu summary: C1, ef = R' = {ef} (recall@10 {plain['config']['recall_at_k']} over 40k queries, "
            f"per set {plain['config'].get('recall_at_k_per_set')}), 10k queries per launch\n\n{desc}\n\n")
    f.write("Algorithmic bytes of one search launch (bench.py counters, exact visited set): "
            f"hops {ctr['hops']:.2f}, n_trav {ctr['n_trav']:.1f}, R' {ctr['n_hp']:.0f} -> B_q = "
            f"{ctr['bytes_per_query']:.0f} B/query, {plain['roofline']['bytes_per_launch'] / 1e9:.3f} GB/launch.\n\n")
    f.write("## launch list (`bench.py --ef %d --steps 5 --warmup 3`, ncu --metrics gpu__time_duration.sum "
            "--clock-control none: cold-cache, serialised; the list also holds the bench's ground-truth GEMMs, "
            "left out here)\n```\n" % ef)
    for name, n, m in vals:
        f.write(f"{name[:58]:58s} launches {n:3d}  mean {m:9.1f} us  share of the path {100 * n * m / tot:5.1f}%\n")
    f.write("```\n(the timed steps launch the `<..., 1>` search variant; `<..., 0>`/`<..., 2>` are the bench's "
            "traced counter runs)\n\n")
    f.write("## search_kernel: ncu --set full --clock-control none --import-source on "
            f"(tools/stage_times.py {ef}, one launch after warm-up)\n\n")
    f.write(f"DRAM traffic per launch (`dram__bytes_read.sum + dram__bytes_write.sum`): {dram / 1e6:.1f} MB "
            f"= {dram / plain['roofline']['bytes_per_launch']:.2f} x the algorithmic bytes (L1 + L2 serve the rest).\n\n")
    f.write(classes + "\n")
    f.write("## executed SASS by opcode (per hop)\n```\n" + opmix + "```\n\n")
    if seed_rows:
        f.write("## seed phase kernels (ncu --set full, same command)\n\n| kernel | us | inst (M) | issue active % "
                "| warps active % | regs | DRAM MB r/w |\n|---|---|---|---|---|---|---|\n")
        for kn, k in seed_rows:
            f.write(f"| {kn} | {float(k['gpu__time_duration.sum']):.1f} | {float(k['smsp__inst_executed.sum']) / 1e6:.1f} | "
                    f"{float(k['smsp__issue_active.avg.pct_of_peak_sustained_active']):.1f} | "
                    f"{float(k['sm__warps_active.avg.pct_of_peak_sustained_active']):.1f} | {k['launch__registers_per_thread']} | "
                    f"{float(k['dram__bytes_read.sum']):.1f} / {float(k['dram__bytes_write.sum']):.1f} |\n")
json.dump({"source": f"profiles/{tag}_ncu_summary.md (ncu --set full, search_kernel, C1 ef={ef})", "ef": ef,
           "search_kernel_dram_bytes_per_launch": int(dram)},
          open(os.path.join(root, "profiles", "ncu_summary.json"), "w"), indent=1)
print(open(os.path.join(root, "profiles", f"{tag}_ncu_summary.md")).read())
