"""Write profiles/<tag>_ncu_summary.md (+ launches csv, bench json) from tools/profile_round.sh outputs.
python tools/profile_summary.py r01_v20 "<one-line kernel description>" """
import csv
import io
import json
import shutil
import subprocess
import sys

tag, desc = sys.argv[1], sys.argv[2]
rep = "gpurun_out/prof_new.ncu-rep"
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
d = dict(zip(r[0], r[2]))
keys = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__maximum_warps_per_active_cycle_pct",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "lts__t_sector_hit_rate.pct",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__warps_eligible.avg.per_cycle_active",
        "smsp__average_warp_latency_per_inst_issued.ratio", "sass__inst_executed_local_loads",
        "sass__inst_executed_local_stores"]
stalls = [k for k in d if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
          and d[k] not in ("0", "")]
launches = subprocess.run(["python", "tools/ncu_launches.py", "gpurun_out/launches.csv"], capture_output=True,
                          text=True).stdout
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"], capture_output=True,
                     text=True).stdout
open("/tmp/_src.csv", "w").write(src)
bench = json.load(open("gpurun_out/bench.json"))
hops = bench["roofline"]["counters"]["hops"] * 10000
opmix = subprocess.run(["python", "tools/ncu_opmix.py", "/tmp/_src.csv", str(hops)], capture_output=True, text=True).stdout
lines = subprocess.run(["python", "tools/ncu_lines.py", "/tmp/_src.csv", str(hops), "3.0"], capture_output=True,
                       text=True).stdout
dram = (float(d["dram__bytes_read.sum"]) + float(d["dram__bytes_write.sum"])) * 1e6  # ncu reports MB
with open(f"profiles/{tag}_ncu_summary.md", "w") as f:
    f.write(f"# {tag} ncu summary: C1, ef={bench['config']['ef']} (recall@10 {bench['config']['recall_at_k']}), "
            f"10k queries\n\n{desc}\n\n")
    f.write("## launch list (bench.py --ef <timed> --steps 5 --warmup 3; ncu --metrics gpu__time_duration.sum "
            "--clock-control none; cold-cache, serialised)\n```\n" + launches + "```\n\n")
    f.write("## search_kernel, ncu --set full --clock-control none --import-source on (tools/ab.sh: "
            "sweep_launch.py, first timed launch after 3 warm-ups)\n```\n")
    for k in keys:
        f.write(f"{k:60s} {d.get(k, '')}\n")
    for k in stalls:
        f.write(f"{k:60s} {d[k]}\n")
    f.write("```\n\n## executed SASS by opcode (per hop)\n```\n" + opmix + "```\n\n")
    f.write("## per-line executed instructions / hop (lines >= 3 / hop)\n```\n" + lines + "```\n")
shutil.copy("gpurun_out/launches.csv", f"profiles/{tag}_launches.csv")
shutil.copy("gpurun_out/bench.json", f"profiles/{tag.replace('_v', '_bench_v')}.json")
json.dump({"source": f"profiles/{tag}_ncu_summary.md (ncu --set full, search_kernel, C1 ef={bench['config']['ef']})",
           "search_kernel_dram_bytes_per_launch": int(dram)}, open("profiles/ncu_summary.json", "w"), indent=1)
print("dram bytes per launch", int(dram))
