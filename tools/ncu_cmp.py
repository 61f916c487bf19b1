"""Compare key metrics of several ncu reports: python tools/ncu_cmp.py a.ncu-rep b.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__maximum_warps_per_active_cycle_pct", "lts__t_sector_hit_rate.pct", "dram__bytes_read.sum",
        "smsp__warps_eligible.avg.per_cycle_active", "smsp__average_warp_latency_per_inst_issued.ratio",
        "local_load", "local_store"]
STALL = "smsp__pcsamp_warps_issue_stalled_"


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return dict(zip(r[0], r[2]))


reps = [load(p) for p in sys.argv[1:]]
names = sorted(set().union(*reps))
for n in names:
    if any(k in n for k in KEYS) or (n.startswith(STALL) and not n.endswith("not_issued")):
        print(f"{n:70s} " + " ".join(f"{r.get(n, ''):>16s}" for r in reps))
