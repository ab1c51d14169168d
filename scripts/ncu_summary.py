"""Summarise an ncu --set full capture of one sweep launch for profiles/ (dev tool).

    python scripts/ncu_summary.py REPORT.ncu-rep ALG_BYTES "description" > profiles/<name>.txt

ALG_BYTES = algorithmic bytes of that launch (DESIGN.md §4 per-unit figures x the units
of the launch); prints the raw metrics the roofline uses, the stall breakdown and the
hottest source lines, and writes nothing else."""
import csv
import subprocess
import sys

rep, alg, desc = sys.argv[1], float(sys.argv[2]), sys.argv[3]
raw = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                     text=True).stdout.splitlines()))
h, units, v = raw[0], raw[1], raw[2]
get = lambda k: v[h.index(k)]
print(desc)
print("kernel:", get("Kernel Name")[:110])
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct"]
for k in keys:
    print(f"{k:60s} {get(k):>16s} {units[h.index(k)]}")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rd = float(get("dram__bytes_read.sum")) * scale[units[h.index("dram__bytes_read.sum")]]
wr = float(get("dram__bytes_write.sum")) * scale[units[h.index("dram__bytes_write.sum")]]
us = float(get("gpu__time_duration.sum")) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[units[h.index("gpu__time_duration.sum")]]
print(f"dram traffic per launch: {(rd + wr) / 1e6:.1f} MB; algorithmic bytes per launch: {alg / 1e6:.1f} MB; "
      f"traffic/algorithmic = {(rd + wr) / alg:.3f}")
print(f"dram GB/s under ncu (cold L2, serialised): {(rd + wr) / (us * 1e-6) / 1e9:.0f}; "
      f"algorithmic GB/s: {alg / (us * 1e-6) / 1e9:.0f}")
print("stall reasons (warps per issue):")
st = [(float(v[i]), n) for i, n in enumerate(h)
      if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio")]
for val, n in sorted(st, reverse=True)[:10]:
    print(f"  {n.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):24s} {val:.2f}")
