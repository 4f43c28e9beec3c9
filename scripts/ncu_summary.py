"""Summarise an ncu --set full report into the committed per-kernel CSV
(selected metrics) and the per-launch DRAM bytes bench.py reads.
python scripts/ncu_summary.py REPORT.ncu-rep OUT_CSV [TRAFFIC_JSON]"""
import csv
import io
import json
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
           "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           # north-star evidence: warp execution efficiency (active threads per
           # warp instruction, of 32), pipe utilisation, L1 hit rate, stalls
           "smsp__thread_inst_executed_per_inst_executed.ratio",
           "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
           "l1tex__t_sector_hit_rate.pct", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio"]
rep, out_csv = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
idx = {h: i for i, h in enumerate(hdr)}
with open(out_csv, "w", newline="") as fh:
    w = csv.writer(fh)
    w.writerow(["Kernel Name"] + METRICS)
    w.writerow([""] + [units[idx[m]] if m in idx else "" for m in METRICS])
    traffic = {}
    for r in rows[2:]:
        name = r[idx["Kernel Name"]]
        w.writerow([name] + [r[idx[m]] if m in idx else "" for m in METRICS])
        short = name.split("(")[0].split("<")[0].replace("void ", "").strip()
        try:
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            b = sum(float(r[idx[m]]) * mult.get(units[idx[m]], 1) for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        except (KeyError, ValueError):
            continue
        traffic.setdefault(short, int(b))
if len(sys.argv) > 3:
    json.dump({"source": f"{out_csv} (ncu --set full, rings 2x7.5M, min query; cold cache per replay)",
               "per_launch_dram_bytes": traffic}, open(sys.argv[3], "w"), indent=2)
print(json.dumps(traffic, indent=1))
