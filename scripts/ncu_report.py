"""Headline summary of one `ncu --set full` capture of the K2 assign kernel:
launch config, duration, issue/occupancy, pipe utilisation, stall reasons,
DRAM traffic, and the per-section instruction/stall shares (source markers
`// ---- name ----` in kernels_fast_main.cuh). Usage: ncu_report.py REPORT"""
import csv, io, json, subprocess, sys

rep = sys.argv[1]


def ncu(args):
    return subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout


rows = list(csv.reader(io.StringIO(ncu(["--page", "raw", "--csv"]))))
h, u, v = rows[0], rows[1], rows[2]
raw = {k: (u[i], v[i]) for i, k in enumerate(h)}
print("kernel:", raw.get("Kernel Name", ("", "?"))[1])
print("grid x block:", raw.get("Grid Size", ("", "?"))[1], "x", raw.get("Block Size", ("", "?"))[1])
keys = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
for k in keys:
    if k in raw:
        print(f"  {k:58s} {raw[k][1]:>16s} {raw[k][0]}")
print("stall reasons (warp-cycles per issued instruction):")
st = []
for k, (unit, val) in raw.items():
    if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
        try:
            st.append((float(val), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        except ValueError:
            pass
for val, name in sorted(st, reverse=True)[:10]:
    print(f"  {name:28s} {val:6.3f}")
