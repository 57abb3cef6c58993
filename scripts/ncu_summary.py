"""Summarise an ncu report: headline metrics + per-source-line instruction and
stall shares (needs -lineinfo builds and --import-source on)."""
import csv, io, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
def run(args):
    return subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout

raw = list(csv.reader(io.StringIO(run(["--page", "raw", "--csv"]))))
if len(raw) > 2:
    h, v = raw[0], raw[2]
    print("kernel:", v[h.index("Kernel Name")] if "Kernel Name" in h else "?")
    for w in ["gpu__time_duration.sum", "smsp__inst_executed.sum", "launch__registers_per_thread",
              "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
              "launch__shared_mem_per_block_dynamic",
              "sm__warps_active.avg.pct_of_peak_sustained_active",
              "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
              "dram__bytes_read.sum", "dram__bytes_write.sum"]:
        if w in h:
            print(f"  {w:58s} {v[h.index(w)]} {raw[1][h.index(w)]}")
    print("stall reasons (warp-cycles per issued instruction):")
    st = []
    for i, name in enumerate(h):
        if name.startswith("smsp__average_warps_issue_stalled_") and name.endswith(
                "_per_issue_active.ratio"):
            try:
                st.append((float(v[i]), name[len("smsp__average_warps_issue_stalled_"):
                                             -len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    for val, name in sorted(st, reverse=True)[:10]:
        print(f"  {name:28s} {val:.3f}")
det = run(["--page", "details", "--csv"])
keys = ["Duration", "Executed Ipc Active", "Issue Slots Busy", "Warp Cycles Per Issued Instruction",
        "No Eligible", "Registers Per Thread", "Achieved Occupancy", "DRAM Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Dynamic Shared Memory Per Block", "Memory Throughput"]
for row in csv.reader(io.StringIO(det)):
    if len(row) > 3 and row[-3] in keys:
        print(f"{row[-3]:40s} {row[-1]:>14s} {row[-2]}")
src = run(["--page", "source", "--csv", "--print-source=cuda,sass"])
rows = list(csv.reader(io.StringIO(src)))
hdr = next((r for r in rows if "Instructions Executed" in r), None)
if hdr is None:
    sys.exit(0)
ie = hdr.index("Instructions Executed"); ss = hdr.index("Warp Stall Sampling (All Samples)")
agg = defaultdict(lambda: [0, 0, ""])
cur_file, cur = "?", "?"
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] and r[0].isdigit():
        cur = f"{cur_file}:{r[0]}"
        agg[cur][2] = r[1].strip()[:80]
        continue
    if len(r) > ss and r[2].startswith("0x"):
        agg[cur][0] += int(r[ie] or 0)
        agg[cur][1] += int(r[ss] or 0)
tot = sum(v[0] for v in agg.values()) or 1; st = sum(v[1] for v in agg.values()) or 1
print("total warp instrs %.4g, stall samples %d" % (tot, st))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:n]:
    print(f"{k:>28s} instr {100*v[0]/tot:5.1f}% stall {100*v[1]/st:5.1f}%  {v[2]}")
