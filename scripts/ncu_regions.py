import subprocess, csv, io, sys, re
from collections import defaultdict
rep = sys.argv[1]
src = subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source=cuda,sass"],capture_output=True,text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = next(r for r in rows if "Instructions Executed" in r)
ie = hdr.index("Instructions Executed"); ss = hdr.index("Warp Stall Sampling (All Samples)")
agg = defaultdict(lambda: [0, 0, ""]); cur_file = "?"; cur = ("?", 0)
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur_file = r[1].split("/")[-1]; continue
    if r[0] and r[0].isdigit(): cur = (cur_file, int(r[0])); agg[cur][2] = r[1].strip()[:70]; continue
    if len(r) > ss and r[2].startswith("0x"):
        agg[cur][0] += int(r[ie] or 0); agg[cur][1] += int(r[ss] or 0)
tot = sum(v[0] for v in agg.values()); st = sum(v[1] for v in agg.values())
# map source markers in kernels_fast_main.cuh to regions by scanning the file for tags
lines = open("paper_1806_08741_b200/csrc/kernels_fast_main.cuh").read().splitlines()
marks = []
for i, l in enumerate(lines, 1):
    m = re.search(r"// ---- (.*?) ----", l)
    if m: marks.append((i, m.group(1)[:40]))
def region(ln):
    name = "prologue"
    for i, nm in marks:
        if ln >= i: name = nm
    return name
reg = defaultdict(lambda: [0, 0])
for (f, ln), v in agg.items():
    key = region(ln) if f == "kernels_fast_main.cuh" else "(inlined helpers: " + f + ")"
    reg[key][0] += v[0]; reg[key][1] += v[1]
print(f"total warp instrs {tot:.4g}, stall samples {st}")
for k, v in sorted(reg.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:45s} instr {100*v[0]/tot:5.1f}%  stall {100*v[1]/st:5.1f}%")
