"""Per-source-line instruction and stall-sample shares of an ncu report,
sorted by instructions (needs -lineinfo and --import-source on)."""
import csv, io, subprocess, sys
from collections import defaultdict
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 60
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = next(r for r in rows if "Instructions Executed" in r)
ie = hdr.index("Instructions Executed"); ss = hdr.index("Warp Stall Sampling (All Samples)")
agg = defaultdict(lambda: [0, 0, ""]); cur_file = "?"; cur = ("?", 0)
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur_file = r[1].split("/")[-1]; continue
    if r[0] and r[0].isdigit(): cur = (cur_file, int(r[0])); agg[cur][2] = r[1].strip()[:80]; continue
    if len(r) > ss and r[2].startswith("0x"):
        agg[cur][0] += int(r[ie] or 0); agg[cur][1] += int(r[ss] or 0)
tot = sum(v[0] for v in agg.values()); st = sum(v[1] for v in agg.values())
for (f, ln), v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{f[:22]:>22s}:{ln:<5d} instr {100*v[0]/tot:5.2f}%  stall {100*v[1]/st:5.2f}%  {v[2]}")
