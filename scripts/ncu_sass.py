"""Per-SASS-instruction execution profile of one kernel from an ncu report.

python scripts/ncu_sass.py report.ncu-rep [--ranges a:b,c:d] [--top N]

Prints executed warp-instructions per launch, the hottest instructions, the
opcode mix weighted by execution count, and (--ranges, offsets in hex) the
share of address ranges, e.g. the sweep loop vs. the per-box body."""
import csv
import io
import re
import subprocess
import sys
from collections import Counter


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia, isrc, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
    ist = hdr.index("Warp Stall Sampling (All Samples)")
    ins = []
    base = None
    for r in rows[2:]:
        if len(r) <= iex or not r[ia].startswith("0x"):
            continue
        a = int(r[ia], 16)
        base = a if base is None else base
        ins.append((a - base, r[isrc].strip(), int(r[iex] or 0), int(r[ist] or 0)))
    return ins


def main():
    ins = load(sys.argv[1])
    total = sum(e for _, _, e, _ in ins)
    stalls = sum(s for _, _, _, s in ins)
    print(f"{len(ins)} static instructions, {total:.4e} executed warp-instructions, "
          f"{stalls} stall samples")
    ops = Counter()
    for _, src, e, _ in ins:
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", src)
        ops[m.group(2) if m else src] += e
    print("opcode mix (executed):")
    for op, e in ops.most_common(30):
        print(f"  {op:12s} {100 * e / total:5.1f}%")
    # loops: backward branches
    print("backward branches (loop ranges) by executed instructions inside:")
    loops = []
    for off, src, e, _ in ins:
        m = re.search(r"BRA.*?0x([0-9a-f]+)", src)
        if m:
            pass
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
    print(f"hottest {top}:")
    for off, src, e, s in sorted(ins, key=lambda x: -x[2])[:top]:
        print(f"  {off:#07x} {100 * e / total:5.2f}% st {100 * s / max(stalls, 1):5.2f}%  {src}")
    if "--ranges" in sys.argv:
        for rg in sys.argv[sys.argv.index("--ranges") + 1].split(","):
            a, b = (int(x, 16) for x in rg.split(":"))
            e = sum(x for off, _, x, _ in ins if a <= off <= b)
            s = sum(x for off, _, _, x in ins if a <= off <= b)
            print(f"range {a:#x}..{b:#x}: {100 * e / total:5.1f}% of instructions, "
                  f"{100 * s / max(stalls, 1):5.1f}% of stalls")
    if "--dump" in sys.argv:
        for off, src, e, s in ins:
            print(f"{off:#07x} {e:12d} {s:7d}  {src}")


main()
