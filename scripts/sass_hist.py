"""SASS opcode histogram and loop map of one kernel (cuobjdump -sass text).

python scripts/sass_hist.py <file.sass> [--loops]
Static counts; --loops lists backward branches (target..source ranges) with
their static size, to locate the sweep loop and the per-box body."""
import re
import sys
from collections import Counter

LINE = re.compile(r"^\s+/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?\s*(.*?);")


def parse(path):
    ins = []
    for ln in open(path):
        m = LINE.match(ln)
        if m:
            ins.append((int(m.group(1), 16), m.group(3), (m.group(4) or ""), m.group(5)))
    return ins


def main():
    ins = parse(sys.argv[1])
    c = Counter(op for _, op, _, _ in ins)
    print(f"{len(ins)} instructions")
    for op, n in c.most_common(45):
        print(f"{n:6d} {op}")
    if "--loops" in sys.argv:
        for addr, op, _, rest in ins:
            if op == "BRA":
                m = re.search(r"0x([0-9a-f]+)", rest)
                if m and int(m.group(1), 16) < addr:
                    t = int(m.group(1), 16)
                    body = [o for a, o, _, _ in ins if t <= a <= addr]
                    print(f"loop {t:#x}..{addr:#x}: {len(body)} instrs")


main()
