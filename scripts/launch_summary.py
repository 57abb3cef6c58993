"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum
--csv), from the last launch whose name contains START on.
python scripts/launch_summary.py gpurun_out/cc_launches.csv [START]"""
import collections
import csv
import sys

path = sys.argv[1]
start_name = sys.argv[2] if len(sys.argv) > 2 else None
lines = [l for l in open(path) if not l.startswith("==")]
seq = []
for row in csv.DictReader(lines):
    v = float(row["Metric Value"].replace(",", ""))
    u = row["Metric Unit"]
    ms = v / 1e6 if u.startswith("n") else (v / 1e3 if u.startswith("u") else v)
    seq.append((row["Kernel Name"].split("(")[0][-48:], ms))
start = 0
if start_name:
    start = [i for i, (n, _) in enumerate(seq) if start_name in n][-1]
agg = collections.OrderedDict()
tot = 0.0
for n, ms in seq[start:]:
    a = agg.setdefault(n, [0, 0.0])
    a[0] += 1
    a[1] += ms
    tot += ms
for n, (c, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{ms:9.2f} ms  x{c:3d}  {n}")
print(f"{tot:9.2f} ms  total")
