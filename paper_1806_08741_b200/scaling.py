"""Strong-scaling report over GPU counts: the reference's
analysis (bench.hpp:41-262) restated — relative speedup S(p) = T(1)/T(p),
efficiency E(p) = S(p)/p, the Amdahl bounds, the least-squares serial
fraction fit, and the CSV / markdown emitters — applied to bench.py lines
measured at 1/2/4/8 GPUs (one process per GPU) instead of CPU worker counts.

    python -m paper_1806_08741_b200.scaling --gpus 1 2 4 8 --config 3

runs bench.py under torch.distributed.run once per GPU count (each a fresh
job), takes T(p) = ms_per_step (the iteration) and, with --e2e, the end-to-end
seconds, and prints the markdown table; --csv writes the CSV.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
from dataclasses import dataclass, field
from typing import List, Optional


@dataclass
class TimingRecord:
    workers: int
    time_seconds: float
    with_connectivity: bool = False


@dataclass
class ScalingReport:
    records: List[TimingRecord] = field(default_factory=list)
    speedups: List[float] = field(default_factory=list)
    efficiencies: List[float] = field(default_factory=list)
    alpha: float = 0.0


def relative_speedup(t1: float, tp: float) -> float:
    """bench.hpp:43-47"""
    if not (t1 > 0.0) or not (tp > 0.0):
        raise ValueError("relative_speedup: times must be positive")
    return t1 / tp


def relative_efficiency(speedup: float, p: int) -> float:
    """bench.hpp:49-52"""
    if p < 1:
        raise ValueError("relative_efficiency: p must be >= 1")
    return speedup / float(p)


def amdahl_bound(alpha: float, p: int) -> float:
    """bench.hpp:55-60: 1 / (alpha + (1 - alpha) / p)"""
    if alpha < 0.0 or alpha > 1.0 or p < 1:
        raise ValueError("amdahl_bound: alpha outside [0,1] or p < 1")
    return 1.0 / (alpha + (1.0 - alpha) / float(p))


def amdahl_efficiency_bound(alpha: float, p: int) -> float:
    """bench.hpp:63-68: 1 / (1 + alpha (p - 1))"""
    if alpha < 0.0 or alpha > 1.0 or p < 1:
        raise ValueError("amdahl_efficiency_bound: alpha outside [0,1] or p < 1")
    return 1.0 / (1.0 + alpha * float(p - 1))


def fit_alpha(records: List[TimingRecord]) -> float:
    """bench.hpp:74-97: least squares of y = alpha x with x = 1 - 1/p and
    y = T(p)/T(1) - 1/p, accumulated in record order, clamped to [0, 1]."""
    t1 = 0.0
    for r in records:
        if r.workers == 1:
            t1 = r.time_seconds
    if not (t1 > 0.0):
        raise ValueError("fit_alpha: need a record with p = 1")
    sxx = sxy = 0.0
    above = 0
    for r in records:
        if r.workers < 1 or not (r.time_seconds > 0.0):
            raise ValueError("fit_alpha: invalid record")
        inv_p = 1.0 / float(r.workers)
        x = 1.0 - inv_p
        y = r.time_seconds / t1 - inv_p
        sxx += x * x
        sxy += x * y
        above += r.workers > 1
    if above == 0:
        raise ValueError("fit_alpha: need at least two distinct worker counts")
    return min(max(sxy / sxx, 0.0), 1.0)


def make_report(records: List[TimingRecord]) -> ScalingReport:
    """bench.hpp:103-125: per-series speedups/efficiencies (baseline p = 1 of
    the same series), alpha fitted on the without-connectivity series."""
    rep = ScalingReport(records=list(records))
    t1 = [0.0, 0.0]
    for r in rep.records:
        if r.workers == 1:
            t1[1 if r.with_connectivity else 0] = r.time_seconds
    for r in rep.records:
        sp = relative_speedup(t1[1 if r.with_connectivity else 0], r.time_seconds)
        rep.speedups.append(sp)
        rep.efficiencies.append(relative_efficiency(sp, r.workers))
    primary = [r for r in rep.records if not r.with_connectivity] or list(rep.records)
    rep.alpha = fit_alpha(primary) if any(r.workers > 1 for r in primary) else 1.0
    return rep


def _g17(x: float) -> str:
    return format(x, ".17g")  # ostream precision(17), default float format


def emit_scaling_csv(rep: ScalingReport) -> str:
    """bench.hpp:169-181"""
    out = ["p,time_s,speedup,efficiency,connectivity\n"]
    for r, s, e in zip(rep.records, rep.speedups, rep.efficiencies):
        out.append(f"{r.workers},{_g17(r.time_seconds)},{_g17(s)},{_g17(e)},"
                   f"{1 if r.with_connectivity else 0}\n")
    out.append(f"# alpha,{_g17(rep.alpha)}\n")
    return "".join(out)


def parse_scaling_csv(text: str) -> ScalingReport:
    """bench.hpp:189-213"""
    lines = text.split("\n")
    if not lines or lines[0] != "p,time_s,speedup,efficiency,connectivity":
        raise ValueError("parse_scaling_csv: missing header row")
    rep = ScalingReport()
    for line in lines[1:]:
        if not line:
            continue
        if line.startswith("# alpha,"):
            rep.alpha = float(line[8:])
            continue
        f = line.split(",")
        if len(f) != 5:
            raise ValueError("parse_scaling_csv: malformed row: " + line)
        rep.records.append(TimingRecord(int(f[0]), float(f[1]), int(f[4]) != 0))
        rep.speedups.append(float(f[2]))
        rep.efficiencies.append(float(f[3]))
    return rep


def emit_scaling_markdown(rep: ScalingReport, unit: str = "GPUs") -> str:
    """bench.hpp:222-262 (fixed, 6 decimals); the first column is the GPU
    count here (the reference's 'Threads')."""
    both = any(r.with_connectivity for r in rep.records) and \
        any(not r.with_connectivity for r in rep.records)
    col = "Threads" if unit == "Threads" else unit
    out = []
    if both:
        out.append(f"| {col} | Time (sec) | Efficiency | Speedup | Time (sec) | Efficiency | Speedup |\n")
        out.append("|---|---|---|---|---|---|---|\n")
        out.append("| | Without Connectivity | | | With Connectivity | | |\n")
        for p in [r.workers for r in rep.records if not r.with_connectivity]:
            row = f"| {p} |"
            for conn in (False, True):
                for r, s, e in zip(rep.records, rep.speedups, rep.efficiencies):
                    if r.workers == p and r.with_connectivity == conn:
                        row += f" {r.time_seconds:.6f} | {e:.6f} | {s:.6f} |"
                        break
            out.append(row + "\n")
    else:
        out.append(f"| {col} | Time (sec) | Efficiency | Speedup |\n")
        out.append("|---|---|---|---|\n")
        for r, s, e in zip(rep.records, rep.speedups, rep.efficiencies):
            out.append(f"| {r.workers} | {r.time_seconds:.6f} | {e:.6f} | {s:.6f} |\n")
    out.append(f"\nSerial fraction (Amdahl fit): alpha = {rep.alpha:.6f}\n")
    return "".join(out)


def measure(gpus: List[int], config: int, steps: int, warmup: int, e2e: bool,
            port: int = 29611) -> List[TimingRecord]:
    """One bench.py job per GPU count (torch.distributed.run, one process per
    GPU); T(p) is the step time or, with e2e, the end-to-end call time."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    recs = []
    for i, p in enumerate(gpus):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={p}", "--master-addr", "127.0.0.1",
               f"--master-port={port + i}", os.path.join(root, "bench.py"), "--gpus", str(p),
               "--config", str(config), "--steps", str(steps), "--warmup", str(warmup),
               "--no-cpu"] + ([] if e2e else ["--no-e2e"])
        out = subprocess.run(cmd, capture_output=True, text=True, check=True).stdout
        line = json.loads([l for l in out.splitlines() if l.startswith("{")][-1])
        t = line["e2e"]["seconds_per_call"] if e2e else line["ms_per_step"] / 1e3
        recs.append(TimingRecord(p, float(t)))
    return recs


def main(argv: Optional[List[str]] = None) -> None:
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--steps", type=int, default=7)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--e2e", action="store_true")
    ap.add_argument("--csv")
    a = ap.parse_args(argv)
    if 1 not in a.gpus:
        raise SystemExit("the GPU list must contain 1 (the baseline of the relative metrics)")
    rep = make_report(measure(a.gpus, a.config, a.steps, a.warmup, a.e2e))
    if a.csv:
        with open(a.csv, "w") as f:
            f.write(emit_scaling_csv(rep))
    print(emit_scaling_markdown(rep))


if __name__ == "__main__":
    main()
