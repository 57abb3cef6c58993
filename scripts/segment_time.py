"""Whole pipeline, host image in -> host labels out, connectivity ON
(tools/sslic.cpp's segment: run_slic + enforce_connectivity): sslic_segment on
one B200 against the reference's run_slic + enforce_connectivity on the host
cores, outputs compared bitwise.

python scripts/segment_time.py --config 1 [--no-ref] [--reps N]"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1806_08741_b200 as s  # noqa: E402
from bench import CONFIGS, SEED  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--no-ref", action="store_true")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
dims, ch, dtype, grid, m, iters = CONFIGS[a.config]
n = int(np.prod(dims))
tdt = {np.uint8: torch.uint8, np.uint16: torch.int16, np.float32: torch.float32}[dtype]
buf = torch.empty(n * ch, dtype=tdt, device="cuda")
z1 = dims[-1] if len(dims) == 3 else 1
s.synth_generate(a.config, dims, dtype, ch, SEED, 0, z1, buf.data_ptr())
host = buf.cpu().numpy().view(dtype)
del buf
img = s.NDImage(dims, ch, host)
p = s.SlicParams(grid=list(grid), weight_m=m, max_iterations=iters, enforce_connectivity=True)
times = []
for _ in range(a.reps + 1):
    t0 = time.perf_counter()
    res, nxt = s.segment(img, p)
    times.append(time.perf_counter() - t0)
t = min(times[1:])
print(f"config {a.config} {'x'.join(map(str, dims))}: sslic_segment {t * 1e3:.2f} ms per call "
      f"(pageable host buffers, min of {a.reps} after a warm-up call), next label {nxt}", flush=True)
if not a.no_ref:
    import oracle
    ref = oracle.Reference()
    w = os.cpu_count()
    t0 = time.perf_counter()
    rl, rc, rr = ref.run_slic(host, dims, ch, grid, weight_m=m, max_iterations=iters, workers=w)[:3]
    t1 = time.perf_counter()
    ro = ref.enforce_connectivity(dims, rl, rc, ch, grid, workers=w)
    t2 = time.perf_counter()
    print(f"reference ({w} threads): run_slic {(t1 - t0) * 1e3:.1f} ms + enforce_connectivity "
          f"{(t2 - t1) * 1e3:.1f} ms = {(t2 - t0) * 1e3:.1f} ms; labels bitwise equal: "
          f"{np.array_equal(res.labels, ro)}; ratio {(t2 - t0) / t:.0f}x")
