"""Time connectivity enforcement (enforce_connectivity, connectivity.hpp:265-273)
on a BASELINE config volume: ours (GPU CCL + finalize + component-graph
fixpoint; SSLIC_TIMING=1 prints the device phase and the component count)
against the reference's multi-threaded enforce_connectivity on the same
label map, with the outputs compared bitwise.

python scripts/conn_time.py --config 3 [--planes Z0 Z1] [--no-ref]"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("SSLIC_TIMING", "1")
import torch  # noqa: E402

import paper_1806_08741_b200 as s  # noqa: E402
from bench import CONFIGS, SEED  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--planes", type=int, nargs=2, default=None)
ap.add_argument("--no-ref", action="store_true")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
dims, ch, dtype, grid, m, iters = CONFIGS[a.config]
z0, z1 = a.planes if a.planes else (0, dims[-1] if len(dims) == 3 else 1)
idims = tuple(dims[:-1]) + (z1 - z0,) if len(dims) == 3 else dims
n = int(np.prod(idims))
tdt = {np.uint8: torch.uint8, np.uint16: torch.int16, np.float32: torch.float32}[dtype]
buf = torch.empty(n * ch, dtype=tdt, device="cuda")
s.synth_generate(a.config, dims, dtype, ch, SEED, z0, z1, buf.data_ptr())
host = buf.cpu().numpy().view(dtype)
del buf
img = s.NDImage(idims, ch, host)
p = s.SlicParams(grid=list(grid), weight_m=m, max_iterations=iters, enforce_connectivity=False)
r0 = s.run_slic(img, p)
print(f"config {a.config} {'x'.join(map(str, idims))}: run_slic done", flush=True)
times = []
for _ in range(a.reps):
    t0 = time.perf_counter()
    out = s.enforce_connectivity(r0.labels, idims, r0.centers, p)
    times.append(time.perf_counter() - t0)
t = min(times)
print(f"ours: enforce_connectivity {t:.3f} s (host buffers, min of {a.reps}) over {n} voxels "
      f"({n / t / 1e6:.1f} Mvox/s)", flush=True)
if not a.no_ref:
    import oracle
    ref = oracle.Reference()
    t0 = time.perf_counter()
    ro = ref.enforce_connectivity(idims, r0.labels, r0.centers.data, ch, grid,
                                  workers=os.cpu_count())
    t1 = time.perf_counter()
    print(f"reference: enforce_connectivity {t1 - t0:.3f} s with {os.cpu_count()} threads "
          f"({n / (t1 - t0) / 1e6:.1f} Mvox/s); bitwise equal: {np.array_equal(out, ro)}")
