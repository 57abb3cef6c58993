"""Time connectivity enforcement on a BASELINE config volume: our
sslic_segment (GPU CCL + finalize, host sweep; SSLIC_TIMING=1 prints the
phase split) and, on a z-subvolume, the reference's enforce_connectivity."""
import argparse, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("SSLIC_TIMING", "1")
import torch
import paper_1806_08741_b200 as s
from bench import CONFIGS  # noqa

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--ref-planes", type=int, default=0)
a = ap.parse_args()
dims, ch, dtype, grid, m, iters = CONFIGS[a.config]
n = int(np.prod(dims))
tdt = {np.uint8: torch.uint8, np.uint16: torch.int16, np.float32: torch.float32}[dtype]
buf = torch.empty(n * ch, dtype=tdt, device="cuda")
s.synth_generate(a.config, dims, dtype, ch, 1234, 0, dims[-1] if len(dims) == 3 else 1, buf.data_ptr())
host = buf.cpu().numpy().view(dtype)
del buf
img = s.NDImage(dims, ch, host)
p = s.SlicParams(grid=list(grid), weight_m=m, max_iterations=iters, enforce_connectivity=True)
t0 = time.perf_counter()
res, nxt = s.segment(img, p)
t1 = time.perf_counter()
print(f"config {a.config}: segment (with connectivity) {t1 - t0:.3f} s, next label {nxt}")
p0 = s.SlicParams(grid=list(grid), weight_m=m, max_iterations=iters)
t0 = time.perf_counter()
r0 = s.run_slic(img, p0)
t1 = time.perf_counter()
print(f"config {a.config}: run_slic alone {t1 - t0:.3f} s")
t0 = time.perf_counter()
out = s.enforce_connectivity(r0.labels, dims, r0.centers, p0)
t1 = time.perf_counter()
print(f"config {a.config}: enforce_connectivity {t1 - t0:.3f} s over {n} voxels "
      f"({n / (t1 - t0) / 1e6:.1f} Mvox/s)")
if a.ref_planes:
    import oracle
    ref = oracle.Reference()
    sd = list(dims[:-1]) + [a.ref_planes]
    ns = int(np.prod(sd))
    lab = np.ascontiguousarray(r0.labels.reshape(-1)[:ns])
    t0 = time.perf_counter()
    ro = ref.enforce_connectivity(sd, lab, r0.centers.data, ch, grid, workers=os.cpu_count())
    t1 = time.perf_counter()
    print(f"reference enforce_connectivity on {sd}: {t1 - t0:.3f} s ({ns / (t1 - t0) / 1e6:.1f} Mvox/s)")
