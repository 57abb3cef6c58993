"""run_slic / segment through the public API with ordinary (pageable) numpy
buffers -- what a caller of the reference holds (std::vector storage) -- on a
BASELINE config: seconds per call, to compare with the pinned-buffer e2e of
bench.py. usage: python scripts/pageable_e2e.py [config] [calls] [f64]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("SSLIC_TIMING", "1")
import torch  # noqa: E402

import paper_1806_08741_b200 as s  # noqa: E402
from bench import CONFIGS, SEED  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 3
as_f64 = len(sys.argv) > 3 and sys.argv[3] == "f64"  # the reference's storage: doubles
dims, ch, dtype, grid, m, iters = CONFIGS[cfg]
n = int(np.prod(dims))
tdt = {np.uint8: torch.uint8, np.uint16: torch.int16, np.float32: torch.float32}[dtype]
dev = torch.empty(n * ch, dtype=tdt, device="cuda")
s.synth_generate(cfg, dims, dtype, ch, SEED, 0, dims[-1] if len(dims) == 3 else 1, dev.data_ptr())
host = dev.cpu().numpy().view(dtype).copy()  # pageable
if as_f64:
    host = host.astype(np.float64)
del dev
torch.cuda.empty_cache()
p = s.SlicParams(grid=list(grid), weight_m=m, max_iterations=iters)
img = s.NDImage(dims, ch, host)
for i in range(calls):
    t0 = time.perf_counter()
    res = s.run_slic(img, p)
    t = time.perf_counter() - t0
    print(f"config {cfg} run_slic, pageable {'fp64' if as_f64 else 'native'} buffers, call {i}: {t:.3f} s "
          f"({n * iters / t / 1e9:.2f} G voxel-iterations/s), residual[-1] {res.residuals[-1]:.6g}",
          flush=True)
