"""Config 5 at its stated parameters (2048x1216x7000 RGB u8 = 17.4 G voxels,
S = 32, m = 10, 5 iterations, connectivity ON) through the public pipeline
sslic_segment on ONE B200: host image in, host labels out. The connectivity
pass runs on 2^32+ voxels (64-bit offsets, CCL slabs stitched across their
faces, connectivity.cu). Prints the phase timings (SSLIC_TIMING) and a few
size-independent checks of the output."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("SSLIC_TIMING", "1")
import torch  # noqa: E402

import paper_1806_08741_b200 as s  # noqa: E402
from bench import CONFIGS, SEED  # noqa: E402

dims, ch, dtype, grid, m, iters = CONFIGS[5]
n = int(np.prod(dims))
plane = dims[0] * dims[1]
host = np.empty(n * ch, np.uint8)
t0 = time.perf_counter()
step = 512
buf = torch.empty(step * plane * ch, dtype=torch.uint8, device="cuda")
for z0 in range(0, dims[2], step):
    z1 = min(dims[2], z0 + step)
    s.synth_generate(5, dims, dtype, ch, SEED, z0, z1, buf.data_ptr())
    host[z0 * plane * ch:z1 * plane * ch] = buf[: (z1 - z0) * plane * ch].cpu().numpy()
del buf
torch.cuda.empty_cache()
print(f"generated {n} voxels ({host.nbytes / 1e9:.1f} GB) in {time.perf_counter() - t0:.1f} s",
      flush=True)
p = s.SlicParams(grid=list(grid), weight_m=m, max_iterations=iters, enforce_connectivity=True)
t0 = time.perf_counter()
res, nxt = s.segment(s.NDImage(dims, ch, host), p)
t = time.perf_counter() - t0
print(f"config 5 segment (connectivity on): {t:.1f} s end to end, next label {nxt}, "
      f"residuals {['%.4g' % r for r in res.residuals]}", flush=True)
lab = res.labels
mx = int(lab.max())
print(f"max label {mx} < next label {nxt}: {mx < nxt}; labels >= k (fresh): "
      f"{int(np.count_nonzero(lab >= res.centers.count()))}")
