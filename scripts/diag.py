"""Per-iteration diagnostics of the assign kernel on a BASELINE config:
device time, label changes, fp64 re-decisions, evaluations per voxel."""
import argparse, sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1806_08741_b200 as s
from bench import CONFIGS, SEED

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--exact", action="store_true")
a = ap.parse_args()
dims, ch, dtype, grid, m, _ = CONFIGS[a.config]
n = int(np.prod(dims))
tdt = {np.uint8: torch.uint8, np.uint16: torch.int16, np.float32: torch.float32}[dtype]
img = torch.empty(n * ch, dtype=tdt, device="cuda")
s.synth_generate(a.config, dims, dtype, ch, SEED, 0, dims[-1] if len(dims) == 3 else 1, img.data_ptr())
e = s.Engine(dims, ch, dtype, img.data_ptr(), s.SlicParams(grid=list(grid), weight_m=m, max_iterations=a.iters))
if a.exact:
    e.set_exact(True)
e.init(); e.commit(); e.set_stats(True)
for it in range(a.iters):
    e.assign()
    amb, crowd, chg = e.fast_stats()
    ev, win = e.eval_stats()
    e.update()
    torch.cuda.synchronize()
    print(f"iter {it}: assign {e.assign_ms(it):8.3f} ms  changed {chg/n:7.4f}  redecided {amb/n:.2e}  "
          f"evals/vox {ev/n:5.2f}  window/vox {win/n:5.2f}  crowded {crowd:.0f}")
print("residuals", ["%.4g" % r for r in e.residuals()])
