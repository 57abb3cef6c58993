"""Assign-kernel time on fp64 images: the fast path (f32 working copy) vs
the exact fp64 kernel, config-4-like and config-2-like (Lab ranges)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1806_08741_b200 as s

for name, dims, ch, grid, m, cfg in (("config4 f64", (512, 512, 256), 4, (8, 8, 8), 20.0, 4),
                                     ("config2 Lab f64", (2048, 1216), 3, (32, 32), 10.0, 2)):
    n = int(np.prod(dims))
    base = torch.empty(n * ch, dtype=torch.float32, device="cuda")
    s.synth_generate(cfg, dims, np.float32, ch, 99, 0, dims[-1] if len(dims) == 3 else 1,
                     base.data_ptr())
    x = base.double()
    if cfg == 2:
        x = (x.view(-1, 3) * torch.tensor([100.0, 160.0, 160.0], device="cuda")
             - torch.tensor([0.0, 80.0, 80.0], device="cuda")).view(-1)
    x = x + (torch.rand_like(x) - 0.5) * 2e-7
    for exact in (False, True):
        p = s.SlicParams(grid=list(grid), weight_m=m, max_iterations=10)
        e = s.Engine(dims, ch, np.float64, x.data_ptr(), p)
        if exact:
            e.set_exact(True)
        e.init(); e.commit()
        for _ in range(10):
            e.assign(); e.update()
        torch.cuda.synchronize()
        ms = [e.assign_ms(i) for i in range(3, 10)]
        print(f"{name}: {'exact' if exact else 'fast '} assign {np.mean(ms):8.3f} ms/iter "
              f"({n / np.mean(ms) / 1e6:6.2f} Gvox/s)")
        e.close()
