"""BASELINE sizes (size-independent properties): at the full
config-3 (1024^3 uint16) and config-4 (512x512x256 4-channel f32) sizes, and
on a 384-plane z-subvolume of config 5 (2048x1216 RGB uint8; two full-size
engines would not fit one GPU), the fast kernel must equal the exact fp64
kernel bit for bit at every iteration (labels, centres, undefined counts),
and the centres must be the fp64 means of their members recomputed
independently from the label map (torch index_add over the volume;
reduce_and_update, slic.hpp:352-372: count > 0 -> sums / count)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [
    # config, dims, channels, dtype, grid, m, iterations
    (3, (1024, 1024, 1024), 1, np.uint16, (16, 16, 16), 10.0, 3),
    (4, (512, 512, 256), 4, np.float32, (8, 8, 8), 20.0, 3),
    (5, (2048, 1216, 384), 3, np.uint8, (32, 32, 32), 10.0, 3),
]


def _recomputed_centres(torch, img, labels, dims, ch, k, shift):
    """fp64 means of (intensities, coordinates) per label, exactly as the
    engine's fixed-point sums would produce them (integer data: exact)."""
    n = int(np.prod(dims))
    lab = labels.to(torch.int64)
    if img.dtype == torch.int16:
        vals = (img.to(torch.int32) & 0xFFFF).to(torch.float64)
    else:
        vals = img.to(torch.float64)
    stride = ch + len(dims)
    sums = torch.zeros((k, stride), dtype=torch.float64, device="cuda")
    cnt = torch.zeros(k, dtype=torch.float64, device="cuda")
    cnt.index_add_(0, lab, torch.ones(n, dtype=torch.float64, device="cuda"))
    for c in range(ch):
        sums[:, c].index_add_(0, lab, vals[c::ch])
    idx = torch.arange(n, device="cuda", dtype=torch.int64)
    rem = idx
    for a, d in enumerate(dims):
        sums[:, ch + a].index_add_(0, lab, (rem % d).to(torch.float64))
        rem = rem // d
    return sums, cnt


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"cfg{c[0]}-{'x'.join(map(str, c[1]))}")
def test_fullsize_fast_equals_exact(sslic, case):
    import torch
    s = sslic
    cfg, dims, ch, dtype, grid, m, iters = case
    n = int(np.prod(dims))
    tdt = {np.uint8: torch.uint8, np.uint16: torch.int16, np.float32: torch.float32}[dtype]
    img = torch.empty(n * ch, dtype=tdt, device="cuda")
    s.synth_generate(cfg, dims, dtype, ch, 1806, 0, dims[-1], img.data_ptr())
    torch.cuda.synchronize()
    p = s.SlicParams(grid=list(grid), weight_m=m, max_iterations=iters)
    fast = s.Engine(dims, ch, dtype, img.data_ptr(), p)
    exact = s.Engine(dims, ch, dtype, img.data_ptr(), p)
    exact.set_exact(True)
    la = torch.empty(n, dtype=torch.int32, device="cuda")
    lb = torch.empty(n, dtype=torch.int32, device="cuda")
    for e in (fast, exact):
        e.init()
        e.commit()
    for it in range(iters):
        fast.assign()
        exact.assign()
        assert fast.undefined_count() == exact.undefined_count() == 0
        fast.update()
        exact.update()
        fast.labels_to(la.data_ptr())
        exact.labels_to(lb.data_ptr())
        torch.cuda.synchronize()
        diff = int((la != lb).sum().item())
        assert diff == 0, f"iteration {it}: {diff} labels differ"
        assert np.array_equal(fast.centers(), exact.centers()), f"iteration {it}: centres"
    np.testing.assert_allclose(fast.residuals(), exact.residuals(), rtol=1e-12)
    exact.close()
    if dtype != np.float32:  # integer data: the recomputed means are exact
        k = fast.k
        sums, cnt = _recomputed_centres(torch, img, la, dims, ch, k, 0)
        cen = torch.from_numpy(fast.centers().reshape(k, -1)).cuda()
        have = cnt > 0
        mean = sums[have] / cnt[have].unsqueeze(1)
        assert torch.equal(mean, cen[have]), "centres are not the means of their members"
    fast.close()
    del img, la, lb
    torch.cuda.empty_cache()
