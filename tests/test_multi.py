"""Multi-GPU run_slic behind the C ABI (csrc/multi.cu).

CPU: the native z-slab split (sslic_slab_bounds) equals sharded.slab_bounds,
which the gloo tests drive. GPU: the NCCL path on one device (a 1-rank
communicator: ncclCommInitAll / ncclCommInitRank, allreduces on the engine
stream, inside the captured graph) is bitwise the single-GPU run_slic. More
than one device cannot be exercised here (one GPU per box); the slab engines
that the N-device path runs are pinned by test_gpu_fast.py's slab tests."""
import numpy as np
import pytest


def test_native_slab_bounds_match_python():
    import paper_1806_08741_b200 as s
    from paper_1806_08741_b200.sharded import slab_bounds
    rng = np.random.default_rng(7)
    for _ in range(300):
        last = int(rng.integers(1, 9000))
        world = int(rng.integers(1, 9))
        align = int(rng.choice([1, 8, 16, 32]))
        for r in range(world):
            assert s.slab_bounds_native(last, world, r, align) == slab_bounds(last, world, r,
                                                                              align)


def test_multi_rejects_bad_arguments():
    import paper_1806_08741_b200 as s
    img = s.NDImage((16, 16), 1, np.zeros(256, np.uint8))
    p = s.SlicParams(grid=[4, 4], max_iterations=1)
    with pytest.raises(s.InvalidArgument):  # 2-D images do not split into z-slabs
        s.run_slic_multi(img, p, [0, 1])
    with pytest.raises(s.InvalidArgument):
        s.slab_bounds_native(10, 2, 2, 1)


def _volume(dtype, dims, seed):
    rng = np.random.default_rng(seed)
    n = int(np.prod(dims))
    if dtype == np.uint16:
        base = rng.integers(5000, 60000, 64)
        cell = (np.arange(n) // 977) % 64
        return (base[cell] + rng.normal(0, 200, n)).clip(0, 65535).astype(np.uint16)
    return rng.random(n).astype(np.float32)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [np.uint16, np.float32])
def test_multi_one_device_nccl_equals_run_slic(sslic, dtype):
    s = sslic
    dims = (64, 48, 40)
    img = s.NDImage(dims, 1, _volume(dtype, dims, 3))
    p = s.SlicParams(grid=[8, 8, 8], weight_m=10.0, max_iterations=4,
                     enforce_connectivity=False)
    ref = s.run_slic(img, p, device=0)
    got = s.run_slic_multi(img, p, [0])
    assert np.array_equal(got.labels, ref.labels)
    assert np.array_equal(got.centers.data, ref.centers.data)
    assert got.residuals == ref.residuals


@pytest.mark.gpu
def test_run_slic_rank_world1_equals_run_slic(sslic):
    s = sslic
    dims = (64, 48, 40)
    img = s.NDImage(dims, 1, _volume(np.uint16, dims, 4))
    p = s.SlicParams(grid=[8, 8, 8], weight_m=10.0, max_iterations=3,
                     enforce_connectivity=False)
    ref = s.run_slic(img, p, device=0)
    for uid in (None, s.nccl_unique_id()):
        lab, cen, res = s.run_slic_rank(img, p, 0, 1, uid, device=0)
        assert np.array_equal(lab, ref.labels)
        assert np.array_equal(cen.data, ref.centers.data)
        assert res == ref.residuals


@pytest.mark.gpu
def test_engine_with_nccl_graph_equals_plain_engine(sslic):
    """attach_nccl + start + iterate_graph (the allreduce captured as a graph
    node) against a plain engine: labels and centres bitwise."""
    import torch
    s = sslic
    dims = (96, 64, 48)
    data = _volume(np.uint16, dims, 5)
    img = torch.from_numpy(data.view(np.int16)).cuda()
    p = s.SlicParams(grid=[16, 16, 16], weight_m=10.0, max_iterations=5)
    stream = torch.cuda.Stream()
    a = s.Engine(dims, 1, np.uint16, img.data_ptr(), p, stream=stream.cuda_stream)
    b = s.Engine(dims, 1, np.uint16, img.data_ptr(), p)
    a.attach_nccl(s.nccl_unique_id(), 0, 1)
    a.start()
    a.iterate_graph(5)
    b.init()
    b.commit()
    b.iterate(5)
    n = int(np.prod(dims))
    la = torch.empty(n, dtype=torch.int32, device="cuda")
    lb = torch.empty(n, dtype=torch.int32, device="cuda")
    a.labels_to(la.data_ptr())
    b.labels_to(lb.data_ptr())
    torch.cuda.synchronize()
    assert torch.equal(la, lb)
    assert np.array_equal(a.centers(), b.centers())
    assert a.residuals() == b.residuals()
