"""World-size-2 gloo test of the z-slab sharding driver
(paper_1806_08741_b200/sharded.py) on CPU.

Each rank runs the driver over an oracle-backed engine that owns one slab:
it assigns and accumulates only its slab's voxels, contributes only the
clusters whose initial cell centre lies in its slab to the init table, and
relies on the driver's SUM allreduces to assemble the centre table and the
per-cluster int64 partials. The concatenated slab labels and the centres
must equal the single-process oracle run bit for bit — the multi-GPU
determinism contract (the reference's "bitwise identical for any worker
count", parallel.hpp:1-8)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class OracleSlabEngine:
    """CPU stand-in for the CUDA engine, same protocol as sharded.ShardedLoop."""

    def __init__(self, oracle, data, dims, ch, grid, m, slab):
        import torch
        self.torch = torch
        self.o, self.data, self.dims, self.ch = oracle, data, tuple(dims), ch
        self.grid, self.m, self.slab = tuple(grid), m, slab
        n = int(np.prod(dims))
        self.plane = n // dims[-1]
        self.labels = np.full(n, 0xFFFFFFFF, np.uint32)
        self.dists = np.full(n, np.inf)
        self.k = oracle.cluster_count(dims, grid)
        self.stride = ch + len(dims)
        self.centers = None
        self.partials = None

    def init(self):
        full = self.o.init_centers(self.data, self.dims, self.ch, self.grid, perturb=True)
        # ownership by the initial (pre-perturbation) cell centre's last coordinate
        init = self.o.init_centers(self.data, self.dims, self.ch, self.grid, perturb=False)
        zc = init[:, -1]
        own = (zc >= self.slab[0]) & (zc < self.slab[1])
        full[~own] = 0.0
        self.centers = self.torch.from_numpy(full.reshape(-1).copy())

    def centers_tensor(self):
        return self.centers

    def value_range(self):
        plane = self.plane * self.ch
        return float(np.abs(self.data[self.slab[0] * plane: self.slab[1] * plane]).max())

    def set_value_range(self, v):
        self.synced_range = v

    def commit(self):
        pass

    def assign(self):
        c = self.centers.numpy().reshape(self.k, self.stride)
        lab, dist = self.o.assign(self.data, self.dims, self.ch, c, self.grid, self.m,
                                  self.labels, self.dists)
        lo, hi = self.slab[0] * self.plane, self.slab[1] * self.plane
        self.labels[lo:hi] = lab[lo:hi]
        self.dists[lo:hi] = dist[lo:hi]
        # int64 partial sums over this slab only (integer intensities: exact)
        part = np.zeros((self.k, self.stride + 1), np.int64)
        idx = np.arange(lo, hi)
        coords = []
        rem = idx.copy()
        for d in self.dims:
            coords.append(rem % d)
            rem //= d
        vals = self.data.reshape(-1, self.ch)[lo:hi].astype(np.int64)
        L = self.labels[lo:hi].astype(np.int64)
        for c in range(self.ch):
            np.add.at(part[:, c], L, vals[:, c])
        for a, co in enumerate(coords):
            np.add.at(part[:, self.ch + a], L, co)
        np.add.at(part[:, self.stride], L, 1)
        self.partials = self.torch.from_numpy(part.reshape(-1))

    def partials_tensor(self):
        return self.partials

    def labels_tensor(self):
        plane = self.plane
        return self.torch.from_numpy(
            self.labels[self.slab[0] * plane: self.slab[1] * plane].astype(np.int64))

    def update(self):
        part = self.partials.numpy().reshape(self.k, self.stride + 1)
        sums = part[:, : self.stride].astype(np.float64)
        counts = part[:, self.stride].copy()
        c = self.centers.numpy().reshape(self.k, self.stride)
        new, _ = self.o.update(c, sums, counts)
        self.centers = self.torch.from_numpy(new.reshape(-1).copy())


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import oracle
    from paper_1806_08741_b200.sharded import ShardedLoop, slab_bounds

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(5)
        dims, ch, grid, m, iters = (24, 20, 18), 2, (6, 5, 4), 10.0, 4
        data = rng.integers(0, 256, int(np.prod(dims)) * ch).astype(np.float64)
        o = oracle.Oracle()
        slab = slab_bounds(dims[-1], world, rank, align=grid[-1])
        eng = OracleSlabEngine(o, data, dims, ch, grid, m, slab)
        loop = ShardedLoop(eng, lambda t: dist.all_reduce(t), world)
        loop.init()
        for _ in range(iters):
            loop.iterate()
        plane = int(np.prod(dims[:-1]))
        # connectivity once, on rank 0, over the slabs gathered there
        def gather(t, parts, dst):
            dist.gather(t, gather_list=parts, dst=dst)
        full = loop.gather_labels(gather, dims[-1], plane, align=grid[-1], rank=rank)
        cc = loop.segment(gather,
                          lambda f: o.enforce_connectivity(dims, f.numpy().astype(np.uint32),
                                                           eng.centers.numpy().reshape(eng.k, -1),
                                                           ch, grid),
                          dims[-1], plane, align=grid[-1], rank=rank)
        assert (full is None) == (rank != 0) and (cc is None) == (rank != 0)
        mine = eng.labels[slab[0] * plane: slab[1] * plane].copy()
        parts = [None] * world
        # every rank adopted the MAX of the ranks' value ranges (gloo MAX)
        assert eng.synced_range == float(np.abs(data).max())
        dist.all_gather_object(parts, (slab, mine, eng.centers.numpy().copy(), cc))
        if rank == 0:
            labels = np.concatenate([p[1] for p in sorted(parts, key=lambda p: p[0][0])])
            ref_l, ref_c, _ = o.run_slic(data, dims, ch, grid, m, max_iterations=iters)
            ok_l = np.array_equal(labels, ref_l) and np.array_equal(full.numpy(), ref_l)
            ok_c = all(np.array_equal(p[2], ref_c.reshape(-1)) for p in parts)
            ref_cc = o.enforce_connectivity(dims, ref_l, ref_c, ch, grid)
            ok_cc = np.array_equal(cc, ref_cc)
            q.put((ok_l and ok_cc, ok_c, [p[0] for p in parts]))
    finally:
        dist.destroy_process_group()


def test_slab_bounds():
    from paper_1806_08741_b200.sharded import all_slabs, data_bounds, slab_bounds
    assert all_slabs(1024, 8, align=16) == [(i * 128, (i + 1) * 128) for i in range(8)]
    s = all_slabs(7000, 8, align=32)
    assert s[0][0] == 0 and s[-1][1] == 7000
    assert all(a[1] == b[0] for a, b in zip(s, s[1:]))
    assert all(lo % 32 == 0 for lo, _ in s)
    assert all_slabs(3, 4) == [(0, 0), (0, 1), (1, 2), (2, 3)]
    assert data_bounds(100, (40, 60)) == (38, 62)
    assert data_bounds(100, (0, 10)) == (0, 12)
    with pytest.raises(ValueError):
        slab_bounds(10, 2, 2)


def test_two_rank_gloo_matches_single_process():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    assert all(p.exitcode == 0 for p in procs)
    ok_l, ok_c, slabs = q.get(timeout=5)
    assert slabs == [(0, 8), (8, 18)] or len(slabs) == 2
    assert ok_l, "sharded labels differ from the single-process oracle"
    assert ok_c, "sharded centres differ from the single-process oracle"
