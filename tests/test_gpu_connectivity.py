"""The device sweep (connectivity.cu: component-graph fixpoint + the exact
serial prefix) against the CPU oracle's raster sweep (sslic_oracle.c, pinned
bit for bit to connectivity.hpp:182-261 by test_oracle_pinning.py).

Each case checks the relabelled map AND the next unused label. The inputs are
chosen to reach every branch of the recurrence: noise-dominated SLIC maps
(config-3-like: most voxels outside finalized components, many fills that
grow through merged specks), random label fields on ranks 1-4 (the pending
cascade at offset 0, the whole-image component), and maps holding ids >= k
(the fully serial path)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _check(s, o, dims, lab, cen, ch, grid):
    t = s.ClusterTable(ch, len(dims), np.ascontiguousarray(cen, np.float64).reshape(-1))
    p = s.SlicParams(grid=list(grid), weight_m=10.0)
    out, nxt = s.enforce_connectivity(lab, dims, t, p, return_next=True)
    ref, rnxt = o.enforce_connectivity(dims, lab, np.asarray(cen).reshape(len(cen), -1), ch,
                                       list(grid), return_next=True)
    assert nxt == rnxt, f"next label {nxt} != {rnxt}"
    bad = int((out != ref).sum())
    assert bad == 0, f"{bad} of {out.size} labels differ"
    return out


def _noisy_volume(rng, dims, ncell):
    """Voronoi cells with U[5000, 60000] means and sigma = sqrt(mean) noise
    (the config-3 construction at a small size)."""
    r = len(dims)
    seeds = rng.random((ncell, r)) * np.asarray(dims)
    means = rng.uniform(5000, 60000, ncell)
    grids = np.meshgrid(*[np.arange(d, dtype=np.float32) for d in reversed(dims)],
                        indexing="ij")
    coords = np.stack([g.reshape(-1) for g in reversed(grids)], -1)
    best = np.full(coords.shape[0], np.inf, np.float32)
    idx = np.zeros(coords.shape[0], np.int32)
    for i in range(ncell):
        d = ((coords - seeds[i]) ** 2).sum(-1)
        mk = d < best
        best[mk] = d[mk]
        idx[mk] = i
    mu = means[idx]
    return np.clip(np.rint(mu + rng.normal(0, 1, mu.size) * np.sqrt(mu)), 0, 65535).astype(
        np.uint16)


@pytest.mark.parametrize("seed,dims,grid,m", [
    (1, (96, 96, 96), (16, 16, 16), 10.0),
    (2, (64, 80, 72), (8, 8, 8), 10.0),
    (3, (160, 128, 64), (16, 16, 16), 10.0),
    (4, (100, 90, 80), (16, 16, 16), 1.0),
    (5, (512, 384), (16, 16), 10.0),
])
def test_noisy_slic_maps(sslic, oracle_lib, seed, dims, grid, m):
    rng = np.random.default_rng(seed)
    data = _noisy_volume(rng, dims, max(8, int(np.prod(dims)) // 16000))
    p = sslic.SlicParams(grid=list(grid), weight_m=m, max_iterations=10,
                         enforce_connectivity=False)
    res = sslic.run_slic(sslic.NDImage(dims, 1, data), p)
    _check(sslic, oracle_lib, dims, res.labels, res.centers.data.reshape(-1, 1 + len(dims)), 1,
           grid)


def _random_field(rng, dims, k, blob):
    """Piecewise-constant random labels (blob-sized patches) with speckle."""
    coarse = [max(1, d // blob) for d in dims]
    base = rng.integers(0, k, size=tuple(reversed(coarse)))
    idx = np.ix_(*[np.minimum(np.arange(d) // blob, c - 1)
                   for d, c in zip(reversed(dims), reversed(coarse))])
    lab = base[idx].reshape(-1).astype(np.uint32)
    speck = rng.random(lab.size) < 0.3
    lab[speck] = rng.integers(0, k, int(speck.sum()))
    return lab


def _random_centres(rng, dims, k, ch):
    c = np.empty((k, ch + len(dims)))
    c[:, :ch] = rng.random((k, ch))
    c[:, ch:] = rng.random((k, len(dims))) * (np.asarray(dims) - 1)
    return c


@pytest.mark.parametrize("seed", range(40))
def test_random_label_fields_ranks_1_to_4(sslic, oracle_lib, seed):
    rng = np.random.default_rng(1000 + seed)
    rank = 1 + seed % 4
    ext = {1: (200, 4000), 2: (12, 90), 3: (6, 30), 4: (4, 12)}[rank]
    dims = tuple(int(x) for x in rng.integers(ext[0], ext[1], rank))
    grid = tuple(int(rng.integers(1, min(d, 6) + 1)) for d in dims)
    k = int(rng.integers(2, 40))
    lab = _random_field(rng, dims, k, int(rng.integers(1, 5)))
    _check(sslic, oracle_lib, dims, lab, _random_centres(rng, dims, k, 1), 1, grid)


@pytest.mark.parametrize("seed", range(6))
def test_ids_at_or_above_k_take_the_serial_sweep(sslic, oracle_lib, seed):
    rng = np.random.default_rng(2000 + seed)
    dims = (int(rng.integers(8, 40)), int(rng.integers(8, 40)))
    k = int(rng.integers(2, 10))
    lab = _random_field(rng, dims, k + 6, 3)  # ids up to k + 5
    _check(sslic, oracle_lib, dims, lab, _random_centres(rng, dims, k, 2), 2, (4, 4))


def test_whole_image_component(sslic, oracle_lib):
    dims = (17, 9, 5)
    lab = np.zeros(int(np.prod(dims)), np.uint32)
    cen = np.array([[0.5, 30.0, 30.0, 30.0], [0.5, 8.0, 4.0, 2.0]])  # no seed for id 0
    _check(sslic, oracle_lib, dims, lab, cen, 1, (3, 3, 3))
    cen2 = np.array([[0.5, 8.0, 4.0, 2.0], [0.5, 30.0, 30.0, 30.0]])
    _check(sslic, oracle_lib, dims, lab, cen2, 1, (3, 3, 3))


def test_rank4_map_is_face_connected_in_w(sslic, oracle_lib):
    """a rank-4 sweep must probe all four axes and never
    fold w into z."""
    rng = np.random.default_rng(44)
    dims = (6, 5, 4, 7)
    k = 9
    lab = _random_field(rng, dims, k, 2)
    out = _check(sslic, oracle_lib, dims, lab, _random_centres(rng, dims, k, 1), 1, (2, 2, 2, 2))
    assert out.size == int(np.prod(dims))


class _env:
    """Temporarily set environment switches the C library reads per call."""

    def __init__(self, **kv):
        self.kv = kv

    def __enter__(self):
        import os
        self.old = {k: os.environ.get(k) for k in self.kv}
        os.environ.update({k: str(v) for k, v in self.kv.items()})

    def __exit__(self, *a):
        import os
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _stitch_cases():
    out = []
    for seed in range(12):
        rng = np.random.default_rng(3000 + seed)
        rank = 1 + seed % 4
        ext = {1: (200, 3000), 2: (12, 80), 3: (6, 28), 4: (4, 10)}[rank]
        dims = tuple(int(x) for x in rng.integers(ext[0], ext[1], rank))
        grid = tuple(int(rng.integers(1, min(d, 6) + 1)) for d in dims)
        k = int(rng.integers(2, 40))
        out.append((seed, dims, grid, k, int(rng.integers(1, 4))))
    return out


@pytest.mark.parametrize("case", _stitch_cases(), ids=lambda c: f"seed{c[0]}-rank{len(c[1])}")
def test_slab_stitched_ccl_equals_whole_volume(sslic, oracle_lib, case):
    """The >= 2^32-voxel path labels components slab by slab and stitches them
    across the slab faces (connectivity.cu). Forced onto small volumes with 2,
    3 or more slabs (SSLIC_CC_SLAB_PLANES), with 32- and 64-bit offsets
    (SSLIC_CC_FORCE64), the output equals the whole-volume result and the
    oracle's raster sweep bit for bit."""
    seed, dims, grid, k, blob = case
    rng = np.random.default_rng(seed)
    lab = _random_field(rng, dims, k, blob)
    cen = _random_centres(rng, dims, k, 1)
    whole = _check(sslic, oracle_lib, dims, lab, cen, 1, grid)
    last = dims[-1]
    for planes in sorted({1, 2, max(1, last // 3), max(1, last // 2)}):
        for force64 in (False, True):
            env = {"SSLIC_CC_SLAB_PLANES": planes}
            if force64:
                env["SSLIC_CC_FORCE64"] = 1
            with _env(**env):
                got = _check(sslic, oracle_lib, dims, lab, cen, 1, grid)
            assert np.array_equal(got, whole), (planes, force64)


def test_slab_stitched_noisy_volume(sslic, oracle_lib):
    """A config-3-like noisy SLIC map (most voxels outside finalized
    components) cut into 5 slabs, 64-bit offsets: equal to the oracle."""
    rng = np.random.default_rng(77)
    dims, grid = (96, 80, 72), (16, 16, 16)
    data = _noisy_volume(rng, dims, 40)
    p = sslic.SlicParams(grid=list(grid), weight_m=10.0, max_iterations=10,
                         enforce_connectivity=False)
    res = sslic.run_slic(sslic.NDImage(dims, 1, data), p)
    cen = res.centers.data.reshape(-1, 4)
    with _env(SSLIC_CC_SLAB_PLANES=15, SSLIC_CC_FORCE64=1):
        _check(sslic, oracle_lib, dims, res.labels, cen, 1, grid)


@pytest.mark.parametrize("seed,dims,blob", [
    (0, (70, 21, 19), 3), (1, (33, 9, 9), 2), (2, (64, 16, 16), 5), (3, (32, 8, 8), 1),
    (4, (97, 40, 23), 9), (5, (16, 70, 33), 4), (6, (129, 37), 6), (7, (40, 300), 2),
    (8, (5000,), 7), (9, (65, 17, 41), 30), (10, (200, 9, 17), 12), (11, (31, 64, 64), 8),
])
def test_tiled_ccl_and_edge_list_equal_whole_slab_union_find(sslic, oracle_lib, seed, dims, blob):
    """The CCL labels 32x8x8 tiles in shared memory and unites the tile faces
    afterwards (k_cc_tile / k_cc_seams), and the fixpoint rounds walk a list
    of candidate edges (k_edge_list / k_edges_list). On
    volumes that cut tiles on every axis, with components from specks to
    blobs spanning many tiles: equal to the oracle's raster sweep, and equal
    to the whole-slab union-find with whole-map edge passes
    (SSLIC_CC_NO_TILES, SSLIC_CC_NO_LIST), also with slabs and 64-bit offsets."""
    rng = np.random.default_rng(9100 + seed)
    k = int(rng.integers(2, 30))
    grid = tuple(int(rng.integers(1, min(d, 6) + 1)) for d in dims)
    lab = _random_field(rng, dims, k, blob)
    cen = _random_centres(rng, dims, k, 1)
    out = _check(sslic, oracle_lib, dims, lab, cen, 1, grid)
    with _env(SSLIC_CC_NO_TILES=1, SSLIC_CC_NO_LIST=1):
        plain = _check(sslic, oracle_lib, dims, lab, cen, 1, grid)
    assert np.array_equal(out, plain)
    with _env(SSLIC_CC_SLAB_PLANES=max(1, dims[-1] // 3), SSLIC_CC_FORCE64=1):
        slabs = _check(sslic, oracle_lib, dims, lab, cen, 1, grid)
    assert np.array_equal(out, slabs)
    # the edge list kept in the output map (what a volume that fills the
    # device does), whole and in slabs; fields with more edges than room fall
    # back to the map scans after the list was started
    with _env(SSLIC_CC_LIST_IN_OUTPUT=1):
        inout = _check(sslic, oracle_lib, dims, lab, cen, 1, grid)
    assert np.array_equal(out, inout)
    with _env(SSLIC_CC_LIST_IN_OUTPUT=1, SSLIC_CC_SLAB_PLANES=max(1, dims[-1] // 2),
              SSLIC_CC_FORCE64=1):
        inout = _check(sslic, oracle_lib, dims, lab, cen, 1, grid)
    assert np.array_equal(out, inout)
