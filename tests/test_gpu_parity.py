"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
outputs and the CPU oracle. Bit-exact for labels, centres and (where the
reference sums in the same exact integer domain) everything else; residuals
are compared at rtol 1e-12 because the device reduces the per-cluster squared
displacements in a fixed tree order instead of the reference's sequential
(k, i) order."""
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_cases

pytestmark = pytest.mark.gpu

RES_RTOL = 1e-12


def _img(s, data, dims, ch):
    return s.NDImage(tuple(int(d) for d in dims), int(ch), data)


@pytest.mark.parametrize("corpus", ["corpus_acceptance", "corpus_run_slic",
                                    "corpus_connectivity"])
def test_run_slic_matches_reference_corpus(sslic, corpus):
    # acceptance.cpp:96-113 (C1), test_slic.cpp:376-397
    for i, c in enumerate(load_cases(corpus)):
        img = _img(sslic, c["data"], c["dims"], c["channels"])
        p = sslic.SlicParams(grid=[int(g) for g in c["grid"]], weight_m=float(c["weight_m"]))
        r = sslic.run_slic(img, p)
        assert np.array_equal(r.labels, c["labels"]), (corpus, i)
        assert np.array_equal(r.centers.data.reshape(-1), c["centers"].reshape(-1)), (corpus, i)
        np.testing.assert_allclose(r.residuals, c["residuals"], rtol=RES_RTOL, atol=0)


@pytest.mark.parametrize("corpus", ["corpus_acceptance", "corpus_connectivity"])
def test_enforce_connectivity_matches_reference(sslic, corpus):
    # acceptance.cpp:115-140 (C2), test_connectivity.cpp:185-216
    for i, c in enumerate(load_cases(corpus)):
        p = sslic.SlicParams(grid=[int(g) for g in c["grid"]], weight_m=float(c["weight_m"]))
        t = sslic.ClusterTable(int(c["channels"]), len(c["dims"]), c["centers"])
        out = sslic.enforce_connectivity(c["labels"], c["dims"], t, p)
        assert np.array_equal(out, c["labels_cc"]), (corpus, i)


def test_single_pass_bit_exact(sslic):
    # test_slic.cpp:199-246: labels AND dists bitwise given identical centres.
    z = np.load(os.path.join(GOLDEN, "single_pass.npz"))
    img = _img(sslic, z["data"], z["dims"], 1)
    p = sslic.SlicParams(grid=[6, 6])
    t = sslic.ClusterTable(1, 2, z["centers"])
    lab = np.full(144, sslic.UNDEFINED, np.uint32)
    dist = np.full(144, np.inf)
    sslic.assign_labels(img, t, p, lab, dist)
    assert np.array_equal(lab, z["labels"])
    assert np.array_equal(dist, z["dists"])


def test_single_pass_random_centres_bit_exact(sslic, oracle_lib):
    # Arbitrary (drifted, fractional) centre tables and carried-over state.
    rng = np.random.default_rng(11)
    for trial in range(30):
        rank = int(rng.integers(1, 4))
        ch = int(rng.integers(1, 4))
        dims = rng.integers(2, 20, rank)
        grid = np.array([rng.integers(1, d + 1) for d in dims])
        data = rng.integers(0, 65535, int(np.prod(dims)) * ch) / 256.0
        k = int(np.prod([(d + s - 1) // s for d, s in zip(dims, grid)]))
        cen = np.concatenate([rng.uniform(0, 255, (k, ch)),
                              np.stack([rng.uniform(-1, d, k) for d in dims], 1)], 1)
        lab0 = rng.integers(0, k, int(np.prod(dims))).astype(np.uint32)
        dist0 = rng.uniform(0, 2e4, int(np.prod(dims)))
        exp_l, exp_d = oracle_lib.assign(data, dims, ch, cen, grid, 7.5, lab0, dist0)
        img = _img(sslic, data, dims, ch)
        lab, dist = lab0.copy(), dist0.copy()
        sslic.assign_labels(img, sslic.ClusterTable(ch, rank, cen),
                            sslic.SlicParams(grid=list(grid), weight_m=7.5), lab, dist)
        assert np.array_equal(lab, exp_l), trial
        assert np.array_equal(dist, exp_d), trial


def test_configlike_native_dtypes(sslic):
    # u8 / u16 / f32 native inputs shaped like BASELINE configs 1-5.
    for c in load_cases("configlike"):
        img = _img(sslic, c["data"], c["dims"], c["channels"])
        p = sslic.SlicParams(grid=[int(g) for g in c["grid"]], weight_m=float(c["weight_m"]),
                             max_iterations=int(c["iterations"]))
        r, nxt = sslic.segment(img, p)
        assert np.array_equal(r.labels, c["labels_cc"]), c["name"]
        assert nxt >= len(c["centers"])
        np.testing.assert_allclose(r.centers.data.reshape(-1), c["centers"].reshape(-1),
                                   rtol=1e-12, atol=1e-12)


def test_configlike_pre_connectivity(sslic):
    for c in load_cases("configlike"):
        img = _img(sslic, c["data"], c["dims"], c["channels"])
        p = sslic.SlicParams(grid=[int(g) for g in c["grid"]], weight_m=float(c["weight_m"]),
                             max_iterations=int(c["iterations"]))
        r = sslic.run_slic(img, p)
        assert np.array_equal(r.labels, c["labels"]), c["name"]
        if c["data"].dtype.kind == "u":
            # integer intensities: int64 sums are exact -> bitwise centres
            assert np.array_equal(r.centers.data.reshape(-1), c["centers"].reshape(-1))
        else:
            # float32 intensities are summed in 2^-shift fixed point
            np.testing.assert_allclose(r.centers.data.reshape(-1), c["centers"].reshape(-1),
                                       rtol=1e-12, atol=1e-12)


def test_known_answers(sslic):
    s = sslic
    # init_centers (test_slic.cpp:23-45)
    t = s.init_centers(s.NDImage.zeros((100, 100), 1), s.SlicParams(grid=[50, 50]))
    assert [tuple(np.rint(r[1:]).astype(int)) for r in t.data] == [(25, 25), (75, 25),
                                                                   (25, 75), (75, 75)]
    t = s.init_centers(s.NDImage.zeros((7,), 1), s.SlicParams(grid=[3]))
    assert list(t.data[:, 1]) == [1.0, 4.0, 6.0]
    img = s.NDImage((6, 6), 2, np.array([[x, y] for y in range(6) for x in range(6)], float))
    t = s.init_centers(img, s.SlicParams(grid=[6, 6]))
    assert t.data[0, 0] == 3.0 and t.data[0, 1] == 3.0
    with pytest.raises(s.InvalidArgument):
        s.init_centers(img, s.SlicParams(grid=[7, 6]))
    # perturb (test_slic.cpp:65-111)
    z = s.NDImage.zeros((5, 5), 1)
    t = s.perturb_centers(z, s.init_centers(z, s.SlicParams(grid=[5, 5])))
    assert tuple(t.data[0, 1:]) == (1.0, 1.0)
    ridge = s.NDImage((5, 5), 1, [100.0 if x == 2 else 0.0 for y in range(5) for x in range(5)])
    t = s.perturb_centers(ridge, s.init_centers(ridge, s.SlicParams(grid=[5, 5])))
    assert tuple(t.data[0, 1:]) == (2.0, 1.0) and t.data[0, 0] == 100.0
    tiny = s.NDImage.zeros((2, 2), 1)
    t = s.perturb_centers(tiny, s.init_centers(tiny, s.SlicParams(grid=[1, 1])))
    assert np.all((t.data[:, 1:] >= 0) & (t.data[:, 1:] < 2))
    # squared_distance 0 / 100 / 25 (test_slic.cpp:113-129)
    p = s.SlicParams(grid=[7, 5], weight_m=10.0)
    assert s.squared_distance([10, 20, 3, 4], [10, 20], [3, 4], p) == 0.0
    assert s.squared_distance([10, 20, 3, 4], [10, 20], [10, 4], p) == 100.0
    assert s.squared_distance([50, 10, 5, 2, 2], [53, 14, 5], [2, 2], p) == 25.0
    # gradient (test_color.cpp:85-106)
    flat = s.NDImage((5, 5), 1, np.full(25, 3.5))
    assert np.all(s.gradient_magnitude_sq(flat, [[x, y] for y in range(5)
                                                 for x in range(5)]) == 0.0)
    ramp = s.NDImage((5, 4), 1, [float(x) for y in range(4) for x in range(5)])
    assert s.gradient_magnitude_sq(ramp, [2, 1]) == 1.0
    assert s.gradient_magnitude_sq(ramp, [1, 2]) == 1.0
    two = s.NDImage((3, 3), 2, [[float(x), 2.0 * y] for y in range(3) for x in range(3)])
    assert s.gradient_magnitude_sq(two, [1, 1]) == 5.0
    with pytest.raises(s.OutOfRange):
        s.gradient_magnitude_sq(two, [3, 0])


def test_assign_covers_window_and_ties(sslic):
    s = sslic
    # single cluster claims its whole window (test_slic.cpp:170-179)
    img = s.NDImage.zeros((8, 8), 1)
    p = s.SlicParams(grid=[8, 8])
    lab = np.full(64, s.UNDEFINED, np.uint32)
    dist = np.full(64, np.inf)
    s.assign_labels(img, s.init_centers(img, p), p, lab, dist)
    assert np.all(lab == 0)
    # equidistant pixel keeps the lower id (test_slic.cpp:181-197)
    img = s.NDImage.zeros((8, 1), 1)
    p = s.SlicParams(grid=[4, 1])
    t = s.ClusterTable(1, 2, [[0.0, 1.0, 0.0], [0.0, 5.0, 0.0]])
    lab = np.full(8, s.UNDEFINED, np.uint32)
    dist = np.full(8, np.inf)
    s.assign_labels(img, t, p, lab, dist)
    assert lab[3] == 0


def test_accumulate_and_reduce(sslic):
    s = sslic
    # four constant pixels (test_slic.cpp:250-262)
    img = s.NDImage((2, 2), 1, np.full(4, 7.0))
    sums, counts = s.accumulate_region(img, np.zeros(4, np.uint32))
    assert counts[0] == 4 and list(sums[0]) == [28.0, 2.0, 2.0]
    # undefined labels are a loud error (test_slic.cpp:272-276)
    with pytest.raises(s.LogicError):
        s.accumulate_region(s.NDImage.zeros((2, 2), 1), np.full(4, s.UNDEFINED, np.uint32), k=1)
    # reduce: single point and empty cluster (test_slic.cpp:304-346)
    t = s.ClusterTable(1, 2, [[5.0, 2.0, 3.0]])
    nt, r = s.reduce_and_update(t, [(np.array([[5.0, 2.0, 3.0]]), np.array([1]))])
    assert list(nt.data[0]) == [5.0, 2.0, 3.0] and r == 0.0
    t = s.ClusterTable(1, 1, [[1.0, 4.0], [9.0, 8.0]])
    nt, r = s.reduce_and_update(t, [(np.array([[10.0, 20.0]]), np.array([1]))])
    assert list(nt.data[0]) == [10.0, 20.0] and list(nt.data[1]) == [9.0, 8.0]
    assert r == np.sqrt(81.0 + 256.0)


def test_uniform_image_and_monotone(sslic, oracle_lib):
    s = sslic
    # uniform image converges to the init cells (test_slic.cpp:399-411)
    r = s.run_slic(s.NDImage((40, 30), 1, np.full(1200, 9.0)), s.SlicParams(grid=[10, 10]))
    exp = [(x // 10) + 4 * (y // 10) for y in range(30) for x in range(40)]
    assert list(r.labels) == exp
    # acceptance C6 (acceptance.cpp:285-302): 4 cells after connectivity
    res, _ = s.segment(s.NDImage((100, 100), 1, np.full(10000, 42.0)),
                       s.SlicParams(grid=[50, 50]))
    exp = [(0 if x < 50 else 1) + (0 if y < 50 else 2) for y in range(100) for x in range(100)]
    assert list(res.labels) == exp
    # residual threshold (test_slic.cpp:476-490)
    rng = np.random.default_rng(606)
    img = s.NDImage((16, 13), 1, rng.integers(0, 65280, 208) / 256.0)
    r = s.run_slic(img, s.SlicParams(grid=[4, 4], max_iterations=10,
                                     residual_threshold=np.finfo(float).max))
    assert len(r.residuals) == 1
    r = s.run_slic(img, s.SlicParams(grid=[4, 4], max_iterations=10))
    assert len(r.residuals) == 10


def test_errors(sslic):
    s = sslic
    img = s.NDImage.zeros((8, 8), 1)
    with pytest.raises(s.InvalidArgument):
        s.run_slic(img, s.SlicParams(grid=[9, 8]))
    with pytest.raises(s.InvalidArgument):
        s.run_slic(img, s.SlicParams(grid=[4, 4], weight_m=0.0))
    with pytest.raises(s.InvalidArgument):
        s.run_slic(img, s.SlicParams(grid=[4, 4]), workers=0)


def test_convert_image_to_lab_matches_reference(sslic, reference_lib):
    """GPU sRGB -> Lab against the unmodified reference:
    u8 images, integral f64 and fractional f32 data. The transfer function
    of integral inputs is the reference's bit for bit (host table); the cube
    root is the device's, so Lab is compared at 1e-12 absolute."""
    s = sslic
    rng = np.random.default_rng(11)
    dims = (37, 23, 5)
    n = int(np.prod(dims))
    cases = [rng.integers(0, 256, size=n * 3).astype(np.uint8),
             rng.integers(0, 256, size=n * 3).astype(np.float64),
             rng.uniform(0.0, 255.0, size=n * 3).astype(np.float32)]
    for x in cases:
        ours = s.convert_image_to_lab(s.NDImage(dims, 3, x))
        ref = reference_lib.convert_to_lab(dims, x.astype(np.float64))
        got = np.asarray(ours.data, np.float64).reshape(-1)
        # (glibc's and the device's cbrt are each within 1 ulp, neither is
        # correctly rounded, so ties to the last bit are not expected)
        assert np.max(np.abs(got - ref)) < 1e-12
    with pytest.raises(s.InvalidArgument):
        s.convert_image_to_lab(s.NDImage((2, 2), 1, np.zeros(4)))


def test_mask_label_contour_matches_oracle(sslic, oracle_lib):
    """GPU label-contour mask (io.hpp:432-454): bitwise equal to the oracle on
    random 2-D/3-D label maps and native dtypes; label dims must match."""
    s = sslic
    rng = np.random.default_rng(13)
    for dims, ch, dt in (((40, 30), 3, np.uint8), ((17, 9, 11), 1, np.uint16),
                         ((12, 10, 6), 4, np.float32)):
        n = int(np.prod(dims))
        x = (rng.integers(0, 200, size=n * ch) if dt != np.float32
             else rng.uniform(0, 1, size=n * ch)).astype(dt)
        lab = rng.integers(0, 3, size=n).astype(np.uint32)
        ours = s.mask_label_contour(s.NDImage(dims, ch, x), lab)
        ref = oracle_lib.mask_label_contour(dims, ch, x.astype(np.float64), lab)
        assert np.array_equal(np.asarray(ours.data, np.float64), ref)
    with pytest.raises(s.InvalidArgument):
        s.mask_label_contour(s.NDImage((2, 2), 1, np.zeros(4)), np.zeros(6, np.uint32), (3, 2))


def _pipeline_fuzz(n=24, seed=18060874):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        rank = int(rng.integers(2, 4))
        ch = int(rng.integers(1, 5))
        dtype = [np.uint8, np.uint16][int(rng.integers(0, 2))]
        dims = tuple(int(x) for x in rng.integers(24, 160 if rank == 2 else 48, size=rank))
        grid = tuple(int(rng.integers(3, min(d, 16) + 1)) for d in dims)
        m = float(rng.choice([2.0, 10.0, 30.0]))
        iters = int(rng.integers(2, 6))
        out.append((dims, ch, dtype, grid, m, iters, int(rng.integers(0, 1 << 30))))
    return out


@pytest.mark.parametrize("case", _pipeline_fuzz(), ids=lambda c: f"r{len(c[0])}c{c[1]}-"
                         f"{np.dtype(c[2]).name}-{'x'.join(map(str, c[0]))}")
def test_segment_matches_oracle_fuzz(sslic, oracle_lib, case):
    """The whole product pipeline (sslic_segment: upload, init + perturb, the
    iterations, connectivity) against the CPU oracle on seeded random
    volumes: labels after connectivity and centres bit for bit, residuals at
    rtol 1e-12."""
    s = sslic
    dims, ch, dtype, grid, m, iters, seed = case
    rng = np.random.default_rng(seed)
    hi = 255 if dtype == np.uint8 else 65535
    n = int(np.prod(dims))
    coarse = [max(1, d // 6) for d in dims]
    base = rng.integers(0, hi + 1, size=tuple(reversed(coarse)) + (ch,))
    idx = np.ix_(*[np.minimum(np.arange(d) // max(1, d // c), c - 1)
                   for d, c in zip(reversed(dims), reversed(coarse))])
    vol = base[idx] + rng.normal(0, 0.05 * hi, size=tuple(reversed(dims)) + (ch,))
    data = np.clip(np.rint(vol), 0, hi).astype(dtype).reshape(-1)
    p = s.SlicParams(grid=list(grid), weight_m=m, max_iterations=iters)
    res, _ = s.segment(s.NDImage(dims, ch, data), p, device=0)
    lab, cen, rs = oracle_lib.run_slic(data.astype(np.float64), dims, ch, list(grid), m,
                                       max_iterations=iters)
    assert np.array_equal(res.centers.data.reshape(-1), cen.reshape(-1)), "centres"
    np.testing.assert_allclose(res.residuals, rs, rtol=RES_RTOL)
    cc = oracle_lib.enforce_connectivity(dims, lab, cen, ch, list(grid))
    assert np.array_equal(res.labels, cc), f"{int((res.labels != cc).sum())} labels differ"


@pytest.mark.parametrize("conn", [True, False])
def test_segment_write_files(sslic, oracle_lib, tmp_path, conn):
    """sslic_segment_write: the labels file equals segment()'s map with the
    reference's "label count" header comment (write_labels, io.hpp:396-412),
    and the contour file equals write_volume(mask_label_contour(img, labels))
    in float32 (io.hpp:432-454, 362-392) -- both from the fused final pass."""
    s = sslic
    rng = np.random.default_rng(909)
    dims = (70, 52, 33)
    data = rng.integers(0, 255, int(np.prod(dims)) * 3).astype(np.uint8)
    img = s.NDImage(dims, 3, data)
    p = s.SlicParams(grid=[8, 8, 8], weight_m=10.0, max_iterations=4, enforce_connectivity=conn)
    ref, nxt = s.segment(img, p)
    lp, cp = str(tmp_path / "labels.hdr"), str(tmp_path / "contour.hdr")
    cen, res, nxt2 = s.segment_write(img, p, lp, cp)
    assert nxt2 == nxt and cen == ref.centers and res == ref.residuals
    lab, ldims = s.read_labels(lp)
    assert tuple(ldims) == dims and np.array_equal(lab.reshape(-1), ref.labels)
    head = open(lp).read()
    assert f"label count: {int(ref.labels.max()) + 1}" in head
    vol = s.read_volume(cp)
    want = oracle_lib.mask_label_contour(dims, 3, data.astype(np.float64), ref.labels)
    assert np.array_equal(np.asarray(vol.data, np.float32), want.astype(np.float32))
