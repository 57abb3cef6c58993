"""Pins the CPU oracle (oracle/sslic_oracle.c) to the reference.

CPU-only. The oracle must reproduce, bit for bit, the golden outputs that the
UNMODIFIED reference produced (tests/golden/make_golden.py) and, when the
reference build oracle/_ref is present, the live reference on fresh cases.
Known-answer cases are the reference's own (test_slic.cpp, test_color.cpp,
test_connectivity.cpp).
"""
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_cases


@pytest.mark.parametrize("corpus", ["corpus_acceptance", "corpus_run_slic",
                                    "corpus_connectivity"])
def test_oracle_matches_reference_corpus(oracle_lib, corpus):
    # acceptance.cpp:96-113 (C1) / test_slic.cpp:376-397: bitwise labels.
    for i, c in enumerate(load_cases(corpus)):
        lab, cen, res = oracle_lib.run_slic(c["data"], c["dims"], c["channels"], c["grid"],
                                            c["weight_m"])
        assert np.array_equal(lab, c["labels"]), (corpus, i)
        assert np.array_equal(cen.reshape(-1), c["centers"].reshape(-1)), (corpus, i)
        assert np.array_equal(res, c["residuals"]), (corpus, i)
        if "labels_cc" in c:
            cc = oracle_lib.enforce_connectivity(c["dims"], lab, cen, c["channels"], c["grid"])
            assert np.array_equal(cc, c["labels_cc"]), (corpus, i)


def test_oracle_single_pass_golden(oracle_lib):
    # test_slic.cpp:199-246: one pass, labels AND dists bitwise.
    z = np.load(os.path.join(GOLDEN, "single_pass.npz"))
    lab, dist = oracle_lib.assign(z["data"].astype(np.float64), z["dims"], 1, z["centers"],
                                  z["grid"], 10.0)
    assert np.array_equal(lab, z["labels"])
    assert np.array_equal(dist, z["dists"])


def test_oracle_configlike_golden(oracle_lib):
    for c in load_cases("configlike"):
        lab, cen, res = oracle_lib.run_slic(c["data"].astype(np.float64), c["dims"],
                                            c["channels"], c["grid"], c["weight_m"],
                                            max_iterations=int(c["iterations"]))
        assert np.array_equal(lab, c["labels"]), c["name"]
        assert np.array_equal(cen.reshape(-1), c["centers"].reshape(-1)), c["name"]
        assert np.array_equal(res, c["residuals"]), c["name"]
        cc = oracle_lib.enforce_connectivity(c["dims"], lab, cen, c["channels"], c["grid"])
        assert np.array_equal(cc, c["labels_cc"]), c["name"]


def test_oracle_vs_live_reference(oracle_lib, reference_lib):
    # Fresh cases beyond the fixtures, including rank 4 (kMaxRank, image.hpp:25).
    rng = np.random.default_rng(7)
    for trial in range(40):
        rank = int(rng.integers(1, 5))
        ch = int(rng.integers(1, 4))
        dims = rng.integers(1, 12 if rank < 4 else 6, rank)
        grid = np.array([rng.integers(1, d + 1) for d in dims])
        data = rng.integers(0, 255 * 256, int(np.prod(dims)) * ch) / 256.0
        w = float(rng.integers(1, 80)) / 2
        a = oracle_lib.run_slic(data, dims, ch, grid, w)
        b = reference_lib.run_slic(data, dims, ch, grid, w, workers=3)
        for x, y in zip(a, b):
            assert np.array_equal(np.asarray(x).reshape(-1), np.asarray(y).reshape(-1)), trial
        cc_a = oracle_lib.enforce_connectivity(dims, a[0], a[1], ch, grid)
        cc_b = reference_lib.enforce_connectivity(dims, b[0], b[1], ch, grid, workers=2)
        assert np.array_equal(cc_a, cc_b), trial


def test_oracle_known_answers(oracle_lib):
    o = oracle_lib
    # init_centers known answers (test_slic.cpp:23-45)
    four = o.init_centers(np.zeros(100 * 100), (100, 100), 1, (50, 50))
    assert [tuple(np.rint(r[1:]).astype(int)) for r in four] == [(25, 25), (75, 25), (25, 75),
                                                                 (75, 75)]
    line = o.init_centers(np.zeros(7), (7,), 1, (3,))
    assert list(line[:, 1]) == [1.0, 4.0, 6.0]
    # perturb: constant image -> row-major first pixel (test_slic.cpp:69-73)
    t = o.init_centers(np.zeros(25), (5, 5), 1, (5, 5), perturb=True)
    assert tuple(t[0, 1:]) == (1.0, 1.0)
    # ridge (test_slic.cpp:75-96): argmin at (2,1)
    img = np.array([100.0 if x == 2 else 0.0 for y in range(5) for x in range(5)])
    t = o.init_centers(img, (5, 5), 1, (5, 5), perturb=True)
    assert tuple(t[0, 1:]) == (2.0, 1.0) and t[0, 0] == 100.0
    # squared_distance known answers 0 / 100 / 25 (test_slic.cpp:113-129)
    assert o.distance([10, 20, 3, 4], [10, 20], [3, 4], [7, 5], 10.0) == 0.0
    assert o.distance([10, 20, 3, 4], [10, 20], [10, 4], [7, 5], 10.0) == 100.0
    assert o.distance([50, 10, 5, 2, 2], [53, 14, 5], [2, 2], [7, 5], 10.0) == 25.0
    # gradient known answers (test_color.cpp:85-106)
    ramp = np.array([float(x) for y in range(4) for x in range(5)])
    assert o.gradient_sq(ramp, (5, 4), 1, (2, 1)) == 1.0
    two = np.array([[float(x), 2.0 * y] for y in range(3) for x in range(3)]).reshape(-1)
    assert o.gradient_sq(two, (3, 3), 2, (1, 1)) == 5.0
    # size_threshold (test_connectivity.cpp:31-35)
    assert o.size_threshold((10, 10)) == 25 and o.size_threshold((5, 4, 3)) == 15
    assert o.size_threshold((3,)) == 0


def test_oracle_sweep_known_answers(oracle_lib):
    o = oracle_lib
    # orphan island absorbs the surrounding label (test_connectivity.cpp:136-155)
    lab = np.zeros(36, np.uint32)
    mk = np.ones(36, np.uint8)
    for x, y in [(2, 2), (3, 2), (2, 3), (3, 3)]:
        lab[y * 6 + x] = 9
        mk[y * 6 + x] = 0
    out, mk2, nxt = o.sweep((6, 6), lab, mk, 4, 1)
    assert nxt == 1 and np.all(out == 0) and np.all(mk2 == 1)
    # big non-final component gets a fresh label (test_connectivity.cpp:157-173)
    lab = np.zeros(12, np.uint32)
    mk = np.ones(12, np.uint8)
    for y in range(2):
        for x in range(3, 6):
            lab[y * 6 + x] = 4
            mk[y * 6 + x] = 0
    out, _, nxt = o.sweep((6, 2), lab, mk, 4, 10)
    assert nxt == 11 and all(out[y * 6 + x] == 10 for y in range(2) for x in range(3, 6))


def test_oracle_lab_pinned_and_known_answers(oracle_lib, reference_lib):
    """sRGB -> CIE-Lab (color.hpp:21-66): the C restatement equals the
    unmodified reference bitwise (integral and fractional inputs) and meets
    the reference suite's anchors (test_color.cpp:11-83)."""
    rng = np.random.default_rng(7)
    xi = rng.integers(0, 256, size=(2000, 3)).astype(np.float64)
    xf = rng.uniform(0.0, 255.0, size=(2000, 3))
    for x in (xi, xf):
        assert np.array_equal(oracle_lib.srgb_to_lab(x), reference_lib.convert_to_lab((2000,), x))
    white, black, red = oracle_lib.srgb_to_lab(
        np.array([[255.0, 255, 255], [0, 0, 0], [255, 0, 0]])).reshape(3, 3)
    assert abs(white[0] - 100.0) < 0.01 and abs(white[1]) < 0.01 and abs(white[2]) < 0.01
    assert abs(black[0]) < 1e-12 and black[1] == 0.0 and black[2] == 0.0
    assert np.allclose(red, [53.24, 80.09, 67.20], atol=0.01)
    grays = oracle_lib.srgb_to_lab(np.repeat(np.arange(256.0), 3)).reshape(256, 3)
    assert np.all(np.abs(grays[:, 1:]) < 0.01) and np.all(np.diff(grays[:, 0]) > 0)


def test_oracle_mask_label_contour_known_answers(oracle_lib):
    """mask_label_contour (io.hpp:432-454), the reference suite's cases
    (test_io.cpp:212-262) restated: uniform labels copy through, a 2x1 split
    blacks both pixels, a checkerboard blacks everything, a half split blacks
    exactly the two boundary columns in every channel."""
    rng = np.random.default_rng(5)
    img = rng.integers(0, 256, size=4 * 4 * 3).astype(np.float64)
    assert np.array_equal(oracle_lib.mask_label_contour((4, 4), 3, img, np.full(16, 2)), img)
    assert list(oracle_lib.mask_label_contour((2, 1), 1, [5.0, 6.0], [0, 1])) == [0.0, 0.0]
    x, y = np.meshgrid(np.arange(4), np.arange(4), indexing="xy")
    cb = ((x + y) % 2).reshape(-1)
    assert np.all(oracle_lib.mask_label_contour((4, 4), 1, np.full(16, 200.0), cb) == 0.0)
    img = rng.integers(0, 256, size=8 * 8 * 3).astype(np.float64)
    x, y = np.meshgrid(np.arange(8), np.arange(8), indexing="xy")
    lab = (x >= 4).astype(np.uint32).reshape(-1)
    out = oracle_lib.mask_label_contour((8, 8), 3, img, lab).reshape(64, 3)
    boundary = ((x == 3) | (x == 4)).reshape(-1)
    assert np.all(out[boundary] == 0.0)
    assert np.array_equal(out[~boundary], img.reshape(64, 3)[~boundary])
