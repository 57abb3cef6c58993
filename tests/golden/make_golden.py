"""Generates tests/golden/*.npz from the UNMODIFIED reference.

Runs in the build container only (needs /root/reference to build
oracle/_ref/libsslic_ref.so). The fixtures are committed so the GPU box —
where /root/reference does not exist — checks against the reference's own
outputs. Every case is drawn exactly as the reference test suite draws it
(std::mt19937_64 + libstdc++ distributions, via ref_harness.cpp):

* corpus_acceptance: acceptance.cpp:73-87 make_corpus(seed 0x55110C), first
  N cases (max extent 24), run_slic + enforce_connectivity outputs.
* corpus_run_slic: test_slic.cpp:376-386 (seed 60902, 25 cases, extent 14).
* corpus_connectivity: test_connectivity.cpp:185-197 (seed 90125, 30 cases).
* single_pass: test_slic.cpp:199-246 (seed 2024): one assign pass, labels and
  dists from the reference.
* configlike_*: small seeded images shaped like BASELINE configs 1-5 (native
  dtypes u8/u16/f32), reference run_slic (+ connectivity) outputs.

Usage: python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import Reference  # noqa: E402


def pack_cases(cases):
    """Flattens a list of dict cases into one npz-able dict."""
    out = {"n": np.array(len(cases))}
    for i, c in enumerate(cases):
        for key, v in c.items():
            out[f"{i}_{key}"] = np.asarray(v)
    return out


def corpus_cases(ref, seed, count, max_extent, connectivity=True):
    cases = []
    for data, dims, ch, grid, w in ref.corpus(seed, count, max_extent=max_extent):
        lab, cen, res = ref.run_slic(data, dims, ch, grid, w, workers=2)
        c = {"data_x256": np.round(data * 256).astype(np.uint16), "dims": dims,
             "channels": ch, "grid": grid, "weight_m": w, "labels": lab, "centers": cen,
             "residuals": res}
        assert np.array_equal(c["data_x256"].astype(np.float64) / 256.0, data)
        if connectivity:
            c["labels_cc"] = ref.enforce_connectivity(dims, lab, cen, ch, grid, workers=2)
        cases.append(c)
    return cases


def single_pass_case(ref):
    lib = ref.lib
    rng = lib.ref_rng_new(2024)
    dims = np.zeros(2, np.int64)
    vals = np.zeros(12 * 12)
    import ctypes as C
    lib.ref_random_image(rng, 2, 12, 1, dims.ctypes.data_as(C.POINTER(C.c_int64)),
                         vals.ctypes.data_as(C.POINTER(C.c_double)))
    img = np.array([lib.ref_rng_uniform_int32(rng, 0, 255) for _ in range(144)], np.float64)
    lib.ref_rng_free(rng)
    dims = np.array([12, 12], np.int64)
    grid = np.array([6, 6], np.int64)
    cen = ref.init_centers(img, dims, 1, grid, perturb=False)
    lab, dist = ref.assign_pass(img, dims, 1, grid, 10.0, cen)
    return {"data": img.astype(np.uint8), "dims": dims, "grid": grid, "centers": cen,
            "labels": lab, "dists": dist}


def voronoi(rng, dims, ncells):
    pts = np.stack([rng.uniform(0, d, ncells) for d in dims], 1)
    grids = np.meshgrid(*[np.arange(d) + 0.5 for d in dims], indexing="ij")
    coords = np.stack([g.reshape(-1) for g in grids], 1)
    best = np.full(coords.shape[0], np.inf)
    idx = np.zeros(coords.shape[0], np.int64)
    for i, p in enumerate(pts):
        d = ((coords - p) ** 2).sum(1)
        m = d < best
        best[m] = d[m]
        idx[m] = i
    # meshgrid "ij" puts axis 0 slowest; the reference layout is axis 0 fastest.
    return idx.reshape(dims).transpose(*reversed(range(len(dims)))).reshape(-1)


def configlike(seed):
    rng = np.random.default_rng(seed)
    out = []
    # config-1-like: 2D RGB u8, ramp + noise 8, S=16, m=10
    dims = (128, 96)
    cell = voronoi(rng, dims, 40)
    means = rng.uniform(0, 255, (40, 3))
    x = np.tile(np.arange(dims[0]), dims[1])
    v = means[cell] + (40 * x / dims[0] - 20)[:, None] + rng.normal(0, 8, (cell.size, 3))
    out.append(("c1", np.clip(np.rint(v), 0, 255).astype(np.uint8), dims, 3, (16, 16), 10.0, 0))
    # config-2-like: 2D RGB f32, shading 0.1 + noise 0.03, S=32
    dims = (160, 128)
    cell = voronoi(rng, dims, 60)
    means = rng.uniform(0, 1, (60, 3))
    x = np.tile(np.arange(dims[0]), dims[1])
    y = np.repeat(np.arange(dims[1]), dims[0])
    shade = 0.1 * np.sin(2 * np.pi * x / 64) * np.cos(2 * np.pi * y / 48)
    v = means[cell] + shade[:, None] + rng.normal(0, 0.03, (cell.size, 3))
    out.append(("c2", v.astype(np.float32), dims, 3, (32, 32), 10.0, 0))
    # config-3-like: 3D u16 grey, membranes, Poisson-like noise, S=16 (3 iterations)
    dims = (48, 40, 32)
    cell = voronoi(rng, dims, 30)
    means = rng.uniform(5000, 60000, 30)
    lvl = means[cell]
    v = lvl + np.sqrt(lvl) * rng.normal(0, 1, cell.size)
    out.append(("c3", np.clip(np.rint(v), 0, 65535).astype(np.uint16), dims, 1, (16, 16, 16),
                10.0, 3))
    # config-4-like: 3D 4-ch f32, near-zero channels, S=8, m=20 (3 iterations)
    dims = (32, 24, 16)
    cell = voronoi(rng, dims, 24)
    means = rng.uniform(0, 1, (24, 4))
    dark = rng.uniform(size=24) < 0.3
    for i in np.nonzero(dark)[0]:
        means[i, rng.uniform(size=4) < 0.5] *= 0.02
    v = means[cell] + rng.normal(0, 0.05, (cell.size, 4))
    out.append(("c4", v.astype(np.float32), dims, 4, (8, 8, 8), 20.0, 3))
    # config-5-like: 3D RGB u8, z drift, S=32 (smaller grid: 16), 3 iterations
    dims = (64, 48, 40)
    cell = voronoi(rng, dims, 12)
    means = rng.uniform(20, 235, (12, 3))
    z = np.repeat(np.arange(dims[2]), dims[0] * dims[1])
    drift = np.stack([30 * z / dims[2], -20 * z / dims[2], 0 * z], 1)
    v = means[cell] + drift + rng.normal(0, 6, (cell.size, 3))
    out.append(("c5", np.clip(np.rint(v), 0, 255).astype(np.uint8), dims, 3, (16, 16, 16),
                10.0, 3))
    return out


def main():
    ref = Reference()
    np.savez_compressed(os.path.join(HERE, "corpus_acceptance.npz"),
                        **pack_cases(corpus_cases(ref, 0x55110C, 200, 24)))
    np.savez_compressed(os.path.join(HERE, "corpus_run_slic.npz"),
                        **pack_cases(corpus_cases(ref, 60902, 25, 14, connectivity=False)))
    np.savez_compressed(os.path.join(HERE, "corpus_connectivity.npz"),
                        **pack_cases(corpus_cases(ref, 90125, 30, 12)))
    np.savez_compressed(os.path.join(HERE, "single_pass.npz"), **single_pass_case(ref))
    cases = []
    for name, data, dims, ch, grid, m, iters in configlike(1806):
        dd = np.array(dims, np.int64)
        gg = np.array(grid, np.int64)
        lab, cen, res = ref.run_slic(data.astype(np.float64), dd, ch, gg, m,
                                     max_iterations=iters, workers=4)
        cc = ref.enforce_connectivity(dd, lab, cen, ch, gg, workers=4)
        cases.append({"name": name, "data": data, "dims": dd, "channels": ch, "grid": gg,
                      "weight_m": m, "iterations": iters, "labels": lab, "centers": cen,
                      "residuals": res, "labels_cc": cc})
    np.savez_compressed(os.path.join(HERE, "configlike.npz"), **pack_cases(cases))
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
