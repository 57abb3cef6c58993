"""TEST INFRASTRUCTURE ONLY — numpy front end for the CPU oracle.

Two checkers live here, both CPU-only:

* ``Oracle``    — ctypes binding of ``oracle/liboracle.so``, the plain-C
  restatement of the reference algorithm (``sslic_oracle.c``; every function
  cites the reference file:line it follows).
* ``Reference`` — ctypes binding of ``oracle/_ref/libsslic_ref.so``, the
  UNMODIFIED reference headers behind a C shim (``ref_harness.cpp``), built
  from ``/root/reference`` by ``oracle/Makefile``. Used to pin ``Oracle`` and
  to generate ``tests/golden``; also the CPU baseline of ``bench.py``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package. The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsslic_ref.so")

_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_u32p = C.POINTER(C.c_uint32)
_u8p = C.POINTER(C.c_uint8)


def build(force: bool = False) -> None:
    """Compile liboracle.so (and _ref when /root/reference exists)."""
    if force or not os.path.exists(ORACLE_SO) or (
        os.path.isdir("/root/reference/proj") and not os.path.exists(REF_SO)
    ):
        subprocess.run(["make", "-s", "-C", HERE], check=True)


def _p(a, t):
    return a.ctypes.data_as(t)


def _dims(dims):
    return np.ascontiguousarray(dims, dtype=np.int64)


class Oracle:
    """The C restatement; numpy in, numpy out."""

    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            build()
        lib = C.CDLL(ORACLE_SO)
        lib.orc_cluster_count.restype = C.c_int64
        lib.orc_cluster_count.argtypes = [C.c_int, _i64p, _i64p]
        lib.orc_init_centers.argtypes = [C.c_int, _i64p, C.c_int, _f64p, _i64p, _f64p]
        lib.orc_gradient_sq.restype = C.c_double
        lib.orc_gradient_sq.argtypes = [C.c_int, _i64p, C.c_int, _f64p, _i64p]
        lib.orc_perturb_centers.argtypes = [C.c_int, _i64p, C.c_int, _f64p, _f64p, C.c_int64]
        lib.orc_distance.restype = C.c_double
        lib.orc_distance.argtypes = [_f64p, _f64p, _i64p, C.c_int, C.c_int, _i64p, C.c_double]
        lib.orc_assign.argtypes = [C.c_int, _i64p, C.c_int, _f64p, _f64p, C.c_int64, _i64p,
                                   C.c_double, _u32p, _f64p]
        lib.orc_accumulate.restype = C.c_int
        lib.orc_accumulate.argtypes = [C.c_int, _i64p, C.c_int, _f64p, _u32p, C.c_int64,
                                       C.c_int64, _f64p, _i64p]
        lib.orc_update.restype = C.c_double
        lib.orc_update.argtypes = [_f64p, C.c_int64, C.c_int, _f64p, _i64p]
        lib.orc_run_slic.restype = C.c_int
        lib.orc_run_slic.argtypes = [C.c_int, _i64p, C.c_int, _f64p, _i64p, C.c_double, C.c_int,
                                     C.c_int, C.c_double, _u32p, _f64p, _f64p,
                                     C.POINTER(C.c_int)]
        lib.orc_srgb_to_lab.argtypes = [C.c_int64, _f64p, _f64p]
        lib.orc_mask_label_contour.argtypes = [C.c_int, _i64p, C.c_int, _f64p, _u32p, _f64p]
        lib.orc_size_threshold.restype = C.c_int64
        lib.orc_size_threshold.argtypes = [C.c_int, _i64p]
        lib.orc_finalize.argtypes = [C.c_int, _i64p, _u32p, _f64p, C.c_int, C.c_int64, _i64p,
                                     _u8p]
        lib.orc_sweep.restype = C.c_uint32
        lib.orc_sweep.argtypes = [C.c_int, _i64p, _u32p, _u8p, C.c_int64, C.c_uint32]
        lib.orc_enforce_connectivity.restype = C.c_uint32
        lib.orc_enforce_connectivity.argtypes = [C.c_int, _i64p, _u32p, _f64p, C.c_int,
                                                 C.c_int64, _i64p, _u32p]
        lib.orc_synth_generate.restype = C.c_int
        lib.orc_synth_generate.argtypes = [C.c_int, C.c_int, _i64p, C.c_int, C.c_uint64,
                                           C.c_int64, C.c_int64, C.c_void_p, C.c_int]
        self.lib = lib

    def synth_generate(self, config, dims, dtype, channels, seed, z_begin=0, z_end=None,
                       threads=None):
        """Planes [z_begin, z_end) of a seeded config volume (the device
        generator's bytes), as a flat numpy array of the native dtype."""
        d = _dims(dims)
        if len(dims) == 2:
            z_begin, z_end = 0, 1
        elif z_end is None:
            z_end = int(dims[-1])
        plane = int(np.prod(dims[:2])) if len(dims) == 3 else int(np.prod(dims))
        out = np.empty(plane * (z_end - z_begin) * channels, dtype=dtype)
        st = self.lib.orc_synth_generate(int(config), len(d), _p(d, _i64p), int(channels),
                                         int(seed), int(z_begin), int(z_end),
                                         out.ctypes.data_as(C.c_void_p),
                                         int(threads or os.cpu_count() or 1))
        if st != 0:
            raise ValueError(f"synth_generate: bad shape for config {config}")
        return out

    # -- helpers -----------------------------------------------------------
    @staticmethod
    def _img(data, dims, channels):
        d = np.ascontiguousarray(data, dtype=np.float64).reshape(-1)
        assert d.size == int(np.prod(dims)) * channels
        return d

    def cluster_count(self, dims, grid):
        dims, grid = _dims(dims), _dims(grid)
        return int(self.lib.orc_cluster_count(len(dims), _p(dims, _i64p), _p(grid, _i64p)))

    def init_centers(self, data, dims, channels, grid, perturb=False):
        dims, grid = _dims(dims), _dims(grid)
        d = self._img(data, dims, channels)
        k = self.cluster_count(dims, grid)
        c = np.zeros(k * (channels + len(dims)), dtype=np.float64)
        self.lib.orc_init_centers(len(dims), _p(dims, _i64p), channels, _p(d, _f64p),
                                  _p(grid, _i64p), _p(c, _f64p))
        if perturb:
            self.lib.orc_perturb_centers(len(dims), _p(dims, _i64p), channels, _p(d, _f64p),
                                         _p(c, _f64p), k)
        return c.reshape(k, channels + len(dims))

    def perturb_centers(self, data, dims, channels, centers):
        dims = _dims(dims)
        d = self._img(data, dims, channels)
        c = np.ascontiguousarray(centers, dtype=np.float64).copy()
        self.lib.orc_perturb_centers(len(dims), _p(dims, _i64p), channels, _p(d, _f64p),
                                     _p(c, _f64p), c.shape[0])
        return c

    def gradient_sq(self, data, dims, channels, coord):
        dims = _dims(dims)
        d = self._img(data, dims, channels)
        co = _dims(coord)
        return self.lib.orc_gradient_sq(len(dims), _p(dims, _i64p), channels, _p(d, _f64p),
                                        _p(co, _i64p))

    def distance(self, center, pixel, coord, grid, weight_m):
        center = np.ascontiguousarray(center, dtype=np.float64)
        pixel = np.ascontiguousarray(pixel, dtype=np.float64)
        coord, grid = _dims(coord), _dims(grid)
        return self.lib.orc_distance(_p(center, _f64p), _p(pixel, _f64p), _p(coord, _i64p),
                                     pixel.size, coord.size, _p(grid, _i64p),
                                     float(weight_m) * float(weight_m))

    def assign(self, data, dims, channels, centers, grid, weight_m, labels=None, dists=None):
        dims, grid = _dims(dims), _dims(grid)
        d = self._img(data, dims, channels)
        n = int(np.prod(dims))
        c = np.ascontiguousarray(centers, dtype=np.float64)
        lab = (np.full(n, 0xFFFFFFFF, np.uint32) if labels is None
               else np.ascontiguousarray(labels, dtype=np.uint32).reshape(-1).copy())
        dis = (np.full(n, np.inf) if dists is None
               else np.ascontiguousarray(dists, dtype=np.float64).reshape(-1).copy())
        self.lib.orc_assign(len(dims), _p(dims, _i64p), channels, _p(d, _f64p), _p(c, _f64p),
                            c.shape[0], _p(grid, _i64p), float(weight_m), _p(lab, _u32p),
                            _p(dis, _f64p))
        return lab, dis

    def accumulate(self, data, dims, channels, labels, k, slab_rows=0):
        dims = _dims(dims)
        d = self._img(data, dims, channels)
        lab = np.ascontiguousarray(labels, dtype=np.uint32).reshape(-1)
        s = np.zeros(k * (channels + len(dims)))
        cnt = np.zeros(k, dtype=np.int64)
        st = self.lib.orc_accumulate(len(dims), _p(dims, _i64p), channels, _p(d, _f64p),
                                     _p(lab, _u32p), k, slab_rows, _p(s, _f64p), _p(cnt, _i64p))
        if st == -1:
            raise RuntimeError("accumulate: pixel with undefined label")
        if st == -2:
            raise RuntimeError("accumulate: label out of range")
        return s.reshape(k, -1), cnt

    def update(self, centers, sums, counts):
        c = np.ascontiguousarray(centers, dtype=np.float64).copy()
        s = np.ascontiguousarray(sums, dtype=np.float64)
        cnt = np.ascontiguousarray(counts, dtype=np.int64)
        r = self.lib.orc_update(_p(c, _f64p), c.shape[0], c.shape[1], _p(s, _f64p),
                                _p(cnt, _i64p))
        return c, r

    def run_slic(self, data, dims, channels, grid, weight_m=10.0, max_iterations=0,
                 residual_threshold=None):
        dims, grid = _dims(dims), _dims(grid)
        d = self._img(data, dims, channels)
        n = int(np.prod(dims))
        k = self.cluster_count(dims, grid)
        iters = max_iterations if max_iterations > 0 else (10 if len(dims) <= 2 else 5)
        lab = np.empty(n, np.uint32)
        cen = np.empty(k * (channels + len(dims)))
        res = np.empty(iters)
        done = C.c_int(0)
        st = self.lib.orc_run_slic(len(dims), _p(dims, _i64p), channels, _p(d, _f64p),
                                   _p(grid, _i64p), float(weight_m), int(max_iterations),
                                   int(residual_threshold is not None),
                                   float(residual_threshold or 0.0), _p(lab, _u32p),
                                   _p(cen, _f64p), _p(res, _f64p), C.byref(done))
        if st == -3:
            raise ValueError("invalid parameters")
        if st == -1:
            raise RuntimeError("pixel with undefined label")
        return lab, cen.reshape(k, -1), res[: done.value]

    def mask_label_contour(self, dims, channels, img, labels):
        dims = _dims(dims)
        d = np.ascontiguousarray(img, dtype=np.float64).reshape(-1)
        lab = np.ascontiguousarray(labels, dtype=np.uint32).reshape(-1)
        out = np.empty_like(d)
        self.lib.orc_mask_label_contour(len(dims), _p(dims, _i64p), channels, _p(d, _f64p),
                                        _p(lab, _u32p), _p(out, _f64p))
        return out

    def srgb_to_lab(self, rgb):
        """orc_srgb_to_lab: interleaved RGB (n*3) -> Lab (n*3)."""
        d = np.ascontiguousarray(rgb, dtype=np.float64).reshape(-1)
        out = np.empty_like(d)
        self.lib.orc_srgb_to_lab(d.size // 3, _p(d, _f64p), _p(out, _f64p))
        return out

    def size_threshold(self, grid):
        grid = _dims(grid)
        return int(self.lib.orc_size_threshold(len(grid), _p(grid, _i64p)))

    def finalize(self, dims, labels, centers, channels, grid):
        dims, grid = _dims(dims), _dims(grid)
        lab = np.ascontiguousarray(labels, dtype=np.uint32).reshape(-1)
        c = np.ascontiguousarray(centers, dtype=np.float64)
        mk = np.zeros(lab.size, np.uint8)
        self.lib.orc_finalize(len(dims), _p(dims, _i64p), _p(lab, _u32p), _p(c, _f64p),
                              channels, c.shape[0], _p(grid, _i64p), _p(mk, _u8p))
        return mk

    def sweep(self, dims, labels, markers, min_size, k_start):
        dims = _dims(dims)
        lab = np.ascontiguousarray(labels, dtype=np.uint32).reshape(-1).copy()
        mk = np.ascontiguousarray(markers, dtype=np.uint8).reshape(-1).copy()
        nxt = self.lib.orc_sweep(len(dims), _p(dims, _i64p), _p(lab, _u32p), _p(mk, _u8p),
                                 int(min_size), int(k_start))
        return lab, mk, int(nxt)

    def enforce_connectivity(self, dims, labels, centers, channels, grid, return_next=False):
        dims, grid = _dims(dims), _dims(grid)
        lab = np.ascontiguousarray(labels, dtype=np.uint32).reshape(-1)
        c = np.ascontiguousarray(centers, dtype=np.float64)
        out = np.empty_like(lab)
        nxt = self.lib.orc_enforce_connectivity(len(dims), _p(dims, _i64p), _p(lab, _u32p),
                                                _p(c, _f64p), channels, c.shape[0],
                                                _p(grid, _i64p), _p(out, _u32p))
        return (out, int(nxt)) if return_next else out


class Reference:
    """The unmodified reference headers behind ref_harness.cpp."""

    def __init__(self):
        if not os.path.exists(REF_SO):
            build()
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        lib = C.CDLL(REF_SO)
        lib.ref_run_slic.restype = C.c_int
        lib.ref_run_slic.argtypes = [C.c_int, _i64p, C.c_int, _f64p, _i64p, C.c_double, C.c_int,
                                     C.c_int, C.c_double, C.c_int, _u32p, _f64p, _f64p,
                                     C.POINTER(C.c_int)]
        lib.ref_init_perturb.restype = C.c_int
        lib.ref_init_perturb.argtypes = [C.c_int, _i64p, C.c_int, _f64p, _i64p, C.c_int, _f64p]
        lib.ref_assign_pass.restype = C.c_int
        lib.ref_assign_pass.argtypes = [C.c_int, _i64p, C.c_int, _f64p, _i64p, C.c_double,
                                        _f64p, C.c_int64, _u32p, _f64p]
        lib.ref_enforce_connectivity.restype = C.c_int
        lib.ref_enforce_connectivity.argtypes = [C.c_int, _i64p, _u32p, C.c_int, _f64p,
                                                 C.c_int64, _i64p, C.c_int, _u32p]
        lib.ref_rng_new.restype = C.c_void_p
        lib.ref_rng_new.argtypes = [C.c_uint64]
        lib.ref_rng_free.argtypes = [C.c_void_p]
        lib.ref_rng_raw.restype = C.c_uint64
        lib.ref_rng_raw.argtypes = [C.c_void_p]
        lib.ref_rng_uniform_int.restype = C.c_int64
        lib.ref_rng_uniform_int.argtypes = [C.c_void_p, C.c_int64, C.c_int64]
        lib.ref_rng_uniform_int32.restype = C.c_int
        lib.ref_rng_uniform_int32.argtypes = [C.c_void_p, C.c_int, C.c_int]
        lib.ref_random_image.restype = C.c_int64
        lib.ref_random_image.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_int, _i64p, _f64p]
        lib.ref_random_grid.argtypes = [C.c_void_p, C.c_int, _i64p, _i64p]
        lib.ref_random_weight.restype = C.c_double
        lib.ref_random_weight.argtypes = [C.c_void_p]
        lib.ref_scaling_report.restype = C.c_int
        lib.ref_scaling_report.argtypes = [C.c_int, C.POINTER(C.c_int), _f64p, C.POINTER(C.c_int),
                                           C.POINTER(C.c_double), _f64p, _f64p, C.c_char_p,
                                           C.c_int64, C.c_char_p, C.c_int64]
        lib.ref_amdahl_bound.restype = C.c_double
        lib.ref_amdahl_bound.argtypes = [C.c_double, C.c_int]
        lib.ref_amdahl_efficiency_bound.restype = C.c_double
        lib.ref_amdahl_efficiency_bound.argtypes = [C.c_double, C.c_int]
        lib.ref_convert_to_lab.restype = C.c_int
        lib.ref_convert_to_lab.argtypes = [C.c_int, _i64p, _f64p, _f64p]
        lib.ref_time_iterations.restype = C.c_int
        lib.ref_time_iterations.argtypes = [C.c_int, _i64p, C.c_int, _f64p, _i64p, C.c_double,
                                            C.c_int, C.c_int, _f64p, _f64p, _u32p, _f64p]
        self.lib = lib

    def run_slic(self, data, dims, channels, grid, weight_m=10.0, max_iterations=0,
                 residual_threshold=None, workers=1):
        dims, grid = _dims(dims), _dims(grid)
        d = np.ascontiguousarray(data, dtype=np.float64).reshape(-1)
        n = int(np.prod(dims))
        k = int(np.prod([(a + s - 1) // s for a, s in zip(dims, grid)]))
        iters = max_iterations if max_iterations > 0 else (10 if len(dims) <= 2 else 5)
        lab = np.empty(n, np.uint32)
        cen = np.empty(k * (channels + len(dims)))
        res = np.empty(iters)
        done = C.c_int(0)
        st = self.lib.ref_run_slic(len(dims), _p(dims, _i64p), channels, _p(d, _f64p),
                                   _p(grid, _i64p), float(weight_m), int(max_iterations),
                                   int(residual_threshold is not None),
                                   float(residual_threshold or 0.0), int(workers),
                                   _p(lab, _u32p), _p(cen, _f64p), _p(res, _f64p),
                                   C.byref(done))
        if st != 0:
            raise RuntimeError(f"reference run_slic failed with status {st}")
        return lab, cen.reshape(k, -1), res[: done.value]

    def init_centers(self, data, dims, channels, grid, perturb=False):
        dims, grid = _dims(dims), _dims(grid)
        d = np.ascontiguousarray(data, dtype=np.float64).reshape(-1)
        k = int(np.prod([(a + s - 1) // s for a, s in zip(dims, grid)]))
        cen = np.empty(k * (channels + len(dims)))
        st = self.lib.ref_init_perturb(len(dims), _p(dims, _i64p), channels, _p(d, _f64p),
                                       _p(grid, _i64p), int(perturb), _p(cen, _f64p))
        if st != 0:
            raise RuntimeError(f"reference init failed with status {st}")
        return cen.reshape(k, -1)

    def assign_pass(self, data, dims, channels, grid, weight_m, centers, labels=None,
                    dists=None):
        dims, grid = _dims(dims), _dims(grid)
        d = np.ascontiguousarray(data, dtype=np.float64).reshape(-1)
        n = int(np.prod(dims))
        c = np.ascontiguousarray(centers, dtype=np.float64)
        lab = (np.full(n, 0xFFFFFFFF, np.uint32) if labels is None
               else np.ascontiguousarray(labels, dtype=np.uint32).reshape(-1).copy())
        dis = (np.full(n, np.inf) if dists is None
               else np.ascontiguousarray(dists, dtype=np.float64).reshape(-1).copy())
        st = self.lib.ref_assign_pass(len(dims), _p(dims, _i64p), channels, _p(d, _f64p),
                                      _p(grid, _i64p), float(weight_m), _p(c, _f64p),
                                      c.shape[0], _p(lab, _u32p), _p(dis, _f64p))
        if st != 0:
            raise RuntimeError(f"reference assign failed with status {st}")
        return lab, dis

    def enforce_connectivity(self, dims, labels, centers, channels, grid, workers=1):
        dims, grid = _dims(dims), _dims(grid)
        lab = np.ascontiguousarray(labels, dtype=np.uint32).reshape(-1)
        c = np.ascontiguousarray(centers, dtype=np.float64)
        out = np.empty_like(lab)
        st = self.lib.ref_enforce_connectivity(len(dims), _p(dims, _i64p), _p(lab, _u32p),
                                               channels, _p(c, _f64p), c.shape[0],
                                               _p(grid, _i64p), int(workers), _p(out, _u32p))
        if st != 0:
            raise RuntimeError(f"reference connectivity failed with status {st}")
        return out

    def scaling_report(self, workers, times, conn):
        """bench.hpp make_report + emit_scaling_csv/markdown of the reference."""
        n = len(workers)
        w = np.asarray(workers, np.int32)
        t = np.asarray(times, np.float64)
        c = np.asarray(conn, np.int32)
        alpha = C.c_double()
        sp, ef = np.empty(n), np.empty(n)
        csv = C.create_string_buffer(1 << 16)
        md = C.create_string_buffer(1 << 16)
        st = self.lib.ref_scaling_report(n, w.ctypes.data_as(C.POINTER(C.c_int)), _p(t, _f64p),
                                         c.ctypes.data_as(C.POINTER(C.c_int)), C.byref(alpha),
                                         _p(sp, _f64p), _p(ef, _f64p), csv, 1 << 16, md, 1 << 16)
        if st != 0:
            raise ValueError(f"reference scaling report failed with status {st}")
        return alpha.value, sp, ef, csv.value.decode(), md.value.decode()

    def convert_to_lab(self, dims, rgb):
        """convert_image_to_lab (color.hpp:54-66) of the unmodified reference."""
        dims = _dims(dims)
        d = np.ascontiguousarray(rgb, dtype=np.float64).reshape(-1)
        out = np.empty_like(d)
        st = self.lib.ref_convert_to_lab(len(dims), _p(dims, _i64p), _p(d, _f64p), _p(out, _f64p))
        if st != 0:
            raise ValueError(f"reference convert_image_to_lab failed with status {st}")
        return out

    def time_iterations(self, data, dims, channels, grid, weight_m, iterations, workers):
        dims, grid = _dims(dims), _dims(grid)
        d = np.ascontiguousarray(data, dtype=np.float64).reshape(-1)
        ti = C.c_double(0)
        tt = np.zeros(max(int(iterations), 1))
        st = self.lib.ref_time_iterations(len(dims), _p(dims, _i64p), channels, _p(d, _f64p),
                                          _p(grid, _i64p), float(weight_m), int(iterations),
                                          int(workers), C.byref(ti), _p(tt, _f64p), None, None)
        if st != 0:
            raise RuntimeError(f"reference timing failed with status {st}")
        return ti.value, list(tt[: int(iterations)])

    # -- the reference test-suite corpora (std::mt19937_64, libstdc++) ------
    def corpus(self, seed, count, rank_range=(1, 3), max_extent=24, channels_rule="parity",
               connectivity_seed=False):
        """Replays the draw order of acceptance.cpp:73-87 (make_corpus) /
        test_slic.cpp:376-386: rank, channels, random_image, random_grid,
        random_weight. Yields (data, dims, channels, grid, weight_m)."""
        lib = self.lib
        rng = lib.ref_rng_new(seed)
        try:
            for _ in range(count):
                rank = lib.ref_rng_uniform_int32(rng, rank_range[0], rank_range[1])
                channels = 1 if lib.ref_rng_raw(rng) % 2 == 0 else 3
                dims = np.zeros(rank, np.int64)
                vals = np.zeros(max_extent ** rank * channels)
                n = lib.ref_random_image(rng, rank, max_extent, channels, _p(dims, _i64p),
                                         _p(vals, _f64p))
                grid = np.zeros(rank, np.int64)
                lib.ref_random_grid(rng, rank, _p(dims, _i64p), _p(grid, _i64p))
                w = lib.ref_random_weight(rng)
                yield vals[: n * channels].copy(), dims.copy(), channels, grid.copy(), w
        finally:
            lib.ref_rng_free(rng)
