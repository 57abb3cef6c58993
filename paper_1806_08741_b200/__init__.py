"""B200-native SSLIC hot path — Python mirror of the reference C++ interface.

The reference (``/root/reference/proj/include/sslic``) is a header-only C++
library; its public surface for the hot path is ``SlicParams``, ``NDImage``,
``ClusterTable``, ``run_slic``, ``enforce_connectivity`` and the lower-level
``init_centers`` / ``perturb_centers`` / ``assign_labels`` /
``accumulate_region`` / ``reduce_and_update`` / ``squared_distance`` /
``gradient_magnitude_sq`` / ``size_threshold``. This module mirrors those names,
argument meanings and error classes (``InvalidArgument`` for
``std::invalid_argument``, ``LogicError`` for ``std::logic_error``,
``OutOfRange`` for ``std::out_of_range``) on top of the C ABI in
``include/sslic_b200.h``, implemented by the CUDA library
``libsslic_b200.so`` built in-tree for sm_100a.

There is no CPU fallback: if the library or a CUDA device is missing, every
compute entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

__all__ = [
    "NDImage", "SlicParams", "ClusterTable", "SlicResult", "Engine",
    "run_slic", "segment", "enforce_connectivity", "init_centers", "perturb_centers",
    "assign_labels", "accumulate_region", "reduce_and_update", "squared_distance",
    "gradient_magnitude_sq", "size_threshold", "cluster_count", "synth_generate",
    "InvalidArgument", "LogicError", "OutOfRange", "CudaError", "UNDEFINED", "lib",
]

HERE = os.path.dirname(os.path.abspath(__file__))
# (SSLIC_B200_LIB: another in-tree build of the same library, for A/B timing)
LIB_PATH = os.environ.get("SSLIC_B200_LIB") or os.path.join(HERE, "libsslic_b200.so")
UNDEFINED = 0xFFFFFFFF  # LabelMap::kUndefined (image.hpp:291)

U8, U16, F32, F64 = 0, 1, 2, 3
_DT = {np.dtype(np.uint8): U8, np.dtype(np.uint16): U16, np.dtype(np.float32): F32,
       np.dtype(np.float64): F64}


class InvalidArgument(ValueError):
    """std::invalid_argument"""


class LogicError(RuntimeError):
    """std::logic_error"""


class OutOfRange(IndexError):
    """std::out_of_range"""


class CudaError(RuntimeError):
    """CUDA failure or no usable device (there is no CPU fallback)."""


class IoError(OSError):
    """io_error (io.hpp:40-56); ``code`` is the io_errc name."""

    def __init__(self, code: str, msg: str):
        super().__init__(msg)
        self.code = code


_IO_CODES = {-10: "file_not_found", -11: "malformed_header", -12: "size_mismatch",
             -13: "unsupported_type", -14: "write_failed"}


class _VolumeInfo(C.Structure):
    _fields_ = [("rank", C.c_int), ("dims", C.c_int64 * 4), ("channels", C.c_int),
                ("dtype", C.c_int), ("label_map", C.c_int)]


class _Image(C.Structure):
    _fields_ = [("rank", C.c_int), ("dims", C.c_int64 * 4), ("channels", C.c_int),
                ("dtype", C.c_int), ("data", C.c_void_p)]


class _Params(C.Structure):
    _fields_ = [("grid", C.c_int64 * 4), ("weight_m", C.c_double), ("max_iterations", C.c_int),
                ("enforce_connectivity", C.c_int), ("has_residual_threshold", C.c_int),
                ("residual_threshold", C.c_double)]


_lib = None


def lib():
    """Loads libsslic_b200.so (fails loudly when it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA library first "
            "(python -c 'import __graft_entry__ as g; g.build()')")
    L = C.CDLL(LIB_PATH)
    i64p, f64p, u32p = C.POINTER(C.c_int64), C.POINTER(C.c_double), C.POINTER(C.c_uint32)
    ip, vp = C.POINTER(_Image), C.c_void_p
    pp = C.POINTER(_Params)
    sig = {
        "sslic_last_error": (C.c_char_p, []),
        "sslic_version": (C.c_char_p, []),
        "sslic_cluster_count": (C.c_int64, [C.c_int, i64p, i64p]),
        "sslic_iterations_for": (C.c_int, [pp, C.c_int]),
        "sslic_run_slic": (C.c_int, [ip, pp, C.c_int, u32p, f64p, f64p, C.POINTER(C.c_int)]),
        "sslic_segment": (C.c_int, [ip, pp, C.c_int, u32p, f64p, f64p, C.POINTER(C.c_int),
                                    u32p]),
        "sslic_init_centers": (C.c_int, [ip, pp, C.c_int, C.c_int, f64p]),
        "sslic_perturb_centers": (C.c_int, [ip, f64p, C.c_int64, C.c_int]),
        "sslic_gradient_sq": (C.c_int, [ip, i64p, C.c_int64, C.c_int, f64p]),
        "sslic_convert_image_to_lab": (C.c_int, [ip, C.c_int, f64p]),
        "sslic_mask_label_contour": (C.c_int, [ip, C.c_int, i64p, u32p, C.c_int, f64p]),
        "sslic_volume_info_read": (C.c_int, [C.c_char_p, C.POINTER(_VolumeInfo)]),
        "sslic_volume_read": (C.c_int, [C.c_char_p, C.c_int64, C.c_int64, vp, C.c_int]),
        "sslic_volume_write": (C.c_int, [C.c_char_p, ip]),
        "sslic_labels_write": (C.c_int, [C.c_char_p, C.c_int, i64p, u32p]),
        "sslic_labels_read": (C.c_int, [C.c_char_p, u32p]),
        "sslic_squared_distance": (C.c_int, [C.c_int, C.c_int, i64p, C.c_double, C.c_int64,
                                             f64p, f64p, i64p, C.c_int, f64p]),
        "sslic_assign_pass": (C.c_int, [ip, pp, f64p, C.c_int64, C.c_int, u32p, f64p]),
        "sslic_accumulate": (C.c_int, [ip, u32p, C.c_int64, C.c_int, f64p, i64p]),
        "sslic_reduce_and_update": (C.c_int, [f64p, C.c_int64, C.c_int, f64p, i64p, C.c_int,
                                              f64p]),
        "sslic_enforce_connectivity": (C.c_int, [C.c_int, i64p, u32p, f64p, C.c_int, C.c_int64,
                                                 i64p, C.c_int, u32p, u32p]),
        "sslic_engine_create": (C.c_int, [ip, pp, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                                          C.c_int64, vp, C.POINTER(vp)]),
        "sslic_engine_destroy": (C.c_int, [vp]),
        "sslic_engine_value_range": (C.c_int, [vp, C.POINTER(C.c_double)]),
        "sslic_engine_set_value_range": (C.c_int, [vp, C.c_double]),
        "sslic_engine_init": (C.c_int, [vp]),
        "sslic_engine_reset": (C.c_int, [vp]),
        "sslic_engine_centers_buffer": (C.c_int, [vp, C.POINTER(vp), i64p]),
        "sslic_engine_commit_centers": (C.c_int, [vp]),
        "sslic_engine_assign": (C.c_int, [vp]),
        "sslic_engine_partials": (C.c_int, [vp, C.POINTER(vp), i64p]),
        "sslic_engine_update": (C.c_int, [vp]),
        "sslic_engine_iterate": (C.c_int, [vp, C.c_int]),
        "sslic_engine_iterate_graph": (C.c_int, [vp, C.c_int, C.POINTER(C.c_float)]),
        "sslic_engine_iterations_done": (C.c_int, [vp]),
        "sslic_engine_residuals": (C.c_int, [vp, f64p]),
        "sslic_engine_labels": (C.c_int, [vp, vp]),
        "sslic_engine_centers": (C.c_int, [vp, f64p]),
        "sslic_engine_undefined_count": (C.c_int64, [vp]),
        "sslic_engine_launch_count": (C.c_int64, [vp]),
        "sslic_engine_eval_stats": (C.c_int, [vp, f64p, f64p]),
        "sslic_engine_set_stats": (C.c_int, [vp, C.c_int]),
        "sslic_engine_set_exact": (C.c_int, [vp, C.c_int]),
        "sslic_engine_fast_stats": (C.c_int, [vp, f64p, f64p, f64p]),
        "sslic_engine_assign_ms": (C.c_int, [vp, C.c_int, C.POINTER(C.c_float),
                                             C.POINTER(C.c_int)]),
        "sslic_synth_generate": (C.c_int, [C.c_int, C.c_int, i64p, C.c_int, C.c_int, C.c_uint64,
                                           C.c_int64, C.c_int64, vp, vp]),
        "sslic_run_slic_multi": (C.c_int, [ip, pp, C.c_int, C.POINTER(C.c_int), u32p, f64p, f64p,
                                           C.POINTER(C.c_int)]),
        "sslic_run_slic_rank": (C.c_int, [ip, pp, C.c_int, C.c_int, vp, C.c_int, C.c_int64, u32p,
                                          f64p, f64p, C.POINTER(C.c_int)]),
        "sslic_device_count": (C.c_int, []),
        "sslic_segment_write": (C.c_int, [ip, pp, C.c_int, C.c_char_p, C.c_char_p, f64p, f64p,
                                          C.POINTER(C.c_int), u32p]),
        "sslic_nccl_unique_id": (C.c_int, [vp, C.c_int64]),
        "sslic_slab_bounds": (C.c_int, [C.c_int64, C.c_int, C.c_int, C.c_int64, i64p, i64p]),
        "sslic_engine_attach_nccl": (C.c_int, [vp, vp, C.c_int, C.c_int]),
        "sslic_engine_start": (C.c_int, [vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def _check(status: int) -> None:
    if status == 0:
        return
    msg = lib().sslic_last_error().decode(errors="replace")
    if status == -1:
        raise InvalidArgument(msg)
    if status == -2:
        raise LogicError(msg)
    if status == -3:
        raise OutOfRange(msg)
    if status == -5:
        raise MemoryError(msg)
    if status in _IO_CODES:
        raise IoError(_IO_CODES[status], msg)
    raise CudaError(f"status {status}: {msg}")


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


# --------------------------------------------------------------------------
# Types (image.hpp:236-338, slic.hpp:34-103)
# --------------------------------------------------------------------------
class NDImage:
    """n-dimensional image, axis 0 fastest, channels interleaved
    (image.hpp:1-5, 236-285). ``data`` keeps its native dtype (uint8, uint16,
    float32 or float64); conversion to the reference's fp64 is exact."""

    def __init__(self, dims: Sequence[int], channels: int, data):
        dims = tuple(int(d) for d in dims)
        if len(dims) < 1 or len(dims) > 4:
            raise InvalidArgument("NDImage: rank must be in [1, 4]")
        if any(d < 1 for d in dims):
            raise InvalidArgument("NDImage: extents must be positive")
        if channels < 1:
            raise InvalidArgument("NDImage: channels must be >= 1")
        arr = np.asarray(data)
        if arr.dtype not in _DT:
            arr = arr.astype(np.float64)
        arr = np.ascontiguousarray(arr).reshape(-1)
        if arr.size != channels * int(np.prod(dims)):
            raise InvalidArgument("NDImage: data length must be channels * product(dims)")
        if arr.dtype.kind == "f" and not np.all(np.isfinite(arr)):
            raise InvalidArgument("NDImage: non-finite value")
        self.dims, self.channels, self.data = dims, int(channels), arr

    @staticmethod
    def zeros(dims, channels):
        return NDImage(dims, channels, np.zeros(int(np.prod(dims)) * channels))

    @property
    def rank(self):
        return len(self.dims)

    def pixel_count(self):
        return int(np.prod(self.dims))

    def _desc(self, data_ptr=None):
        d = _Image()
        d.rank = self.rank
        for a in range(4):
            d.dims[a] = self.dims[a] if a < self.rank else 1
        d.channels = self.channels
        d.dtype = _DT[self.data.dtype]
        d.data = self.data.ctypes.data if data_ptr is None else data_ptr
        return d


@dataclass
class SlicParams:
    """SlicParams (slic.hpp:34-65)."""
    grid: Sequence[int]
    weight_m: float = 10.0
    max_iterations: int = 0
    enforce_connectivity: bool = True
    residual_threshold: Optional[float] = None

    def iterations_for(self, rank: int) -> int:
        if self.max_iterations > 0:
            return self.max_iterations
        return 10 if rank <= 2 else 5

    def validate(self, dims):
        if len(self.grid) != len(dims):
            raise InvalidArgument("SlicParams: grid rank does not match image rank")
        for i, (s, d) in enumerate(zip(self.grid, dims)):
            if s < 1:
                raise InvalidArgument("SlicParams: grid sizes must be >= 1")
            if s > d:
                raise InvalidArgument(f"SlicParams: grid size exceeds image extent on axis {i}")
        if not self.weight_m > 0.0:
            raise InvalidArgument("SlicParams: weight_m must be positive")
        if self.max_iterations < 0:
            raise InvalidArgument(
                "SlicParams: max_iterations must be positive (or 0 for default)")

    def _c(self):
        p = _Params()
        for a in range(4):
            p.grid[a] = int(self.grid[a]) if a < len(self.grid) else 1
        p.weight_m = float(self.weight_m)
        p.max_iterations = int(self.max_iterations)
        p.enforce_connectivity = int(bool(self.enforce_connectivity))
        p.has_residual_threshold = int(self.residual_threshold is not None)
        p.residual_threshold = float(self.residual_threshold or 0.0)
        return p


class ClusterTable:
    """k x (c + n) fp64 centres [intensity | index coords] (slic.hpp:69-103)."""

    def __init__(self, channels: int, rank: int, count_or_data):
        self.channels, self.rank = int(channels), int(rank)
        if np.isscalar(count_or_data):
            self.data = np.zeros((int(count_or_data), self.stride()), np.float64)
        else:
            self.data = np.ascontiguousarray(count_or_data, np.float64).reshape(-1, self.stride())

    def stride(self):
        return self.channels + self.rank

    def count(self):
        return self.data.shape[0]

    def center(self, k):
        return self.data[k]

    def coordinate(self, k, axis):
        return self.data[k, self.channels + axis]

    def __eq__(self, o):
        return (isinstance(o, ClusterTable) and self.channels == o.channels
                and self.rank == o.rank and np.array_equal(self.data, o.data))


@dataclass
class SlicResult:
    """SlicResult (slic.hpp:374-378); labels are the flat LabelMap."""
    labels: np.ndarray
    centers: ClusterTable
    residuals: list = field(default_factory=list)


def size_threshold(grid) -> int:
    """connectivity.hpp:34-38"""
    return int(np.prod([int(s) for s in grid])) // 4


def cluster_count(dims, grid) -> int:
    d = np.asarray(dims, np.int64)
    g = np.asarray(grid, np.int64)
    return int(lib().sslic_cluster_count(len(d), _p(d, C.c_int64), _p(g, C.c_int64)))


# --------------------------------------------------------------------------
# Entry points (each runs the CUDA path on `device`)
# --------------------------------------------------------------------------
def run_slic(img: NDImage, params: SlicParams, workers: int = 1, device: int = 0) -> SlicResult:
    """run_slic (slic.hpp:384-415). `workers` is accepted for signature
    parity and must be >= 1 (slic.hpp:386); the device does the work."""
    params.validate(img.dims)
    if workers < 1:
        raise InvalidArgument("run_slic: workers must be >= 1")
    L = lib()
    n = img.pixel_count()
    k = cluster_count(img.dims, params.grid)
    iters = params.iterations_for(img.rank)
    labels = np.empty(n, np.uint32)
    centers = np.empty(k * (img.channels + img.rank))
    res = np.empty(max(iters, 1))
    done = C.c_int(0)
    d, p = img._desc(), params._c()
    _check(L.sslic_run_slic(C.byref(d), C.byref(p), device, _p(labels, C.c_uint32),
                            _p(centers, C.c_double), _p(res, C.c_double), C.byref(done)))
    return SlicResult(labels, ClusterTable(img.channels, img.rank, centers),
                      list(res[: done.value]))


def run_slic_multi(img: NDImage, params: SlicParams, devices: Sequence[int]) -> SlicResult:
    """run_slic over several GPUs of this process (sslic_run_slic_multi):
    z-slabs of a 3-D volume, one per device, one NCCL allreduce of the int64
    per-cluster partials per iteration; bitwise the single-GPU result."""
    params.validate(img.dims)
    L = lib()
    n = img.pixel_count()
    k = cluster_count(img.dims, params.grid)
    iters = params.iterations_for(img.rank)
    labels = np.empty(n, np.uint32)
    centers = np.empty(k * (img.channels + img.rank))
    res = np.empty(max(iters, 1))
    done = C.c_int(0)
    devs = (C.c_int * len(devices))(*[int(d) for d in devices])
    d, p = img._desc(), params._c()
    _check(L.sslic_run_slic_multi(C.byref(d), C.byref(p), len(devices), devs,
                                  _p(labels, C.c_uint32), _p(centers, C.c_double),
                                  _p(res, C.c_double), C.byref(done)))
    return SlicResult(labels, ClusterTable(img.channels, img.rank, centers),
                      list(res[: done.value]))


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId (128 bytes), to be shared with every rank."""
    buf = C.create_string_buffer(128)
    _check(lib().sslic_nccl_unique_id(buf, 128))
    return buf.raw


def slab_bounds_native(last: int, world: int, rank: int, align: int = 1):
    """The C ABI's z-slab split (sslic_slab_bounds)."""
    lo, hi = C.c_int64(), C.c_int64()
    _check(lib().sslic_slab_bounds(int(last), int(world), int(rank), int(align), C.byref(lo),
                                   C.byref(hi)))
    return lo.value, hi.value


def run_slic_rank(img: NDImage, params: SlicParams, rank: int, world: int, uid: bytes,
                  device: int = 0, labels_out=None, host_planes=None):
    """One rank of a one-process-per-GPU run (sslic_run_slic_rank). img: the
    full volume, or (host_planes=(dims, data_ptr, first_plane)) a raw host
    buffer holding planes [first_plane, ...) of it, e.g. pinned memory with
    just this rank's slab and halo. Returns (slab labels, centres, residuals);
    labels_out: optional preallocated uint32 buffer (numpy or pinned torch)."""
    L = lib()
    if host_planes is None:
        params.validate(img.dims)
        desc, first, dims, ch = img._desc(), 0, img.dims, img.channels
    else:
        dims, data_ptr, first, ch, dtype = host_planes
        desc = _Image()
        desc.rank = len(dims)
        for a in range(4):
            desc.dims[a] = dims[a] if a < len(dims) else 1
        desc.channels = ch
        desc.dtype = _DT[np.dtype(dtype)]
        desc.data = data_ptr
    k = cluster_count(dims, params.grid)
    iters = params.iterations_for(len(dims))
    lo, hi = (slab_bounds_native(dims[-1], world, rank, params.grid[-1]) if world > 1
              else (0, dims[-1]))
    plane = int(np.prod(dims[:-1]))
    labels = labels_out if labels_out is not None else np.empty((hi - lo) * plane, np.uint32)
    centers = np.empty(k * (ch + len(dims)))
    res = np.empty(max(iters, 1))
    done = C.c_int(0)
    p = params._c()
    ub = C.create_string_buffer(uid, 128) if uid else None
    lp = (_p(labels, C.c_uint32) if isinstance(labels, np.ndarray)
          else C.cast(C.c_void_p(labels.data_ptr()), C.POINTER(C.c_uint32)))
    _check(L.sslic_run_slic_rank(C.byref(desc), C.byref(p), int(rank), int(world), ub,
                                 int(device), int(first), lp, _p(centers, C.c_double),
                                 _p(res, C.c_double), C.byref(done)))
    return labels, ClusterTable(ch, len(dims), centers), list(res[: done.value])


def segment(img: NDImage, params: SlicParams, device: int = 0):
    """run_slic followed by enforce_connectivity when params asks for it
    (tools/sslic.cpp:104-108). Returns (SlicResult, next_label)."""
    params.validate(img.dims)
    L = lib()
    n = img.pixel_count()
    k = cluster_count(img.dims, params.grid)
    iters = params.iterations_for(img.rank)
    labels = np.empty(n, np.uint32)
    centers = np.empty(k * (img.channels + img.rank))
    res = np.empty(max(iters, 1))
    done, nxt = C.c_int(0), C.c_uint32(0)
    d, p = img._desc(), params._c()
    _check(L.sslic_segment(C.byref(d), C.byref(p), device, _p(labels, C.c_uint32),
                           _p(centers, C.c_double), _p(res, C.c_double), C.byref(done),
                           C.byref(nxt)))
    return (SlicResult(labels, ClusterTable(img.channels, img.rank, centers),
                       list(res[: done.value])), int(nxt.value))


def segment_write(img: NDImage, params: SlicParams, labels_path: str,
                  contour_path: Optional[str] = None, device: int = 0):
    """tools/sslic.cpp's segment pipeline writing its files (sslic_segment_write):
    run_slic, enforce_connectivity, write_labels(labels_path) and optionally
    write_volume(contour_path, mask_label_contour(img, labels)) as float32; the
    label count and the contour come out of the final device pass. Returns
    (ClusterTable, residuals, next_label)."""
    params.validate(img.dims)
    k = cluster_count(img.dims, params.grid)
    iters = params.iterations_for(img.rank)
    centers = np.empty(k * (img.channels + img.rank))
    res = np.empty(max(iters, 1))
    done, nxt = C.c_int(0), C.c_uint32(0)
    d, p = img._desc(), params._c()
    _check(lib().sslic_segment_write(C.byref(d), C.byref(p), device, os.fsencode(labels_path),
                                     os.fsencode(contour_path) if contour_path else None,
                                     _p(centers, C.c_double), _p(res, C.c_double),
                                     C.byref(done), C.byref(nxt)))
    return (ClusterTable(img.channels, img.rank, centers), list(res[: done.value]),
            int(nxt.value))


def init_centers(img: NDImage, params: SlicParams, device: int = 0) -> ClusterTable:
    """init_centers (slic.hpp:206-230)."""
    params.validate(img.dims)
    k = cluster_count(img.dims, params.grid)
    out = np.empty(k * (img.channels + img.rank))
    d, p = img._desc(), params._c()
    _check(lib().sslic_init_centers(C.byref(d), C.byref(p), 0, device, _p(out, C.c_double)))
    return ClusterTable(img.channels, img.rank, out)


def perturb_centers(img: NDImage, table: ClusterTable, workers: int = 1,
                    device: int = 0) -> ClusterTable:
    """perturb_centers (slic.hpp:236-267): returns a new table."""
    out = table.data.copy()
    d = img._desc()
    _check(lib().sslic_perturb_centers(C.byref(d), _p(out, C.c_double), out.shape[0], device))
    return ClusterTable(table.channels, table.rank, out)


def convert_image_to_lab(img: NDImage, device: int = 0) -> NDImage:
    """convert_image_to_lab (color.hpp:54-66): pixelwise sRGB (D65, values in
    [0, 255]) to CIE-Lab, computed on the GPU; returns an fp64 NDImage.
    Raises InvalidArgument unless the image has 3 channels."""
    if img.channels != 3:
        raise InvalidArgument("convert_image_to_lab: image must have 3 channels")
    out = np.empty(img.pixel_count() * 3, np.float64)
    _check(lib().sslic_convert_image_to_lab(C.byref(img._desc()), device, _p(out, C.c_double)))
    return NDImage(img.dims, 3, out)


def mask_label_contour(img: NDImage, labels: np.ndarray, label_dims=None,
                       device: int = 0) -> NDImage:
    """mask_label_contour (io.hpp:432-454): fp64 copy of the image with every
    voxel on a label boundary (a face neighbour with a different label) zeroed
    in all channels. Raises InvalidArgument when the label dims differ."""
    ld = np.asarray(img.dims if label_dims is None else label_dims, np.int64)
    lab = np.ascontiguousarray(labels, np.uint32).reshape(-1)
    if lab.size != int(np.prod(ld)):
        raise InvalidArgument("mask_label_contour: label map size does not match its dims")
    out = np.empty(img.pixel_count() * img.channels, np.float64)
    _check(lib().sslic_mask_label_contour(C.byref(img._desc()), len(ld), _p(ld, C.c_int64),
                                          _p(lab, C.c_uint32), device, _p(out, C.c_double)))
    return NDImage(img.dims, img.channels, out)


_NP_OF_DT = {0: np.uint8, 1: np.uint16, 2: np.float32}


def read_volume_info(path) -> dict:
    """parse_volume_header (io.hpp:123-190) of a detached-header volume."""
    info = _VolumeInfo()
    _check(lib().sslic_volume_info_read(os.fsencode(path), C.byref(info)))
    return {"dims": tuple(int(info.dims[a]) for a in range(info.rank)),
            "channels": int(info.channels), "label_map": bool(info.label_map),
            "dtype": None if info.label_map else _NP_OF_DT[info.dtype]}


def read_volume(path) -> NDImage:
    """read_volume (io.hpp:337-360) for the detached-header format, keeping
    the stored type (uint8 / uint16 / float32) instead of widening to fp64
    (the values are the same). uint32 files are label maps: IoError."""
    info = read_volume_info(path)
    if info["label_map"]:
        raise IoError("unsupported_type", "uint32 volumes are label maps; use read_labels")
    out = np.empty(int(np.prod(info["dims"])) * info["channels"], info["dtype"])
    _check(lib().sslic_volume_read(os.fsencode(path), 0, info["dims"][-1],
                                   C.c_void_p(out.ctypes.data), -1))
    return NDImage(info["dims"], info["channels"], out)


def read_volume_planes(path, plane_begin: int, plane_end: int, dst_ptr: int,
                       device: int = 0) -> None:
    """Planes [plane_begin, plane_end) of the last axis straight into device
    memory (a z-slab rank's share), streamed through pinned staging."""
    _check(lib().sslic_volume_read(os.fsencode(path), int(plane_begin), int(plane_end),
                                   C.c_void_p(dst_ptr), int(device)))


def write_volume(path, img: NDImage) -> None:
    """write_volume (io.hpp:362-392) in the image's stored type."""
    _check(lib().sslic_volume_write(os.fsencode(path), C.byref(img._desc())))


def write_labels(path, labels: np.ndarray, dims) -> None:
    """write_labels (io.hpp:396-412)."""
    d = np.asarray(dims, np.int64)
    lab = np.ascontiguousarray(labels, np.uint32).reshape(-1)
    if lab.size != int(np.prod(d)):
        raise InvalidArgument("write_labels: label count does not match dims")
    _check(lib().sslic_labels_write(os.fsencode(path), len(d), _p(d, C.c_int64),
                                    _p(lab, C.c_uint32)))


def read_labels(path):
    """read_labels (io.hpp:414-428): (flat uint32 labels, dims)."""
    info = read_volume_info(path)
    out = np.empty(int(np.prod(info["dims"])), np.uint32)
    _check(lib().sslic_labels_read(os.fsencode(path), _p(out, C.c_uint32)))
    return out, info["dims"]


def gradient_magnitude_sq(img: NDImage, coord, device: int = 0):
    """gradient_magnitude_sq (color.hpp:71-102) at one coordinate or an
    (n, rank) array of coordinates."""
    co = np.ascontiguousarray(coord, np.int64)
    single = co.ndim == 1
    co = co.reshape(-1, img.rank)
    out = np.empty(co.shape[0])
    d = img._desc()
    _check(lib().sslic_gradient_sq(C.byref(d), _p(co, C.c_int64), co.shape[0], device,
                                   _p(out, C.c_double)))
    return float(out[0]) if single else out


def squared_distance(center, pixel_value, pixel_coord, params: SlicParams, device: int = 0):
    """squared_distance (slic.hpp:189-200). Accepts one triple or batches
    (center (n, c+r), pixel (n, c), coord (n, r))."""
    ctr = np.ascontiguousarray(center, np.float64)
    pix = np.ascontiguousarray(pixel_value, np.float64)
    co = np.ascontiguousarray(pixel_coord, np.int64)
    single = co.ndim == 1
    rank = co.shape[-1]
    ch = pix.shape[-1]
    if ctr.shape[-1] != ch + rank:
        raise InvalidArgument("squared_distance: center size must be channels + rank")
    if len(params.grid) != rank:
        raise InvalidArgument("squared_distance: grid rank mismatch")
    ctr, pix, co = ctr.reshape(-1, ch + rank), pix.reshape(-1, ch), co.reshape(-1, rank)
    g = np.asarray(params.grid, np.int64)
    out = np.empty(co.shape[0])
    _check(lib().sslic_squared_distance(ch, rank, _p(g, C.c_int64), float(params.weight_m),
                                        co.shape[0], _p(ctr, C.c_double), _p(pix, C.c_double),
                                        _p(co, C.c_int64), device, _p(out, C.c_double)))
    return float(out[0]) if single else out


def assign_labels(img: NDImage, table: ClusterTable, params: SlicParams, labels: np.ndarray,
                  dists: np.ndarray, device: int = 0) -> None:
    """assign_labels (slic.hpp:275-310) over the whole image; mutates the
    caller-owned flat uint32 labels / float64 dists in place."""
    if labels.dtype != np.uint32 or dists.dtype != np.float64:
        raise InvalidArgument("assign_labels: labels must be uint32, dists float64")
    if not (labels.flags.c_contiguous and dists.flags.c_contiguous):
        raise InvalidArgument("assign_labels: maps must be contiguous")
    d, p = img._desc(), params._c()
    c = np.ascontiguousarray(table.data, np.float64)
    _check(lib().sslic_assign_pass(C.byref(d), C.byref(p), _p(c, C.c_double), c.shape[0],
                                   device, _p(labels, C.c_uint32), _p(dists, C.c_double)))


def accumulate_region(img: NDImage, labels: np.ndarray, k: Optional[int] = None,
                      device: int = 0):
    """accumulate_region (slic.hpp:315-346) over the whole image: returns
    (sums (k, c+n) float64, counts (k,) int64). Undefined labels raise
    LogicError like the reference."""
    lab = np.ascontiguousarray(labels, np.uint32).reshape(-1)
    if k is None:
        valid = lab[lab != UNDEFINED]
        k = int(valid.max()) + 1 if valid.size else 0
    stride = img.channels + img.rank
    sums = np.zeros(k * stride)
    counts = np.zeros(k, np.int64)
    d = img._desc()
    _check(lib().sslic_accumulate(C.byref(d), _p(lab, C.c_uint32), k, device,
                                  _p(sums, C.c_double), _p(counts, C.c_int64)))
    return sums.reshape(k, stride), counts


def reduce_and_update(table: ClusterTable, partials, device: int = 0):
    """reduce_and_update (slic.hpp:352-372). `partials` is a list of
    (sums, counts) pairs merged in order; returns (new_table, residual)."""
    k, stride = table.count(), table.stride()
    sums = np.zeros((k, stride))
    counts = np.zeros(k, np.int64)
    for s, n in partials:
        m = min(k, len(n))
        sums[:m] += np.asarray(s)[:m]
        counts[:m] += np.asarray(n)[:m]
    out = table.data.copy()
    r = C.c_double(0.0)
    _check(lib().sslic_reduce_and_update(_p(out, C.c_double), k, stride, _p(sums, C.c_double),
                                         _p(counts, C.c_int64), device, C.byref(r)))
    return ClusterTable(table.channels, table.rank, out), float(r.value)


def enforce_connectivity(labels: np.ndarray, dims, table: ClusterTable, params: SlicParams,
                         workers: int = 1, device: int = 0, return_next: bool = False):
    """enforce_connectivity (connectivity.hpp:265-273): returns a relabelled
    copy of the flat label map (and, with return_next, the next unused label
    that sweep_relabel returns, connectivity.hpp:182)."""
    lab = np.ascontiguousarray(labels, np.uint32).reshape(-1)
    dd = np.asarray(dims, np.int64)
    g = np.asarray(params.grid, np.int64)
    c = np.ascontiguousarray(table.data, np.float64)
    out = np.empty_like(lab)
    nxt = C.c_uint32(0)
    _check(lib().sslic_enforce_connectivity(len(dd), _p(dd, C.c_int64), _p(lab, C.c_uint32),
                                            _p(c, C.c_double), table.channels, c.shape[0],
                                            _p(g, C.c_int64), device, _p(out, C.c_uint32),
                                            C.byref(nxt)))
    return (out, int(nxt.value)) if return_next else out


def synth_generate(config: int, dims, dtype, channels: int, seed: int, z_begin: int,
                   z_end: int, dev_ptr: int, stream: int = 0) -> None:
    """Seeded synthetic BASELINE config volume written straight into device
    memory (planes [z_begin, z_end) of the last axis)."""
    dd = np.asarray(dims, np.int64)
    _check(lib().sslic_synth_generate(int(config), len(dd), _p(dd, C.c_int64), int(channels),
                                      _DT[np.dtype(dtype)], C.c_uint64(seed), int(z_begin),
                                      int(z_end), C.c_void_p(dev_ptr), C.c_void_p(stream)))


class _DevArray:
    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None}


def _torch_view(ptr, n, typestr, device):
    import torch
    return torch.as_tensor(_DevArray(ptr, n, typestr), device=f"cuda:{device}")


class Engine:
    """Device-resident iteration engine over one z-slab (the last axis) of a
    volume already in HBM (see sslic_engine_* in include/sslic_b200.h).

    data_ptr points at planes [data_begin, data_end) of the full image
    described by (dims, channels, dtype)."""

    def __init__(self, dims, channels, dtype, data_ptr: int, params: SlicParams,
                 slab=None, data_range=None, device: int = 0, stream: int = 0):
        dims = tuple(int(d) for d in dims)
        last = dims[-1]
        slab = slab or (0, last)
        data_range = data_range or (0, last)
        d = _Image()
        d.rank = len(dims)
        for a in range(4):
            d.dims[a] = dims[a] if a < len(dims) else 1
        d.channels = channels
        d.dtype = _DT[np.dtype(dtype)]
        d.data = data_ptr
        self._params = params._c()
        h = C.c_void_p()
        _check(lib().sslic_engine_create(C.byref(d), C.byref(self._params), device, slab[0],
                                         slab[1], data_range[0], data_range[1],
                                         C.c_void_p(stream), C.byref(h)))
        self.h = h
        self.device = device
        self.dims, self.channels, self.slab = dims, channels, slab
        self.k = cluster_count(dims, params.grid)
        self.iterations = params.iterations_for(len(dims))

    def close(self):
        if self.h:
            lib().sslic_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def reset(self):
        """Back to iteration 0 for another whole run (labels undefined)."""
        _check(lib().sslic_engine_reset(self.h))

    def attach_nccl(self, uid: bytes, rank: int, world: int):
        """NCCL communicator for this engine (collective over the ranks):
        start / iterate / iterate_graph then run the allreduces natively."""
        ub = C.create_string_buffer(uid, 128) if uid else None
        _check(lib().sslic_engine_attach_nccl(self.h, ub, int(rank), int(world)))

    def start(self):
        """init + perturb, the (allreduced) table and its anchors / bins."""
        _check(lib().sslic_engine_start(self.h))

    def init(self):
        _check(lib().sslic_engine_init(self.h))

    def centers_buffer(self):
        p, n = C.c_void_p(), C.c_int64()
        _check(lib().sslic_engine_centers_buffer(self.h, C.byref(p), C.byref(n)))
        return p.value, n.value

    def commit(self):
        _check(lib().sslic_engine_commit_centers(self.h))

    def assign(self):
        _check(lib().sslic_engine_assign(self.h))

    def partials(self):
        p, n = C.c_void_p(), C.c_int64()
        _check(lib().sslic_engine_partials(self.h, C.byref(p), C.byref(n)))
        return p.value, n.value

    def update(self):
        _check(lib().sslic_engine_update(self.h))

    def iterate(self, n: int = 1):
        _check(lib().sslic_engine_iterate(self.h, n))

    def iterate_graph(self, n: int) -> float:
        """n iterations captured in one CUDA graph and launched once; returns
        the launch's device time in ms."""
        ms = C.c_float(0)
        _check(lib().sslic_engine_iterate_graph(self.h, int(n), C.byref(ms)))
        return float(ms.value)

    def iterations_done(self):
        return lib().sslic_engine_iterations_done(self.h)

    def residuals(self):
        n = self.iterations_done()
        out = np.empty(max(n, 1))
        _check(lib().sslic_engine_residuals(self.h, _p(out, C.c_double)))
        return list(out[:n])

    def labels_to(self, dev_ptr: int):
        _check(lib().sslic_engine_labels(self.h, C.c_void_p(dev_ptr)))

    def centers(self):
        out = np.empty(self.k * (self.channels + len(self.dims)))
        _check(lib().sslic_engine_centers(self.h, _p(out, C.c_double)))
        return out.reshape(self.k, -1)

    def undefined_count(self):
        v = lib().sslic_engine_undefined_count(self.h)
        if v < 0:
            _check(-4)
        return v

    def launch_count(self):
        return lib().sslic_engine_launch_count(self.h)

    def assign_ms(self, i: int) -> float:
        ms, n = C.c_float(), C.c_int()
        _check(lib().sslic_engine_assign_ms(self.h, int(i), C.byref(ms), C.byref(n)))
        return float(ms.value)

    def assign_calls(self) -> int:
        ms, n = C.c_float(), C.c_int()
        lib().sslic_engine_assign_ms(self.h, -1, None, C.byref(n))
        return int(n.value)

    # zero-copy torch views of the engine's device buffers (for NCCL)
    def centers_tensor(self):
        p, n = self.centers_buffer()
        return _torch_view(p, n, "<f8", self.device)

    def partials_tensor(self):
        p, n = self.partials()
        return _torch_view(p, n, "<i8", self.device)

    def labels_tensor(self):
        """This slab's labels (plain LabelMap values, int32 bit patterns of
        the uint32 labels) in a new device tensor (sharded.gather_labels)."""
        import torch
        plane = int(np.prod(self.dims[:-1]))
        t = torch.empty((self.slab[1] - self.slab[0]) * plane, dtype=torch.int32,
                        device=f"cuda:{self.device}")
        self.labels_to(t.data_ptr())
        return t

    def value_range(self) -> float:
        """max |value| over this engine's planes (float dtypes; the dtype
        maximum for u8/u16), see sslic_engine_value_range."""
        v = C.c_double()
        _check(lib().sslic_engine_value_range(self.h, C.byref(v)))
        return float(v.value)

    def set_value_range(self, absmax: float):
        """Multi-GPU: every rank sets the MAX over ranks (before init)."""
        _check(lib().sslic_engine_set_value_range(self.h, C.c_double(absmax)))

    def set_exact(self, exact: bool = True):
        _check(lib().sslic_engine_set_exact(self.h, int(exact)))

    def fast_stats(self):
        """(voxels re-decided in fp64, crowded CTAs, voxels whose label value
        changed) of the last assign (fast path, with set_stats(True))."""
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        _check(lib().sslic_engine_fast_stats(self.h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def set_stats(self, on: bool = True):
        _check(lib().sslic_engine_set_stats(self.h, int(on)))

    def eval_stats(self):
        a, b = C.c_double(), C.c_double()
        _check(lib().sslic_engine_eval_stats(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value
