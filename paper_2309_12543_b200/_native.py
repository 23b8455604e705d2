"""ctypes binding of the C ABI in ``include/linksdf_b200.h``.

The extension is a plain shared library built in-tree by ``build.py``
(``_lib/liblinksdf_b200.so``); device memory comes from torch tensors (their
``data_ptr()``), work is enqueued on torch's current stream.  There is no CPU
fallback: if the library or a CUDA device is missing, every compute call
raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

from . import errors

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "liblinksdf_b200.so"

MAX_LINKS = 32

# --------------------------------------------------------------------------- structs


class EnvGridT(C.Structure):
    _fields_ = [("extent", C.c_double * 3), ("resolution", C.c_double * 3),
                ("dims", C.c_int32 * 3), ("pad_", C.c_int32)]


class LinkT(C.Structure):
    _fields_ = [("kind", C.c_int32), ("parent", C.c_int32), ("q_col", C.c_int32),
                ("geom_slot", C.c_int32), ("joint_R", C.c_double * 9), ("joint_t", C.c_double * 3),
                ("skew", C.c_double * 9), ("outer", C.c_double * 9), ("R_axis", C.c_double * 3),
                ("link_R", C.c_double * 9), ("link_t", C.c_double * 3)]


class LinkGridT(C.Structure):
    _fields_ = [("values_dev", C.c_void_p), ("packed_dev", C.c_void_p), ("dims", C.c_int32 * 3), ("d_far", C.c_float),
                ("extent", C.c_double * 3), ("resolution", C.c_double * 3), ("core_radius", C.c_float),
                ("seg_kappa_lo", C.c_float), ("seg_kappa_hi", C.c_float), ("seg_len", C.c_float),
                ("seg_a", C.c_float * 3), ("seg_u", C.c_float * 3)]


class TmlpTrainT(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("w1", "b1", "w2", "b2", "m_w1", "m_b1", "m_w2", "m_b2",
                                         "v_w1", "v_b1", "v_w2", "v_b2", "points")] + [
        ("hidden", C.c_int32), ("n_out", C.c_int64), ("lr", C.c_float), ("beta1", C.c_float),
        ("beta2", C.c_float), ("eps", C.c_float), ("step", C.c_void_p), ("ld_w2", C.c_int64)]


class WindowT(C.Structure):
    _fields_ = [("W", C.c_int32 * 3), ("n_masked", C.c_int32), ("e_r", C.c_double),
                ("P_dev", C.c_void_p), ("Wmax", C.c_int32), ("pad_", C.c_int32),
                ("zrange_dev", C.c_void_p), ("mask_bits_dev", C.c_void_p),
                ("shell_cells_dev", C.c_void_p), ("shell_radius_dev", C.c_void_p)]


_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64
_D = C.c_double
_F = C.c_float

_SIGS = {
    "lsdf_fk_align": [C.POINTER(LinkT), _I32, _I32, _P, _I64, _I32, _P, C.POINTER(EnvGridT),
                      C.POINTER(_I32), _P, _P, _P, _P, _P, _P, _P],
    "lsdf_fk_align_link_major": [C.POINTER(LinkT), _I32, _I32, _P, _I64, _I32, _P, C.POINTER(EnvGridT),
                                 C.POINTER(_I32), _P, _P, _P, _P, _P, _P, _P],
    "lsdf_fk_align_ex": [C.POINTER(LinkT), _I32, _I32, _P, _I64, _I32, _P, C.POINTER(EnvGridT),
                         C.POINTER(_I32), _P, _P, _P, _P, _P, _P, _I32, _P],
    "lsdf_align": [_P, _I64, C.POINTER(EnvGridT), C.POINTER(_I32), _P, _P, _P, _P],
    "lsdf_occupancy_bytes": [C.POINTER(EnvGridT)],
    "lsdf_voxelize": [_P, _I32, _I64, C.POINTER(EnvGridT), _P, _P, _P],
    "lsdf_voxelize_bitmap": [_P, _I32, _I64, C.POINTER(EnvGridT), _P, _P],
    "lsdf_occupancy_prefix": [C.POINTER(EnvGridT), _P, _P],
    "lsdf_occupancy_merge": [_P, _I32, _P, _I64, C.POINTER(EnvGridT), _P, _P],
    "lsdf_occupancy_from_indices": [_P, _I64, _I32, C.POINTER(EnvGridT), _P, _P],
    "lsdf_voxel_index": [_P, _I64, C.POINTER(EnvGridT), _P, _P, _P],
    "lsdf_query_direct": [_P, _P, _P, _I64, _I32, C.POINTER(LinkGridT), C.POINTER(WindowT),
                          C.POINTER(EnvGridT), _P, _I32, _D, _P, _P, _P, _P, _P, _P],
    "lsdf_query_scan": [_P, _P, _P, _I64, _I32, C.POINTER(LinkGridT), C.POINTER(WindowT),
                          C.POINTER(EnvGridT), _P, _I32, _D, _P, _P, _P, _P, _P, _P],
    "lsdf_query_finalize": [_P, _P, _P, _I64, _I32, C.POINTER(LinkGridT), C.POINTER(WindowT),
                          C.POINTER(EnvGridT), _P, _I32, _D, _P, _P, _P, _P, _P, _P],
    "lsdf_query_workspace_bytes": [_I64, _I32],
    "lsdf_pack_corners": [_P, C.POINTER(_I32), _P, _P],
    "lsdf_materialize_vm": [_P, _P, _P, _I64, _I32, C.POINTER(LinkGridT), C.POINTER(WindowT),
                            C.POINTER(EnvGridT), _D, _P, _P],
    "lsdf_query_vm": [_P, _P, _P, _P, _I64, _I32, C.POINTER(LinkGridT), C.POINTER(WindowT), C.POINTER(EnvGridT),
                      _P, _P, _I64, _D, _P, _P, _P, _P, _P],
    "lsdf_place_windows": [_P, _P, _I64, _I32, C.POINTER(LinkGridT), C.POINTER(WindowT), _P, _P],
    "lsdf_place_windows_g": [_P, _I64, _P, _I32, _P, _P, _I64, _I32, C.POINTER(LinkGridT), C.POINTER(WindowT), _P,
                             _P],
    "lsdf_assemble": [_P, _P, _P, _I64, C.POINTER(_I32), C.POINTER(EnvGridT), _I64, _D, _P, _P],
    "lsdf_query_dense": [_P, _I64, C.POINTER(EnvGridT), _P, _I64, _P, _P, _P],
    "lsdf_per_link_fields": [_P, _P, _P, _P, _P, _I64, C.POINTER(_I32), _I32, C.POINTER(EnvGridT),
                             _P, _P, _P],
    "lsdf_fill": [_P, _I64, _F, _P],
    "lsdf_link_at_voxel": [_P, _P, _I64, _I32, C.POINTER(_I32), _P, _P, _P, _F, _P, _P, _P],
    "lsdf_sphere_baseline": [_P, _P, _I64, _I32, _P, _P, _P, _I32, _P, _I64, C.POINTER(EnvGridT),
                             _P, _P],
    "lsdf_trilinear": [C.POINTER(LinkGridT), _P, _I64, _D, _P, _P],
    "lsdf_grid_transform_exact": [_P, _P, _I64, _P, _I64, _D, _P, _P],
    "lsdf_build_primitive": [_I32, C.POINTER(_D), C.POINTER(_D), C.POINTER(_D), C.POINTER(_I32), _P, _P],
    "lsdf_primitive_points": [_I32, C.POINTER(_D), _P, _I64, _P, _P],
    "lsdf_build_mesh": [_P, _I32, _I32, C.POINTER(_D), C.POINTER(_D), C.POINTER(_I32), _P, _P],
    "lsdf_mesh_points": [_P, _I32, _I32, _P, _I64, _P, _P],
    "lsdf_mlp_predict": [_P, _P, _P, _P, _P, _I32, _I64, _P, _I64, _P, _I64, _I32, _P],
    "lsdf_mlp_packed_bytes": [_I32, _I64],
    "lsdf_mlp_pack": [_P, _I32, _I64, _P, _P],
    "lsdf_mlp_place_packed_bytes": [_I32, _I64],
    "lsdf_mlp_place_pack": [_P, _I32, _I64, _P, _P],
    "lsdf_mlp_place": [_P, _P, _P, _P, _I32, _I64, _P, _P, _P, _I64, _I32, C.POINTER(LinkGridT), C.POINTER(WindowT),
                       _P, _P],
    "lsdf_host_device_pointer": [_P, C.POINTER(C.c_void_p)],
    "lsdf_tmlp_train_workspace_bytes": [_I32, _I32],
    "lsdf_tmlp_train_step": [C.POINTER(TmlpTrainT), _P, _I32, _P, _P],
    "lsdf_sample_rotations": [C.c_uint64, C.c_uint64, _I64, _P, _P],
    "lsdf_l2_reserve": [C.c_size_t, C.POINTER(C.c_size_t)],
}

QUERY_BY_POSITION = 1        # lsdf_query_* flags word (include/linksdf_b200.h)
QUERY_POSES_LINK_MAJOR = 2
QUERY_DENSE_HINT = 4
FK_LINK_MAJOR = 1            # lsdf_fk_align_ex options
FK_FLAGS_SELF_RESET = 2

EXPORTS = tuple(_SIGS) + ("lsdf_version", "lsdf_last_error", "lsdf_launch_count")

_ERRORS = {
    1: errors.ValidationError,
    2: errors.OutOfBoundsError,
    3: errors.NoOverlapError,
    5: errors.NonWatertightError,
    6: errors.GridMismatchError,
    7: errors.DimensionMismatchError,
    100: errors.CudaError,
    101: errors.ValidationError,
}

_lock = threading.Lock()
_lib = None


def load_library(path: Path | None = None):
    """Load (once) and type the shared library; raises if it is missing."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        # LINKSDF_B200_LIB: an alternative build of the same library (A/B timing)
        p = Path(path) if path else Path(os.environ.get("LINKSDF_B200_LIB", LIB_PATH))
        if not p.exists():
            raise ImportError(
                f"linksdf-b200 CUDA extension not built ({p}); run "
                "`python -m paper_2309_12543_b200.build` (nvcc, sm_100a)")
        lib = C.CDLL(str(p))
        alternative = path is None and "LINKSDF_B200_LIB" in os.environ
        for name, argtypes in _SIGS.items():
            if alternative and not hasattr(lib, name):  # an older build in an A/B run: skip newer entries
                continue
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = C.c_int64 if name.endswith("_bytes") else C.c_int
        lib.lsdf_version.restype = C.c_char_p
        lib.lsdf_last_error.restype = C.c_char_p
        lib.lsdf_launch_count.restype = C.c_uint64
        _lib = lib
        return lib


def lib():
    return _lib if _lib is not None else load_library()


def call(name: str, *args) -> int:
    """Invoke an entry point; CUDA tensors may be passed directly (their
    pointers are taken here, and ``args`` keeps them alive until the launch
    is enqueued, so temporaries cannot be recycled under a pending copy)."""
    t = _torch
    if t is not None:
        cargs = [a.data_ptr() if isinstance(a, t.Tensor) else a for a in args]
    else:
        cargs = args
    rc = getattr(lib(), name)(*cargs)
    if rc != 0:
        msg = lib().lsdf_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, errors.LinkSdfError)(f"{name}: {msg}")
    return rc


# --------------------------------------------------------------------------- device helpers

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t

        _torch = t
    return _torch


def device():
    """The CUDA device every tensor lives on; raises without one (no CPU path)."""
    t = torch()
    if not t.cuda.is_available():
        raise errors.CudaError("linksdf-b200 needs a CUDA device (B200, sm_100a); none is visible")
    load_library()
    return t.device("cuda", t.cuda.current_device())


def stream() -> int:
    return torch().cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def to_device(a, dtype=None):
    """numpy array or tensor → contiguous CUDA tensor (dtype optional)."""
    t = torch()
    if isinstance(a, t.Tensor):
        out = a.to(device=device(), dtype=dtype) if dtype is not None else a.to(device=device())
        return out.contiguous()
    arr = np.ascontiguousarray(a)
    if not arr.flags.writeable:
        arr = arr.copy()
    out = t.from_numpy(arr).to(device(), non_blocking=False)
    if dtype is not None:
        out = out.to(dtype)
    return out.contiguous()


def empty(shape, dtype):
    return torch().empty(shape, dtype=dtype, device=device())


def zeros(shape, dtype):
    return torch().zeros(shape, dtype=dtype, device=device())


def mapped_pointer(host_tensor) -> int:
    """Device address of a pinned host tensor (zero-copy access from kernels)."""
    out = C.c_void_p()
    call("lsdf_host_device_pointer", host_tensor.data_ptr(), C.byref(out))
    return int(out.value)


def env_struct(grid) -> EnvGridT:
    e = EnvGridT()
    e.extent[:] = [float(v) for v in grid.extent]
    e.resolution[:] = [float(v) for v in grid.resolution]
    e.dims[:] = [int(v) for v in grid.dims]
    return e


def i32x3(v) -> C.Array:
    arr = (C.c_int32 * 3)()
    arr[:] = [int(x) for x in v]
    return arr


def f64s(v, n: int) -> C.Array:
    arr = (C.c_double * n)()
    vals = [float(x) for x in np.ravel(v)]
    arr[: len(vals)] = vals
    return arr


def l2_reserve(nbytes: int) -> int:
    """Persisting-L2 set-aside on the current device (lsdf_l2_reserve); returns the bytes granted."""
    got = C.c_size_t(0)
    call("lsdf_l2_reserve", int(nbytes), C.byref(got))
    return int(got.value)
