"""ctypes binding of the in-tree CUDA library (include/radsplat.h).

There is no CPU fallback: importing the renderer on a host without the built
library or without a CUDA device raises immediately (``NativeUnavailable``).
Status codes map onto the reference's exception classes (core.py:20-37).
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

from .core import InvalidParameterError, InvalidSceneError

LIB_PATH = Path(__file__).resolve().parent / "libradsplat_b200.so"

RS_OK, RS_EINVAL, RS_ENONFINITE, RS_ENOMEM_WORKSPACE, RS_ECUDA, RS_EOVERFLOW = range(6)
RS_FLAG_COUNT_EVALS = 1
RS_FLAG_BLEND_1PX = 2
RS_F32, RS_F64 = 0, 1
ABI_VERSION = 2


class NativeUnavailable(RuntimeError):
    """The CUDA library or a CUDA device is missing (no fallback exists)."""


class WorkspaceTooSmall(RuntimeError):
    pass


class PairOverflow(RuntimeError):
    pass


class RsScene(C.Structure):
    _fields_ = [("planes", C.c_void_p), ("sh", C.c_void_p), ("n", C.c_int64), ("plane_stride", C.c_int64),
                ("sh_degree", C.c_int32), ("dtype", C.c_int32)]


class RsCamera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double), ("R", C.c_double * 9), ("t", C.c_double * 3),
                ("center", C.c_double * 3)]


class RsOptions(C.Structure):
    _fields_ = [(n, C.c_double) for n in
                ("alpha_max", "alpha_cut", "tau_stop", "near_limit", "lowpass", "sigma_bound")] + \
               [("precision", C.c_int32), ("_pad", C.c_int32)]


class RsOutputs(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("rgb", "alpha", "depth", "count", "rgb64", "alpha64", "count64", "tau",
                                          "last")]


class RsStats(C.Structure):
    _fields_ = [("n_items", C.c_uint32), ("n_visible", C.c_uint32), ("n_pairs", C.c_uint32),
                ("overflow", C.c_uint32), ("evals", C.c_uint64), ("composites", C.c_uint64),
                ("pairs_needed", C.c_uint64), ("bad_index", C.c_uint32), ("_pad", C.c_uint32)]


class RsBuffers(C.Structure):
    _fields_ = [("records", C.c_void_p), ("records64", C.c_void_p), ("items_sorted", C.c_void_p),
                ("pair_items", C.c_void_p),
                ("ranges", C.c_void_p), ("counters", C.c_void_p), ("tiles_x", C.c_int32),
                ("tiles_y", C.c_int32)]


# every symbol include/radsplat.h declares, with (restype, argtypes)
_vp, _i64, _i32, _u32, _sz = C.c_void_p, C.c_int64, C.c_int32, C.c_uint32, C.c_size_t
SIGNATURES = {
    "rs_abi_version": (_i32, []),
    "rs_status_string": (C.c_char_p, [_i32]),
    "rs_workspace_size": (_sz, [_i64, _i64, _i32, _i32]),
    "rs_workspace_create": (_i32, [_vp, _sz, _i64, _i64, _i32, _i32, C.POINTER(_vp)]),
    "rs_workspace_destroy": (None, [_vp]),
    "rs_render": (_i32, [_vp, C.POINTER(RsScene), _vp, _i64, C.POINTER(RsCamera), C.POINTER(RsOptions),
                         _vp, _vp, _vp, _vp, _vp, _u32, _vp]),
    "rs_render_ex": (_i32, [_vp, C.POINTER(RsScene), _vp, _i64, C.POINTER(RsCamera), C.POINTER(RsOptions),
                            C.POINTER(RsOutputs), _vp, _u32, _vp]),
    "rs_project": (_i32, [_vp, C.POINTER(RsScene), _vp, _i64, C.POINTER(RsCamera), C.POINTER(RsOptions), _vp]),
    "rs_project_full": (_i32, [_vp, C.POINTER(RsScene), _vp, _i64, C.POINTER(RsCamera), C.POINTER(RsOptions),
                               _vp, _vp, _vp]),
    "rs_bin": (_i32, [_vp, _vp]),
    "rs_set_camera": (_i32, [_vp, C.POINTER(RsCamera), _vp]),
    "rs_blend": (_i32, [_vp, C.POINTER(RsOptions), _vp, _vp, _vp, _vp, _vp, _u32, _vp]),
    "rs_blend_ex": (_i32, [_vp, C.POINTER(RsOptions), C.POINTER(RsOutputs), _vp, _u32, _vp]),
    "rs_read_stats": (_i32, [_vp, C.POINTER(RsStats), _vp]),
    "rs_read_overflow": (_i32, [_vp, C.POINTER(_u32), C.POINTER(C.c_uint64), _i32, _vp]),
    "rs_read_sticky": (_i32, [_vp, C.POINTER(_u32), C.POINTER(C.c_uint64), C.POINTER(_u32), _i32, _vp]),
    "rs_get_buffers": (_i32, [_vp, C.POINTER(RsBuffers)]),
    "rs_compact_workspace_size": (_sz, [_i64]),
    "rs_compact": (_i32, [_vp, _i64, _vp, _vp, _vp, _sz, _vp]),
    "rs_compact_bits": (_i32, [_vp, _i64, _vp, _vp, _vp, _sz, _vp]),
    "rs_check_finite": (_i32, [C.POINTER(RsScene), _vp, _vp]),
    "rs_max_merge": (_i32, [_vp, _vp, _i64, _vp]),
    "rs_backward": (_i32, [_vp, C.POINTER(RsScene), _vp, _i64, C.POINTER(RsOptions), _vp, _vp, _vp, _vp, _vp, _vp,
                           _vp, _vp, _vp, _vp, _vp]),
    "rs_rspl_unpack": (_i32, [_vp, _i64, _vp, _i64, _vp, _vp, _vp]),
    "rs_rspl_pack": (_i32, [_vp, _i64, _vp, _i64, _vp, _vp]),
    "rs_pack_bits": (_i32, [_vp, _i64, _vp, _vp]),
    "rs_nearest_cluster": (_i32, [_vp, _i32, _vp, _i64, _vp, _vp]),
    "rs_sq_diff_sum": (_i32, [_vp, _vp, _i64, _vp, _vp]),
    "rs_ssim_workspace_size": (_sz, [_i32, _i32, _i32, _i32]),
    "rs_ssim": (_i32, [_vp, _vp, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _sz, _vp]),
}

_lib = None


def load(require_cuda: bool = True):
    """Load the library (and bind every signature). Raises NativeUnavailable."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise NativeUnavailable(f"{LIB_PATH.name} is not built (python -m paper_2403_13806_b200.build)")
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.rs_abi_version() != ABI_VERSION:
            raise NativeUnavailable("ABI version mismatch")
        _lib = lib
    if require_cuda:
        import torch
        if not torch.cuda.is_available():
            raise NativeUnavailable("no CUDA device: the B200 path has no CPU fallback")
    return _lib


def check(status: int, what: str = "") -> None:
    if status == RS_OK:
        return
    msg = f"{what}: {_lib.rs_status_string(status).decode()}" if _lib else str(status)
    if status == RS_EINVAL:
        raise InvalidParameterError(msg)
    if status == RS_ENONFINITE:
        raise InvalidSceneError(msg)
    if status == RS_ENOMEM_WORKSPACE:
        raise WorkspaceTooSmall(msg)
    if status == RS_EOVERFLOW:
        raise PairOverflow(msg)
    raise RuntimeError(msg)
