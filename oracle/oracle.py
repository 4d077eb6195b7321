"""ctypes wrapper of the CPU oracle (oracle/cpu_ref.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and
bench.py's CPU-baseline legs as the checker; the product package never
imports it. ``dtype=np.float32`` selects the Tier-A fp32 contract the CUDA
path's RS_F32 frames reproduce bit for bit; ``np.float64`` the Tier-B
restatement pinned against the reference's own outputs (tests/golden);
``"c64"`` the Tier-C fp64 contract (Tier B with the contract exp and the
culling-box gate) that RS_F64 frames reproduce bit for bit.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "libcpu_ref.so"


def build(force: bool = False) -> Path:
    src = HERE / "cpu_ref.cpp"
    if force or not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.check_call(["make", "-s", "-C", str(HERE)])
    return LIB


class ProjOut(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in (
        "valid", "mx", "my", "a", "b", "c", "ia", "ib", "ic", "radius", "depth", "color",
        "opacity", "x0", "x1", "y0", "y1", "na", "nb", "nc", "cut2", "cx0", "cx1", "cy0", "cy1", "bin", "ell")]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        _lib = C.CDLL(str(LIB))
        vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int
        for suf in ("f32", "f64", "c64"):
            getattr(_lib, f"orc_project_{suf}").argtypes = [vp] * 5 + [i64, i32, vp, vp, C.POINTER(ProjOut)]
            getattr(_lib, f"orc_order_{suf}").argtypes = [vp] * 5 + [i64, i32, vp, vp, vp, vp]
            getattr(_lib, f"orc_order_{suf}").restype = i64
            getattr(_lib, f"orc_bin_{suf}").argtypes = [vp] * 5 + [i64, i32, vp, vp, vp, vp, vp, vp, i64]
            getattr(_lib, f"orc_bin_{suf}").restype = i64
            getattr(_lib, f"orc_render_{suf}").argtypes = [vp] * 5 + [i64, i32, vp, vp, vp, i32] + [vp] * 6
            getattr(_lib, f"orc_views_{suf}").argtypes = [vp] * 5 + [i64, i32, vp, i64, vp, i32, i32, vp, vp, vp]
        _lib.orc_exp2_contract.argtypes = [vp, vp, i64]
        _lib.orc_exp_contract.argtypes = [vp, vp, i64]
        _lib.orc_exp64_contract.argtypes = [vp, vp, i64]
        _lib.orc_log2_contract.argtypes = [vp, vp, i64]
        _lib.orc_depth_key.argtypes = [C.c_float]
        _lib.orc_depth_key.restype = C.c_uint32
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _suf(dtype):
    if isinstance(dtype, str) and dtype == "c64":
        return "c64"
    return "f32" if np.dtype(dtype) == np.float32 else "f64"


def _np(dtype):
    """numpy value type of a tier (Tier C computes in float64)."""
    return np.float64 if isinstance(dtype, str) and dtype == "c64" else np.dtype(dtype).type


class _Scene:
    def __init__(self, scene, dtype):
        dtype = _np(dtype)
        f = lambda a, shape: np.ascontiguousarray(np.asarray(a).reshape(shape), dtype=dtype)  # noqa: E731
        n = np.asarray(scene.positions).shape[0]
        self.n = n
        self.pos = f(scene.positions, (n, 3))
        self.logit = f(scene.opacity_logits, (n,))
        self.sh = f(scene.sh, (n, 3, 16))
        self.ls = f(scene.log_scales, (n, 3))
        self.quat = f(scene.quaternions, (n, 4))
        self.deg = int(scene.active_sh_degree)

    def args(self):
        return [_p(self.pos), _p(self.logit), _p(self.sh), _p(self.ls), _p(self.quat), self.n, self.deg]


def pack_camera(cam, dtype=np.float32) -> np.ndarray:
    dtype = _np(dtype)
    """[W, H, fx, fy, cx, cy, R(9), t(3), C(3)]; C = -R^T t computed in fp64."""
    R = np.asarray(cam.rotation, np.float64)
    t = np.asarray(cam.translation, np.float64)
    c = -R.T @ t
    v = np.concatenate([[cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy], R.ravel(), t, c])
    return np.ascontiguousarray(v, dtype=dtype)


def pack_options(opts=None, dtype=np.float32) -> np.ndarray:
    dtype = _np(dtype)
    if opts is None:
        v = [0.99, 1.0 / 255.0, 1e-4, 0.01, 0.3, 3.0]
    elif isinstance(opts, (list, tuple, np.ndarray)):
        v = list(opts)
    else:
        v = [opts.alpha_max, opts.alpha_cut, opts.tau_stop, opts.near_limit, opts.lowpass, opts.sigma_bound]
    return np.ascontiguousarray(v, dtype=dtype)


def project(scene, cam, opts=None, dtype=np.float32) -> dict:
    s = _Scene(scene, dtype)
    n = s.n
    out = dict(valid=np.zeros(n, np.uint8), x0=np.zeros(n, np.int32), x1=np.zeros(n, np.int32),
               y0=np.zeros(n, np.int32), y1=np.zeros(n, np.int32), color=np.zeros((n, 3), _np(dtype)),
               na=np.zeros(n, np.float32), nb=np.zeros(n, np.float32), nc=np.zeros(n, np.float32),
               cut2=np.zeros(n, np.float32), cx0=np.zeros(n, np.int32), cx1=np.zeros(n, np.int32),
               cy0=np.zeros(n, np.int32), cy1=np.zeros(n, np.int32), bin=np.zeros(n, np.uint8),
               ell=np.zeros(n, np.uint8))
    for k in ("mx", "my", "a", "b", "c", "ia", "ib", "ic", "radius", "depth", "opacity"):
        out[k] = np.zeros(n, _np(dtype))
    po = ProjOut()
    for k, _ in ProjOut._fields_:
        setattr(po, k, out[k].ctypes.data)
    getattr(lib(), f"orc_project_{_suf(dtype)}")(*s.args(), _p(pack_camera(cam, dtype)),
                                                   _p(pack_options(opts, dtype)), C.byref(po))
    out["valid"] = out["valid"].astype(bool)
    out["bin"] = out["bin"].astype(bool)
    out["ell"] = out["ell"].astype(bool)
    return out


def order(scene, cam, opts=None, dtype=np.float32, active=None) -> np.ndarray:
    s = _Scene(scene, dtype)
    o = np.zeros(s.n, np.int64)
    act = None if active is None else np.ascontiguousarray(active, np.uint8)
    m = getattr(lib(), f"orc_order_{_suf(dtype)}")(*s.args(), _p(pack_camera(cam, dtype)),
                                                   _p(pack_options(opts, dtype)), _p(act), _p(o))
    return o[:m]


def bin_tiles(scene, cam, opts=None, dtype=np.float32, active=None) -> dict:
    """64-bit (tile << 32 | depth_key) keys, Gaussian indices and per-tile ranges."""
    s = _Scene(scene, dtype)
    tiles = ((cam.width + 15) // 16) * ((cam.height + 15) // 16)
    ranges = np.zeros((tiles, 2), np.uint32)
    act = None if active is None else np.ascontiguousarray(active, np.uint8)
    fn = getattr(lib(), f"orc_bin_{_suf(dtype)}")
    cp, op = pack_camera(cam, dtype), pack_options(opts, dtype)
    P = fn(*s.args(), _p(cp), _p(op), _p(act), None, None, _p(ranges), 0)
    keys, vals = np.zeros(P, np.uint64), np.zeros(P, np.uint32)
    fn(*s.args(), _p(cp), _p(op), _p(act), _p(keys), _p(vals), _p(ranges), P)
    return dict(keys=keys, vals=vals, ranges=ranges, P=int(P))


def render(scene, cam, opts=None, dtype=np.float32, active=None, method: int = 0,
           contrib: np.ndarray | None = None) -> dict:
    """Render one view: img (H,W,3), alpha, depth, count, contrib (N,), E, C."""
    s = _Scene(scene, dtype)
    H, W = cam.height, cam.width
    vt = _np(dtype)
    img = np.zeros((H, W, 3), vt)
    alpha = np.zeros((H, W), vt)
    depth = np.zeros((H, W), vt)
    count = np.zeros((H, W), np.int32)
    contrib = np.zeros(s.n, vt) if contrib is None else contrib
    assert contrib.dtype == np.dtype(vt) and contrib.flags.c_contiguous
    k = np.zeros(2, np.int64)
    act = None if active is None else np.ascontiguousarray(active, np.uint8)
    getattr(lib(), f"orc_render_{_suf(dtype)}")(*s.args(), _p(pack_camera(cam, dtype)),
                                                _p(pack_options(opts, dtype)), _p(act), method,
                                                _p(img), _p(alpha), _p(depth), _p(count), _p(contrib), _p(k))
    return dict(img=img, alpha=alpha, depth=depth, count=count, contrib=contrib, E=int(k[0]), C=int(k[1]))


def views(scene, cams, opts=None, dtype=np.float32, threads: int | None = None,
          scores: bool = True, images: bool = False) -> dict:
    """All views over a thread pool; per-Gaussian max contributions merged."""
    s = _Scene(scene, dtype)
    threads = threads or os.cpu_count() or 1
    cp = np.ascontiguousarray(np.stack([pack_camera(c, dtype) for c in cams]))
    contrib = np.zeros(s.n, _np(dtype)) if scores else None
    last = np.zeros((cams[-1].height, cams[-1].width, 3), _np(dtype)) if images else None
    k = np.zeros(2, np.int64)
    getattr(lib(), f"orc_views_{_suf(dtype)}")(*s.args(), _p(cp), len(cams), _p(pack_options(opts, dtype)),
                                               int(threads), int(images), _p(contrib), _p(last), _p(k))
    return dict(contrib=contrib, img_last=last, E=int(k[0]), C=int(k[1]), threads=threads)


def exp2_contract(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    y = np.empty_like(x)
    lib().orc_exp2_contract(_p(x), _p(y), x.size)
    return y


def exp64_contract(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float64)
    y = np.empty_like(x)
    lib().orc_exp64_contract(_p(x), _p(y), x.size)
    return y


def exp_contract(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    y = np.empty_like(x)
    lib().orc_exp_contract(_p(x), _p(y), x.size)
    return y


def log2_contract(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    y = np.empty_like(x)
    lib().orc_log2_contract(_p(x), _p(y), x.size)
    return y


def depth_key(d: float) -> int:
    return int(lib().orc_depth_key(float(d)))
