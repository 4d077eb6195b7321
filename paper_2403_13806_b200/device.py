"""Device residency: scenes in HBM, workspaces, and the frame launcher.

* ``DeviceScene`` -- the scene in HBM: 11 geometry planes of N values plus N
  SH rows of 48 values (the layout ``rs_scene`` documents), stored as fp32 when
  every value is exactly an fp32 number (synthetic scenes, RSPL files) and as
  fp64 otherwise (the reference's float64 arrays), so no frame ever sees
  rounded inputs. Reference scenes are immutable and carry a ``generation``
  tag (core.py:467-485), so an uploaded copy is cached per (object,
  generation) and reused by every later call on the same scene.
* Precision: every frame runs in fp64 (the reference's arithmetic, RS_F64:
  bit-identical to the oracle's Tier C, ~1e-15 from the reference) unless its
  options ask for ``precision="fp32"`` (the fast fp32 contract, Tier A).
* ``Renderer`` -- one per device: owns the workspace (grown on demand; a pair
  overflow re-runs the frame with the capacity the device reported), the
  stream, and launches ``rs_render`` / ``rs_project_full`` / ``rs_compact``.

Everything here calls the CUDA library; nothing computes on the CPU.
"""

from __future__ import annotations

import ctypes as C
import weakref

import numpy as np
import torch

from . import _native as N
from .core import InvalidParameterError, InvalidSceneError

PLANES = 11  # positions(3), opacity logit, log scales(3), quaternion(4); SH rows are separate
DEFAULT_PRECISION = "fp64"
_PRECISIONS = {"fp64": N.RS_F64, "f64": N.RS_F64, "float64": N.RS_F64, "double": N.RS_F64,
               "fp32": N.RS_F32, "f32": N.RS_F32, "float32": N.RS_F32, "float": N.RS_F32}


def precision_of(opts) -> int:
    """RS_F32 / RS_F64 of a RasterizeOptions-like object (``precision`` attribute;
    objects without one -- e.g. the reference's own RasterizeOptions -- get fp64)."""
    p = getattr(opts, "precision", None) or DEFAULT_PRECISION
    try:
        return _PRECISIONS[str(p).lower()]
    except KeyError:
        raise InvalidParameterError(f"precision must be 'fp32' or 'fp64', got {p!r}") from None


def value_dtype(precision: int) -> torch.dtype:
    return torch.float64 if precision == N.RS_F64 else torch.float32


def _arrays(scene):
    return (scene.positions, scene.opacity_logits, scene.log_scales, scene.quaternions, scene.sh)


def storage_dtype(scene) -> np.dtype:
    """float32 when every value is exactly representable in fp32, else float64."""
    for a in _arrays(scene):
        a = np.asarray(a)
        if a.dtype == np.float32 or a.size == 0:
            continue
        if a.dtype != np.float64 or not np.array_equal(a.astype(np.float32).astype(np.float64), a):
            return np.dtype(np.float64)
    return np.dtype(np.float32)


def pack_planes(scene, dtype=np.float32) -> np.ndarray:
    """(11, N) plane-major geometry of a scene-like object."""
    pos = np.asarray(scene.positions)
    n = pos.shape[0]
    out = np.empty((PLANES, n), dtype)
    out[0:3] = pos.reshape(n, 3).T
    out[3] = np.asarray(scene.opacity_logits).reshape(n)
    out[4:7] = np.asarray(scene.log_scales).reshape(n, 3).T
    out[7:11] = np.asarray(scene.quaternions).reshape(n, 4).T
    return out


def pack_sh(scene, dtype=np.float32) -> np.ndarray:
    """(N, 48) SH rows, channel-major [c][b] (core.py:480)."""
    sh = np.asarray(scene.sh)
    return np.ascontiguousarray(sh.reshape(sh.shape[0], 48), dtype=dtype)


class DeviceScene:
    """A scene resident in HBM (fp32 or fp64 planes) plus its ``rs_scene`` descriptor."""

    def __init__(self, scene, device: torch.device | None = None, check_finite: bool = True, dtype=None):
        lib = N.load()
        self.device = torch.device(device or torch.device("cuda", torch.cuda.current_device()))
        dt = np.dtype(dtype) if dtype is not None else storage_dtype(scene)
        host = torch.from_numpy(pack_planes(scene, dt))
        host_sh = torch.from_numpy(pack_sh(scene, dt))
        self.n = int(host.shape[1])
        self.sh_degree = int(scene.active_sh_degree)
        if not 0 <= self.sh_degree <= 3:
            raise InvalidParameterError("active SH degree must be in 0..3")
        self.generation = getattr(scene, "generation", None)
        with torch.cuda.device(self.device):
            if self.n:
                self.planes = host.pin_memory().to(self.device, non_blocking=True)
                self.sh = host_sh.pin_memory().to(self.device, non_blocking=True)
            else:
                self.planes = torch.zeros((PLANES, 1), dtype=host.dtype, device=self.device)
                self.sh = torch.zeros((1, 48), dtype=host.dtype, device=self.device)
        self.struct = N.RsScene(self.planes.data_ptr(), self.sh.data_ptr(), self.n, max(self.n, 1),
                                self.sh_degree, self.dtype_code)
        if check_finite and self.n:
            with torch.cuda.device(self.device):
                bad = torch.zeros(1, dtype=torch.int32, device=self.device)
                N.check(lib.rs_check_finite(C.byref(self.struct), bad.data_ptr(),
                                            torch.cuda.current_stream(self.device).cuda_stream), "check_finite")
                if int(bad.item()) != 0:
                    raise InvalidSceneError("scene contains non-finite parameters")

    @classmethod
    def from_tensors(cls, planes: torch.Tensor, sh: torch.Tensor, sh_degree: int, n: int | None = None,
                     generation=None, check_finite: bool = True) -> "DeviceScene":
        """Wrap device tensors already in the scene layout ((11, N) planes, (N, 48) SH rows),
        e.g. an RSPL payload unpacked on the device (io.load_scene_device)."""
        self = cls.__new__(cls)
        lib = N.load()
        self.device = planes.device
        self.n = int(planes.shape[1]) if n is None else int(n)
        self.sh_degree = int(sh_degree)
        if not 0 <= self.sh_degree <= 3:
            raise InvalidParameterError("active SH degree must be in 0..3")
        self.generation = generation
        self.planes, self.sh = planes, sh
        if planes.dtype not in (torch.float32, torch.float64) or sh.dtype != planes.dtype:
            raise InvalidParameterError("scene planes / SH must be float32 or float64 (same dtype)")
        self.struct = N.RsScene(planes.data_ptr(), sh.data_ptr(), self.n, max(self.n, 1), self.sh_degree,
                                self.dtype_code)
        if check_finite and self.n:
            with torch.cuda.device(self.device):
                bad = torch.zeros(1, dtype=torch.int32, device=self.device)
                N.check(lib.rs_check_finite(C.byref(self.struct), bad.data_ptr(),
                                            torch.cuda.current_stream(self.device).cuda_stream), "check_finite")
                if int(bad.item()) != 0:
                    raise InvalidSceneError("scene contains non-finite parameters")
        return self

    @property
    def dtype_code(self) -> int:
        return N.RS_F64 if self.planes.dtype == torch.float64 else N.RS_F32

    def __len__(self):
        return self.n


_scene_cache: dict = {}


def device_scene(scene, device: torch.device | None = None, dtype=None) -> DeviceScene:
    """Upload once per (scene object, generation, device, storage dtype); later calls
    reuse it. ``dtype`` None = exact storage (storage_dtype)."""
    if isinstance(scene, DeviceScene):
        if dtype is None or np.dtype(dtype) == (np.float64 if scene.dtype_code == N.RS_F64 else np.float32):
            return scene
        raise InvalidParameterError("a DeviceScene cannot change its storage dtype")
    N.load()  # raises NativeUnavailable without the library or a CUDA device (no CPU fallback)
    dev = torch.device(device or torch.device("cuda", torch.cuda.current_device()))
    key = (id(scene), dev, None if dtype is None else np.dtype(dtype).str)
    hit = _scene_cache.get(key)
    gen = getattr(scene, "generation", None)
    if hit is not None and hit.generation == gen and hit.n == len(scene.positions):
        return hit
    ds = DeviceScene(scene, dev, dtype=dtype)
    _scene_cache[key] = ds
    try:
        weakref.finalize(scene, _scene_cache.pop, key, None)
    except TypeError:  # not weak-referenceable: keep only the latest such scene
        pass
    return ds


def camera_struct(cam) -> N.RsCamera:
    """fp64 camera packet (the reference's values); centre = -R^T t (core.py:351-354).
    The library rounds it once for fp32 frames."""
    R = np.asarray(cam.rotation, np.float64).reshape(3, 3)
    t = np.asarray(cam.translation, np.float64).reshape(3)
    c = -R.T @ t
    s = N.RsCamera()
    s.width, s.height = int(cam.width), int(cam.height)
    s.fx, s.fy, s.cx, s.cy = (float(v) for v in (cam.fx, cam.fy, cam.cx, cam.cy))
    s.R[:] = [float(v) for v in R.ravel()]
    s.t[:] = [float(v) for v in t]
    s.center[:] = [float(v) for v in c]
    return s


def options_struct(opts) -> N.RsOptions:
    return N.RsOptions(*(float(getattr(opts, k)) for k in
                         ("alpha_max", "alpha_cut", "tau_stop", "near_limit", "lowpass", "sigma_bound")),
                       precision_of(opts), 0)


class Renderer:
    """Frame launcher bound to one CUDA device."""

    def __init__(self, device: torch.device | None = None):
        self.lib = N.load()
        self.device = torch.device(device or torch.device("cuda", torch.cuda.current_device()))
        self.buf = None
        self.handle = C.c_void_p()
        self.caps = (0, 0, 0, 0)
        self.frame_id = 0  # frames launched on this workspace (rs_backward needs the latest one)

    # -- workspace ---------------------------------------------------------
    def ensure(self, n: int, pairs: int, width: int, height: int) -> None:
        cn, cp, cw, ch = self.caps
        if n <= cn and pairs <= cp and width <= cw and height <= ch:
            return
        caps = (max(n, cn, 1), max(pairs, cp, 1 << 16), max(width, cw), max(height, ch))
        size = self.lib.rs_workspace_size(*caps)
        if size == 0:
            raise InvalidParameterError(f"unsupported workspace shape {caps}")
        self.close()
        self.frame_id += 1  # a new workspace holds no frame: a cached backward must redo its forward
        with torch.cuda.device(self.device):
            self.buf = torch.empty(size, dtype=torch.uint8, device=self.device)
        N.check(self.lib.rs_workspace_create(self.buf.data_ptr(), size, *caps, C.byref(self.handle)),
                "workspace_create")
        self.caps = caps

    def close(self) -> None:
        if self.handle:
            torch.cuda.synchronize(self.device)
            self.lib.rs_workspace_destroy(self.handle)
            self.handle = C.c_void_p()
        self.buf = None
        self.caps = (0, 0, 0, 0)

    def __del__(self):
        try:
            if self.handle:
                self.lib.rs_workspace_destroy(self.handle)
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    def stats(self) -> N.RsStats:
        st = N.RsStats()
        N.check(self.lib.rs_read_stats(self.handle, C.byref(st), self.stream), "read_stats")
        return st

    def read_overflow(self, reset: bool = True) -> tuple[bool, int]:
        """(did any frame since the last reset overflow, largest P it needed); synchronizes.
        Raises InvalidParameterError if one of those frames had an out-of-range active index."""
        o, p, b = C.c_uint32(), C.c_uint64(), C.c_uint32()
        N.check(self.lib.rs_read_sticky(self.handle, C.byref(o), C.byref(p), C.byref(b), int(reset), self.stream),
                "read_sticky")
        if b.value:
            raise InvalidParameterError("active index list holds an index outside the scene")
        return bool(o.value), int(p.value)

    def clear_sticky(self) -> None:
        o, p, b = C.c_uint32(), C.c_uint64(), C.c_uint32()
        N.check(self.lib.rs_read_sticky(self.handle, C.byref(o), C.byref(p), C.byref(b), 1, self.stream),
                "read_sticky")

    def buffers(self) -> N.RsBuffers:
        b = N.RsBuffers()
        N.check(self.lib.rs_get_buffers(self.handle, C.byref(b)), "get_buffers")
        return b

    def view(self, ptr: int, count: int, dtype: torch.dtype) -> torch.Tensor:
        """A tensor view of `count` elements at device pointer `ptr` inside the workspace."""
        off = int(ptr) - self.buf.data_ptr()
        size = torch.empty((), dtype=dtype).element_size()
        assert 0 <= off and off + count * size <= self.buf.numel()
        return self.buf[off:off + count * size].view(dtype)

    def frame_arrays(self) -> dict:
        """Binning state of the last frame, copied to host (parity tests)."""
        st, b = self.stats(), self.buffers()
        T = b.tiles_x * b.tiles_y
        return dict(
            stats=st, tiles_x=b.tiles_x, tiles_y=b.tiles_y,
            records=self.view(b.records, 16 * st.n_items, torch.float32).view(-1, 16).cpu().numpy(),
            records64=self.view(b.records64, 24 * st.n_items, torch.float32).view(-1, 24).cpu().numpy(),
            items_sorted=self.view(b.items_sorted, st.n_items, torch.int32).cpu().numpy().view(np.uint32),
            pair_items=self.view(b.pair_items, st.n_pairs, torch.int32).cpu().numpy().view(np.uint32),
            ranges=self.view(b.ranges, 2 * T, torch.int32).cpu().numpy().view(np.uint32).reshape(T, 2))

    # -- frames --------------------------------------------------------------
    def alloc_outputs(self, cam, color: bool = True, precision: int = N.RS_F32) -> dict:
        """Device images of a frame: float32 (RS_F32) or float64 (RS_F64) rgb/alpha/depth."""
        H, W = int(cam.height), int(cam.width)
        if not color:
            return {}
        d, vt = self.device, value_dtype(precision)
        return dict(rgb=torch.empty((H, W, 3), dtype=vt, device=d),
                    alpha=torch.empty((H, W), dtype=vt, device=d),
                    depth=torch.empty((H, W), dtype=vt, device=d),
                    count=torch.empty((H, W), dtype=torch.int32, device=d))

    @staticmethod
    def outputs_struct(out: dict) -> N.RsOutputs:
        """rs_outputs over the image tensors present in ``out`` (fp32 device images
        rgb/alpha/depth/count and/or reference-typed rgb64/alpha64/count64, which may
        live in pinned host memory)."""
        return N.RsOutputs(*(out[k].data_ptr() if k in out else None for k in
                             ("rgb", "alpha", "depth", "count", "rgb64", "alpha64", "count64", "tau", "last")))

    def launch(self, ds: DeviceScene, cam_s: N.RsCamera, opt_s: N.RsOptions, out: dict,
               scores: torch.Tensor | None = None, active_idx: torch.Tensor | None = None,
               m: int = 0, flags: int = 0) -> None:
        """Enqueue one frame (no host synchronization)."""
        self.frame_id += 1
        N.check(self.lib.rs_render_ex(
            self.handle, C.byref(ds.struct), active_idx.data_ptr() if active_idx is not None else None,
            int(m), C.byref(cam_s), C.byref(opt_s), C.byref(self.outputs_struct(out)),
            scores.data_ptr() if scores is not None else None, flags, self.stream), "render")

    @staticmethod
    def check_scores(scores: torch.Tensor | None, precision: int, ds: "DeviceScene | None" = None) -> None:
        """A score vector holds the frame's value type (float32 / float64, non-negative), one
        entry per Gaussian of the scene, on the scene's device."""
        if scores is not None and ds is not None and (scores.numel() < ds.n or not scores.is_contiguous()
                                                      or scores.device != torch.device(ds.device)):
            raise InvalidParameterError(f"scores must be a contiguous vector of >= {ds.n} entries on {ds.device}")
        if scores is not None and scores.dtype not in (value_dtype(precision), torch.int32, torch.int64):
            raise InvalidParameterError(f"scores must be {value_dtype(precision)} for this precision")
        if scores is not None and scores.element_size() != (8 if precision == N.RS_F64 else 4):
            raise InvalidParameterError("scores element size does not match the precision")

    @staticmethod
    def check_outputs(out: dict, cam, precision: int, device) -> None:
        """Caller-provided images must hold the frame (dtype, element count, contiguity; the
        float64/int64 reference-typed ones may be pinned host memory) -- the kernels write
        through the raw pointers."""
        H, W = int(cam.height), int(cam.width)
        vt = value_dtype(precision)
        spec = {"rgb": (vt, 3), "alpha": (vt, 1), "depth": (vt, 1), "count": (torch.int32, 1),
                "rgb64": (torch.float64, 3), "alpha64": (torch.float64, 1), "count64": (torch.int64, 1),
                "tau": (torch.float32, 1), "last": (torch.int32, 1)}
        for k, t in out.items():
            if k not in spec:
                raise InvalidParameterError(f"unknown output {k!r}")
            dt, ch = spec[k]
            if t.dtype != dt or t.numel() < H * W * ch or not t.is_contiguous():
                raise InvalidParameterError(f"output {k!r} must be a contiguous {dt} tensor of >= {H * W * ch} "
                                            f"elements for this frame and precision")
            if k in ("rgb64", "alpha64", "count64"):
                if not (t.is_cuda or t.is_pinned()):
                    raise InvalidParameterError(f"output {k!r} must be device or pinned host memory")
            elif not t.is_cuda or t.device != torch.device(device):
                raise InvalidParameterError(f"output {k!r} must live on {device}")

    def render(self, ds: DeviceScene, cam, opts, *, color: bool = True, scores: torch.Tensor | None = None,
               active_idx: torch.Tensor | None = None, m: int | None = None, count_evals: bool = False,
               out: dict | None = None) -> tuple[dict, N.RsStats]:
        """One frame with overflow handling (reads the counters: synchronizes)."""
        items = ds.n if active_idx is None else int(m if m is not None else active_idx.numel())
        W, H = int(cam.width), int(cam.height)
        self.ensure(items, self.caps[1] or max(4 * items, 1 << 20), W, H)
        cam_s, opt_s = camera_struct(cam), options_struct(opts)
        self.check_scores(scores, opt_s.precision, ds)
        if out is not None:
            self.check_outputs(out, cam, opt_s.precision, ds.device)
        out = out if out is not None else self.alloc_outputs(cam, color, opt_s.precision)
        flags = N.RS_FLAG_COUNT_EVALS if count_evals else 0
        snapshot = scores.clone() if scores is not None else None
        for _ in range(4):
            self.launch(ds, cam_s, opt_s, out, scores, active_idx, items, flags)
            st = self.stats()
            if st.bad_index:
                self.clear_sticky()  # reported here: later passes must not re-raise it
                raise InvalidParameterError("active index list holds an index outside the scene")
            if not st.overflow:
                return out, st
            self.ensure(items, int(st.pairs_needed * 1.15) + 1024, W, H)
            if snapshot is not None:
                scores.copy_(snapshot)
        raise N.PairOverflow("tile pair capacity could not be satisfied")

    def score_views(self, ds: DeviceScene, cams, opts, scores: torch.Tensor) -> None:
        """Score-only frames of every camera max-merged into ``scores`` (fp32 bits viewed
        as int32), launched back to back with no host sync per view; the pass is checked
        for pair overflow once and, if a view overflowed, re-run from a snapshot with the
        capacity the device reported."""
        cams = list(cams)
        if not cams:
            return
        W, H = max(int(c.width) for c in cams), max(int(c.height) for c in cams)
        self.ensure(ds.n, self.caps[1] or max(4 * ds.n, 1 << 20), W, H)
        opt_s = options_struct(opts)
        self.check_scores(scores, opt_s.precision, ds)
        structs = [camera_struct(c) for c in cams]
        snapshot = scores.clone()
        self.read_overflow(reset=True)
        for _ in range(4):
            for cs in structs:
                self.launch(ds, cs, opt_s, {}, scores)
            over, need = self.read_overflow(reset=True)
            if not over:
                return
            self.ensure(ds.n, int(need * 1.15) + 1024, W, H)
            scores.copy_(snapshot)
        raise N.PairOverflow("tile pair capacity could not be satisfied")

    def capture(self, ds: DeviceScene, cam, opts, *, color: bool = True, scores: torch.Tensor | None = None,
                active_idx: torch.Tensor | None = None, pairs_hint: int | None = None) -> FrameGraph:
        """Capture one frame into a CUDA graph (workspace sized first, no overflow check at
        replay time: size it with ``pairs_hint`` or a checked ``render`` beforehand)."""
        items = ds.n if active_idx is None else int(active_idx.numel())
        self.ensure(items, max(self.caps[1], pairs_hint or 0, 1 << 16), int(cam.width), int(cam.height))
        out = self.alloc_outputs(cam, color, precision_of(opts))
        torch.cuda.synchronize(self.device)
        self.frame_id += 1  # capture records a frame without running it
        return FrameGraph(self, ds, cam, opts, out, scores, active_idx, items)

    def project_full(self, ds: DeviceScene, cam, opts) -> tuple[np.ndarray, np.ndarray]:
        """ProjectedGaussian fields for every Gaussian (render.py:161-211), in the
        frame's value type."""
        self.ensure(ds.n, self.caps[1] or (1 << 16), int(cam.width), int(cam.height))
        n = max(ds.n, 1)
        self.frame_id += 1  # the projection replaces the workspace's frame
        full = torch.empty((n, 16), dtype=value_dtype(precision_of(opts)), device=self.device)
        bbox = torch.empty((n, 4), dtype=torch.int32, device=self.device)
        N.check(self.lib.rs_project_full(self.handle, C.byref(ds.struct), None, 0, C.byref(camera_struct(cam)),
                                         C.byref(options_struct(opts)), full.data_ptr(), bbox.data_ptr(),
                                         self.stream), "project_full")
        if self.stats().bad_index:
            self.clear_sticky()
            raise InvalidParameterError("active index list holds an index outside the scene")
        return full[:ds.n].cpu().numpy(), bbox[:ds.n].cpu().numpy()

    def compact(self, flags: torch.Tensor, bits: bool = False, n: int | None = None) -> torch.Tensor:
        """Ascending indices of non-zero flags (or set bits), on device."""
        n = int(flags.numel() if n is None else n)
        nbytes = self.lib.rs_compact_workspace_size(n)
        scratch = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.device)
        idx = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        cnt = torch.empty(1, dtype=torch.int32, device=self.device)
        fn = self.lib.rs_compact_bits if bits else self.lib.rs_compact
        N.check(fn(flags.data_ptr() if n else None, n, idx.data_ptr(), cnt.data_ptr(), scratch.data_ptr(),
                   scratch.numel(), self.stream), "compact")
        return idx[:int(cnt.item())]


class FrameGraph:
    """One frame (rs_render) captured into a CUDA graph.

    The camera lives in the workspace (``rs_set_camera``, a stream-ordered copy
    enqueued before each replay), so ``replay(cam)`` renders a new view without
    re-capture: the whole frame (memset and ~12 kernels) is one graph launch.
    """

    def __init__(self, r: "Renderer", ds: DeviceScene, cam, opts, out: dict, scores=None,
                 active_idx=None, m: int = 0):
        self.r, self.ds, self.out, self.scores = r, ds, out, scores
        self.buf = r.buf
        self.width, self.height = int(cam.width), int(cam.height)
        self.opt_s = options_struct(opts)
        self.set_camera(cam)
        side = torch.cuda.Stream(r.device)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.device(r.device):
            side.wait_stream(torch.cuda.current_stream(r.device))
            with torch.cuda.graph(self.graph, stream=side):
                N.check(r.lib.rs_render_ex(
                    r.handle, C.byref(ds.struct), active_idx.data_ptr() if active_idx is not None else None,
                    int(m), None, C.byref(self.opt_s), C.byref(r.outputs_struct(out)),
                    scores.data_ptr() if scores is not None else None, 0, side.cuda_stream), "render(capture)")

    def set_camera(self, cam) -> None:
        if int(cam.width) != self.width or int(cam.height) != self.height:
            raise InvalidParameterError("a captured frame graph is bound to its image size")
        cs = camera_struct(cam)
        N.check(self.r.lib.rs_set_camera(self.r.handle, C.byref(cs), self.r.stream), "set_camera")

    def replay(self, cam=None) -> None:
        """Enqueue the frame (optionally after uploading a new camera) on the current stream."""
        if self.r.buf is not self.buf:
            raise RuntimeError("the workspace was re-allocated after capture; capture again")
        if cam is not None:
            self.set_camera(cam)
        self.r.frame_id += 1
        self.graph.replay()


def pack_bits_device(flags: torch.Tensor) -> torch.Tensor:
    """(n,) bool/uint8 CUDA tensor -> LSB-first bitset bytes (np.packbits(bitorder="little"))."""
    lib = N.load()
    n = int(flags.numel())
    out = torch.empty(max((n + 7) // 8, 1), dtype=torch.uint8, device=flags.device)
    f = flags.contiguous().view(torch.uint8)
    with torch.cuda.device(flags.device):
        N.check(lib.rs_pack_bits(f.data_ptr() if n else None, n, out.data_ptr(),
                                 torch.cuda.current_stream(flags.device).cuda_stream), "pack_bits")
    return out[:(n + 7) // 8]


_renderers: dict = {}


def renderer(device: torch.device | None = None) -> Renderer:
    N.load()
    dev = torch.device(device or torch.device("cuda", torch.cuda.current_device()))
    r = _renderers.get(dev)
    if r is None:
        r = _renderers[dev] = Renderer(dev)
    return r
