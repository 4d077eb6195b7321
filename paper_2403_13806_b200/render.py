"""Reference-compatible rasterizer API backed by the sm_100a kernels.

Same names, arguments, return types and error behaviour as the reference's
``fieldsplat.render`` forward path (render.py:37-321), so callers switch by
changing the import:

* ``RasterizeOptions`` (render.py:37-46), ``ProjectedGaussian`` (:49-59),
  ``RenderOutput`` (:62-68; plus a ``depth`` image),
  ``ContributionAccumulator`` (:71-88)
* ``project_gaussian`` / ``project_scene`` (:161-211)
* ``rasterize`` (:290-293), ``rasterize_with_contributions`` (:296-308),
  ``rasterize_filtered`` (:311-315)
* ``rasterize_cached`` (:318-321) and ``rasterize_backward`` (:328-487), the
  training pair

The compute runs on the GPU in fp64 by default -- the reference's own
expressions and composite order, bit-identical to the oracle's Tier C and
within ~1e-15 of the NumPy reference -- or, with
``RasterizeOptions(precision="fp32")``, on the fast fp32 path (bit-identical
to the Tier-A fp32 oracle; DESIGN.md §4 gives its measured distance from the
reference). The training pair (``rasterize_cached`` / ``rasterize_backward``)
is fp32. Device-native entry points that keep everything in HBM
(``render_device``) are what the benchmarks use.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

import ctypes as C
from dataclasses import replace

from . import _native as N
from .core import GaussianScene, ImageBuffer, InvalidParameterError
from .device import DeviceScene, device_scene, options_struct, precision_of, renderer, value_dtype


@dataclass(frozen=True)
class RasterizeOptions:
    """render.py:37-46, plus the arithmetic precision of the GPU frame: "fp64"
    (default; the reference's arithmetic) or "fp32" (the fast contract)."""
    alpha_max: float = 0.99
    alpha_cut: float = 1.0 / 255.0
    tau_stop: float = 1e-4
    near_limit: float = 0.01
    lowpass: float = 0.3
    sigma_bound: float = 3.0
    precision: str = "fp64"


def fp32_options(options) -> RasterizeOptions:
    """The same options on the fp32 path (the training pair's precision)."""
    return RasterizeOptions(*(float(getattr(options, k)) for k in
                              ("alpha_max", "alpha_cut", "tau_stop", "near_limit", "lowpass", "sigma_bound")),
                            precision="fp32")


@dataclass(frozen=True)
class ProjectedGaussian:
    index: int
    mean2d: np.ndarray
    cov2d: np.ndarray
    depth: float
    color: np.ndarray
    opacity: float
    bbox: tuple


class RenderOutput:
    """color (ImageBuffer, (H,W,3) float64), alpha (H,W) float64, count (H,W) int64,
    plus ``depth`` (H,W) = sum of w * camera z -- not in the reference; copied from
    the device on first access only."""

    def __init__(self, color: ImageBuffer, alpha: np.ndarray, count: np.ndarray, depth=None):
        self.color, self.alpha, self.count = color, alpha, count
        self._depth = depth

    @property
    def depth(self):
        if isinstance(self._depth, torch.Tensor):
            self._depth = self._depth.double().cpu().numpy()
        return self._depth


class ContributionAccumulator:
    """Per-Gaussian running max of alpha*tau (float64, caller-owned)."""

    def __init__(self, n: int):
        self.values = np.zeros(n, dtype=np.float64)

    def __len__(self) -> int:
        return self.values.shape[0]

    def update(self, other) -> None:
        np.maximum(self.values, other, out=self.values)

    def merge(self, other: "ContributionAccumulator") -> None:
        self.update(other.values)


def _check_scene(scene) -> DeviceScene:
    """Device copy of the scene. Finiteness (render.py:229-230) is checked by
    the rs_check_finite kernel once per upload: scenes are immutable and the
    upload is cached per generation, so this equals a check per render."""
    return device_scene(scene)


def render_device(scene, camera, options: RasterizeOptions = RasterizeOptions(), *, color: bool = True,
                  scores: torch.Tensor | None = None, active_idx: torch.Tensor | None = None,
                  count_evals: bool = False):
    """Render one view on the GPU; returns (dict of device tensors, rs_stats).

    ``scores`` is an (N,) CUDA tensor of the frame's value type (float32 for
    fp32 frames, float64 for fp64 frames) max-merged in place (bit-level
    atomicMax on non-negative values)."""
    ds = _check_scene(scene)
    r = renderer(ds.device)
    return r.render(ds, camera, options, color=color, scores=scores, active_idx=active_idx,
                    count_evals=count_evals)


def _render_host(scene, camera, options, *, scores: torch.Tensor | None = None,
                 active_idx: torch.Tensor | None = None) -> RenderOutput:
    """One frame whose reference-typed results (float64 colour/alpha, int64 count)
    the blend kernel writes straight into pinned host memory (no device-side
    widening pass, no staging copy); depth stays on the device until read."""
    ds = _check_scene(scene)
    r = renderer(ds.device)
    H, W = int(camera.height), int(camera.width)
    out = dict(rgb64=torch.empty((H, W, 3), dtype=torch.float64, pin_memory=True),
               alpha64=torch.empty((H, W), dtype=torch.float64, pin_memory=True),
               count64=torch.empty((H, W), dtype=torch.int64, pin_memory=True),
               depth=torch.empty((H, W), dtype=value_dtype(precision_of(options)), device=ds.device))
    r.render(ds, camera, options, scores=scores, active_idx=active_idx, out=out)  # synchronizes
    return RenderOutput(color=ImageBuffer.trusted(out["rgb64"].numpy()), alpha=out["alpha64"].numpy(),
                        count=out["count64"].numpy(), depth=out["depth"])


def rasterize(scene, camera, options: RasterizeOptions = RasterizeOptions()) -> RenderOutput:
    """Render over a black background, front to back (render.py:290-293)."""
    return _render_host(scene, camera, options)


def rasterize_with_contributions(scene, camera, accumulator: ContributionAccumulator,
                                 options: RasterizeOptions = RasterizeOptions()) -> RenderOutput:
    """Same image as ``rasterize``; max-merges alpha*tau into ``accumulator``."""
    if len(accumulator) != len(scene):
        raise InvalidParameterError("accumulator length must equal scene size")
    ds = _check_scene(scene)
    scores = torch.zeros(max(ds.n, 1), dtype=value_dtype(precision_of(options)), device=ds.device)
    res = _render_host(ds, camera, options, scores=scores)
    accumulator.update(scores[:ds.n].cpu().numpy().astype(np.float64))
    return res


def active_indices(scene, active, device=None) -> torch.Tensor:
    """Bool indicator over scene order -> ascending int32 index list on device
    (compacted by the rs_compact kernel)."""
    a = np.asarray(active, dtype=bool)
    if a.shape != (len(scene),):
        raise InvalidParameterError("indicator list length must equal scene size")
    ds = _check_scene(scene)
    flags = torch.from_numpy(a.view(np.uint8)).to(ds.device)
    return renderer(ds.device).compact(flags)


def rasterize_filtered(scene, camera, active, options: RasterizeOptions = RasterizeOptions()) -> RenderOutput:
    """Render only the active Gaussians; only those are projected."""
    idx = active_indices(scene, active)
    return _render_host(scene, camera, options, active_idx=idx)


# ---------------------------------------------------------------------------
# training: forward with cache + backward (render.py:318-487)
# ---------------------------------------------------------------------------
def _fp32_scene(scene) -> DeviceScene:
    """The scene as the training pair reads it: fp32 storage (rounded once if needed)."""
    ds = _check_scene(scene)
    if ds.dtype_code == N.RS_F32 or isinstance(scene, DeviceScene):
        if ds.dtype_code != N.RS_F32:
            raise InvalidParameterError("the training pair needs an fp32 device scene")
        return ds
    return device_scene(scene, ds.device, dtype=np.float32)


def _training_forward(ds: DeviceScene, camera, options, active_idx=None):
    r = renderer(ds.device)
    options = fp32_options(options)
    out = r.alloc_outputs(camera)
    H, W = int(camera.height), int(camera.width)
    out["tau"] = torch.empty((H, W), dtype=torch.float32, device=ds.device)
    out["last"] = torch.empty((H, W), dtype=torch.int32, device=ds.device)
    r.render(ds, camera, options, out=out, active_idx=active_idx)
    return out, r.frame_id


def rasterize_cached(scene, camera, options: RasterizeOptions = RasterizeOptions(), *,
                     device_outputs: bool = False):
    """Forward render keeping what the backward pass needs (render.py:318-321):
    returns (RenderOutput, cache). The cache holds, on the device, the per-pixel
    final transmittance and last composite; the binning stays in the workspace.
    The training pair runs on the fp32 path (fp32 scene storage).

    ``device_outputs=True`` (a device-resident training loop: the scene a
    ``DeviceScene.from_tensors`` over parameter tensors updated in place, the loss
    on the device) returns the device images dict (rgb, alpha, depth, count)
    instead of host arrays."""
    ds = _fp32_scene(scene)
    out, frame = _training_forward(ds, camera, options)
    if device_outputs:
        return {k: out[k] for k in ("rgb", "alpha", "depth", "count")}, \
            dict(options=options, device_out=out, frame=frame, camera=camera)
    H, W = int(camera.height), int(camera.width)
    res = RenderOutput(color=ImageBuffer.trusted(out["rgb"].double().cpu().numpy().reshape(H, W, 3)),
                       alpha=out["alpha"].double().cpu().numpy(), count=out["count"].long().cpu().numpy(),
                       depth=out["depth"])
    return res, dict(options=options, device_out=out, frame=frame, camera=camera)


def rasterize_backward(scene, camera, cache: dict, grad_image, *, device: bool = False) -> dict:
    """Analytic gradients of a scalar loss through the rendered image
    (render.py:328-394 + _chain_to_parameters :397-487). ``grad_image`` =
    dL/d(colour image), (H, W, 3). Returns float64 gradients w.r.t. positions,
    sh, log_scales, quaternions, opacity_logits, plus ``mean2d_grad_norm`` and
    ``touched`` -- the reference's dict, computed by rs_backward in fp32.

    ``device=True``: ``grad_image`` may be a CUDA tensor (used in place) and the
    gradients stay on the device as fp32 tensors (positions (n,3), sh (n,3,16),
    log_scales (n,3), quaternions (n,4), opacity_logits, mean2d_grad_norm, touched)
    -- no host round trip per optimizer step."""
    ds = _fp32_scene(scene)
    r = renderer(ds.device)
    options = fp32_options(cache["options"])
    out = cache["device_out"]
    if r.frame_id != cache["frame"]:  # the workspace rendered something else since: redo the forward
        out, cache["frame"] = _training_forward(ds, camera, options)
        cache["device_out"] = out
    H, W = int(camera.height), int(camera.width)
    dev = ds.device
    if isinstance(grad_image, torch.Tensor):
        grad = grad_image.to(device=dev, dtype=torch.float32).contiguous()
        if tuple(grad.shape) != (H, W, 3):
            raise InvalidParameterError(f"grad_image must be ({H}, {W}, 3)")
    else:
        g = np.asarray(grad_image, dtype=np.float32)
        if g.shape != (H, W, 3):
            raise InvalidParameterError(f"grad_image must be ({H}, {W}, 3)")
        grad = torch.from_numpy(np.ascontiguousarray(g)).to(dev)
    n = max(ds.n, 1)
    o = dict(positions=torch.empty((n, 3), device=dev), sh=torch.empty((n, 48), device=dev),
             log_scales=torch.empty((n, 3), device=dev), quaternions=torch.empty((n, 4), device=dev),
             opacity_logits=torch.empty(n, device=dev), mean2d_grad_norm=torch.empty(n, device=dev),
             touched=torch.empty(n, dtype=torch.uint8, device=dev))
    N.check(r.lib.rs_backward(r.handle, C.byref(ds.struct), None, 0, C.byref(options_struct(options)),
                              grad.data_ptr(), out["tau"].data_ptr(), out["last"].data_ptr(),
                              *(o[k].data_ptr() for k in ("positions", "sh", "log_scales", "quaternions",
                                                         "opacity_logits", "mean2d_grad_norm", "touched")),
                              r.stream), "backward")
    if device:
        o = {k: v[:ds.n] for k, v in o.items()}
        o["sh"] = o["sh"].view(ds.n, 3, 16)
        o["touched"] = o["touched"].bool()
        return o
    res = {k: v[:ds.n].cpu().numpy() for k, v in o.items()}
    grads = {k: res[k].astype(np.float64) for k in ("positions", "log_scales", "quaternions", "opacity_logits",
                                                  "mean2d_grad_norm")}
    grads["sh"] = res["sh"].astype(np.float64).reshape(ds.n, 3, 16)
    grads["touched"] = res["touched"].astype(bool)
    return grads


def _project_all(scene, camera, options):
    ds = _check_scene(scene)
    full, bbox = renderer(ds.device).project_full(ds, camera, options)
    return full.astype(np.float64), bbox.astype(np.int64)


def project_scene(scene, camera, options: RasterizeOptions = RasterizeOptions()):
    """List of ProjectedGaussian (culled omitted) plus the raw arrays."""
    full, bbox = _project_all(scene, camera, options)
    proj = dict(mx=full[:, 0], my=full[:, 1], a=full[:, 2], b=full[:, 3], c=full[:, 4],
                inv_a=full[:, 5], inv_b=full[:, 6], inv_c=full[:, 7], radius=full[:, 8],
                depth=full[:, 9], color=full[:, 10:13], opacity=full[:, 13], valid=full[:, 14] > 0.5,
                x0=bbox[:, 0], x1=bbox[:, 1], y0=bbox[:, 2], y1=bbox[:, 3])
    out = []
    for i in np.nonzero(proj["valid"])[0]:
        out.append(ProjectedGaussian(
            index=int(i), mean2d=np.array([proj["mx"][i], proj["my"][i]]),
            cov2d=np.array([[proj["a"][i], proj["b"][i]], [proj["b"][i], proj["c"][i]]]),
            depth=float(proj["depth"][i]), color=proj["color"][i].copy(),
            opacity=float(proj["opacity"][i]),
            bbox=(int(proj["x0"][i]), int(proj["x1"][i]), int(proj["y0"][i]), int(proj["y1"][i]))))
    return out, proj


def project_gaussian(primitive, camera, options: RasterizeOptions = RasterizeOptions(),
                     active_sh_degree: int = 3) -> ProjectedGaussian | None:
    """Project one primitive; None when culled (render.py:161-191)."""
    scene = GaussianScene(positions=np.asarray(primitive.position)[None],
                          opacity_logits=np.array([primitive.opacity_logit]),
                          sh=np.asarray(primitive.sh)[None], log_scales=np.asarray(primitive.log_scale)[None],
                          quaternions=np.asarray(primitive.quaternion)[None], active_sh_degree=active_sh_degree)
    lst, _ = project_scene(scene, camera, options)
    if not lst:
        return None
    g = lst[0]
    return ProjectedGaussian(index=0, mean2d=g.mean2d, cov2d=g.cov2d, depth=g.depth, color=g.color,
                             opacity=g.opacity, bbox=g.bbox)
