"""Scene, camera and error types of the render-and-prune path (host side).

Mirrors the value types the reference rasterizer consumes
(``fieldsplat/core.py``) so reference callers can switch imports without
touching their code:

* exception classes -- ``core.py:20-37``
* ``normalize_quaternion`` / ``quat_to_rotmat`` -- ``core.py:111-139``
* SH constants and ``SH_BANDS_FOR_DEGREE`` -- ``core.py:196-204``
* ``SH_COLOR_OFFSET`` -- ``core.py:288``
* ``PinholeCamera`` (+ ``center`` = -R^T t) -- ``core.py:316-374``
* ``look_at_camera`` (horizontal fov, fx = fy, principal point W/2, H/2)
  -- ``core.py:382-412``
* ``sigmoid`` / ``logit`` -- ``core.py:419-426``
* ``GaussianScene`` (frozen float64 SoA, quaternions normalized on
  construction, ``generation`` staleness tag, ``subset``) -- ``core.py:470-562``

Reference objects are accepted everywhere through duck typing: the device
path only reads ``positions``, ``opacity_logits``, ``sh``, ``log_scales``,
``quaternions``, ``active_sh_degree`` and ``generation`` from a scene and
``width``, ``height``, ``fx``, ``fy``, ``cx``, ``cy``, ``rotation``,
``translation`` from a camera.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np


class InvalidParameterError(ValueError):
    """A primitive or camera parameter violates its domain."""


class InvalidSceneError(ValueError):
    """A scene contains non-finite or otherwise unusable parameters."""


class StaleTableError(RuntimeError):
    """A per-Gaussian table was computed against a different scene revision."""


class FileFormatError(IOError):
    """A persisted file has the wrong magic or an unsupported version (core.py:35-36)."""


SH_C0 = 0.28209479177387814
SH_BANDS_FOR_DEGREE = (1, 4, 9, 16)
SH_COLOR_OFFSET = 0.5


def _frozen(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    a.setflags(write=False)
    return a


def normalize_quaternion(q) -> np.ndarray:
    q = np.asarray(q, dtype=np.float64)
    norm = np.linalg.norm(q, axis=-1, keepdims=True)
    if np.any(norm < 1e-12):
        raise InvalidParameterError("zero quaternion has no direction")
    return q / norm


def quat_to_rotmat(q) -> np.ndarray:
    """(…, 4) wxyz -> (…, 3, 3); the device kernel evaluates the same nine
    entries in fp32 (csrc/project.cu)."""
    q = normalize_quaternion(q)
    w, x, y, z = (q[..., i] for i in range(4))
    r = np.empty(q.shape[:-1] + (3, 3))
    r[..., 0, 0] = 1 - 2 * (y * y + z * z)
    r[..., 0, 1] = 2 * (x * y - w * z)
    r[..., 0, 2] = 2 * (x * z + w * y)
    r[..., 1, 0] = 2 * (x * y + w * z)
    r[..., 1, 1] = 1 - 2 * (x * x + z * z)
    r[..., 1, 2] = 2 * (y * z - w * x)
    r[..., 2, 0] = 2 * (x * z - w * y)
    r[..., 2, 1] = 2 * (y * z + w * x)
    r[..., 2, 2] = 1 - 2 * (x * x + y * y)
    return r


def sigmoid(x):
    x = np.asarray(x, dtype=np.float64)
    with np.errstate(over="ignore"):
        return np.where(x >= 0, 1.0 / (1.0 + np.exp(-x)), np.exp(x) / (1.0 + np.exp(x)))


def logit(p):
    p = np.asarray(p, dtype=np.float64)
    return np.log(p) - np.log1p(-p)


@dataclass(frozen=True)
class ImageBuffer:
    """(H, W, 3) float64 read-only colour image (reference core.py:74-101)."""

    data: np.ndarray

    def __post_init__(self):
        data = np.asarray(self.data, dtype=np.float64)
        if data.ndim != 3 or data.shape[2] != 3:
            raise InvalidParameterError(f"image must be (H, W, 3), got {data.shape}")
        if not np.all(np.isfinite(data)):
            raise InvalidParameterError("image contains non-finite values")
        object.__setattr__(self, "data", _frozen(data))

    @classmethod
    def trusted(cls, data: np.ndarray) -> "ImageBuffer":
        """Wrap a freshly rendered (H, W, 3) float64 array without re-validating it:
        the kernels only produce finite sums of finite products."""
        obj = object.__new__(cls)
        data.setflags(write=False)
        object.__setattr__(obj, "data", data)
        return obj

    @property
    def height(self) -> int:
        return self.data.shape[0]

    @property
    def width(self) -> int:
        return self.data.shape[1]


@dataclass(frozen=True)
class PinholeCamera:
    """World-to-camera rigid transform ``p_cam = R p + t``; +z forward,
    x right, y down (reference ``core.py:316-374``)."""

    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    rotation: np.ndarray
    translation: np.ndarray

    def __post_init__(self):
        if self.width <= 0 or self.height <= 0:
            raise InvalidParameterError("image dimensions must be positive")
        if self.fx <= 0 or self.fy <= 0:
            raise InvalidParameterError("focal lengths must be positive")
        if not (0 <= self.cx < self.width and 0 <= self.cy < self.height):
            raise InvalidParameterError("principal point must lie inside the image")
        rot = np.asarray(self.rotation, dtype=np.float64)
        tr = np.asarray(self.translation, dtype=np.float64).reshape(3)
        if rot.shape != (3, 3):
            raise InvalidParameterError("rotation must be 3x3")
        if np.max(np.abs(rot @ rot.T - np.eye(3))) > 1e-9:
            raise InvalidParameterError("rotation must be orthonormal within 1e-9")
        if abs(np.linalg.det(rot) - 1.0) > 1e-9:
            raise InvalidParameterError("rotation must have det +1 within 1e-9")
        object.__setattr__(self, "rotation", _frozen(rot))
        object.__setattr__(self, "translation", _frozen(tr))

    @property
    def center(self) -> np.ndarray:
        return -self.rotation.T @ self.translation


def look_at_camera(eye, target, up=(0.0, 0.0, 1.0), *, width: int, height: int,
                   fov_deg: float = 60.0) -> PinholeCamera:
    """Camera at ``eye`` looking at ``target``; ``fov_deg`` is horizontal."""
    eye = np.asarray(eye, dtype=np.float64)
    fwd = np.asarray(target, dtype=np.float64) - eye
    n = np.linalg.norm(fwd)
    if n < 1e-12:
        raise InvalidParameterError("eye and target coincide")
    fwd = fwd / n
    right = np.cross(fwd, np.asarray(up, dtype=np.float64))
    if np.linalg.norm(right) < 1e-9:  # up parallel to the view axis
        right = np.cross(fwd, np.array([0.0, 1.0, 0.0]))
    right = right / np.linalg.norm(right)
    rot = np.stack([right, np.cross(fwd, right), fwd])
    u, _, vt = np.linalg.svd(rot)  # exact orthonormality for the 1e-9 gate
    rot = u @ vt
    f = 0.5 * width / np.tan(np.deg2rad(fov_deg) / 2)
    return PinholeCamera(width=width, height=height, fx=f, fy=f,
                         cx=width / 2.0, cy=height / 2.0,
                         rotation=rot, translation=-rot @ eye)


_generation = itertools.count(1)


@dataclass(frozen=True)
class GaussianScene:
    """Ordered Gaussian primitives as frozen float64 struct-of-arrays."""

    positions: np.ndarray       # (N, 3)
    opacity_logits: np.ndarray  # (N,)
    sh: np.ndarray              # (N, 3, 16) channel-major
    log_scales: np.ndarray      # (N, 3)
    quaternions: np.ndarray     # (N, 4) wxyz
    active_sh_degree: int = 0
    metadata: dict = field(default_factory=dict)
    generation: int = field(default_factory=lambda: next(_generation))

    def __post_init__(self):
        n = np.asarray(self.positions).shape[0]
        q = np.asarray(self.quaternions, dtype=np.float64).reshape(n, 4)
        if n > 0:
            q = normalize_quaternion(q)
        if not 0 <= self.active_sh_degree <= 3:
            raise InvalidParameterError("active SH degree must be in 0..3")
        object.__setattr__(self, "positions", _frozen(np.asarray(self.positions, dtype=np.float64).reshape(n, 3)))
        object.__setattr__(self, "opacity_logits", _frozen(np.asarray(self.opacity_logits, dtype=np.float64).reshape(n)))
        object.__setattr__(self, "sh", _frozen(np.asarray(self.sh, dtype=np.float64).reshape(n, 3, 16)))
        object.__setattr__(self, "log_scales", _frozen(np.asarray(self.log_scales, dtype=np.float64).reshape(n, 3)))
        object.__setattr__(self, "quaternions", _frozen(q))

    def __len__(self) -> int:
        return self.positions.shape[0]

    # frozen dataclasses with ndarray fields: identity semantics
    __hash__ = object.__hash__

    def __eq__(self, other):
        return self is other

    @property
    def opacities(self) -> np.ndarray:
        return sigmoid(self.opacity_logits)

    @property
    def scales(self) -> np.ndarray:
        return np.exp(self.log_scales)

    def is_finite(self) -> bool:
        return scene_is_finite(self)

    def subset(self, mask_or_indices) -> "GaussianScene":
        idx = np.asarray(mask_or_indices)
        return GaussianScene(
            positions=self.positions[idx], opacity_logits=self.opacity_logits[idx],
            sh=self.sh[idx], log_scales=self.log_scales[idx],
            quaternions=self.quaternions[idx],
            active_sh_degree=self.active_sh_degree, metadata=dict(self.metadata))


def scene_is_finite(scene) -> bool:
    return all(np.all(np.isfinite(np.asarray(a))) for a in
               (scene.positions, scene.opacity_logits, scene.sh,
                scene.log_scales, scene.quaternions))
