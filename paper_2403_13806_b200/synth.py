"""Seeded synthetic scenes and camera sets for BASELINE.json ``configs[0..4]``.

The reference ships no generator for these workloads; the paper's
datasets (MipNeRF360, Zip-NeRF) are not available offline, so these seeded
scenes with the BASELINE shapes, sizes and value distributions stand in.

Draw order (fixed, documented in DESIGN.md): means, log-scales, quaternions,
opacity logits, SH DC, SH rest -- all from ``numpy.random.default_rng(seed)``
(the reference's own seeding practice, ``pkg/tests/conftest.py:46-48``).
Arrays are stored as float32; the fp64 reference consumes the same values
upcast, exactly as it reads RSPL files (``io.py:163-191``).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .core import GaussianScene, look_at_camera


@dataclass
class SceneArrays:
    """fp32 struct-of-arrays scene (duck-types ``GaussianScene`` for the device
    path). Quaternions are stored normalized (fp64 normalize, then cast)."""

    positions: np.ndarray
    opacity_logits: np.ndarray
    sh: np.ndarray
    log_scales: np.ndarray
    quaternions: np.ndarray
    active_sh_degree: int = 3
    metadata: dict = field(default_factory=dict)
    generation: int = 0

    def __post_init__(self):
        if not self.generation:
            # unique tag so the device cache never confuses two scenes
            from .core import _generation
            self.generation = next(_generation)

    __hash__ = object.__hash__

    def __eq__(self, other):
        return self is other

    def __len__(self):
        return self.positions.shape[0]

    def to_scene(self) -> GaussianScene:
        """fp64 ``GaussianScene`` holding the same (upcast) values."""
        return GaussianScene(
            positions=self.positions.astype(np.float64),
            opacity_logits=self.opacity_logits.astype(np.float64),
            sh=self.sh.astype(np.float64),
            log_scales=self.log_scales.astype(np.float64),
            quaternions=self.quaternions.astype(np.float64),
            active_sh_degree=self.active_sh_degree,
            metadata=dict(self.metadata))

    def subset(self, mask_or_indices) -> "SceneArrays":
        idx = np.asarray(mask_or_indices)
        return SceneArrays(self.positions[idx], self.opacity_logits[idx], self.sh[idx],
                           self.log_scales[idx], self.quaternions[idx],
                           self.active_sh_degree, dict(self.metadata))


def _attributes(rng, means, n, logscale_mu, logscale_sigma, logscale_max=None):
    ls = rng.normal(logscale_mu, logscale_sigma, size=(n, 3))
    if logscale_max is not None:
        ls = np.minimum(ls, logscale_max)
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    logits = rng.normal(0.0, 1.5, size=n)
    sh = np.empty((n, 3, 16))
    sh[:, :, 0] = rng.normal(0.0, 0.5, size=(n, 3))
    sh[:, :, 1:] = rng.normal(0.0, 0.1, size=(n, 3, 15))
    f = np.float32
    return SceneArrays(np.ascontiguousarray(means, f), logits.astype(f), sh.astype(f),
                       ls.astype(f), q.astype(f), 3)


def _clustered_means(rng, n, k=32, sigma=0.15, lo=-2.0, hi=2.0):
    centers = rng.uniform(lo, hi, size=(k, 3))
    labels = rng.integers(0, k, size=n)
    return np.clip(centers[labels] + rng.normal(0.0, sigma, size=(n, 3)), lo, hi)


def fibonacci_eyes(n: int, radius: float = 3.0) -> np.ndarray:
    i = np.arange(n) + 0.5
    z = 1.0 - 2.0 * i / n
    r = np.sqrt(1.0 - z * z)
    phi = i * np.pi * (3.0 - np.sqrt(5.0))
    return radius * np.stack([r * np.cos(phi), r * np.sin(phi), z], axis=1)


def config0(seed: int = 0):
    """4,096 Gaussians, 128x128, fov 50 deg, eye (0,-3,0) on the radius-3 sphere."""
    rng = np.random.default_rng(seed)
    n = 4096
    means = rng.uniform(-1.0, 1.0, size=(n, 3))
    scene = _attributes(rng, means, n, -3.5, 0.4)
    cam = look_at_camera((0.0, -3.0, 0.0), (0.0, 0.0, 0.0), width=128, height=128, fov_deg=50.0)
    return scene, [cam]


def orbit_cameras(n: int, width=1256, height=828, fov_deg=55.0, radius=3.0, height_z=0.6):
    """Orbit at horizontal radius 3, fixed elevation z=0.6 (frame 0 = the SURVEY
    measurement camera (3,0,0.6))."""
    cams = []
    for k in range(n):
        th = 2.0 * np.pi * k / n
        eye = (radius * np.cos(th), radius * np.sin(th), height_z)
        cams.append(look_at_camera(eye, (0.0, 0.0, 0.0), width=width, height=height, fov_deg=fov_deg))
    return cams


def config1(seed: int = 0, n: int = 500_000, n_frames: int = 1000):
    """500k Gaussians in 32 clusters (sigma 0.15) inside [-2,2]^3; 1256x828 orbit."""
    rng = np.random.default_rng(seed)
    means = _clustered_means(rng, n)
    return _attributes(rng, means, n, -3.5, 0.4), orbit_cameras(n_frames)


def config2(seed: int = 0, n: int = 3_000_000, n_views: int = 200):
    """3M Gaussians, log-scales N(-4.0, 0.6); 200 Fibonacci cameras at radius 3."""
    rng = np.random.default_rng(seed)
    means = _clustered_means(rng, n)
    scene = _attributes(rng, means, n, -4.0, 0.6)
    cams = [look_at_camera(e, (0.0, 0.0, 0.0), width=1256, height=828, fov_deg=55.0)
            for e in fibonacci_eyes(n_views)]
    return scene, cams


BOX_LO = np.array([-10.0, -10.0, 0.0])
BOX_HI = np.array([10.0, 10.0, 4.0])


def config3(seed: int = 0, n: int = 6_000_000, n_cams: int = 512, n_frames: int = 300,
            width: int = 1920, height: int = 1080):
    """House scale: half uniform in the 20x20x4 box, half in 256 clusters
    (sigma 0.3); log-scales N(-3.8,0.5). 512 training cameras on 8 random walks
    of 64 steps inside the box; the 300-frame test trajectory runs along the
    same walks, one frame halfway between consecutive training poses (held-out
    in-between views, as test views are taken from a capture path), evenly
    subsampled from the 8 x 63 midpoints in walk order."""
    rng = np.random.default_rng(seed)
    n_uni = n // 2
    uni = rng.uniform(BOX_LO, BOX_HI, size=(n_uni, 3))
    centers = rng.uniform(BOX_LO, BOX_HI, size=(256, 3))
    labels = rng.integers(0, 256, size=n - n_uni)
    clu = np.clip(centers[labels] + rng.normal(0.0, 0.3, size=(n - n_uni, 3)), BOX_LO, BOX_HI)
    scene = _attributes(rng, np.concatenate([uni, clu]), n, -3.8, 0.5)
    walk_rng = np.random.default_rng(seed + 1)
    cams, mids = [], []
    walks, steps = 8, n_cams // 8

    def cam_at(pos, head):
        tgt = pos + np.array([np.cos(head), np.sin(head), -0.1])
        return look_at_camera(pos, tgt, width=width, height=height, fov_deg=55.0)

    for _ in range(walks):
        pos = walk_rng.uniform([-8, -8, 1.0], [8, 8, 3.0])
        head = walk_rng.uniform(0, 2 * np.pi)
        prev = None
        for _ in range(steps):
            head += walk_rng.normal(0.0, 0.3)
            pos = np.clip(pos + 0.4 * np.array([np.cos(head), np.sin(head), 0.0])
                          + walk_rng.normal(0, 0.05, 3), [-9.5, -9.5, 0.5], [9.5, 9.5, 3.5])
            cams.append(cam_at(pos, head))
            if prev is not None:
                mids.append(cam_at(0.5 * (prev[0] + pos), 0.5 * (prev[1] + head)))
            prev = (pos.copy(), head)
    pick = np.round(np.linspace(0, len(mids) - 1, n_frames)).astype(int) if mids else []
    traj = [mids[k] for k in pick]
    return scene, cams, traj


def config4(seed: int = 0, n: int = 1_000_000, n_views: int = 512):
    """1M Gaussians, heavy-tailed anisotropic log-scales N(-3,1) clamped at
    scale <= 0.5 (log-scale <= ln 0.5); 512 Fibonacci views at 1920x1080."""
    rng = np.random.default_rng(seed)
    means = _clustered_means(rng, n)
    scene = _attributes(rng, means, n, -3.0, 1.0, logscale_max=float(np.log(0.5)))
    cams = [look_at_camera(e, (0.0, 0.0, 0.0), width=1920, height=1080, fov_deg=55.0)
            for e in fibonacci_eyes(n_views)]
    return scene, cams
