import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_cuda = torch.cuda.is_available()
    except Exception:
        has_cuda = False
    if has_cuda:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


_cache = {}


def golden(name: str):
    if name not in _cache:
        _cache[name] = dict(np.load(GOLDEN / f"{name}.npz"))
    return _cache[name]


def load_case(d, p):
    """(scene, camera, RasterizeOptions-like values) from a golden npz prefix."""
    from paper_2403_13806_b200.core import GaussianScene, PinholeCamera
    scene = GaussianScene(positions=d[p + "pos"], opacity_logits=d[p + "logit"], sh=d[p + "sh"],
                          log_scales=d[p + "ls"], quaternions=d[p + "quat"], active_sh_degree=int(d[p + "deg"]))
    cam = load_cam(d, p)
    opts = d.get(p + "opts")
    return scene, cam, opts


def load_cam(d, p):
    from paper_2403_13806_b200.core import PinholeCamera
    W, H = (int(v) for v in d[p + "wh"])
    fx, fy, cx, cy = (float(v) for v in d[p + "intr"])
    return PinholeCamera(width=W, height=H, fx=fx, fy=fy, cx=cx, cy=cy, rotation=d[p + "R"],
                         translation=d[p + "t"])


def options_from(vals, precision=None):
    """RasterizeOptions-like values; ``precision`` None = the library default (fp64)."""
    from types import SimpleNamespace
    if vals is None:
        vals = [0.99, 1.0 / 255.0, 1e-4, 0.01, 0.3, 3.0]
    keys = ("alpha_max", "alpha_cut", "tau_stop", "near_limit", "lowpass", "sigma_bound")
    o = SimpleNamespace(**dict(zip(keys, (float(v) for v in vals))))
    if precision is not None:
        o.precision = precision
    return o


def with_precision(opts, precision):
    """Copy of RasterizeOptions-like ``opts`` (None = defaults) on the given path."""
    keys = ("alpha_max", "alpha_cut", "tau_stop", "near_limit", "lowpass", "sigma_bound")
    vals = None if opts is None else [getattr(opts, k) for k in keys]
    return options_from(vals, precision)


# the two GPU paths and the oracle tier each must reproduce bit for bit
PRECISIONS = [("fp32", np.float32), ("fp64", "c64")]
PREC_IDS = ["fp32", "fp64"]


def render_cases():
    """(name, scene, cam, opts) for every golden render case."""
    out = []
    for f in ("suite50", "accept50"):
        d = golden(f)
        for c in range(int(d["n_cases"])):
            s, cam, o = load_case(d, f"c{c}_")
            out.append((f"{f}-{c}", s, cam, options_from(o), d, f"c{c}_"))
    d = golden("known")
    for name in ("single", "twolayer", "tie", "iso", "lowpass", "occluder", "occluder1", "behind",
                 "offscreen", "ragged"):
        s, cam, o = load_case(d, name + "_")
        out.append((name, s, cam, options_from(o), d, name + "_"))
    d = golden("config0")
    s, cam, o = load_case(d, "cfg0_")
    out.append(("config0", s, cam, options_from(o), d, "cfg0_"))
    return out


def reference_check_fp64(name, img, alpha, count, contrib, d, p):
    """fp64 path (Tier C bits) vs the fp64 reference's golden output: same
    composite decisions everywhere (count identical), pixels and scores within
    a few ulp -- asserted at 1e-12 (north_star: 1e-4 pixels, 1e-5 scores)."""
    assert np.array_equal(count, d[p + "count"]), (name, int((count != d[p + "count"]).sum()))
    assert np.abs(img - d[p + "img"]).max(initial=0.0) <= 1e-12, name
    assert np.abs(alpha - d[p + "alpha"]).max(initial=0.0) <= 1e-12, name
    ref = d[p + "contrib"]
    assert np.array_equal(contrib > 0, ref > 0), name
    rel = np.abs(contrib - ref) / np.maximum(ref, 1e-300)
    assert rel.max(initial=0.0) <= 1e-12, (name, float(rel.max(initial=0.0)))


def tier_b_check(name, img, alpha, count, contrib, d, p, thresholds=(0.001, 0.01, 0.05)):
    """fp32 result vs the fp64 reference's golden output (Tier B budget).

    * count flips (a threshold decision alpha >= 1/255 or tau >= 1e-4 taken the
      other way in fp32) are rare: <= max(4, pixels / 10^4);
    * every pixel that is not a flip pixel is within the north-star 1e-4 (RGB
      and alpha); flip pixels may differ by up to alpha_cut * tau;
    * importance: >= 99.5% of Gaussians within 1e-5 relative (fp32 tau after
      many near-opaque layers carries ~6e-8 * o/(1-o) relative error per layer);
    * prune / visibility masks identical except where |h - t| <= 1e-4 * t.
    """
    ref_count = d[p + "count"]
    flips = count != ref_count
    assert flips.sum() <= max(4, ref_count.size // 10000), (name, int(flips.sum()))
    err = np.abs(img - d[p + "img"]).max(axis=-1)
    assert np.all(err[~flips] <= 1e-4), (name, float(err[~flips].max()))
    aerr = np.abs(alpha - d[p + "alpha"])
    assert np.all(aerr[~flips] <= 1e-4), (name, float(aerr[~flips].max()))
    ref = d[p + "contrib"]
    rel = np.abs(contrib - ref) / np.maximum(ref, 1e-30)
    assert np.mean(rel <= 1e-5) >= 0.995, (name, float(rel.max()))
    assert np.all(rel <= 1e-3) or flips.any(), (name, float(rel.max()))
    for t in thresholds:
        diff = (contrib >= t) != (ref >= t)
        assert np.all(np.abs(ref[diff] - t) <= 1e-4 * t), (name, t)
