"""Backward pass (render.py:318-487) on the GPU vs the reference's own fp64
gradients (tests/golden/grad.npz, made by tests/golden/make_golden.py grad).

fp32 with atomic per-Gaussian sums: a tolerance, stated here. Each gradient
array must match the reference within 2e-5 of that array's largest magnitude
(plus 1e-6 absolute) -- the same scale-relative criterion as the reference's
own finite-difference check (test_render.py:183-222, rel 1e-4 in fp64);
touched flags exactly."""

import numpy as np
import pytest
import torch

from conftest import golden, load_case, load_cam, options_from

pytestmark = pytest.mark.gpu

REL = 2e-5
KEYS = ("positions", "sh", "log_scales", "quaternions", "opacity_logits", "mean2d_grad_norm")


def _cases():
    return [str(c) for c in golden("grad")["cases"]]


@pytest.mark.parametrize("name", _cases())
def test_backward_matches_reference_gradients(name):
    from paper_2403_13806_b200.render import rasterize_backward, rasterize_cached
    d = golden("grad")
    p = name + "_"
    scene, cam, o = load_case(d, p)
    opts = options_from(o)
    out, cache = rasterize_cached(scene, cam, opts)
    assert np.abs(out.color.data - d[p + "img"]).max() < 1e-4
    g = rasterize_backward(scene, cam, cache, d[p + "w"])
    assert np.array_equal(g["touched"], d[p + "g_touched"]), name
    for k in KEYS:
        ref = d[p + "g_" + k]
        got = g[k]
        scale = np.abs(ref).max()
        err = np.abs(got - ref).max()
        assert err <= REL * scale + 1e-6, f"{name}.{k}: max err {err} vs scale {scale}"
    untouched = ~g["touched"]
    for k in KEYS:
        assert np.all(g[k][untouched] == 0)


def test_backward_after_other_frames_recomputes_the_forward():
    """A cache whose workspace rendered other frames since is re-forwarded, not misread."""
    from paper_2403_13806_b200.render import rasterize, rasterize_backward, rasterize_cached
    d = golden("grad")
    p = "deg3_"
    scene, cam, o = load_case(d, p)
    opts = options_from(o)
    _, cache = rasterize_cached(scene, cam, opts)
    g1 = rasterize_backward(scene, cam, cache, d[p + "w"])
    rasterize(scene, load_cam(golden("known"), "single_"), opts)  # another frame on the same workspace
    g2 = rasterize_backward(scene, cam, cache, d[p + "w"])
    for k in KEYS:
        assert np.allclose(g1[k], g2[k], rtol=1e-5, atol=1e-6)
