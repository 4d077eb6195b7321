"""Image metrics on the device (metrics.py:34-117) vs the reference's own values
(tests/golden/metrics.npz). float64 on both sides; only the summation order
differs, so: MSE / PSNR / SSIM within 1e-12 relative, the SSIM gradient within
1e-12 of its largest magnitude."""

import math

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["render", "rand", "gray"])
def test_metrics_match_reference(name):
    from paper_2403_13806_b200 import metrics as M
    d = golden("metrics")
    a, b = d[name + "_a"], d[name + "_b"]
    assert M.mse(a, b) == pytest.approx(float(d[name + "_mse"]), rel=1e-12)
    assert M.psnr(a, b) == pytest.approx(float(d[name + "_psnr"]), rel=1e-12)
    assert M.ssim(a, b) == pytest.approx(float(d[name + "_ssim"]), rel=1e-12)
    assert M.ssim(a, b, win_size=7, sigma=1.0) == pytest.approx(float(d[name + "_ssim7"]), rel=1e-12)
    v, g = M.ssim_with_grad(a, b)
    assert v == pytest.approx(float(d[name + "_ssim"]), rel=1e-12)
    ref = d[name + "_ssim_g"]
    assert g.shape == ref.shape
    assert np.abs(g - ref).max() <= 1e-12 * np.abs(ref).max()


def test_metrics_edge_cases():
    import torch
    from paper_2403_13806_b200 import metrics as M
    from paper_2403_13806_b200.core import InvalidParameterError
    a = np.random.default_rng(0).uniform(size=(12, 12, 3))
    assert M.psnr(a, a) == math.inf
    assert M.ssim(torch.from_numpy(a).cuda(), a) == pytest.approx(1.0, rel=1e-12)
    with pytest.raises(InvalidParameterError):
        M.mse(a, a[:, :11])
    with pytest.raises(InvalidParameterError):
        M.ssim(a[:10], a[:10])
