"""Image metrics on the device (reference ``fieldsplat/metrics.py:34-117``;
SURVEY §8f next #4): ``mse``, ``psnr``, ``ssim``, ``ssim_with_grad`` with the
reference's signatures, errors and float64 formulas, computed by the
``rs_sq_diff_sum`` / ``rs_ssim`` kernels. Inputs may be numpy arrays (as the
reference takes) or CUDA tensors (e.g. rendered frames that never leave HBM).
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np
import torch

from . import _native as N
from .core import InvalidParameterError

SSIM_C1 = 0.01 ** 2
SSIM_C2 = 0.03 ** 2


def _dev(x, device=None) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        t = x.detach()
        if not t.is_cuda:
            t = t.to(device or torch.device("cuda", torch.cuda.current_device()))
        return t.to(torch.float64).contiguous()
    a = np.asarray(getattr(x, "data", x), dtype=np.float64)  # ImageBuffer-like objects carry .data
    return torch.from_numpy(np.ascontiguousarray(a)).to(device or torch.device("cuda", torch.cuda.current_device()))


def _pair(a, b):
    N.load()
    ta = _dev(a)
    tb = _dev(b, ta.device)
    if ta.shape != tb.shape:
        raise InvalidParameterError(f"image shapes differ: {tuple(ta.shape)} vs {tuple(tb.shape)}")
    return ta, tb


def mse(a, b) -> float:
    ta, tb = _pair(a, b)
    out = torch.zeros(1, dtype=torch.float64, device=ta.device)
    with torch.cuda.device(ta.device):
        N.check(N.load().rs_sq_diff_sum(ta.data_ptr(), tb.data_ptr(), ta.numel(), out.data_ptr(),
                                        torch.cuda.current_stream(ta.device).cuda_stream), "sq_diff_sum")
    return float(out.item()) / ta.numel()


def psnr(a, b) -> float:
    """10 log10(1 / MSE) in dB; +inf when the images are identical (metrics.py:40-45)."""
    err = mse(a, b)
    if err == 0.0:
        return math.inf
    return 10.0 * math.log10(1.0 / err)


def gaussian_window(size: int = 11, sigma: float = 1.5) -> np.ndarray:
    """The reference's normalised Gaussian window (metrics.py:48-52), float64."""
    ax = np.arange(size, dtype=np.float64) - (size - 1) / 2.0
    g = np.exp(-0.5 * (ax / sigma) ** 2)
    k = np.outer(g, g)
    return k / k.sum()


def _ssim(a, b, win_size: int, sigma: float, want_grad: bool):
    ta, tb = _pair(a, b)
    if ta.dim() == 2:
        ta, tb = ta[..., None], tb[..., None]
    h, w, ch = ta.shape
    if h < win_size or w < win_size:
        raise InvalidParameterError(f"images must be at least {win_size}x{win_size} for SSIM")
    lib = N.load()
    dev = ta.device
    kern = torch.from_numpy(gaussian_window(win_size, sigma)).to(dev)
    out = torch.zeros(1, dtype=torch.float64, device=dev)
    grad = torch.empty_like(ta) if want_grad else None
    nbytes = lib.rs_ssim_workspace_size(h, w, ch, win_size) if want_grad else 0
    scratch = torch.empty(max(nbytes, 8), dtype=torch.uint8, device=dev) if want_grad else None
    with torch.cuda.device(dev):
        N.check(lib.rs_ssim(ta.data_ptr(), tb.data_ptr(), h, w, ch, win_size, kern.data_ptr(), out.data_ptr(),
                            grad.data_ptr() if want_grad else None, scratch.data_ptr() if want_grad else None,
                            nbytes, torch.cuda.current_stream(dev).cuda_stream), "ssim")
    n_windows = (h - win_size + 1) * (w - win_size + 1) * ch
    value = float(out.item()) / n_windows
    if want_grad:
        return value, grad.cpu().numpy()  # (H, W, C), like the reference (2-D inputs gain C = 1)
    return value, None


def ssim(a, b, win_size: int = 11, sigma: float = 1.5) -> float:
    """Mean local SSIM over valid windows, averaged across channels (metrics.py:59-64)."""
    return _ssim(a, b, win_size, sigma, False)[0]


def ssim_with_grad(a, b, win_size: int = 11, sigma: float = 1.5):
    """(SSIM, dSSIM/da) for gradient-based optimization against target b (metrics.py:67-71)."""
    return _ssim(a, b, win_size, sigma, True)
