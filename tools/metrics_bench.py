"""Device SSIM / PSNR at configs[1] size (1256x828x3, float64) vs the oracle-free
reference formulas restated in numpy+scipy (same as metrics.py:59-117), one JSON line."""
import json
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from paper_2403_13806_b200 import metrics as M

rng = np.random.default_rng(0)
a = rng.uniform(size=(828, 1256, 3))
b = np.clip(a + rng.normal(scale=0.05, size=a.shape), 0, 1)
ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
res = {}
for name, fn in (("psnr", lambda: M.psnr(ta, tb)), ("ssim", lambda: M.ssim(ta, tb)),
                 ("ssim_with_grad", lambda: M.ssim_with_grad(ta, tb))):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    res[name + "_ms"] = 1e3 * (time.perf_counter() - t0) / 10
try:
    from scipy.signal import correlate2d
    k = M.gaussian_window()
    t0 = time.perf_counter()
    x, y = a[..., 0], b[..., 0]
    mu = correlate2d(x, k, mode="valid")
    res["cpu_scipy_one_correlate_ms"] = 1e3 * (time.perf_counter() - t0)
    res["cpu_scipy_ssim_estimate_ms"] = res["cpu_scipy_one_correlate_ms"] * 15  # 5 correlates x 3 channels
except Exception as e:  # noqa: BLE001
    res["cpu_error"] = str(e)
print(json.dumps(res))
