"""Driver for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): a few small
frames through every kernel family of the library, both precisions.

    compute-sanitizer --tool memcheck python tools/sanitize_frames.py

configs[0] frame (fp32 + fp64, scores, host float64 outputs), a 100k-Gaussian binning-stress
frame at 640x480 (cooperative depth sort) and the same with the onesweep launches
(RS_DSORT=0 in the environment), one scoring pass (configs[2] distributions, 4 views), one
backward (forward with cache + rs_backward), a filtered render from a device index list,
compaction, the RSPL unpack and the metrics kernels.
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    from paper_2403_13806_b200 import metrics, synth
    from paper_2403_13806_b200.core import look_at_camera
    from paper_2403_13806_b200.pruning import compute_importance
    from paper_2403_13806_b200.render import (RasterizeOptions, rasterize, rasterize_backward, rasterize_cached,
                                              rasterize_filtered, render_device)
    s0, c0 = synth.config0(0)
    for prec in ("fp32", "fp64"):
        o = RasterizeOptions(near_limit=0.2, precision=prec)
        vt = torch.float32 if prec == "fp32" else torch.float64
        sc = torch.zeros(len(s0), dtype=vt, device="cuda")
        render_device(s0, c0[0], o, scores=sc, count_evals=True)
        out = rasterize(s0, c0[0], o)
        rasterize_filtered(s0, c0[0], np.arange(len(s0)) % 3 == 0, o)
        s1, _ = synth.config1(1, n=100_000, n_frames=1)
        cam = look_at_camera((2.8, -1.1, 0.7), (0.1, 0.0, 0.0), width=640, height=480, fov_deg=55.0)
        render_device(s1, cam, o)
        s2, c2 = synth.config2(0, n=60_000, n_views=4)
        compute_importance(s2, c2, o)
    res, cache = rasterize_cached(s0, c0[0], RasterizeOptions(near_limit=0.2, precision="fp32"))
    rasterize_backward(s0, c0[0], cache, np.ones((128, 128, 3)))
    img = out.color.data
    metrics.psnr(img, np.clip(img + 0.01, 0, 1))
    metrics.ssim_with_grad(img, np.clip(img + 0.01, 0, 1))
    torch.cuda.synchronize()
    print("sanitize frames ok")


if __name__ == "__main__":
    main()
