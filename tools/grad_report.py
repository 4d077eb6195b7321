"""Backward pass vs the reference's fp64 gradients: max error / array scale per case."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np
from conftest import golden, load_case, options_from
from paper_2403_13806_b200.render import rasterize_backward, rasterize_cached
d = golden("grad")
for name in d["cases"]:
    p = str(name) + "_"
    scene, cam, o = load_case(d, p)
    out, cache = rasterize_cached(scene, cam, options_from(o))
    g = rasterize_backward(scene, cam, cache, d[p + "w"])
    errs = {k: float(np.abs(g[k] - d[p + "g_" + k]).max() / max(np.abs(d[p + "g_" + k]).max(), 1e-30))
            for k in ("positions", "sh", "log_scales", "quaternions", "opacity_logits", "mean2d_grad_norm")}
    print(name, len(scene.positions), {k: f"{v:.1e}" for k, v in errs.items()})
