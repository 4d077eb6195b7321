"""ncu driver: a few configs[1] training steps (forward with cache + backward)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
from paper_2403_13806_b200 import synth  # noqa: E402
from paper_2403_13806_b200.render import RasterizeOptions, rasterize_backward, rasterize_cached  # noqa: E402

scene, cams = synth.config1(0, n_frames=8)
opts = RasterizeOptions(near_limit=0.2)
w = np.random.default_rng(0).normal(size=(cams[0].height, cams[0].width, 3))
for f in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    out, cache = rasterize_cached(scene, cams[f], opts)
    g = rasterize_backward(scene, cams[f], cache, w)
print("train ok", int(g["touched"].sum()))
