"""Host-side cost of one Renderer.render() / rasterize() call (cProfile over 50 frames)."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2403_13806_b200 import synth  # noqa: E402
from paper_2403_13806_b200.device import device_scene, renderer  # noqa: E402
from paper_2403_13806_b200.render import RasterizeOptions, rasterize  # noqa: E402

scene, cams = synth.config1(0, n_frames=100)
opts = RasterizeOptions(near_limit=0.2, precision="fp32")
ds = device_scene(scene)
r = renderer(ds.device)
out = r.alloc_outputs(cams[0])
for c in cams[:5]:
    r.render(ds, c, opts, out=out)
torch.cuda.synchronize()
t0 = time.perf_counter()
for c in cams[:50]:
    r.render(ds, c, opts, out=out)
print(f"render(): {1e3 * (time.perf_counter() - t0) / 50:.3f} ms/frame")
pr = cProfile.Profile()
pr.enable()
for c in cams[:50]:
    r.render(ds, c, opts, out=out)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
for c in cams[:5]:
    rasterize(scene, c, opts)
pr = cProfile.Profile()
pr.enable()
for c in cams[:50]:
    rasterize(scene, c, opts)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
