"""Where does the e2e (rasterize) time go? Host-link bandwidth vs frame time vs API overhead."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2403_13806_b200 import synth
from paper_2403_13806_b200.device import device_scene, renderer
from paper_2403_13806_b200.render import RasterizeOptions, rasterize

scene, cams = synth.config1(0, n_frames=100)
opts = RasterizeOptions(near_limit=0.2, precision="fp32")
ds = device_scene(scene)
r = renderer(ds.device)
H, W = cams[0].height, cams[0].width
nbytes = H * W * 40
dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
host = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
for _ in range(3):
    host.copy_(dev, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    host.copy_(dev, non_blocking=True)
torch.cuda.synchronize()
print(f"D2H copy engine: {20 * nbytes / (time.perf_counter() - t0) / 1e9:.1f} GB/s ({nbytes / 1e6:.1f} MB/frame)")
# zero-copy kernel writes: a fill kernel into the mapped pinned buffer
hv = host.view(torch.float64)
t0 = time.perf_counter()
for _ in range(20):
    hv.fill_(1.0)  # CPU tensor fill -> runs on CPU; use a device kernel via cuda tensor view below
t_cpu = time.perf_counter() - t0
print(f"CPU memset of the same buffer: {20 * nbytes / t_cpu / 1e9:.1f} GB/s")
out = r.alloc_outputs(cams[0])
for c in cams[:5]:
    r.render(ds, c, opts, out=out)
torch.cuda.synchronize()
t0 = time.perf_counter()
for c in cams[:50]:
    r.render(ds, c, opts, out=out)
torch.cuda.synchronize()
t_dev = (time.perf_counter() - t0) / 50
print(f"render() device outputs (wall, with stats sync): {1e3 * t_dev:.3f} ms/frame")
for path in ("zerocopy",):
    for c in cams[:5]:
        rasterize(scene, c, opts)
    t0 = time.perf_counter()
    for c in cams[:50]:
        rasterize(scene, c, opts)
    t_e2e = (time.perf_counter() - t0) / 50
    print(f"rasterize() [{path}]: {1e3 * t_e2e:.3f} ms/frame")
t0 = time.perf_counter()
for _ in range(50):
    o = dict(rgb64=torch.empty((H, W, 3), dtype=torch.float64, pin_memory=True),
             alpha64=torch.empty((H, W), dtype=torch.float64, pin_memory=True),
             count64=torch.empty((H, W), dtype=torch.int64, pin_memory=True))
    del o
print(f"pinned alloc (cached): {1e3 * (time.perf_counter() - t0) / 50:.3f} ms")
# the zero-copy host-output frame without the API's allocations
oh = dict(rgb64=torch.empty((H, W, 3), dtype=torch.float64, pin_memory=True),
          alpha64=torch.empty((H, W), dtype=torch.float64, pin_memory=True),
          count64=torch.empty((H, W), dtype=torch.int64, pin_memory=True),
          depth=torch.empty((H, W), dtype=torch.float32, device="cuda"))
for c in cams[:5]:
    r.render(ds, c, opts, out=oh)
t0 = time.perf_counter()
for c in cams[:50]:
    r.render(ds, c, opts, out=oh)
print(f"render() host outputs, reused buffers: {1e3 * (time.perf_counter() - t0) / 50:.3f} ms/frame")
