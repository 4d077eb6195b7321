"""Where one rasterize() call's time goes (configs[1] frames): pinned output allocation, the
frame on the device (CUDA events around the launches, host outputs included), the host sync /
stats read and the Python around it. RS_E2E_BANDS selects the host-output path."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2403_13806_b200 import synth
from paper_2403_13806_b200.device import device_scene, renderer
from paper_2403_13806_b200.render import RasterizeOptions, rasterize

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
scene, cams = synth.config1(0, n_frames=100)
opts = RasterizeOptions(near_limit=0.2, precision=prec)
ds = device_scene(scene)
r = renderer(ds.device)
H, W = cams[0].height, cams[0].width
for c in cams[:5]:
    rasterize(scene, c, opts)
torch.cuda.synchronize()
n = 60
t0 = time.perf_counter()
for c in cams[:n]:
    rasterize(scene, c, opts)
t_ras = (time.perf_counter() - t0) / n
t0 = time.perf_counter()
for c in cams[:n]:
    out = dict(rgb64=torch.empty((H, W, 3), dtype=torch.float64, pin_memory=True),
               alpha64=torch.empty((H, W), dtype=torch.float64, pin_memory=True),
               count64=torch.empty((H, W), dtype=torch.int64, pin_memory=True))
t_alloc = (time.perf_counter() - t0) / n
vt = torch.float64 if prec == "fp64" else torch.float32
out = dict(rgb64=torch.empty((H, W, 3), dtype=torch.float64, pin_memory=True),
           alpha64=torch.empty((H, W), dtype=torch.float64, pin_memory=True),
           count64=torch.empty((H, W), dtype=torch.int64, pin_memory=True),
           depth=torch.empty((H, W), dtype=vt, device="cuda"))
for c in cams[:3]:
    r.render(ds, c, opts, out=out)
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
t0 = time.perf_counter()
for i, c in enumerate(cams[:n]):
    ev[i][0].record()
    r.render(ds, c, opts, out=out)
    ev[i][1].record()
t_render = (time.perf_counter() - t0) / n
torch.cuda.synchronize()
t_dev = sum(a.elapsed_time(b) for a, b in ev) / n / 1e3
print(f"{prec}: rasterize {t_ras*1e3:.3f} ms ({1/t_ras:.0f} fps) | pinned alloc x3 {t_alloc*1e3:.3f} ms | "
      f"render(prealloc) {t_render*1e3:.3f} ms | device span {t_dev*1e3:.3f} ms")
# frames launched back to back (no host sync per frame): the device-bound rate of host-output frames
from paper_2403_13806_b200.device import camera_struct, options_struct  # noqa: E402
opt_s = options_struct(opts)
structs = [camera_struct(c) for c in cams[:n]]
for cs in structs[:3]:
    r.launch(ds, cs, opt_s, out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for cs in structs:
    r.launch(ds, cs, opt_s, out)
e1.record()
torch.cuda.synchronize()
print(f"{prec}: back-to-back host-output frames {e0.elapsed_time(e1) / n:.3f} ms/frame (device-bound)")
