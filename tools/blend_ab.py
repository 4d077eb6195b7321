"""A/B of blend variants on configs[1] frames: project+bin once, then time rs_blend per flag.

    python tools/blend_ab.py [frames] [render|score] [fp32|fp64]
"""
import ctypes as C
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2403_13806_b200 import _native as N, synth  # noqa: E402
from paper_2403_13806_b200.device import camera_struct, device_scene, options_struct, renderer  # noqa: E402
from paper_2403_13806_b200.render import RasterizeOptions  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 20
kind = sys.argv[2] if len(sys.argv) > 2 else "render"
prec = sys.argv[3] if len(sys.argv) > 3 else "fp32"
opts = RasterizeOptions(near_limit=0.2, precision=prec)
scene, cams = synth.config1(0) if kind == "render" else synth.config2(0)
ds = device_scene(scene)
r = renderer(ds.device)
out = r.alloc_outputs(cams[0], precision=0 if prec == "fp32" else 1)
sc = torch.zeros(len(scene), dtype=torch.float32 if prec == "fp32" else torch.float64, device=ds.device)
for f in range(frames):
    r.render(ds, cams[f], opts, out=out, color=kind == "render", scores=None if kind == "render" else sc)
os_ = options_struct(opts)
st = torch.cuda.current_stream().cuda_stream
outs = r.outputs_struct(out) if kind == "render" else N.RsOutputs()
res = {0: [], N.RS_FLAG_BLEND_1PX: []} if prec == "fp32" else {0: []}
ref = {}
for f in range(frames):
    N.check(r.lib.rs_project(r.handle, C.byref(ds.struct), None, 0, C.byref(camera_struct(cams[f])), C.byref(os_), st))
    N.check(r.lib.rs_bin(r.handle, st))
    for rep in range(3):
        for flag in res:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            sc.zero_()
            a.record()
            N.check(r.lib.rs_blend_ex(r.handle, C.byref(os_), C.byref(outs), sc.data_ptr() if kind != "render" else None,
                                      flag, st))
            b.record()
            torch.cuda.synchronize()
            if rep:
                res[flag].append(a.elapsed_time(b))
            if kind == "render":
                ref.setdefault((f, flag), out["rgb"].clone())
            else:
                ref.setdefault((f, flag), sc.clone())
for f in range(frames):
    if prec == "fp32" and not os.environ.get("BLEND_AB_NOCHECK"):
        assert torch.equal(ref[(f, 0)], ref[(f, N.RS_FLAG_BLEND_1PX)]), f
for flag, v in res.items():
    print(kind, prec, "2px" if flag == 0 else "1px", f"{1e3 * sum(v) / len(v):.1f} us")
