"""Small deterministic driver for ncu: a few configs[1] frames (or configs[2] views).

    python tools/profile_frame.py [render|score|batch] [frames] [fp32|fp64]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2403_13806_b200 import synth  # noqa: E402
from paper_2403_13806_b200.device import device_scene, renderer  # noqa: E402
from paper_2403_13806_b200.render import RasterizeOptions  # noqa: E402


def main():
    kind = sys.argv[1] if len(sys.argv) > 1 else "render"
    frames = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    prec = sys.argv[3] if len(sys.argv) > 3 else "fp32"
    opts = RasterizeOptions(near_limit=0.2, precision=prec)
    if kind == "render":
        scene, cams = synth.config1(0)
    elif kind == "batch":
        scene, cams = synth.config4(0, n_views=16)
    else:
        scene, cams = synth.config2(0)
    ds = device_scene(scene)
    r = renderer(ds.device)
    scores = torch.zeros(len(scene), dtype=torch.float32 if prec == "fp32" else torch.float64, device=ds.device)
    out = r.alloc_outputs(cams[0], precision=0 if prec == "fp32" else 1)
    for f in range(frames):
        if kind in ("render", "batch"):
            _, st = r.render(ds, cams[f], opts, out=out)
        else:
            _, st = r.render(ds, cams[f], opts, color=False, scores=scores)
    torch.cuda.synchronize()
    print(kind, "ok", st.n_visible, st.n_pairs)


if __name__ == "__main__":
    main()
