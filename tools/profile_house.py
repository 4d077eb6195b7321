"""ncu driver: configs[3]-sized filtered frames (1920x1080, a 1.7k-Gaussian index list of the
6M house scene: a random 1.7k subset) and unfiltered ones.

    python tools/profile_house.py [filtered|unfiltered] [frames]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2403_13806_b200 import synth  # noqa: E402
from paper_2403_13806_b200.device import device_scene, renderer  # noqa: E402
from paper_2403_13806_b200.render import RasterizeOptions  # noqa: E402


def main():
    kind = sys.argv[1] if len(sys.argv) > 1 else "filtered"
    frames = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    scene, _, traj = synth.config3(0)
    opts = RasterizeOptions(near_limit=0.2, precision="fp32")
    ds = device_scene(scene)
    r = renderer(ds.device)
    idx = None
    if kind == "filtered":  # 1.7k random Gaussians (the config rule's list size)
        pick = np.random.default_rng(0).choice(len(scene), 1700, replace=False)
        idx = torch.from_numpy(np.sort(pick).astype(np.int32)).to(ds.device)
    out = r.alloc_outputs(traj[0])
    for f in range(frames):
        _, st = r.render(ds, traj[f], opts, out=out, active_idx=idx)
    torch.cuda.synchronize()
    print(kind, "ok", st.n_visible, st.n_pairs)


if __name__ == "__main__":
    main()
