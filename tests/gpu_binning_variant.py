"""Subprocess body of tests/test_gpu_expand_paths.py: the binning stress cases with the
expansion / launch knobs of the environment (RS_EXPAND_DENSE, RS_EXPAND_MAJOR, RS_PDL are
read once per process), checked bit for bit against the oracle. Exit 0 = all equal."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2403_13806_b200.core import look_at_camera  # noqa: E402
from paper_2403_13806_b200.device import renderer  # noqa: E402
from paper_2403_13806_b200.render import RasterizeOptions, render_device  # noqa: E402
from paper_2403_13806_b200.synth import config1, config4  # noqa: E402


def check(scene, cam, opts, tier):
    n = len(scene)
    sc = torch.zeros(n, dtype=torch.float32 if tier is np.float32 else torch.float64, device="cuda")
    out, st = render_device(scene, cam, opts, scores=sc)
    fa = renderer().frame_arrays()
    ob = O.bin_tiles(scene, cam, opts, tier)
    assert st.n_pairs == ob["P"], (st.n_pairs, ob["P"])
    assert np.array_equal(fa["ranges"], ob["ranges"])
    assert np.array_equal(fa["pair_items"], ob["vals"])
    ref = O.views(scene, [cam], opts, tier, scores=True, images=True)
    assert np.array_equal(out["rgb"].cpu().numpy(), ref["img_last"])
    assert np.array_equal(sc.cpu().numpy(), ref["contrib"])


def main():
    for prec, tier in (("fp32", np.float32), ("fp64", "c64")):
        opts = RasterizeOptions(near_limit=0.2, precision=prec)
        for n, W, H, fov in ((50_000, 33, 17, 60.0), (100_000, 640, 480, 55.0), (60_000, 1920, 1080, 55.0)):
            scene, _ = config1(n, n=n, n_frames=1)
            check(scene, look_at_camera((2.8, -1.1, 0.7), (0.1, 0.0, 0.0), width=W, height=H, fov_deg=fov), opts,
                  tier)
        scene, cams = config4(0, n=20_000, n_views=4)  # heavy tails: long row segments (dense chunks)
        check(scene, cams[1], opts, tier)
    print("ok")


if __name__ == "__main__":
    main()
