"""configs[3] geometry on the GPU: cameras inside a house-scale cloud (near-plane culls,
huge near-camera footprints), visibility bakes and filtered trajectory frames.

Scene: synth.config3 scaled to 300k Gaussians (the same 20x20x4 box, half uniform, half
in 256 clusters), cameras at 480x270 with the configs[3] intrinsics (fov 55 deg). Checked
against the CPU oracle for both precisions:
* the device bake's per-cluster visible-index lists == np.nonzero of the oracle's
  indicators (max alpha*tau over the member cameras > t, visibility.py:204);
* trajectory frames, unfiltered and rendered from the nearest cluster's list: images,
  scores, the 64-bit tile keys' order and per-tile ranges bit-exact.
"""

import numpy as np
import pytest
import torch

from conftest import PREC_IDS, PRECISIONS

pytestmark = pytest.mark.gpu


def _small(cam, w=480, h=270):
    import math

    from paper_2403_13806_b200.core import look_at_camera
    R, t = np.asarray(cam.rotation, np.float64), np.asarray(cam.translation, np.float64)
    eye = -R.T @ t
    fov = math.degrees(2.0 * math.atan(cam.width / (2.0 * cam.fx)))
    return look_at_camera(eye, eye + R[2], width=w, height=h, fov_deg=fov)


@pytest.fixture(scope="module")
def house():
    from paper_2403_13806_b200 import synth
    scene, train, traj = synth.config3(0, n=300_000)
    return scene, [_small(c) for c in train[:48]], [_small(c) for c in traj[::100]]


@pytest.mark.parametrize("prec,tier", PRECISIONS, ids=PREC_IDS)
def test_config3_bake_lists_and_filtered_frames(house, prec, tier):
    from oracle import oracle as O
    from paper_2403_13806_b200.device import renderer
    from paper_2403_13806_b200.render import RasterizeOptions, render_device
    from paper_2403_13806_b200.visibility import _center, bake_visibility, cluster_cameras
    scene, train, traj = house
    opts = RasterizeOptions(near_limit=0.2, precision=prec)
    cl = cluster_cameras(np.array([_center(c) for c in train]), 4, seed=0)
    vis = bake_visibility(scene, cl, train, t_cluster=0.01, aux_per_camera=0, seed=0, options=opts)
    ind = np.zeros((cl.k, len(scene)), bool)
    for j in range(cl.k):  # the oracle's bake: max over the members, strict > (visibility.py:204)
        members = [train[i] for i in cl.cluster_members(j)]
        h = O.views(scene, members, opts, tier, scores=True)["contrib"]
        ind[j] = h.astype(np.float64) > 0.01
        assert np.array_equal(vis.visible_indices(j).cpu().numpy(), np.nonzero(ind[j])[0]), j
    assert np.array_equal(vis.indicators, ind)
    vt = torch.float32 if prec == "fp32" else torch.float64
    for cam in traj:
        j = vis.nearest_cluster(_center(cam))
        for active in (None, ind[j]):
            idx = None if active is None else vis.visible_indices(j)
            sc = torch.zeros(len(scene), dtype=vt, device="cuda")
            out, st = render_device(scene, cam, opts, scores=sc, active_idx=idx)
            fa = renderer().frame_arrays()
            ob = O.bin_tiles(scene, cam, opts, tier, active=active)
            ref = O.render(scene, cam, opts, tier, active=active)
            assert st.n_pairs == ob["P"]
            assert np.array_equal(fa["ranges"], ob["ranges"])
            if active is None:  # item ids are scene indices only for the unfiltered frame
                assert np.array_equal(fa["pair_items"], ob["vals"])
            else:
                assert np.array_equal(idx.cpu().numpy()[fa["pair_items"]], ob["vals"])
            assert np.array_equal(out["rgb"].cpu().numpy(), ref["img"])
            assert np.array_equal(out["count"].cpu().numpy(), ref["count"])
            assert np.array_equal(sc.cpu().numpy(), ref["contrib"])
        # near-plane culls happen here (cameras inside the cloud)
        assert st.n_items > st.n_visible
