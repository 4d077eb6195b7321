"""Generate the golden fixtures that pin the oracle (run in the build container).

Imports the UNMODIFIED reference package from /root/reference (read-only)
with a two-line ``matplotlib`` stub (``__init__.py:80`` ->
``pipeline.py:49`` -> ``plots.py:7`` imports matplotlib, which this image
lacks), runs the reference's own public calls on the reference test suites'
seeded inputs plus the BASELINE configs[0] scene, and writes inputs and
outputs to ``tests/golden/*.npz``. Nothing at run time reads
/root/reference; the GPU box only sees these npz files.

    python tests/golden/make_golden.py
"""

import os
import sys
import types
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("RADSPLAT_REFERENCE", "/root/reference"))
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))


def import_reference():
    mpl = types.ModuleType("matplotlib")
    mpl.use = lambda *a, **k: None
    sys.modules.setdefault("matplotlib", mpl)
    sys.modules.setdefault("matplotlib.pyplot", types.ModuleType("matplotlib.pyplot"))
    sys.path.insert(0, str(REF / "pkg" / "src"))
    sys.path.insert(0, str(REF / "pkg" / "tests"))
    import fieldsplat  # noqa: F401
    import conftest  # reference test fixtures: random_scene, facing_camera
    import oracles  # reference per-pixel composite oracle
    return fieldsplat, conftest, oracles


def pack_scene(d, p, scene):
    d[p + "pos"] = np.asarray(scene.positions, np.float64)
    d[p + "logit"] = np.asarray(scene.opacity_logits, np.float64)
    d[p + "sh"] = np.asarray(scene.sh, np.float64)
    d[p + "ls"] = np.asarray(scene.log_scales, np.float64)
    d[p + "quat"] = np.asarray(scene.quaternions, np.float64)
    d[p + "deg"] = np.int64(scene.active_sh_degree)


def pack_cam(d, p, cam):
    d[p + "R"] = np.asarray(cam.rotation, np.float64)
    d[p + "t"] = np.asarray(cam.translation, np.float64)
    d[p + "intr"] = np.array([cam.fx, cam.fy, cam.cx, cam.cy], np.float64)
    d[p + "wh"] = np.array([cam.width, cam.height], np.int64)


def pack_opts(d, p, o):
    d[p + "opts"] = np.array([o.alpha_max, o.alpha_cut, o.tau_stop, o.near_limit,
                              o.lowpass, o.sigma_bound], np.float64)


def pack_render(d, p, out, acc=None):
    d[p + "img"] = np.asarray(out.color.data, np.float64)
    d[p + "alpha"] = np.asarray(out.alpha, np.float64)
    d[p + "count"] = np.asarray(out.count, np.int64)
    if acc is not None:
        d[p + "contrib"] = np.asarray(acc.values, np.float64)


def pack_proj(d, p, fs, scene, cam, opts):
    proj = fs.render._project_arrays(scene, cam, opts)
    for k in ("valid", "mx", "my", "a", "b", "c", "inv_a", "inv_b", "inv_c", "radius",
              "x0", "x1", "y0", "y1", "depth", "color", "opacity"):
        d[p + "proj_" + k] = np.asarray(proj[k])
    d[p + "order"] = fs.render._composite_order(proj).astype(np.int64)


def render_case(fs, d, p, scene, cam, opts, active=None):
    pack_scene(d, p, scene)
    pack_cam(d, p, cam)
    pack_opts(d, p, opts)
    if active is None:
        acc = fs.render.ContributionAccumulator(len(scene))
        out = fs.render.rasterize_with_contributions(scene, cam, acc, opts)
        pack_render(d, p, out, acc)
    else:
        d[p + "active"] = np.asarray(active, bool)
        pack_render(d, p, fs.render.rasterize_filtered(scene, cam, active, opts))
    pack_proj(d, p, fs, scene, cam, opts)


def main():
    fs, cf, orc = import_reference()
    R = fs.render
    opts = R.RasterizeOptions()

    # A: test_render.py:273-291 -- 50 random scenes (bit-exact suite)
    d = {}
    master = np.random.default_rng(2024)
    for case in range(50):
        rng = np.random.default_rng(master.integers(2 ** 63))
        n = int(rng.integers(1, 11))
        scene = cf.random_scene(rng, n, sh_degree=int(rng.integers(0, 4)))
        cam = cf.facing_camera(int(rng.integers(6, 13)), int(rng.integers(6, 13)),
                               distance=float(rng.uniform(3.0, 5.0)))
        render_case(fs, d, f"c{case}_", scene, cam, opts)
        img, alpha, count, contrib = orc.composite_oracle(scene, cam, opts)
        assert np.array_equal(img, d[f"c{case}_img"]) and np.array_equal(contrib, d[f"c{case}_contrib"])
    d["n_cases"] = np.int64(50)
    np.savez_compressed(HERE / "suite50.npz", **d)

    # B: test_acceptance.py:149-171 -- second 50-scene suite (default fov/distance)
    d = {}
    rng = np.random.default_rng(2024)
    for case in range(50):
        n = int(rng.integers(1, 11))
        scene = cf.random_scene(rng, n, sh_degree=int(rng.integers(0, 3)))
        cam = cf.facing_camera(int(rng.integers(4, 13)), int(rng.integers(4, 13)))
        render_case(fs, d, f"c{case}_", scene, cam, opts)
    d["n_cases"] = np.int64(50)
    np.savez_compressed(HERE / "accept50.npz", **d)

    # C/D/E: filtered subset, importance, known-answer cases
    d = {}
    rng = np.random.default_rng(1234)  # conftest rng fixture
    scene = cf.random_scene(rng, 12)
    active = rng.uniform(size=12) > 0.4
    render_case(fs, d, "filtered_", scene, cf.facing_camera(12, 12, distance=4.0), opts, active)

    rng = np.random.default_rng(1234)
    scene = cf.random_scene(rng, 8)
    cams = [cf.facing_camera(10, 10, distance=dd) for dd in (3.5, 4.5)]
    table = fs.pruning.compute_importance(scene, cams)
    pack_scene(d, "imp_", scene)
    for i, cam in enumerate(cams):
        pack_cam(d, f"imp_cam{i}_", cam)
    d["imp_values"] = table.values

    import test_render as tr  # reference helper single_gaussian_scene
    import test_pruning as tp  # reference helper occluder_scene
    kc = {
        "single": (tr.single_gaussian_scene((0, 0, 0), opacity=0.8, scale=0.5), cf.facing_camera(17, 17, distance=4.0)),
        "twolayer": (fs.GaussianScene.from_primitives([
            tr.single_gaussian_scene((0, 0, -1.0), (0.9, 0.1, 0.1), 0.5, 0.5).primitive(0),
            tr.single_gaussian_scene((0, 0, 1.0), (0.1, 0.1, 0.9), 0.8, 0.5).primitive(0)]),
            cf.facing_camera(17, 17, distance=4.0)),
        "tie": (fs.GaussianScene.from_primitives([
            tr.single_gaussian_scene((0, 0, 0), (1.0, 0.0, 0.0), 0.9, 0.4).primitive(0),
            tr.single_gaussian_scene((0, 0, 0), (0.0, 0.0, 1.0), 0.9, 0.4).primitive(0)]),
            cf.facing_camera(9, 9, distance=4.0)),
        "iso": (tr.single_gaussian_scene((0, 0, 0), scale=0.2), cf.facing_camera(32, 32, distance=5.0)),
        "lowpass": (tr.single_gaussian_scene((0, 0, 0), scale=1e-5), cf.facing_camera(16, 16, distance=4.0)),
        "occluder": (tp.occluder_scene(), cf.facing_camera(16, 16, distance=4.0)),
        "occluder1": (tp.occluder_scene().subset(np.array([True, False, False, False])),
                      cf.facing_camera(17, 17, distance=4.0)),
        "behind": (tr.single_gaussian_scene((0.0, 0.0, -8.0)), cf.facing_camera(16, 16, distance=4.0)),
        "offscreen": (tr.single_gaussian_scene((50.0, 0.0, 0.0), scale=0.1),
                      cf.facing_camera(16, 16, distance=4.0, fov_deg=30)),
    }
    for name, (scene, cam) in kc.items():
        render_case(fs, d, name + "_", scene, cam, opts)
    # ragged / multi-tile random scene: 300 Gaussians at 70x45 (5x3 tiles, ragged edges)
    rng = np.random.default_rng(77)
    scene = cf.random_scene(rng, 300, sh_degree=3, scale_range=(0.02, 0.2))
    render_case(fs, d, "ragged_", scene, cf.facing_camera(70, 45, distance=3.5, fov_deg=60.0), opts)
    np.savez_compressed(HERE / "known.npz", **d)

    # F: BASELINE configs[0] (seeded synth), near_limit 0.2
    from paper_2403_13806_b200.synth import config0
    arrs, cams = config0(0)
    scene = fs.GaussianScene(positions=arrs.positions.astype(np.float64),
                             opacity_logits=arrs.opacity_logits.astype(np.float64),
                             sh=arrs.sh.astype(np.float64), log_scales=arrs.log_scales.astype(np.float64),
                             quaternions=arrs.quaternions.astype(np.float64), active_sh_degree=3)
    cam = fs.look_at_camera((0.0, -3.0, 0.0), (0.0, 0.0, 0.0), width=128, height=128, fov_deg=50.0)
    assert np.array_equal(cam.rotation, cams[0].rotation) and np.array_equal(cam.translation, cams[0].translation)
    d = {}
    render_case(fs, d, "cfg0_", scene, cam, R.RasterizeOptions(near_limit=0.2))
    np.savez_compressed(HERE / "config0.npz", **d)

    # G: two-room visibility fixture (synthetic.py:179-259; test_visibility.py, test_acceptance.py:303-329)
    d = {}
    V = fs.visibility
    for seed, aux in ((0, 2), (5, 3)):
        spec = fs.synthetic.SyntheticSpec(kind="two_room", image_size=24, n_per_room=48)
        scene = fs.synthetic.make_two_room_scene(spec, np.random.default_rng(seed))
        cams = fs.synthetic.two_room_cameras(spec, 6)
        p = f"room{seed}_"
        pack_scene(d, p, scene)
        d[p + "n_per_room"] = np.int64(scene.metadata["n_per_room"])
        for i, cam in enumerate(cams):
            pack_cam(d, f"{p}cam{i}_", cam)
        d[p + "n_cams"] = np.int64(len(cams))
        clustering = V.cluster_cameras(np.array([c.center for c in cams]), k=2, seed=0)
        d[p + "centers"] = clustering.centers
        d[p + "assignment"] = clustering.assignment.astype(np.int64)
        vis = V.bake_visibility(scene, clustering, cams, t_cluster=0.001, aux_per_camera=aux, seed=0)
        d[p + "aux"] = np.int64(aux)
        d[p + "indicators"] = vis.indicators
        vis0 = V.bake_visibility(scene, clustering, cams, t_cluster=0.0, aux_per_camera=0)
        d[p + "indicators_t0_aux0"] = vis0.indicators
        d[p + "importance"] = fs.pruning.compute_importance(scene, cams).values
        d[p + "importance_left"] = fs.pruning.compute_importance(scene, cams[:len(cams) // 2]).values
        for i, cam in enumerate(cams):
            out, n_act, j = V.render_from_viewpoint(scene, vis, cam)
            d[f"{p}cam{i}_filtered_img"] = out.color.data
            d[f"{p}cam{i}_full_img"] = R.rasterize(scene, cam).color.data
            d[f"{p}cam{i}_cluster"] = np.int64(j)
            d[f"{p}cam{i}_n_active"] = np.int64(n_act)
    np.savez_compressed(HERE / "two_room.npz", **d)

    # H: viewer parity bundle (frontend/scripts/make_fixtures.py:67-101), frames kept as fp32 like the script
    d = {}
    sys.path.insert(0, str(REF / "pkg" / "frontend" / "scripts"))
    import make_fixtures as mf
    scene = mf.make_scene(np.random.default_rng(42))
    cams = mf.make_cameras()
    clustering = V.cluster_cameras(np.array([c.center for c in cams]), k=2, seed=0)
    vis = V.bake_visibility(scene, clustering, cams, t_cluster=0.001, aux_per_camera=1, seed=0)
    pack_scene(d, "", scene)
    shared = [cams[0], cams[2], cams[5],
              fs.look_at_camera((-6.0, 1.0, 2.0), (-3.0, 0.0, 0.0), width=mf.SIZE, height=mf.SIZE, fov_deg=55.0),
              fs.look_at_camera((6.2, -0.8, 1.5), (3.0, 0.2, 0.0), width=mf.SIZE, height=mf.SIZE, fov_deg=55.0)]
    d["centers"] = vis.centers
    d["indicators"] = vis.indicators
    for i, cam in enumerate(shared):
        pack_cam(d, f"pose{i}_", cam)
        d[f"pose{i}_frame"] = R.rasterize(scene, cam).color.data.astype("<f4")
        out, n_act, j = V.render_from_viewpoint(scene, vis, cam)
        d[f"pose{i}_filtered"] = out.color.data.astype("<f4")
        d[f"pose{i}_active"] = np.int64(n_act)
        d[f"pose{i}_cluster"] = np.int64(j)
    # cross-check against the committed reference cases.json (active counts / clusters)
    import json
    cases = json.loads((REF / "pkg/frontend/tests/fixtures/parity/cases.json").read_text())
    for i, c in enumerate(cases["cases"]):
        assert c["active_count"] == d[f"pose{i}_active"] and c["cluster_index"] == d[f"pose{i}_cluster"]
    np.savez_compressed(HERE / "viewer_parity.npz", **d)

    make_io(fs, cf)
    make_grad(fs, cf)
    make_grad_c0(fs)
    make_metrics(fs, cf)
    make_scale(fs)
    print("golden fixtures written to", HERE)


def make_io(fs, conftest):
    """I: wire formats (io.py:128-243): reference-written RSPL / RVIS bytes."""
    import tempfile
    d = {}
    with tempfile.TemporaryDirectory() as tmp:
        rng = np.random.default_rng(1234)
        for name, scene in (("s17", conftest.random_scene(rng, 17, sh_degree=2)),
                            ("s1", conftest.random_scene(rng, 1, sh_degree=0)),
                            ("room", fs.synthetic.make_two_room_scene(
                                fs.synthetic.SyntheticSpec(kind="two_room", image_size=24, n_per_room=48),
                                np.random.default_rng(0)))):
            scene.metadata["prune_removed"] = 7
            path = Path(tmp) / f"{name}.rspl"
            fs.io.save_scene(scene, path, sidecar={"stage": "golden"})
            d[name + "_rspl"] = np.frombuffer(path.read_bytes(), np.uint8)
            d[name + "_json"] = np.frombuffer((Path(str(path) + ".json")).read_bytes(), np.uint8)
            back = fs.io.load_scene(path)
            pack_scene(d, name + "_", back)
        vis = fs.visibility.ClusterVisibility(centers=rng.uniform(-5, 5, size=(3, 3)),
                                              indicators=rng.uniform(size=(3, 45)) > 0.5,
                                              t_cluster=0.001, scene_generation=42)
        path = Path(tmp) / "v.rvis"
        fs.io.save_visibility(vis, path)
        d["vis_rvis"] = np.frombuffer(path.read_bytes(), np.uint8)
        d["vis_indicators"] = vis.indicators
        d["vis_centers"] = vis.centers
    np.savez_compressed(HERE / "io.npz", **d)


def make_grad(fs, conftest):
    """J: backward pass (render.py:318-487): reference gradients through the image."""
    R = fs.render
    d = {}
    rng = np.random.default_rng(99)
    cases = []
    cases.append(("deg0", conftest.random_scene(rng, 4, sh_degree=0, opacity_range=(0.3, 0.8),
                                                scale_range=(0.15, 0.4)), conftest.facing_camera(8, 8, distance=4.0)))
    cases.append(("deg2", conftest.random_scene(rng, 3, sh_degree=2, opacity_range=(0.3, 0.8),
                                                scale_range=(0.15, 0.4)), conftest.facing_camera(8, 8, distance=4.0)))
    cases.append(("deg3", conftest.random_scene(rng, 40, sh_degree=3, scale_range=(0.05, 0.3)),
                  conftest.facing_camera(32, 24, distance=4.0)))
    near = conftest.random_scene(rng, 3, scale_range=(0.2, 0.4))
    far = fs.GaussianScene(positions=np.array([[100.0, 0.0, 0.0]]), opacity_logits=np.zeros(1),
                           sh=np.zeros((1, 3, 16)), log_scales=np.full((1, 3), np.log(0.2)),
                           quaternions=np.array([[1.0, 0.0, 0.0, 0.0]]))
    both = fs.GaussianScene.from_primitives([near.primitive(i) for i in range(3)] + [far.primitive(0)])
    cases.append(("touched", both, conftest.facing_camera(8, 8, distance=4.0)))
    s0 = fs.synthetic  # noqa: F841
    sc = conftest.random_scene(rng, 300, sh_degree=3, spread=1.2, scale_range=(0.02, 0.2))
    cases.append(("many", sc, conftest.facing_camera(64, 48, distance=4.0)))
    for name, scene, cam in cases:
        p = name + "_"
        pack_scene(d, p, scene)
        pack_cam(d, p, cam)
        opts = R.RasterizeOptions()
        pack_opts(d, p, opts)
        w = rng.normal(size=(cam.height, cam.width, 3)) if name != "touched" else np.ones((cam.height, cam.width, 3))
        d[p + "w"] = w
        out, cache = R.rasterize_cached(scene, cam)
        g = R.rasterize_backward(scene, cam, cache, w)
        d[p + "img"] = out.color.data
        for k in ("positions", "sh", "log_scales", "quaternions", "opacity_logits", "mean2d_grad_norm", "touched"):
            d[p + "g_" + k] = np.asarray(g[k])
    d["cases"] = np.array([c[0] for c in cases])
    np.savez_compressed(HERE / "grad.npz", **d)


def make_grad_c0(fs):
    """J': backward pass at BASELINE configs[0] scale (4,096 Gaussians, 128x128, SH degree 3,
    near_limit 0.2): the reference's fp64 gradients through a seeded random image weight."""
    R = fs.render
    from paper_2403_13806_b200.synth import config0
    arrs, _ = config0(0)
    scene = fs.GaussianScene(positions=arrs.positions.astype(np.float64),
                             opacity_logits=arrs.opacity_logits.astype(np.float64),
                             sh=arrs.sh.astype(np.float64), log_scales=arrs.log_scales.astype(np.float64),
                             quaternions=arrs.quaternions.astype(np.float64), active_sh_degree=3)
    cam = fs.look_at_camera((0.0, -3.0, 0.0), (0.0, 0.0, 0.0), width=128, height=128, fov_deg=50.0)
    opts = R.RasterizeOptions(near_limit=0.2)
    # the scene is synth.config0(0) and the weight image rng(5).normal: regenerated by the test
    # (the digest pins them); the gradients of the touched Gaussians are stored as float32
    # (rounding ~6e-8 relative, far below the test's 2e-5 of scale)
    import hashlib
    d = {"scene_sha1": np.array(hashlib.sha1(b"".join(np.ascontiguousarray(a).tobytes() for a in (
        arrs.positions, arrs.opacity_logits, arrs.sh, arrs.log_scales, arrs.quaternions))).hexdigest())}
    w = np.random.default_rng(5).normal(size=(cam.height, cam.width, 3))
    out, cache = R.rasterize_cached(scene, cam, opts)
    g = R.rasterize_backward(scene, cam, cache, w)
    t = np.asarray(g["touched"], bool)
    d["img"] = np.asarray(out.color.data, np.float32)
    d["touched"] = t
    for k in ("positions", "sh", "log_scales", "quaternions", "opacity_logits", "mean2d_grad_norm"):
        a = np.asarray(g[k])
        assert np.all(a[~t] == 0)
        d["g_" + k] = a[t].astype(np.float32)
    np.savez_compressed(HERE / "grad_c0.npz", **d)


def make_metrics(fs, conftest):
    """K: image metrics (metrics.py:34-117) on rendered and random images."""
    M = fs.metrics
    d = {}
    rng = np.random.default_rng(7)
    scene = conftest.random_scene(rng, 30, sh_degree=1)
    cam = conftest.facing_camera(40, 32, distance=4.0)
    a = fs.render.rasterize(scene, cam).color.data
    b = np.clip(a + rng.normal(scale=0.05, size=a.shape), 0.0, 1.0)
    cases = {"render": (a, b), "rand": (rng.uniform(size=(24, 27, 3)), rng.uniform(size=(24, 27, 3))),
             "gray": (rng.uniform(size=(16, 20)), rng.uniform(size=(16, 20)))}
    for name, (x, y) in cases.items():
        d[name + "_a"], d[name + "_b"] = x, y
        d[name + "_mse"] = np.float64(M.mse(x, y))
        d[name + "_psnr"] = np.float64(M.psnr(x, y))
        d[name + "_ssim"] = np.float64(M.ssim(x, y))
        v, g = M.ssim_with_grad(x, y)
        d[name + "_ssim_g"] = g
        d[name + "_ssim7"] = np.float64(M.ssim(x, y, win_size=7, sigma=1.0))
    np.savez_compressed(HERE / "metrics.npz", **d)


# ---------------------------------------------------------------------------
# L: BASELINE-scale frames rendered by the reference itself (SURVEY §8d scenes from
# paper_2403_13806_b200.synth, upcast to fp64 exactly like the reference reads RSPL).
# Stored compactly: the full per-pixel composite count (uint16), colour/alpha on a
# seeded sample of pixels, and every non-zero importance score (index + value).
# ---------------------------------------------------------------------------
SCALE_CASES = {
    # name: (config, scene kwargs, camera source, width, height)
    "c1": ("config1", {"n": 500_000}, ("orbit", 137), 628, 414),      # configs[1] frame 137, half res
    "c4": ("config4", {"n": 1_000_000}, ("views", 0), 240, 135),      # configs[4] view 0, 1/8 res
    "c3": ("config3", {"n": 300_000}, ("traj", 0), 480, 270),         # configs[3] scaled to 300k, inside
    "c2": ("config2", {"n": 3_000_000}, ("views", 0), 314, 207),      # configs[2] view 0, 1/4 res
}
SCALE_SAMPLE = 20_000


def scale_case(name):
    """(SceneArrays, camera) of a scale case -- shared by make_golden and the tests."""
    from paper_2403_13806_b200 import synth
    from paper_2403_13806_b200.core import look_at_camera
    cfg, kw, (src, k), w, h = SCALE_CASES[name]
    out = getattr(synth, cfg)(0, **kw)
    scene = out[0]
    cams = out[2] if src == "traj" else out[1]
    c = cams[k]
    R, t = np.asarray(c.rotation, np.float64), np.asarray(c.translation, np.float64)
    eye = -R.T @ t
    fwd = R[2]  # camera z axis in world coordinates (look direction)
    import math
    fov = math.degrees(2.0 * math.atan(c.width / (2.0 * c.fx)))
    cam = look_at_camera(eye, eye + fwd, width=w, height=h, fov_deg=fov)
    return scene, cam


def make_scale(fs, names=None):
    d = {}
    R = fs.render
    opts = R.RasterizeOptions(near_limit=0.2)
    for name in names or SCALE_CASES:
        sa, cam = scale_case(name)
        scene = fs.GaussianScene(positions=sa.positions.astype(np.float64),
                                 opacity_logits=sa.opacity_logits.astype(np.float64),
                                 sh=sa.sh.astype(np.float64), log_scales=sa.log_scales.astype(np.float64),
                                 quaternions=sa.quaternions.astype(np.float64),
                                 active_sh_degree=sa.active_sh_degree)
        rcam = fs.PinholeCamera(rotation=cam.rotation, translation=cam.translation, fx=cam.fx, fy=cam.fy,
                                cx=cam.cx, cy=cam.cy, width=cam.width, height=cam.height)
        acc = R.ContributionAccumulator(len(scene))
        out = R.rasterize_with_contributions(scene, rcam, acc, opts)
        p = name + "_"
        pack_cam(d, p, cam)
        pack_opts(d, p, opts)
        d[p + "count"] = np.asarray(out.count, np.uint16)
        npx = cam.width * cam.height
        pix = np.sort(np.random.default_rng(7).choice(npx, size=min(SCALE_SAMPLE, npx), replace=False))
        d[p + "pix"] = pix.astype(np.int64)
        d[p + "img_s"] = np.asarray(out.color.data, np.float64).reshape(-1, 3)[pix]
        d[p + "alpha_s"] = np.asarray(out.alpha, np.float64).reshape(-1)[pix]
        nz = np.nonzero(acc.values)[0]
        d[p + "score_idx"] = nz.astype(np.int64)
        d[p + "score_val"] = acc.values[nz].astype(np.float64)
        d[p + "n"] = np.int64(len(scene))
        print(name, "visible composites", int(out.count.sum()), "non-zero scores", len(nz), flush=True)
    np.savez_compressed(HERE / "scale.npz", **d)


if __name__ == "__main__":
    if sys.argv[1:2] == ["scale"]:  # only the BASELINE-scale frames (a few minutes)
        fs_, _, _ = import_reference()
        make_scale(fs_, sys.argv[2:] or None)
    elif sys.argv[1:] == ["io"]:  # only the wire-format fixtures
        fs_, conftest_, _ = import_reference()
        make_io(fs_, conftest_)
    elif sys.argv[1:] == ["grad"]:  # only the backward-pass fixtures
        fs_, conftest_, _ = import_reference()
        make_grad(fs_, conftest_)
    elif sys.argv[1:] == ["grad_c0"]:  # only the configs[0]-scale backward fixture
        fs_, _, _ = import_reference()
        make_grad_c0(fs_)
    elif sys.argv[1:] == ["metrics"]:  # only the image-metric fixtures
        fs_, conftest_, _ = import_reference()
        make_metrics(fs_, conftest_)
    else:
        main()
