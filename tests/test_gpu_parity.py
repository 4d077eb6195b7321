"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, both precisions.

fp32 frames vs Tier A and fp64 frames vs Tier C (the oracle's two contracts):
bit-exact -- projection fields, tile keys, per-tile sorted order, ranges,
visible-index lists, RGB/alpha/depth/count, importance scores. The north-star
tolerances (pixels <= 1e-4 abs, scores <= 1e-5 rel) are asserted as well; the
observed difference is exactly zero by construction (same operations, same
order, no FMA contraction, shared exp implementations).
Against the fp64 reference's own outputs (tests/golden, made by the
reference): fp64 frames agree to 1e-12 with identical composite decisions;
fp32 frames within the documented fp32 budget (tier_b_check).
"""

import numpy as np
import pytest
import torch

from conftest import (PREC_IDS, PRECISIONS, golden, load_case, load_cam, options_from, reference_check_fp64,
                      render_cases, tier_b_check, with_precision)

pytestmark = pytest.mark.gpu

PIX_TOL = 1e-4      # north_star: RGB / alpha / depth within 1e-4 absolute (fp32)
SCORE_RTOL = 1e-5   # north_star: importance within 1e-5 relative

CASES = render_cases()
IDS = [c[0] for c in CASES]


def _oracle():
    from oracle import oracle as O
    return O


def _render_gpu(scene, cam, opts, scores=True, count_evals=False):
    from paper_2403_13806_b200.device import device_scene, precision_of, renderer, value_dtype
    from paper_2403_13806_b200.render import render_device
    ds = device_scene(scene)
    vt = value_dtype(precision_of(opts))
    sc = torch.zeros(max(ds.n, 1), dtype=vt, device=ds.device) if scores else None
    out, st = render_device(ds, cam, opts, scores=sc, count_evals=count_evals)
    host = {k: v.cpu().numpy() for k, v in out.items()}
    if scores:
        host["contrib"] = sc[:ds.n].cpu().numpy()
    return host, st, renderer(ds.device)


@pytest.mark.parametrize("prec,tier", PRECISIONS, ids=PREC_IDS)
@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_render_bit_exact_vs_oracle(case, prec, tier):
    name, scene, cam, opts, d, p = case
    opts = with_precision(opts, prec)
    O = _oracle()
    ref = O.render(scene, cam, opts, tier)
    got, st, _ = _render_gpu(scene, cam, opts)
    for k in ("img", "alpha", "depth"):
        g = got["rgb"] if k == "img" else got[k]
        assert np.array_equal(g, ref[k]), f"{name}: {k} max diff {np.abs(g - ref[k]).max()}"
        assert np.abs(g - ref[k]).max() <= PIX_TOL
    assert np.array_equal(got["count"], ref["count"])
    assert np.array_equal(got["contrib"], ref["contrib"]), name
    assert st.composites == 0  # only counted on request


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_render_vs_reference_fp64(case):
    """fp64 frames vs the reference's own output (golden, made by fieldsplat):
    identical composite decisions, pixels and scores within 1e-12."""
    name, scene, cam, opts, d, p = case
    got, _, _ = _render_gpu(scene, cam, with_precision(opts, "fp64"))
    reference_check_fp64(name, got["rgb"], got["alpha"], got["count"], got["contrib"], d, p)


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_render_vs_reference_fp32_budget(case):
    """fp32 frames: within the documented fp32 budget of the reference (tier_b_check)."""
    name, scene, cam, opts, d, p = case
    got, _, _ = _render_gpu(scene, cam, with_precision(opts, "fp32"))
    tier_b_check(name, got["rgb"], got["alpha"], got["count"], got["contrib"], d, p)


@pytest.mark.parametrize("prec,tier", PRECISIONS, ids=PREC_IDS)
@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_projection_bit_exact(case, prec, tier):
    name, scene, cam, opts, d, p = case
    opts = with_precision(opts, prec)
    from paper_2403_13806_b200.render import project_scene
    O = _oracle()
    ref = O.project(scene, cam, opts, tier)
    vt = np.float32 if prec == "fp32" else np.float64
    _, proj = project_scene(scene, cam, opts)
    assert np.array_equal(proj["valid"], ref["valid"])
    v = ref["valid"]
    for k, rk in (("mx", "mx"), ("my", "my"), ("a", "a"), ("b", "b"), ("c", "c"), ("inv_a", "ia"),
                  ("inv_b", "ib"), ("inv_c", "ic"), ("radius", "radius"), ("depth", "depth"),
                  ("opacity", "opacity")):
        assert np.array_equal(proj[k].astype(vt)[v], ref[rk][v]), (name, k)
    assert np.array_equal(proj["color"].astype(vt)[v], ref["color"][v])
    for k in ("x0", "x1", "y0", "y1"):
        assert np.array_equal(proj[k][v], ref[k][v]), (name, k)
    # against the reference's own projection (fp64): bbox/valid decisions agree
    assert np.array_equal(proj["valid"], d[p + "proj_valid"]), name
    if prec == "fp64":
        assert np.allclose(proj["mx"][v], d[p + "proj_mx"][v], rtol=1e-13, atol=1e-12)
    else:
        assert np.allclose(proj["mx"][v], d[p + "proj_mx"][v], rtol=1e-5, atol=1e-4)


@pytest.mark.parametrize("prec,tier", PRECISIONS, ids=PREC_IDS)
@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_binning_bit_exact(case, prec, tier):
    """Tile keys, per-tile (depth, index) order and ranges equal the oracle's."""
    name, scene, cam, opts, d, p = case
    opts = with_precision(opts, prec)
    O = _oracle()
    ob = O.bin_tiles(scene, cam, opts, tier)
    _, st, r = _render_gpu(scene, cam, opts, scores=False)
    fa = r.frame_arrays()
    assert fa["stats"].n_pairs == ob["P"] and not fa["stats"].overflow
    assert np.array_equal(fa["ranges"], ob["ranges"]), name
    assert np.array_equal(fa["pair_items"], ob["vals"]), name
    # reconstruct the 64-bit keys from the GPU's tile lists and depth keys
    rec = fa["records"]
    depth = rec[:, 7] if len(rec) else np.zeros(0, np.float32)
    dk = np.array([O.depth_key(float(z)) for z in depth], np.uint64) if len(depth) else np.zeros(0, np.uint64)
    T = fa["tiles_x"] * fa["tiles_y"]
    tile_of = np.repeat(np.arange(T, dtype=np.uint64), (ob["ranges"][:, 1] - ob["ranges"][:, 0]).astype(np.int64))
    keys = (tile_of << np.uint64(32)) | dk[fa["pair_items"]] if ob["P"] else np.zeros(0, np.uint64)
    assert np.array_equal(keys, ob["keys"]), name
    # global (depth, index) order over visible Gaussians
    nv = fa["stats"].n_visible
    order = O.order(scene, cam, opts, tier)
    assert nv == len(order) <= int(d[p + "proj_valid"].sum())
    assert np.array_equal(fa["items_sorted"][:nv].astype(np.int64), order)


@pytest.mark.parametrize("prec,tier", PRECISIONS, ids=PREC_IDS)
def test_filtered_equals_subset_render(prec, tier):
    from paper_2403_13806_b200.render import rasterize, rasterize_filtered
    d = golden("known")
    scene, cam, o = load_case(d, "filtered_")
    opts = options_from(o, prec)
    active = d["filtered_active"]
    O = _oracle()
    ref = O.render(scene, cam, opts, tier, active=active)
    got = rasterize_filtered(scene, cam, active, opts)
    assert np.array_equal(got.color.data.astype(ref["img"].dtype), ref["img"])
    assert np.array_equal(got.count, ref["count"])
    assert np.abs(got.color.data - d["filtered_img"]).max() <= (1e-5 if prec == "fp32" else 1e-12)
    # all-active filter is the identity (test_render.py:151-156)
    full = rasterize(scene, cam, opts)
    allf = rasterize_filtered(scene, cam, np.ones(len(scene), bool), opts)
    assert np.array_equal(full.color.data, allf.color.data)


@pytest.mark.parametrize("prec,tier", PRECISIONS, ids=PREC_IDS)
def test_compute_importance_matches_oracle_and_reference(prec, tier):
    from paper_2403_13806_b200.core import GaussianScene
    from paper_2403_13806_b200.pruning import compute_importance
    d = golden("known")
    scene = GaussianScene(positions=d["imp_pos"], opacity_logits=d["imp_logit"], sh=d["imp_sh"],
                          log_scales=d["imp_ls"], quaternions=d["imp_quat"], active_sh_degree=int(d["imp_deg"]))
    cams = [load_cam(d, f"imp_cam{i}_") for i in range(2)]
    opts = options_from(None, prec)
    table = compute_importance(scene, cams, opts)
    O = _oracle()
    vt = np.float32 if prec == "fp32" else np.float64
    exp = np.zeros(len(scene), vt)
    for cam in cams:
        exp = np.maximum(exp, O.render(scene, cam, opts, tier)["contrib"])
    assert np.array_equal(table.values.astype(vt), exp)
    assert table.n_cameras == 2
    rel = np.abs(table.values - d["imp_values"]) / np.maximum(d["imp_values"], 1e-30)
    assert rel.max() <= (SCORE_RTOL if prec == "fp32" else 1e-12)
    # duplicate cameras / order invariance (test_pruning.py:54-66)
    assert np.array_equal(compute_importance(scene, cams + cams + cams[:1], opts).values, table.values)
    assert np.array_equal(compute_importance(scene, cams[::-1], opts).values, table.values)


def test_known_answers():
    from paper_2403_13806_b200.pruning import compute_importance
    from paper_2403_13806_b200.render import rasterize, project_scene
    d = golden("known")
    s, cam, _ = load_case(d, "single_")
    out = rasterize(s, cam)
    assert out.alpha[8, 8] == pytest.approx(0.8, abs=1e-3)                    # test_render.py:241-250
    np.testing.assert_allclose(out.color.data[8, 8], 0.8 * np.array([0.8, 0.3, 0.2]), atol=2e-3)
    s, cam, _ = load_case(d, "twolayer_")
    np.testing.assert_allclose(rasterize(s, cam).color.data[8, 8],
                               0.5 * np.array([0.9, 0.1, 0.1]) + 0.4 * np.array([0.1, 0.1, 0.9]), atol=5e-3)
    s, cam, _ = load_case(d, "tie_")
    c = rasterize(s, cam).color.data
    assert c[4, 4, 0] > c[4, 4, 2]                                               # index 0 first on ties
    s, cam, _ = load_case(d, "iso_")
    (p,), _ = project_scene(s, cam)
    assert p.cov2d[0, 0] == pytest.approx((cam.fx * 0.2 / 5.0) ** 2 + 0.3, rel=1e-6)
    s, cam, _ = load_case(d, "lowpass_")
    (p,), _ = project_scene(s, cam)
    assert p.cov2d[0, 0] >= 0.3 and np.linalg.det(p.cov2d) > 0
    s, cam, _ = load_case(d, "occluder_")
    t = compute_importance(s, [cam])
    assert t.values[0] > 0.5 and t.values[3] == 0.0                             # test_pruning.py:68-73
    s, cam, _ = load_case(d, "occluder1_")
    assert compute_importance(s, [cam]).values[0] == 0.99                       # clamp: alpha_max exactly
    assert compute_importance(s, [cam], options_from(None, "fp32")).values[0] == np.float32(0.99)
    for nm in ("behind", "offscreen"):
        s, cam, _ = load_case(d, nm + "_")
        assert project_scene(s, cam)[0] == []


@pytest.mark.parametrize("n", [0, 1, 31, 32, 33, 1000, 8191, 8192, 8193, 100_003])
def test_compaction_bit_exact(n):
    from paper_2403_13806_b200.device import renderer
    rng = np.random.default_rng(n)
    for dens in (0.0, 0.01, 0.5, 1.0):
        flags = rng.uniform(size=n) < dens
        r = renderer()
        got = r.compact(torch.from_numpy(flags.view(np.uint8)).cuda()).cpu().numpy()
        assert np.array_equal(got, np.nonzero(flags)[0]), (n, dens)
        bits = np.packbits(flags, bitorder="little")
        got_b = r.compact(torch.from_numpy(bits).cuda(), bits=True, n=n).cpu().numpy()
        assert np.array_equal(got_b, np.nonzero(flags)[0]), (n, dens)


def test_nonfinite_scene_rejected():
    from paper_2403_13806_b200.core import GaussianScene, InvalidSceneError
    from paper_2403_13806_b200.render import rasterize
    s, cam, _ = load_case(golden("suite50"), "c0_")
    pos = s.positions.copy()
    pos[0, 0] = np.nan
    bad = GaussianScene(positions=pos, opacity_logits=s.opacity_logits, sh=s.sh, log_scales=s.log_scales,
                        quaternions=s.quaternions)
    with pytest.raises(InvalidSceneError):
        rasterize(bad, cam)


def test_accumulator_length_and_active_shape_rejected():
    from paper_2403_13806_b200.core import InvalidParameterError
    from paper_2403_13806_b200.render import (ContributionAccumulator, rasterize_filtered,
                                              rasterize_with_contributions)
    s, cam, _ = load_case(golden("suite50"), "c3_")
    with pytest.raises(InvalidParameterError):
        rasterize_with_contributions(s, cam, ContributionAccumulator(len(s) + 1))
    with pytest.raises(InvalidParameterError):
        rasterize_filtered(s, cam, np.ones(len(s) + 2, bool))


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
@pytest.mark.parametrize("case", CASES[:12] + CASES[-4:], ids=IDS[:12] + IDS[-4:])
def test_rasterize_host_outputs_equal_device_images(case, prec):
    """rasterize(): the blend writes float64 colour/alpha and int64 count straight into
    pinned host memory (rs_outputs rgb64/alpha64/count64) -- exactly the (widened)
    device images, including partial edge tiles."""
    from paper_2403_13806_b200.render import rasterize
    name, scene, cam, opts, d, p = case
    opts = with_precision(opts, prec)
    got, _, _ = _render_gpu(scene, cam, opts, scores=False)
    res = rasterize(scene, cam, opts)
    assert res.color.data.dtype == np.float64 and res.alpha.dtype == np.float64 and res.count.dtype == np.int64
    assert not res.color.data.flags.writeable
    assert np.array_equal(res.color.data, got["rgb"].astype(np.float64)), name
    assert np.array_equal(res.alpha, got["alpha"].astype(np.float64)), name
    assert np.array_equal(res.count, got["count"].astype(np.int64)), name
    assert np.array_equal(res.depth, got["depth"].astype(np.float64)), name


@pytest.mark.parametrize("prec,tier", PRECISIONS, ids=PREC_IDS)
def test_rasterize_host_outputs_odd_sizes(prec, tier):
    """Image sizes that are not tile multiples: the staged row writes clip at W and H."""
    from oracle import oracle as O
    from paper_2403_13806_b200.core import look_at_camera
    from paper_2403_13806_b200.render import RasterizeOptions, rasterize
    from paper_2403_13806_b200.synth import config0
    scene, _ = config0(0)
    opts = RasterizeOptions(near_limit=0.2, precision=prec)
    for w, h in ((1, 1), (17, 5), (33, 47), (130, 97)):
        cam = look_at_camera(np.array([0.0, -3.0, 0.4]), np.zeros(3), width=w, height=h, fov_deg=50.0)
        res = rasterize(scene, cam, opts)
        ref = O.render(scene, cam, opts, tier)
        assert np.array_equal(res.color.data, ref["img"].astype(np.float64)), (w, h)
        assert np.array_equal(res.alpha, ref["alpha"].astype(np.float64)), (w, h)
        assert np.array_equal(res.count, ref["count"].astype(np.int64)), (w, h)


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_score_views_overflow_recovery_matches_per_view_renders(prec):
    """A scoring pass launched without per-view host syncs: a view that overflows the
    pair capacity is detected once per pass (rs_read_overflow) and the pass re-run from a
    snapshot -- the result equals the max over checked single-view renders."""
    from paper_2403_13806_b200.device import Renderer, device_scene
    from paper_2403_13806_b200.render import RasterizeOptions, render_device
    from paper_2403_13806_b200.synth import config2
    scene, cams = config2(0, n=60_000, n_views=6)
    opts = RasterizeOptions(near_limit=0.2, precision=prec)
    vt = torch.float32 if prec == "fp32" else torch.float64
    ds = device_scene(scene)
    ref = torch.zeros(ds.n, dtype=vt, device=ds.device)
    for c in cams:
        render_device(ds, c, opts, color=False, scores=ref)
    r = Renderer(ds.device)
    r.ensure(ds.n, 1 << 16, cams[0].width, cams[0].height)  # far below this pass's P
    pre = torch.rand(ds.n, device=ds.device, dtype=vt) * 1e-3  # an accumulator that already holds values
    got = pre.clone()
    r.score_views(ds, cams, opts, got)
    assert r.caps[1] > (1 << 16)
    assert torch.equal(got, torch.maximum(ref, pre))
    over, _ = r.read_overflow()
    assert not over
    r.close()


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_out_of_range_active_index_rejected(prec):
    """An index list with an entry outside [0, n) is reported by the device
    (rs_stats.bad_index / rs_read_sticky) and raised as InvalidParameterError, the
    reference's error for a bad active mask (render.py:231-234); the bad entries are never
    read."""
    from paper_2403_13806_b200.core import InvalidParameterError
    from paper_2403_13806_b200.device import camera_struct, device_scene, options_struct, renderer
    from paper_2403_13806_b200.render import RasterizeOptions, render_device
    s, cam, _ = load_case(golden("suite50"), "c3_")
    ds = device_scene(s)
    opts = RasterizeOptions(precision=prec)
    for bad in ([0, len(s)], [-1], [0, 1, 2 ** 30]):
        idx = torch.tensor(bad, dtype=torch.int32, device=ds.device)
        with pytest.raises(InvalidParameterError):
            render_device(ds, cam, opts, active_idx=idx)
    # the scoring pass's sticky record too
    r = renderer(ds.device)
    r.read_overflow(reset=True)
    vt = torch.float32 if prec == "fp32" else torch.float64
    sc = torch.zeros(len(s), dtype=vt, device=ds.device)
    r.launch(ds, camera_struct(cam), options_struct(opts), {}, sc,
             torch.tensor([len(s)], dtype=torch.int32, device=ds.device), 1)
    with pytest.raises(InvalidParameterError):
        r.read_overflow(reset=True)
    # a valid list still renders after the errors
    out, st = render_device(ds, cam, opts, active_idx=torch.arange(len(s), dtype=torch.int32, device=ds.device))
    assert st.bad_index == 0


def test_mismatched_caller_outputs_rejected_before_launch():
    """Caller-provided images of the wrong precision / size raise InvalidParameterError
    instead of being written past their end; the renderer keeps working afterwards."""
    from paper_2403_13806_b200.core import InvalidParameterError
    from paper_2403_13806_b200.device import device_scene, renderer
    from paper_2403_13806_b200.render import RasterizeOptions
    from paper_2403_13806_b200 import _native as N
    s, cam, _ = load_case(golden("suite50"), "c3_")
    ds = device_scene(s)
    r = renderer(ds.device)
    f32 = r.alloc_outputs(cam, precision=N.RS_F32)
    with pytest.raises(InvalidParameterError):
        r.render(ds, cam, RasterizeOptions(precision="fp64"), out=f32)
    with pytest.raises(InvalidParameterError):
        r.render(ds, cam, RasterizeOptions(precision="fp32"), scores=torch.zeros(len(s) - 1, device=ds.device))
    out, _ = r.render(ds, cam, RasterizeOptions(precision="fp32"), out=f32)
    torch.cuda.synchronize()
    assert torch.isfinite(out["rgb"]).all()


@pytest.mark.parametrize("prec,tier", PRECISIONS, ids=PREC_IDS)
def test_empty_and_fully_culled_frames(prec, tier):
    """A scene with no Gaussians, and a camera that sees none of them: black image, zero
    counts and scores, no pairs -- and the renderer keeps producing correct frames after."""
    from oracle import oracle as O
    from paper_2403_13806_b200.core import look_at_camera
    from paper_2403_13806_b200.render import RasterizeOptions, rasterize
    from paper_2403_13806_b200.synth import config0
    scene, cams = config0(0)
    cam = cams[0]
    opts = RasterizeOptions(near_limit=0.2, precision=prec)
    empty = scene.subset(np.zeros(len(scene), dtype=bool))
    host, st, _ = _render_gpu(empty, cam, opts)
    assert st.n_visible == 0 and st.n_pairs == 0 and not host["rgb"].any() and not host["count"].any()
    away = look_at_camera(np.array([0.0, -3.0, 0.0]), np.array([0.0, -6.0, 0.0]), width=128, height=128, fov_deg=50.0)
    host, st, _ = _render_gpu(scene, away, opts)
    assert st.n_visible == 0 and st.n_pairs == 0 and not host["rgb"].any() and not host["contrib"].any()
    res = rasterize(scene, cam, opts)  # the next frame is the oracle's
    assert np.array_equal(res.color.data, O.render(scene, cam, opts, tier)["img"].astype(np.float64))


@pytest.mark.parametrize("prec,tier", PRECISIONS, ids=PREC_IDS)
def test_largest_tile_grid_bit_exact(prec, tier):
    """The ABI's largest tile grid (4096 x 4096 px = 65,536 tiles): tile lists, ranges and image
    equal the oracle; one more tile column is refused with InvalidParameterError."""
    from oracle import oracle as O
    from paper_2403_13806_b200.core import InvalidParameterError, look_at_camera
    from paper_2403_13806_b200.device import renderer
    from paper_2403_13806_b200.synth import config1
    from paper_2403_13806_b200.render import RasterizeOptions
    scene, _ = config1(3, n=20_000, n_frames=1)
    opts = RasterizeOptions(near_limit=0.2, precision=prec)
    cam = look_at_camera((2.8, -1.1, 0.7), (0.1, 0.0, 0.0), width=4096, height=4096, fov_deg=55.0)
    host, st, r = _render_gpu(scene, cam, opts)
    fa = r.frame_arrays()
    ob = O.bin_tiles(scene, cam, opts, tier)
    assert st.n_pairs == ob["P"] and np.array_equal(fa["ranges"], ob["ranges"])
    assert np.array_equal(fa["pair_items"], ob["vals"])
    ref = O.views(scene, [cam], opts, tier, scores=True, images=True)
    assert np.array_equal(host["rgb"], ref["img_last"]) and np.array_equal(host["contrib"], ref["contrib"])
    too_wide = look_at_camera((2.8, -1.1, 0.7), (0.1, 0.0, 0.0), width=4112, height=4096, fov_deg=55.0)
    with pytest.raises(InvalidParameterError):
        _render_gpu(scene, too_wide, opts)


@pytest.mark.parametrize("prec,tier", PRECISIONS, ids=PREC_IDS)
def test_depth_ties_at_scale_bit_exact(prec, tier):
    """100k Gaussians on 40 planes facing an axis-aligned camera: every depth is shared by
    ~2,500 Gaussians, so the sorted order is decided by the index (fp32 keys equal, and in
    fp64 frames the fp64 depths equal too): depth order, tile lists and image equal the oracle."""
    from oracle import oracle as O
    from paper_2403_13806_b200.core import look_at_camera
    from paper_2403_13806_b200.device import renderer
    from paper_2403_13806_b200.render import RasterizeOptions
    from paper_2403_13806_b200.synth import SceneArrays, config1
    base, _ = config1(5, n=100_000, n_frames=1)
    pos = base.positions.copy()
    pos[:, 1] = np.round(pos[:, 1] * 10.0).astype(np.float32) / np.float32(10.0)  # 41 depth planes
    scene = SceneArrays(pos, base.opacity_logits, base.sh, base.log_scales, base.quaternions, 3)
    cam = look_at_camera(np.array([0.0, -4.0, 0.0]), np.array([0.0, 0.0, 0.0]), width=640, height=480, fov_deg=60.0)
    opts = RasterizeOptions(near_limit=0.2, precision=prec)
    host, st, r = _render_gpu(scene, cam, opts)
    fa = r.frame_arrays()
    order = O.order(scene, cam, opts, tier)
    assert np.array_equal(fa["items_sorted"][:st.n_visible].astype(np.int64), order)
    ob = O.bin_tiles(scene, cam, opts, tier)
    assert st.n_pairs == ob["P"] and np.array_equal(fa["pair_items"], ob["vals"])
    ref = O.views(scene, [cam], opts, tier, scores=True, images=True)
    assert np.array_equal(host["rgb"], ref["img_last"]) and np.array_equal(host["contrib"], ref["contrib"])
    # the ties are real: many equal depths among the binned items
    depth = ((pos[:, 1].astype(np.float64) + 4.0))[order]
    assert (np.diff(depth) == 0).mean() > 0.9


@pytest.mark.parametrize("prec,tier", PRECISIONS, ids=PREC_IDS)
def test_wide_depth_range_bit_exact(prec, tier):
    """Binned depths from ~1 to ~1e6 (keys spanning more than 2^27 values): the cooperative depth
    sort takes its 4-pass 8-bit-digit path; order, tile lists and image equal the oracle."""
    from oracle import oracle as O
    from paper_2403_13806_b200.core import look_at_camera
    from paper_2403_13806_b200.render import RasterizeOptions
    from paper_2403_13806_b200.synth import SceneArrays, config1
    base, _ = config1(7, n=50_000, n_frames=1)
    pos, ls, lg = base.positions.copy(), base.log_scales.copy(), base.opacity_logits.copy()
    far = np.arange(0, 50_000, 500)  # 100 huge Gaussians far behind the cloud, on the view axis
    rng = np.random.default_rng(1)
    pos[far] = np.stack([rng.uniform(-2e4, 2e4, far.size), rng.uniform(1e5, 1e6, far.size),
                         rng.uniform(-2e4, 2e4, far.size)], 1).astype(np.float32)
    ls[far] = np.float32(9.0)
    lg[far] = np.float32(3.0)
    scene = SceneArrays(pos, lg, base.sh, ls, base.quaternions, 3)
    cam = look_at_camera(np.array([0.0, -4.0, 0.0]), np.array([0.0, 0.0, 0.0]), width=320, height=240, fov_deg=60.0)
    opts = RasterizeOptions(near_limit=0.2, precision=prec)
    host, st, r = _render_gpu(scene, cam, opts)
    fa = r.frame_arrays()
    order = O.order(scene, cam, opts, tier)
    assert np.array_equal(fa["items_sorted"][:st.n_visible].astype(np.int64), order)
    assert np.isin(far, order).sum() > 20  # the far Gaussians are binned
    ob = O.bin_tiles(scene, cam, opts, tier)
    assert st.n_pairs == ob["P"] and np.array_equal(fa["pair_items"], ob["vals"])
    ref = O.views(scene, [cam], opts, tier, scores=True, images=True)
    assert np.array_equal(host["rgb"], ref["img_last"]) and np.array_equal(host["contrib"], ref["contrib"])


@pytest.mark.parametrize("prec,tier", PRECISIONS, ids=PREC_IDS)
def test_precull_border_scene_bit_exact(prec, tier):
    """Culling and binning at the image border: 60k Gaussians whose centres project into a 300-px band around the image
    border (and beyond), at depths from just past the near plane to 40, with log-scales from
    -6 to 4 and strong anisotropy -- order, tile lists and image equal the oracle's; many binned
    Gaussians have their centre outside the image and many are culled."""
    from oracle import oracle as O
    from paper_2403_13806_b200.core import look_at_camera
    from paper_2403_13806_b200.render import RasterizeOptions
    from paper_2403_13806_b200.synth import SceneArrays
    rng = np.random.default_rng(11)
    n, W, H = 60_000, 320, 240
    cam = look_at_camera(np.array([0.0, -4.0, 0.0]), np.array([0.0, 0.0, 0.0]), width=W, height=H, fov_deg=60.0)
    side = rng.integers(0, 4, n)
    u = rng.uniform(-300.0, 300.0, n)
    mx = np.where(side == 0, u, np.where(side == 1, W + u, rng.uniform(-300.0, W + 300.0, n)))
    my = np.where(side == 2, u, np.where(side == 3, H + u, rng.uniform(-300.0, H + 300.0, n)))
    z = np.where(rng.random(n) < 0.1, rng.uniform(0.15, 0.3, n), np.exp(rng.uniform(np.log(0.3), np.log(40.0), n)))
    pc = np.stack([(mx - cam.cx) * z / cam.fx, (my - cam.cy) * z / cam.fy, z], 1)
    pos = ((pc - cam.translation) @ cam.rotation).astype(np.float32)  # R^T (p_cam - t)
    ls = rng.normal(-2.0, 1.5, (n, 3))
    ls[:, 0] += rng.normal(0.0, 2.0, n)  # anisotropy
    ls = np.clip(ls, -6.0, 4.0).astype(np.float32)
    q = rng.normal(size=(n, 4))
    q = (q / np.linalg.norm(q, axis=1, keepdims=True)).astype(np.float32)
    lg = rng.normal(0.0, 2.0, n).astype(np.float32)
    sh = (rng.normal(0.0, 0.3, (n, 3, 16))).astype(np.float32)
    scene = SceneArrays(pos, lg, sh, ls, q, 3)
    opts = RasterizeOptions(near_limit=0.2, precision=prec)
    host, st, r = _render_gpu(scene, cam, opts)
    fa = r.frame_arrays()
    order = O.order(scene, cam, opts, tier)
    assert np.array_equal(fa["items_sorted"][:st.n_visible].astype(np.int64), order)
    ob = O.bin_tiles(scene, cam, opts, tier)
    assert st.n_pairs == ob["P"] and np.array_equal(fa["pair_items"], ob["vals"])
    ref = O.views(scene, [cam], opts, tier, scores=True, images=True)
    assert np.array_equal(host["rgb"], ref["img_last"]) and np.array_equal(host["contrib"], ref["contrib"])
    outside = (mx[order] < 0) | (mx[order] >= W) | (my[order] < 0) | (my[order] >= H)
    assert outside.sum() > 2000 and len(order) < n - 10_000, (outside.sum(), len(order))


def _random_frame(seed: int):
    """A seeded random frame: scene size, distributions (uniform box + clusters, isotropic to
    strongly anisotropic and heavy-tailed scales, SH degree 0-3), camera (outside or inside the
    cloud, any aspect, tiny to 1.5k-wide images, narrow to wide fov) and options (near plane,
    alpha thresholds, low-pass, sigma bound) all drawn from ``seed``."""
    from paper_2403_13806_b200.core import look_at_camera
    from paper_2403_13806_b200.synth import SceneArrays
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(200, 30_000))
    box = float(rng.uniform(0.5, 4.0))
    k = int(rng.integers(1, 40))
    centers = rng.uniform(-box, box, (k, 3))
    pick = rng.integers(0, k, n)
    means = np.where(rng.random((n, 1)) < 0.3, rng.uniform(-box, box, (n, 3)),
                     centers[pick] + rng.normal(0.0, float(rng.uniform(0.02, 0.5)), (n, 3)))
    ls = rng.normal(float(rng.uniform(-5.0, -1.5)), float(rng.uniform(0.1, 1.2)), (n, 3))
    ls[:, 0] += rng.normal(0.0, float(rng.uniform(0.0, 1.5)), n)
    ls = np.minimum(ls, 1.0)
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    lg = rng.normal(0.0, float(rng.uniform(0.5, 3.0)), n)
    sh = rng.normal(0.0, 0.1, (n, 3, 16))
    sh[:, :, 0] = rng.normal(0.0, 0.6, (n, 3))
    deg = int(rng.integers(0, 4))
    scene = SceneArrays(means.astype(np.float32), lg.astype(np.float32), sh.astype(np.float32),
                        ls.astype(np.float32), q.astype(np.float32), deg)
    inside = rng.random() < 0.25
    r = float(rng.uniform(0.1, 0.6) * box) if inside else float(rng.uniform(1.2, 3.0) * box)
    d = rng.normal(size=3)
    eye = d / np.linalg.norm(d) * r
    target = rng.normal(0.0, 0.3 * box, 3)
    W, H = (int(rng.integers(9, 1500)), int(rng.integers(7, 900))) if rng.random() < 0.3 else \
        (int(rng.integers(9, 400)), int(rng.integers(7, 300)))
    cam = look_at_camera(eye, target, width=W, height=H, fov_deg=float(rng.uniform(25.0, 110.0)))
    opts = [float(rng.uniform(0.9, 0.999)), float(rng.choice([1.0 / 255.0, 1e-3, 0.02])),
            float(rng.choice([1e-4, 1e-3, 0.05])), float(rng.uniform(0.01, 0.5)),
            float(rng.choice([0.3, 0.1, 1.0])), float(rng.choice([3.0, 2.5, 4.0]))]
    return scene, cam, opts


@pytest.mark.parametrize("prec,tier", PRECISIONS, ids=PREC_IDS)
@pytest.mark.parametrize("seed", range(64))
def test_random_frames_bit_exact(seed, prec, tier):
    """64 seeded random frames (scene, camera and options all drawn per seed: _random_frame):
    images, counts, scores and tile lists equal the oracle's in both precisions."""
    scene, cam, vals = _random_frame(seed)
    opts = options_from(vals, prec)
    O = _oracle()
    ref = O.render(scene, cam, opts, tier)
    got, st, r = _render_gpu(scene, cam, opts)
    for k in ("img", "alpha", "depth"):
        g = got["rgb"] if k == "img" else got[k]
        assert np.array_equal(g, ref[k]), f"seed {seed}: {k} max diff {np.abs(g - ref[k]).max()}"
    assert np.array_equal(got["count"], ref["count"]), seed
    assert np.array_equal(got["contrib"], ref["contrib"]), seed
    ob = O.bin_tiles(scene, cam, opts, tier)
    fa = r.frame_arrays()
    assert st.n_pairs == ob["P"] and np.array_equal(fa["pair_items"], ob["vals"]), seed
    assert np.array_equal(fa["ranges"], ob["ranges"]), seed


@pytest.mark.parametrize("prec,tier", PRECISIONS, ids=PREC_IDS)
@pytest.mark.parametrize("seed", range(16))
def test_random_filtered_frames_bit_exact(seed, prec, tier):
    """16 seeded random frames rendered through ``rasterize_filtered`` with a random indicator
    (5-90% active): colour, alpha and count equal the oracle's render of the same indicator."""
    from paper_2403_13806_b200.render import rasterize_filtered
    scene, cam, vals = _random_frame(100 + seed)
    opts = options_from(vals, prec)
    rng = np.random.default_rng(seed)
    active = rng.random(len(scene)) < float(rng.uniform(0.05, 0.9))
    ref = _oracle().render(scene, cam, opts, tier, active=active)
    got = rasterize_filtered(scene, cam, active, opts)
    assert np.array_equal(got.color.data.astype(ref["img"].dtype), ref["img"]), seed
    assert np.array_equal(got.alpha.astype(ref["alpha"].dtype), ref["alpha"]), seed
    assert np.array_equal(got.count, ref["count"]), seed


@pytest.mark.parametrize("prec,tier", PRECISIONS, ids=PREC_IDS)
@pytest.mark.parametrize("seed", range(12))
def test_random_scoring_passes_bit_exact(seed, prec, tier):
    """12 seeded random scenes scored by ``compute_importance`` from 2-7 random cameras of
    mixed sizes (one pass, the views launched without a host sync each): the table equals the
    oracle's per-view max-merge; the keep mask at a random threshold follows."""
    from paper_2403_13806_b200.pruning import compute_importance
    scene, _, vals = _random_frame(200 + seed)
    rng = np.random.default_rng(seed)
    cams = [_random_frame(300 + 10 * seed + k)[1] for k in range(int(rng.integers(2, 8)))]
    opts = options_from(vals, prec)
    table = compute_importance(scene, cams, opts)
    vt = np.float32 if prec == "fp32" else np.float64
    exp = np.zeros(len(scene), vt)
    O = _oracle()
    for cam in cams:
        exp = np.maximum(exp, O.render(scene, cam, opts, tier)["contrib"])
    assert np.array_equal(table.values.astype(vt), exp), seed
    h = float(rng.choice([1e-4, 1e-3, 1e-2]))
    assert np.array_equal(table.values >= h, exp.astype(np.float64) >= h)
