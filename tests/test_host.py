"""Host-side logic and the C ABI boundary (CPU only, no GPU needed)."""

import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, golden, load_cam


# ---------------------------------------------------------------------------
# C ABI: the library loads and exports every symbol include/radsplat.h declares
# ---------------------------------------------------------------------------
def _declared():
    src = (ROOT / "include" / "radsplat.h").read_text()
    return sorted(set(re.findall(r"RS_API\s+[\w\s\*]+?\b(rs_\w+)\s*\(", src)))


def test_header_declares_the_documented_entry_points():
    names = _declared()
    for n in ("rs_render", "rs_project", "rs_bin", "rs_blend", "rs_compact", "rs_compact_bits",
              "rs_workspace_size", "rs_workspace_create", "rs_check_finite", "rs_max_merge"):
        assert n in names


def test_library_exports_every_declared_symbol():
    import ctypes

    from paper_2403_13806_b200 import _native
    from paper_2403_13806_b200.build import build
    build()
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    for n in _declared():
        assert hasattr(lib, n), n
    assert set(_declared()) == set(_native.SIGNATURES)
    lib = _native.load(require_cuda=False)
    assert lib.rs_abi_version() == _native.ABI_VERSION == 2
    assert lib.rs_status_string(5) == b"tile pair capacity exceeded"
    assert lib.rs_workspace_size(500_000, 10_000_000, 1256, 828) > 0
    assert lib.rs_workspace_size(-1, 10, 16, 16) == 0
    assert lib.rs_compact_workspace_size(0) > 0


def test_integration_structs_match_header():
    """INTEGRATION.md's documented ctypes structs (the binding a maintainer copies) have
    the header's fields, types and sizes -- i.e. _native.py's mirror of include/radsplat.h."""
    import ctypes
    import re

    from paper_2403_13806_b200 import _native as N
    text = (ROOT / "INTEGRATION.md").read_text()
    block = re.search(r"```python\n(# rs structs \(ABI 2\)\n.*?)```", text, re.S)
    assert block, "INTEGRATION.md lost its struct block"
    ns = {}
    exec(block.group(1), ns)
    for doc, mine in (("rs_scene", N.RsScene), ("rs_camera", N.RsCamera), ("rs_options", N.RsOptions),
                      ("rs_outputs", N.RsOutputs), ("rs_stats", N.RsStats)):
        d = ns[doc]
        assert ctypes.sizeof(d) == ctypes.sizeof(mine), doc
        assert [(n, t) for n, t in d._fields_] == [(n, t) for n, t in mine._fields_], doc
    assert len(N.RsOutputs._fields_) == 9
    # and the header declares the same members in the same order
    hdr = (ROOT / "include" / "radsplat.h").read_text()
    body = re.search(r"typedef struct rs_outputs \{(.*?)\} rs_outputs;", hdr, re.S).group(1)
    members = re.findall(r"\*\s*(\w+);", body)
    assert members == [n for n, _ in N.RsOutputs._fields_]


def test_status_codes_map_to_reference_exceptions():
    from paper_2403_13806_b200 import _native as N
    from paper_2403_13806_b200.core import InvalidParameterError, InvalidSceneError
    N.load(require_cuda=False)
    with pytest.raises(InvalidParameterError):
        N.check(N.RS_EINVAL)
    with pytest.raises(InvalidSceneError):
        N.check(N.RS_ENONFINITE)
    with pytest.raises(N.PairOverflow):
        N.check(N.RS_EOVERFLOW)
    N.check(N.RS_OK)


def test_no_cpu_fallback():
    """The compute path fails loudly without a CUDA device (no silent CPU path)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    from paper_2403_13806_b200 import _native
    from paper_2403_13806_b200.render import rasterize
    from paper_2403_13806_b200.synth import config0
    scene, cams = config0(0)
    with pytest.raises(_native.NativeUnavailable):
        rasterize(scene, cams[0])


def test_product_package_never_imports_the_oracle():
    pkg = ROOT / "paper_2403_13806_b200"
    for f in pkg.rglob("*.py"):
        assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", f.read_text(), re.M), f


# ---------------------------------------------------------------------------
# camera clustering (visibility.py:96-143), restated with the same rng sequence
# ---------------------------------------------------------------------------
def test_cluster_cameras_matches_reference_two_room():
    from paper_2403_13806_b200.visibility import cluster_cameras
    d = golden("two_room")
    for seed in (0, 5):
        p = f"room{seed}_"
        cams = [load_cam(d, f"{p}cam{i}_") for i in range(int(d[p + "n_cams"]))]
        c = cluster_cameras(np.array([cam.center for cam in cams]), k=2, seed=0)
        assert np.array_equal(c.centers, d[p + "centers"])
        assert np.array_equal(c.assignment, d[p + "assignment"])


def test_cluster_cameras_properties():
    from paper_2403_13806_b200.core import InvalidParameterError
    from paper_2403_13806_b200.visibility import cluster_cameras
    rng = np.random.default_rng(1234)
    pts = rng.uniform(-5, 5, size=(6, 3))
    c = cluster_cameras(pts, k=6, seed=0)
    assert c.inertia == pytest.approx(0.0, abs=1e-20) and len(set(c.assignment.tolist())) == 6
    left = rng.normal(size=(10, 3)) + [-20.0, 0, 0]
    right = rng.normal(size=(10, 3)) + [20.0, 0, 0]
    c = cluster_cameras(np.concatenate([left, right]), k=2, seed=1)
    assert len(set(c.assignment[:10].tolist())) == 1 and c.assignment[0] != c.assignment[10]
    np.testing.assert_allclose(sorted(c.centers[:, 0]), sorted([left.mean(0)[0], right.mean(0)[0]]), atol=1e-9)
    pts = rng.uniform(-3, 3, size=(20, 3))
    a, b = cluster_cameras(pts, 4, seed=7), cluster_cameras(pts, 4, seed=7)
    assert np.array_equal(a.centers, b.centers) and np.array_equal(a.assignment, b.assignment)
    assert cluster_cameras(np.zeros((5, 3)), k=3).inertia == 0.0
    with pytest.raises(InvalidParameterError):
        cluster_cameras(pts[:4], k=0)
    with pytest.raises(InvalidParameterError):
        cluster_cameras(pts[:4], k=5)
    c = cluster_cameras(rng.uniform(-2, 2, size=(30, 3)), k=8, seed=3)
    assert all(c.cluster_members(j).size > 0 for j in range(8))


def test_nearest_cluster_ties_lowest_index():
    from paper_2403_13806_b200.visibility import ClusterVisibility
    vis = ClusterVisibility(centers=np.array([[0.0, 0, 0], [10.0, 0, 0]]), indicators=np.ones((2, 3), bool),
                            t_cluster=0.001, scene_generation=0)
    assert vis.nearest_cluster([1.0, 0, 0]) == 0
    assert vis.nearest_cluster([9.0, 0, 0]) == 1
    assert vis.nearest_cluster([5.0, 0, 0]) == 0


def test_aux_cameras_follow_reference_rng_stream():
    """Same seed -> same jittered centres as visibility.py:150-172 (restated)."""
    from paper_2403_13806_b200.visibility import aux_cameras
    d = golden("two_room")
    cams = [load_cam(d, f"room0_cam{i}_") for i in range(3)]
    rng = np.random.default_rng(0)
    aux = aux_cameras(cams, 2, rng)
    centers = np.array([c.center for c in cams])
    sigma = 0.1 * float(np.linalg.norm(centers.std(axis=0)))
    r2 = np.random.default_rng(0)
    exp = [c.center + r2.standard_normal(3) * sigma for c in cams for _ in range(2)]
    assert len(aux) == 6
    for a, e in zip(aux, exp):
        np.testing.assert_allclose(a.center, e, atol=1e-12)


# ---------------------------------------------------------------------------
# ImportanceTable / prune semantics (pruning.py:31-127)
# ---------------------------------------------------------------------------
def _scene(n=5):
    from paper_2403_13806_b200.synth import config0
    return config0(0)[0].subset(np.arange(n)).to_scene()


def test_prune_semantics():
    from paper_2403_13806_b200.core import InvalidParameterError, StaleTableError
    from paper_2403_13806_b200.pruning import ImportanceTable, prune, prune_sweep
    t = ImportanceTable(values=np.array([0.05, 0.049999, 0.0]), scene_generation=0, n_cameras=1)
    assert t.keep_mask(0.05).tolist() == [True, False, False]
    with pytest.raises(InvalidParameterError):
        t.keep_mask(-0.1)
    s = _scene(5)
    tab = ImportanceTable(values=np.array([0.3, 0.0, 0.02, 0.5, 0.01]), scene_generation=s.generation, n_cameras=1)
    pruned, removed = prune(s, tab, 0.01)
    assert removed == 1 and len(pruned) == 4
    assert np.array_equal(pruned.positions, s.positions[[0, 2, 3, 4]])
    assert pruned.metadata["prune_removed"] == 1 and pruned.generation != s.generation
    with pytest.raises(StaleTableError):
        prune(pruned, tab, 0.0)
    with pytest.raises(InvalidParameterError):
        prune(s, tab, 0.9)
    rows = prune_sweep(s, tab, [0.0, 0.01, 0.1, 0.4])
    assert rows[0] == dict(threshold=0.0, kept=5, removed=0)
    assert [r["kept"] for r in rows] == [5, 4, 2, 1]


def test_write_csv(tmp_path):
    from paper_2403_13806_b200.pruning import ImportanceTable
    t = ImportanceTable(values=np.array([0.5, 0.125]), scene_generation=0, n_cameras=1)
    t.write_csv(tmp_path / "imp.csv")
    assert (tmp_path / "imp.csv").read_text().strip().splitlines() == ["primitive,importance", "0,0.5", "1,0.125"]


def test_api_argument_errors_without_gpu():
    from paper_2403_13806_b200.core import InvalidParameterError
    from paper_2403_13806_b200.pruning import compute_importance
    from paper_2403_13806_b200.render import ContributionAccumulator, rasterize_with_contributions
    from paper_2403_13806_b200.visibility import bake_visibility, cluster_cameras
    s = _scene(3)
    cam = load_cam(golden("suite50"), "c0_")
    with pytest.raises(InvalidParameterError):
        compute_importance(s, [])
    with pytest.raises(InvalidParameterError):
        compute_importance(s, ["not a camera"])
    with pytest.raises(InvalidParameterError):
        rasterize_with_contributions(s, cam, ContributionAccumulator(4))
    cl = cluster_cameras(np.array([cam.center]), k=1)
    with pytest.raises(InvalidParameterError):
        bake_visibility(s, cl, [cam, cam])
    with pytest.raises(InvalidParameterError):
        bake_visibility(s, cl, [cam], t_cluster=-1.0)


def test_caller_outputs_and_scores_are_validated():
    """Images / score vectors handed to Renderer.render are checked against the frame before
    any launch (the kernels write through raw pointers): wrong dtype for the precision, too
    few elements, non-contiguous, unknown keys, wrong device."""
    import torch
    from paper_2403_13806_b200 import _native as N
    from paper_2403_13806_b200.core import InvalidParameterError
    from paper_2403_13806_b200.device import Renderer
    cam = load_cam(golden("suite50"), "c0_")
    H, W = int(cam.height), int(cam.width)
    f32 = dict(rgb=torch.empty((H, W, 3)), alpha=torch.empty((H, W)), count=torch.empty((H, W), dtype=torch.int32))
    # CPU tensors: rejected for their device only once dtype and size pass
    with pytest.raises(InvalidParameterError, match="must live on"):
        Renderer.check_outputs(f32, cam, N.RS_F32, "cuda:0")
    with pytest.raises(InvalidParameterError, match="float64"):
        Renderer.check_outputs(f32, cam, N.RS_F64, "cuda:0")
    with pytest.raises(InvalidParameterError, match="elements"):
        Renderer.check_outputs(dict(alpha=torch.empty((H, W - 1))), cam, N.RS_F32, "cuda:0")
    with pytest.raises(InvalidParameterError, match="contiguous"):
        Renderer.check_outputs(dict(rgb=torch.empty((W, H, 3)).transpose(0, 1)), cam, N.RS_F32, "cuda:0")
    with pytest.raises(InvalidParameterError, match="unknown"):
        Renderer.check_outputs(dict(colour=torch.empty(1)), cam, N.RS_F32, "cuda:0")
    with pytest.raises(InvalidParameterError, match="pinned"):
        Renderer.check_outputs(dict(rgb64=torch.empty((H, W, 3), dtype=torch.float64)), cam, N.RS_F32, "cuda:0")

    class _DS:
        n, device = 10, "cuda:0"
    with pytest.raises(InvalidParameterError, match="entries"):
        Renderer.check_scores(torch.zeros(9), N.RS_F32, _DS())
    with pytest.raises(InvalidParameterError):
        Renderer.check_scores(torch.zeros(10, dtype=torch.float64), N.RS_F32)


def test_contribution_accumulator_merge_commutative():
    from paper_2403_13806_b200.render import ContributionAccumulator
    rng = np.random.default_rng(1234)
    a, b, a2 = ContributionAccumulator(5), ContributionAccumulator(5), ContributionAccumulator(5)
    a.values[:] = rng.uniform(size=5)
    b.values[:] = rng.uniform(size=5)
    a2.values[:] = a.values
    a.merge(b)
    b.merge(a2)
    assert np.array_equal(a.values, b.values)


# ---------------------------------------------------------------------------
# core types and the fp32 device packing
# ---------------------------------------------------------------------------
def test_plane_packing_roundtrip():
    from paper_2403_13806_b200.device import pack_planes, pack_sh
    s = _scene(7)
    p = pack_planes(s)
    assert p.shape == (11, 7) and p.dtype == np.float32
    assert np.array_equal(p[0:3].T, s.positions.astype(np.float32))
    assert np.array_equal(p[7:11].T, s.quaternions.astype(np.float32))
    sh = pack_sh(s)
    assert sh.shape == (7, 48) and sh.flags.c_contiguous
    assert np.array_equal(sh.reshape(7, 3, 16), s.sh.astype(np.float32))


def test_camera_struct_center_in_fp64():
    from paper_2403_13806_b200.device import camera_struct
    cam = load_cam(golden("config0"), "cfg0_")
    cs = camera_struct(cam)
    c64 = -np.asarray(cam.rotation).T @ np.asarray(cam.translation)
    assert np.array_equal(np.array(cs.center[:], np.float32), c64.astype(np.float32))
    assert cs.width == 128 and np.float32(cs.fx) == np.float32(cam.fx)


def test_look_at_camera_matches_reference_fixture():
    from paper_2403_13806_b200.core import look_at_camera
    d = golden("config0")
    cam = look_at_camera((0.0, -3.0, 0.0), (0.0, 0.0, 0.0), width=128, height=128, fov_deg=50.0)
    assert np.allclose(cam.rotation, d["cfg0_R"], atol=1e-15) and np.allclose(cam.translation, d["cfg0_t"], atol=1e-15)


def test_synth_generators_deterministic_and_shaped():
    from paper_2403_13806_b200 import synth
    a, ca = synth.config0(0)
    b, _ = synth.config0(0)
    assert np.array_equal(a.positions, b.positions) and np.array_equal(a.sh, b.sh)
    assert a.positions.shape == (4096, 3) and a.sh.shape == (4096, 3, 16) and a.positions.dtype == np.float32
    assert np.allclose(np.linalg.norm(a.quaternions, axis=1), 1, atol=1e-6)
    assert ca[0].width == 128 and np.allclose(np.linalg.norm(ca[0].center), 3.0)
    s1, c1 = synth.config1(0, n=20_000, n_frames=10)
    assert len(c1) == 10 and np.all(np.abs(s1.positions) <= 2.0)
    s4, _ = synth.config4(0, n=10_000, n_views=4)
    assert s4.log_scales.max() <= np.float32(np.log(0.5))
    eyes = synth.fibonacci_eyes(200)
    assert np.allclose(np.linalg.norm(eyes, axis=1), 3.0)


# ---------------------------------------------------------------------------
# multi-process plumbing (gloo, world size 2, CPU)
# ---------------------------------------------------------------------------
def test_shard_range_partitions():
    from paper_2403_13806_b200.dist import shard_range
    for n in (0, 1, 7, 200):
        for w in (1, 2, 3, 8):
            got = [shard_range(n, r, w) for r in range(w)]
            assert got[0][0] == 0 and got[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            assert max(h - lo for lo, h in got) - min(h - lo for lo, h in got) <= 1


def _dist_worker(rank, world, port, q):
    import os

    import torch
    import torch.distributed as dist

    from paper_2403_13806_b200.dist import all_reduce_max, shard_range, world as w
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        assert w() == (rank, world)
        n_views, n = 9, 50
        rng = np.random.default_rng(7)
        per_view = rng.uniform(size=(n_views, n)).astype(np.float32) * (rng.uniform(size=(n_views, n)) > 0.5)
        lo, hi = shard_range(n_views, rank, world)
        local = torch.zeros(n)
        for v in range(lo, hi):  # each rank max-merges its own view slice ...
            local = torch.maximum(local, torch.from_numpy(per_view[v]))
        all_reduce_max(local)  # ... and one MAX all-reduce merges the ranks
        q.put((rank, local.numpy().tobytes(), per_view.max(axis=0).tobytes()))
    finally:
        dist.destroy_process_group()


def test_sharded_scoring_merge_gloo_world2():
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dist_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, got, exp in res:
        assert got == exp  # bit-identical to the single-process max over all views


def _bits_worker(rank, world, port, q):
    import os

    import torch
    import torch.distributed as dist

    from paper_2403_13806_b200.dist import shard_range
    from paper_2403_13806_b200.visibility import gather_cluster_bits
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        k, n = 7, 37
        full = np.random.default_rng(11).uniform(size=(k, n)) > 0.6
        lo, hi = shard_range(k, rank, world)  # this rank "bakes" clusters [lo, hi)
        local = torch.from_numpy(np.packbits(full[lo:hi], axis=1, bitorder="little").reshape(hi - lo, -1))
        got = gather_cluster_bits(local, k, n)
        q.put((rank, got.tobytes(), full.tobytes()))
    finally:
        dist.destroy_process_group()


def test_cluster_bitset_gather_gloo_world2():
    """bake_visibility(shard=True)'s merge: per-rank LSB-first cluster bitsets all-gathered
    into the (k, N) indicators, identical on every rank (visibility.py:195-204)."""
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_bits_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, got, exp in res:
        assert got == exp


def test_bench_roofline_traffic_resolves():
    """bench.py's roofline.traffic comes from the committed ncu captures: every kernel name the
    bench lines look up resolves to the warm frame's DRAM bytes (not null)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", ROOT / "bench.py")
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    for which, kern in (("render_fp32", "blend2_kernel<1, 0, 0, 1, 0>"), ("render_fp64", "blend64_kernel<1, 0, 0, 1>"),
                        ("score_fp32", "blend2_kernel<0,1,0,1,0> (score)"),
                        ("batch_fp32", "blend2_kernel<1, 0, 0, 1, 0>")):
        v = b.profiled_traffic(which, kern)
        assert v is not None and v > 1e6, (which, kern, v)
