"""Scene / visibility wire formats (reference io.py:128-243) against files the
reference itself wrote (tests/golden/io.npz, made by tests/golden/make_golden.py io)."""

import json

import numpy as np
import pytest

from conftest import golden

SCENES = ("s17", "s1", "room")


def _io():
    from paper_2403_13806_b200 import io
    return io


def _write(tmp_path, name, d):
    p = tmp_path / f"{name}.rspl"
    p.write_bytes(d[name + "_rspl"].tobytes())
    (tmp_path / f"{name}.rspl.json").write_bytes(d[name + "_json"].tobytes())
    return p


@pytest.mark.parametrize("name", SCENES)
def test_scene_round_trip_byte_identical_with_reference(tmp_path, name):
    io, d = _io(), golden("io")
    p = _write(tmp_path, name, d)
    s = io.load_scene(p)
    for k, rk in (("positions", "pos"), ("opacity_logits", "logit"), ("log_scales", "ls"), ("quaternions", "quat")):
        assert np.array_equal(np.asarray(getattr(s, k)), d[f"{name}_{rk}"]), k
    assert np.array_equal(np.asarray(s.sh), d[f"{name}_sh"])
    assert s.active_sh_degree == int(d[f"{name}_deg"])
    assert s.metadata["prune_removed"] == 7
    q = tmp_path / "again.rspl"
    io.save_scene(s, q, sidecar={"stage": "golden"})
    assert q.read_bytes() == p.read_bytes()
    got, ref = json.loads((tmp_path / "again.rspl.json").read_text()), json.loads(d[name + "_json"].tobytes())
    for k in ("bbox_min", "bbox_max"):  # the reference's came from the unquantized fp64 scene
        assert np.allclose(got.pop(k), ref.pop(k), rtol=1e-6, atol=1e-7)
    assert got == ref


def test_scene_file_errors(tmp_path):
    from paper_2403_13806_b200.core import FileFormatError
    io, d = _io(), golden("io")
    p = _write(tmp_path, "s17", d)
    good = p.read_bytes()
    p.write_bytes(good + b"\x00")
    with pytest.raises(FileFormatError, match="trailing"):
        io.load_scene(p)
    p.write_bytes(b"RFLD" + good[4:])
    with pytest.raises(FileFormatError, match="magic"):
        io.load_scene(p)
    p.write_bytes(good[:4] + b"\x02\x00\x00\x00" + good[8:])
    with pytest.raises(FileFormatError, match="version"):
        io.load_scene(p)
    p.write_bytes(good[:-4])
    with pytest.raises(FileFormatError, match="truncated"):
        io.load_scene(p)


def test_visibility_round_trip_byte_identical_with_reference(tmp_path):
    from paper_2403_13806_b200.core import InvalidParameterError
    io, d = _io(), golden("io")
    p = tmp_path / "v.rvis"
    p.write_bytes(d["vis_rvis"].tobytes())
    v = io.load_visibility(p)
    assert np.array_equal(v.indicators, d["vis_indicators"])
    assert np.array_equal(v.centers, d["vis_centers"].astype(np.float32).astype(np.float64))
    assert v.t_cluster == np.float32(0.001) and v.scene_generation == -1
    q = tmp_path / "w.rvis"
    io.save_visibility(v, q)
    assert q.read_bytes() == p.read_bytes()
    with pytest.raises(InvalidParameterError):
        io.load_visibility(p, scene=io.load_scene(_write(tmp_path, "s17", d)))


@pytest.mark.gpu
@pytest.mark.parametrize("name", SCENES)
def test_scene_file_straight_to_device(tmp_path, name):
    """RSPL bytes -> one H2D copy -> rs_rspl_unpack equals uploading the reference-loaded
    scene plane for plane; rs_rspl_pack writes the reference's bytes back; frames match."""
    import torch
    from paper_2403_13806_b200.device import DeviceScene
    from paper_2403_13806_b200.render import RasterizeOptions, render_device
    from conftest import load_cam
    io, d = _io(), golden("io")
    p = _write(tmp_path, name, d)
    ds = io.load_scene_device(p)
    ref = DeviceScene(io.load_scene(p), dtype=np.float32)  # RSPL payloads are fp32
    n = ref.n
    assert ds.n == n and ds.sh_degree == ref.sh_degree
    assert torch.equal(ds.planes[:, :n], ref.planes[:, :n]) and torch.equal(ds.sh[:n], ref.sh[:n])
    q = tmp_path / "dev.rspl"
    io.save_scene(ds, q)
    assert q.read_bytes() == p.read_bytes()
    cam = load_cam(golden("known"), "single_")
    a, _ = render_device(ds, cam, RasterizeOptions())
    b, _ = render_device(ref, cam, RasterizeOptions())
    assert torch.equal(a["rgb"], b["rgb"]) and torch.equal(a["count"], b["count"])


@pytest.mark.gpu
def test_visibility_bitsets_straight_to_device_lists(tmp_path):
    import torch
    io, d = _io(), golden("io")
    p = tmp_path / "v.rvis"
    p.write_bytes(d["vis_rvis"].tobytes())
    v = io.load_visibility_device(p)
    for j in range(v.k):
        got = v.visible_indices(j).cpu().numpy()
        assert np.array_equal(got, np.nonzero(d["vis_indicators"][j])[0]), j


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 7, 8, 31, 32, 33, 1000, 100_003])
def test_pack_bits_device_equals_numpy(n):
    import torch
    io = _io()
    flags = np.random.default_rng(n).uniform(size=n) > 0.4
    got = io.pack_bits_device(torch.from_numpy(flags).cuda()).cpu().numpy()
    assert np.array_equal(got, np.packbits(flags, bitorder="little"))
