"""Scene and visibility wire formats (reference ``fieldsplat/io.py:128-243``),
straight to and from HBM.

Byte-identical with the reference: little-endian, 4-byte magic + u32 version,
fp32 payloads, atomic writes (temp file + rename, io.py:46-58), the same
``FileFormatError`` messages and the same JSON sidecar.

* ``save_scene`` / ``load_scene`` (io.py:128-191): host scenes exactly like the
  reference. ``load_scene_device(path)`` reads the 59-float-per-Gaussian
  payload into page-locked memory, makes ONE host-to-device copy, and the
  ``rs_rspl_unpack`` kernel scatters it into the device layout (11 planes + SH
  rows, quaternions normalized in fp64 as the reference's constructor does),
  giving a ``DeviceScene`` without a host-side repack. ``save_scene`` of a
  ``DeviceScene`` packs on the device (``rs_rspl_pack``) and copies once.
* ``save_visibility`` / ``load_visibility`` (io.py:198-243): LSB-first bitsets
  per cluster. ``load_visibility_device`` also turns each cluster's bitset
  straight into its device index list (``rs_compact_bits``), the lists
  ``render_from_viewpoint`` renders from.
"""

from __future__ import annotations

import ctypes as C
import json
import os
import struct
import tempfile
from pathlib import Path

import numpy as np
import torch

from . import _native as N
from .core import FileFormatError, GaussianScene, InvalidParameterError
from .device import PLANES, DeviceScene, pack_bits_device, renderer  # noqa: F401 (re-export)
from .visibility import ClusterVisibility

SCENE_MAGIC = b"RSPL"
VIS_MAGIC = b"RVIS"
SCENE_VERSION = 1
VIS_VERSION = 1
SCENE_HEADER = 17  # magic, version u32, count u64, degree u8
PAYLOAD_ORDER = ("positions", "log_scales", "quaternions", "opacity_logits", "sh")
FLOATS_PER_GAUSSIAN = 3 + 3 + 4 + 1 + 48


def atomic_write_bytes(path, data: bytes) -> None:
    """Write via a temp file in the same directory, then rename (io.py:46-58)."""
    path = Path(path)
    path.parent.mkdir(parents=True, exist_ok=True)
    fd, tmp = tempfile.mkstemp(dir=path.parent, prefix=path.name + ".tmp")
    try:
        with os.fdopen(fd, "wb") as fh:
            fh.write(data)
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def _check_header(data: bytes, magic: bytes, version: int, kind: str) -> None:
    if len(data) < 8 or data[:4] != magic:
        raise FileFormatError(f"not a {kind} file (bad magic)")
    got = struct.unpack_from("<I", data, 4)[0]
    if got != version:
        raise FileFormatError(f"unsupported {kind} version {got}, expected {version}")


# ---------------------------------------------------------------------------
# scene files (RSPL)
# ---------------------------------------------------------------------------
def _host_payload(scene) -> list:
    n = len(scene.positions)
    return [np.ascontiguousarray(scene.positions, dtype="<f4"), np.ascontiguousarray(scene.log_scales, dtype="<f4"),
            np.ascontiguousarray(scene.quaternions, dtype="<f4"),
            np.ascontiguousarray(scene.opacity_logits, dtype="<f4"),
            np.ascontiguousarray(np.asarray(scene.sh).reshape(n, 48), dtype="<f4")]


def _device_payload(ds: DeviceScene) -> np.ndarray:
    """Device scene -> (59 * n,) fp32 payload on the host (packed on the device, one copy)."""
    lib = N.load()
    n = ds.n
    buf = torch.empty(max(FLOATS_PER_GAUSSIAN * n, 4), dtype=torch.float32, device=ds.device)
    # RSPL is fp32 (io.py:128-142): an fp64-stored scene is rounded once, like the reference's writer
    planes, sh = ds.planes.float().contiguous(), ds.sh.float().contiguous()
    with torch.cuda.device(ds.device):
        N.check(lib.rs_rspl_pack(planes.data_ptr(), planes.shape[1], sh.data_ptr(), n, buf.data_ptr(),
                                 torch.cuda.current_stream(ds.device).cuda_stream), "rspl_pack")
    return buf[:FLOATS_PER_GAUSSIAN * n].cpu().numpy()


def save_scene(scene, path, sidecar: dict | None = None) -> None:
    """Write the scene file plus a ``<path>.json`` provenance sidecar (io.py:145-161)."""
    if isinstance(scene, DeviceScene):
        n, degree, metadata = scene.n, scene.sh_degree, {}
        payload = _device_payload(scene)
        pos = payload[:3 * n].reshape(n, 3).astype(np.float64)
        body = payload.astype("<f4").tobytes()
    else:
        n, degree = len(scene.positions), int(scene.active_sh_degree)
        metadata = getattr(scene, "metadata", {}) or {}
        parts = _host_payload(scene)
        pos = np.asarray(scene.positions, np.float64)
        body = b"".join(p.tobytes() for p in parts)
    head = SCENE_MAGIC + struct.pack("<I", SCENE_VERSION) + struct.pack("<Q", n) + struct.pack("<B", degree)
    atomic_write_bytes(path, head + body)
    lo, hi = (pos.min(axis=0), pos.max(axis=0)) if n else (np.zeros(3), np.zeros(3))
    side = dict(bbox_min=lo.tolist(), bbox_max=hi.tolist(), count=n, active_sh_degree=degree,
                metadata={k: v for k, v in metadata.items() if isinstance(v, (str, int, float, bool))})
    side.update(sidecar or {})
    atomic_write_bytes(str(path) + ".json", json.dumps(side, indent=1).encode("utf-8"))


def _read_scene_header(path) -> tuple[int, int, int]:
    with open(path, "rb") as fh:
        head = fh.read(SCENE_HEADER)
        size = os.fstat(fh.fileno()).st_size
    _check_header(head, SCENE_MAGIC, SCENE_VERSION, "scene")
    if len(head) < SCENE_HEADER:
        raise FileFormatError("scene file is truncated")
    n = struct.unpack_from("<Q", head, 8)[0]
    degree = struct.unpack_from("<B", head, 16)[0]
    expect = SCENE_HEADER + 4 * FLOATS_PER_GAUSSIAN * n
    if size > expect:
        raise FileFormatError("scene file has trailing bytes")
    if size < expect:
        raise FileFormatError("scene file is truncated")
    return n, degree, size


def _sidecar_metadata(path) -> dict:
    p = Path(str(path) + ".json")
    return json.loads(p.read_text()).get("metadata", {}) if p.exists() else {}


def load_scene(path) -> GaussianScene:
    """Host scene with the file's fp32 values as float64 (io.py:164-191)."""
    n, degree, _ = _read_scene_header(path)
    data = Path(path).read_bytes()
    shapes = {"positions": (n, 3), "log_scales": (n, 3), "quaternions": (n, 4), "opacity_logits": (n,),
              "sh": (n, 48)}
    off, arrays = SCENE_HEADER, {}
    for key in PAYLOAD_ORDER:
        count = int(np.prod(shapes[key]))
        arrays[key] = np.frombuffer(data, dtype="<f4", count=count, offset=off).reshape(shapes[key]).astype(np.float64)
        off += 4 * count
    return GaussianScene(positions=arrays["positions"], opacity_logits=arrays["opacity_logits"],
                         sh=arrays["sh"].reshape(n, 3, 16), log_scales=arrays["log_scales"],
                         quaternions=arrays["quaternions"], active_sh_degree=int(degree),
                         metadata=_sidecar_metadata(path))


def load_scene_device(path, device: torch.device | None = None) -> DeviceScene:
    """Scene file straight into HBM: payload -> page-locked buffer -> one H2D copy ->
    rs_rspl_unpack. Equal, plane for plane, to uploading ``load_scene(path)``."""
    lib = N.load()
    n, degree, _ = _read_scene_header(path)
    dev = torch.device(device or torch.device("cuda", torch.cuda.current_device()))
    nf = FLOATS_PER_GAUSSIAN * n
    host = torch.empty(max(nf, 4), dtype=torch.float32, pin_memory=True)
    with open(path, "rb") as fh:
        fh.seek(SCENE_HEADER)
        got = fh.readinto(memoryview(host.numpy()).cast("B")[:4 * nf]) if nf else 0
    if got != 4 * nf:
        raise FileFormatError("scene file is truncated")
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev).cuda_stream
        payload = host.to(dev, non_blocking=True)
        planes = torch.empty((PLANES, max(n, 1)), dtype=torch.float32, device=dev)
        sh = torch.empty((max(n, 1), 48), dtype=torch.float32, device=dev)
        bad = torch.zeros(1, dtype=torch.int32, device=dev)
        N.check(lib.rs_rspl_unpack(payload.data_ptr(), n, planes.data_ptr(), max(n, 1), sh.data_ptr(),
                                   bad.data_ptr(), stream), "rspl_unpack")
        if int(bad.item()):
            raise InvalidParameterError("zero quaternion has no direction")
    ds = DeviceScene.from_tensors(planes, sh, degree, n=n)
    ds.metadata = _sidecar_metadata(path)
    return ds


# ---------------------------------------------------------------------------
# visibility files (RVIS)
# ---------------------------------------------------------------------------
def save_visibility(vis: ClusterVisibility, path) -> None:
    """Per cluster: fp32 centre + LSB-first indicator bitset (io.py:198-208)."""
    parts = [VIS_MAGIC, struct.pack("<I", VIS_VERSION), struct.pack("<I", vis.k),
             struct.pack("<Q", vis.scene_size), struct.pack("<f", vis.t_cluster)]
    for j in range(vis.k):
        parts.append(np.asarray(vis.centers[j]).astype("<f4").tobytes())
        parts.append(np.packbits(np.asarray(vis.indicators[j], bool), bitorder="little").tobytes())
    atomic_write_bytes(path, b"".join(parts))


def _read_vis(path):
    data = Path(path).read_bytes()
    _check_header(data, VIS_MAGIC, VIS_VERSION, "visibility")
    k = struct.unpack_from("<I", data, 8)[0]
    size = struct.unpack_from("<Q", data, 12)[0]
    t_cluster = struct.unpack_from("<f", data, 20)[0]
    return data, k, size, t_cluster


def load_visibility(path, scene=None) -> ClusterVisibility:
    """Reload a visibility table, optionally bound to ``scene`` (io.py:211-243)."""
    data, k, size, t_cluster = _read_vis(path)
    off, nbytes = 24, (size + 7) // 8
    centers = np.zeros((k, 3))
    indicators = np.zeros((k, size), dtype=bool)
    for j in range(k):
        centers[j] = np.frombuffer(data, dtype="<f4", count=3, offset=off).astype(np.float64)
        off += 12
        bits = np.frombuffer(data, dtype=np.uint8, count=nbytes, offset=off)
        off += nbytes
        indicators[j] = np.unpackbits(bits, count=size, bitorder="little")
    if scene is not None:
        if len(scene) != size:
            raise InvalidParameterError("visibility file does not match the scene's primitive count")
        generation = scene.generation
    else:
        generation = -1
    return ClusterVisibility(centers=centers, indicators=indicators, t_cluster=float(t_cluster),
                             scene_generation=generation)


def load_visibility_device(path, scene=None, device: torch.device | None = None) -> ClusterVisibility:
    """``load_visibility`` whose per-cluster device index lists (the ones
    ``render_from_viewpoint`` renders from) come straight from the file's bitsets:
    one upload of all bitsets, then ``rs_compact_bits`` per cluster."""
    vis = load_visibility(path, scene)
    data, k, size, _ = _read_vis(path)
    dev = torch.device(device or torch.device("cuda", torch.cuda.current_device()))
    nbytes = (size + 7) // 8
    rec = 12 + nbytes
    raw = np.frombuffer(data, dtype=np.uint8, count=k * rec, offset=24).reshape(k, rec)[:, 12:]
    bits = torch.from_numpy(np.ascontiguousarray(raw)).to(dev)
    r = renderer(dev)
    cache = vis.metadata.setdefault("_device_lists", {})
    for j in range(k):
        cache[(j, dev)] = r.compact(bits[j], bits=True, n=size)
    return vis
