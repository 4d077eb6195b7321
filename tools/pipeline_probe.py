"""Probe: configs[1] frames with 1 or 2 frames in flight (two workspaces, two streams, one
CUDA graph each), device time of K frames from one start event to one end event.

    RS_DSORT=0 python tools/pipeline_probe.py [frames] [fp32|fp64] [flush]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2403_13806_b200 import synth  # noqa: E402
from paper_2403_13806_b200.device import Renderer, device_scene  # noqa: E402
from paper_2403_13806_b200.render import RasterizeOptions  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 100
prec = sys.argv[2] if len(sys.argv) > 2 else "fp32"
flush_on = len(sys.argv) > 3 and sys.argv[3] == "flush"
opts = RasterizeOptions(near_limit=0.2, precision=prec)
scene, cams = synth.config1(0)
dev = torch.device("cuda", 0)
ds = device_scene(scene, dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
rs = [Renderer(dev), Renderer(dev)]
for r in rs:
    for c in cams[:K]:  # size every workspace for all the timed frames (else frames overflow)
        r.render(ds, c, opts)
graphs = [r.capture(ds, cams[0], opts) for r in rs]
streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
main = torch.cuda.current_stream(dev)


def run(inflight):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(main)
    for s in range(0, K, inflight):
        if flush_on:
            flush.zero_()
        ev = torch.cuda.Event()
        ev.record(main)
        for j in range(inflight):
            st = streams[j]
            st.wait_event(ev)
            with torch.cuda.stream(st):
                graphs[j].replay(cams[(s + j) % len(cams)])
        for j in range(inflight):
            main.wait_stream(streams[j])
    b.record(main)
    torch.cuda.synchronize()
    return a.elapsed_time(b)


for inflight in (1, 2, 1, 2):
    for r in rs:
        r.read_overflow(reset=True)
    t = run(inflight)
    assert not any(r.read_overflow()[0] for r in rs), "a timed frame overflowed"
    print(f"{prec} flush={flush_on} inflight={inflight}: {K / (t / 1e3):.0f} frames/s ({t / K * 1e3:.1f} us/frame)")


def bench_style():
    """The bench's loop: flush, event, replay, event per frame; sum of per-frame times."""
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    torch.cuda.synchronize()
    for s in range(K):
        flush.zero_()
        evs[s][0].record(main)
        graphs[0].replay(cams[s % len(cams)])
        evs[s][1].record(main)
    torch.cuda.synchronize()
    t = sum(a.elapsed_time(b) for a, b in evs)
    print(f"{prec} bench-style per-frame events: {K / (t / 1e3):.0f} frames/s ({t / K * 1e3:.1f} us/frame)")


bench_style()
bench_style()
