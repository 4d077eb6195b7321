#!/usr/bin/env python
"""Benchmark: RadSplat render FPS at 1256x828 vs #Gaussians (BASELINE configs[1])
and importance-score views/s (configs[2]) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W]
                    [--workload render|score|house|batch|train] [--precision fp32|fp64]
                    [--impl b200|reference] [--no-cpu-baseline] [--quick]

One JSON line on rank 0 (contract in the task brief). With --gpus N > 1 and no
torchrun environment, the script re-launches itself under
torch.distributed.run (N ranks, one per GPU, NCCL, 127.0.0.1).

* render (default): a step = one 500k-Gaussian 1256x828 frame per rank along
  the 1000-frame orbit (rank r renders frame (s*N + r) mod 1000): replicas,
  weak scaling, value = frames/s over all ranks. Each frame is one CUDA-graph
  replay of rs_render (camera uploaded per frame), device time from CUDA events
  on the launching stream, max over ranks; L2 flushed (256 MB memset) between
  timed frames, outside the events. The same line carries, measured in the
  same run: `fp64` (the reference-arithmetic path), `score` (configs[2]
  views/s: views sharded over the ranks + one NCCL MAX all-reduce, strong
  scaling) and `fps_vs_n` (BASELINE's FPS-vs-#Gaussians sweep at 1256x828).
* score / house / batch / train: one workload per line (see their functions).
* --impl reference: the reference's algorithm on the host CPU (the oracle's
  restatement, oracle/cpu_ref.cpp: the reference itself is NumPy and cannot
  travel to the GPU box), all host threads, same metric/config, rank 0 only.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC_RENDER = "render FPS at 1256x828, 500k Gaussians (configs[1] orbit), 1 frame per GPU per step"
METRIC_SCORE = "importance-score views/s, 3M Gaussians x 200 views at 1256x828 (configs[2])"
METRIC_HOUSE = "house-scale render FPS with visibility filtering, 6M Gaussians, 1920x1080 (configs[3])"
METRIC_BATCH = "batched multi-view render frames/s, 1M heavy-tailed Gaussians, 1920x1080 (configs[4])"
METRIC_TRAIN = "training step (forward with cache + backward) views/s, 500k Gaussians at 1256x828 (configs[1])"
METRICS = {"render": METRIC_RENDER, "score": METRIC_SCORE, "house": METRIC_HOUSE, "batch": METRIC_BATCH,
           "train": METRIC_TRAIN}
WORKLOADS = {"render": "configs[1] orbit render", "score": "configs[2] importance scoring",
             "house": "configs[3] house trajectory", "batch": "configs[4] batched views",
             "train": "configs[1] orbit, forward + backward"}
SWEEP_N = (125_000, 250_000, 500_000, 1_000_000, 2_000_000, 3_000_000)
TRAFFIC = {"render_fp32": "profiles/round2_full_configs1_fp32_traffic.json",
           "render_fp64": "profiles/round2_full_configs1_fp64_traffic.json",
           "score_fp32": "profiles/round2_full_configs2_fp32_traffic.json",
           "batch_fp32": "profiles/round2_full_configs4_fp32_traffic.json"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="default: render 200 frames, score 3 passes, house 300 frames, batch 3 x 64 frames")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", choices=("render", "score", "house", "batch", "train"), default="render")
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--precision", choices=("fp32", "fp64"), default="fp32",
                    help="arithmetic of the headline frames (fp32 = BASELINE configs' dtype)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true", help="render: skip the fp64 / score / fps_vs_n blocks")
    ap.add_argument("--n-gaussians", type=int, default=None, help="override N (debug only)")
    a = ap.parse_args()
    if a.steps is None:
        a.steps = {"render": 200, "score": 3, "house": 300, "batch": 3, "train": 100}[a.workload]
    return a


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def maybe_spawn(args) -> int | None:
    """--gpus N > 1 without a torchrun environment: re-run this command under
    torch.distributed.run with N ranks (one per GPU) and return its exit code."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


# ---------------------------------------------------------------------------
# clocks, peaks, host
# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi -lms 200 during the timed region (clocks + throttle reasons)."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index: int):
        self.index = index
        self.p = None
        self.lines = []

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-i", str(self.index), "-lms", "200"], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p:
            time.sleep(0.25)
            self.p.terminate()
            try:
                out, _ = self.p.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.p.kill()
                out, _ = self.p.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self) -> dict:
        sm, mx, reasons, util_sm = [], None, set(), []
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                s, m, u = float(f[1]), float(f[2]), float(f[8])
            except ValueError:
                continue
            mx = m
            if u > 0:
                util_sm.append(s)
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
            sm.append(s)
        use = util_sm or sm
        return {"sm_mhz": statistics.median(use) if use else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm), "samples_under_load": len(util_sm)}


def peaks():
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        d["_source"] = "MEASURED_PEAKS.json (driver-measured copy bandwidth)"
        return d
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "_source": "fallback (B200_PROFILING.md)"}


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def dict_opts(precision: str = "fp32"):
    from paper_2403_13806_b200.render import RasterizeOptions
    return RasterizeOptions(near_limit=0.2, precision=precision)


def cpu_views(scene, cams, images: bool, threads: int, precision: str = "fp32"):
    """The oracle (the reference's algorithm restated, tile-parallel) on host threads."""
    from oracle import oracle as O
    O.build()
    t0 = time.perf_counter()
    r = O.views(scene, cams, dict_opts(precision), np.float32 if precision == "fp32" else np.float64,
                threads=threads, scores=not images, images=images)
    return time.perf_counter() - t0, r


def crop_camera(cam, frac: int):
    """The central 1/frac x 1/frac window of a camera's image (same intrinsics, shifted
    principal point): a bounded CPU sample of a frame."""
    from paper_2403_13806_b200.core import PinholeCamera
    w, h = cam.width // frac, cam.height // frac
    return PinholeCamera(rotation=cam.rotation, translation=cam.translation, fx=cam.fx, fy=cam.fy,
                         cx=cam.cx - (cam.width - w) / 2.0, cy=cam.cy - (cam.height - h) / 2.0, width=w, height=h)


def bytes_alg_render(n_in, n_vis, P, HW):
    """SURVEY §8d per-frame algorithmic bytes (attributes once, records and pairs written +
    read once, pair values read by the blend, RGB + alpha + depth fp32 written)."""
    return 236 * n_in + 2 * 48 * n_vis + 2 * 12 * P + 4 * P + 20 * HW


def bytes_alg_score(n_in, n_vis, P):
    """SURVEY §8d per-view algorithmic bytes of a scoring view (no SH, no image)."""
    return 44 * n_in + 2 * 36 * n_vis + 2 * 12 * P + 4 * P + 4 * n_vis


def frame_launches(n_items: int, f64: bool) -> int:
    """Kernels per frame: project, depth sort (1 cooperative kernel up to 2^20 items, else
    compaction + 4 onesweep passes), fp64 tie fix, segment rows / scan / placement, chunk
    counts, tile chunks, tile scan, expansion (sparse + dense), blend."""
    sort = 1 if n_items <= (1 << 20) else 5
    return 1 + sort + (1 if f64 else 0) + 3 + 1 + 1 + 1 + 2 + 1


def profiled_traffic(which: str, kernel: str):
    """DRAM bytes per launch of `kernel` (the warm-workspace frame's launch) from the committed
    ncu --set full capture of that workload (profiles/round2_full_*.csv), or None."""
    try:
        table = json.loads((ROOT / TRAFFIC[which]).read_text())
    except (KeyError, OSError, ValueError):
        return None
    # ncu names carry the namespace ("rs::blend2_kernel<1, 0, 0, 1, 0>"); match without it
    want = kernel.split(" (")[0].replace(" ", "").removeprefix("rs::")
    for name, v in table.items():
        if name.replace(" ", "").removeprefix("rs::") == want:
            return v
    return None


def make_config(workload: str, scene_n: int, W: int, H: int, world: int) -> dict:
    """The `config` dict of a line -- identical for the GPU arm and the reference arm."""
    par = ("views sharded over {w} GPU(s) + NCCL all_reduce(MAX)" if workload == "score"
           else "frames split across {w} GPU(s), no communication").format(w=world)
    return {"workload": WORKLOADS[workload], "n_gaussians": scene_n, "width": W, "height": H, "tile": 16,
            "l2": "flushed (256 MB memset) between timed steps", "parallelism": par}


def make_workload(kind: str, n_override=None):
    from paper_2403_13806_b200 import synth
    if kind == "house":
        scene, _, traj = synth.config3(0, n=n_override or 6_000_000)
        return scene, traj
    if kind == "batch":
        return synth.config4(0, n=n_override or 1_000_000)
    if kind in ("render", "train"):
        return synth.config1(0, n=n_override or 500_000)
    return synth.config2(0, n=n_override or 3_000_000)


# ---------------------------------------------------------------------------
# the reference arm
# ---------------------------------------------------------------------------
def run_reference(args):
    """The reference's algorithm on the host's cores (the oracle port: the reference itself is
    NumPy and cannot travel to the GPU box). A step = one bounded sample of the workload."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    scene, cams = make_workload(args.workload, args.n_gaussians)
    threads = os.cpu_count() or 1
    images = args.workload != "score"
    crop = 4 if args.workload == "batch" else 1  # configs[4] frames: the central 1/16 (see sample)
    sample = [crop_camera(c, crop) if crop > 1 else c for c in cams]
    for s in range(args.warmup):
        cpu_views(scene, sample[s:s + 1], images, threads)
    total_t, done, budget = 0.0, 0, float(os.environ.get("RADSPLAT_REF_BUDGET_S", 240))
    for s in range(args.steps):
        dt, _ = cpu_views(scene, [sample[s % len(sample)]], images, threads)
        total_t += dt
        done += 1
        if total_t > budget:
            break
    value = done / total_t / (crop * crop)
    unit = "frames/s" if images else "views/s"
    W, H = cams[0].width, cams[0].height
    line = {
        "metric": METRICS[args.workload], "impl": "reference", "value": value, "unit": unit,
        "n_gpus": world, "steps": args.steps, "steps_completed": done, "warmup": args.warmup,
        "ms_per_step": 1e3 * total_t / done,
        "higher_is_better": True, "scaling": "strong" if args.workload == "score" else "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (seeded, BASELINE configs distributions)",
        "config": make_config(args.workload, len(scene), W, H, world),
        "cpu_baseline": {"value": value, "unit": unit, "cores": threads, "kind": "port",
                         "sample": (f"1 {'frame' if images else 'view'} per step" +
                                    (f" (its central 1/{crop * crop}, rate scaled to whole frames)" if crop > 1
                                     else "") +
                                    f" on {threads} threads (oracle/cpu_ref.cpp fp32 restatement, tile-parallel); "
                                    f"CPU {cpu_model()}")},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU context
# ---------------------------------------------------------------------------
class Ctx:
    def __init__(self, args):
        import torch
        import torch.distributed as dist
        from paper_2403_13806_b200.device import renderer
        self.torch, self.dist = torch, dist
        self.rank, self.world, self.local = dist_env()
        if self.world != args.gpus and not (args.gpus == 1 and self.world == 1):
            raise SystemExit(f"world size {self.world} != --gpus {args.gpus}")
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        if self.world > 1:
            dist.init_process_group("nccl", device_id=self.dev)
        self.r = renderer(self.dev)
        self.lib = self.r.lib
        self.stream = torch.cuda.current_stream(self.dev)
        self.sptr = self.stream.cuda_stream
        self.flush = torch.empty(256 << 20, dtype=torch.uint8, device=self.dev)
        self.pk = peaks()
        self.sms = torch.cuda.get_device_properties(self.dev).multi_processor_count

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()
        self.torch.cuda.synchronize(self.dev)

    def max_over_ranks(self, v: float) -> float:
        t = self.torch.tensor([float(v)], dtype=self.torch.float64, device=self.dev)
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(self, v: float) -> float:
        t = self.torch.tensor([float(v)], dtype=self.torch.float64, device=self.dev)
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return float(t.item())

    def fp32_peak(self) -> float:
        return self.sms * 128 * 2 * self.pk.get("sm_max_mhz", 1965.0) * 1e6 / 1e12

    def fp64_peak(self) -> float:  # B200: 64 FP64 lanes per SM (tools/fma_peak.cu measures 33.6 of 37.2)
        return self.sms * 64 * 2 * self.pk.get("sm_max_mhz", 1965.0) * 1e6 / 1e12

    def hbm(self) -> float:
        return float(self.pk.get("hbm_gbs", 6650.0))

    def events(self, n):
        E = self.torch.cuda.Event
        return [(E(enable_timing=True), E(enable_timing=True)) for _ in range(n)]

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


def check_sticky(ctx):
    """Overflow / bad-index record over every frame since the last reset (the whole timed
    region): an overflowed frame would have been timed as an incomplete one."""
    over, _ = ctx.r.read_overflow(reset=True)
    if over:
        raise RuntimeError("a timed frame overflowed its pair capacity")


def staged_times(ctx, ds, cams, opts, out_ptrs, scores=None, flags=0):
    """Per-stage device times (project / sort / blend, ms per frame) of `cams`, the three
    C-ABI stages launched one by one with events between them."""
    from paper_2403_13806_b200 import _native as N
    from paper_2403_13806_b200.device import camera_struct, options_struct
    torch = ctx.torch
    opt_s = options_struct(opts)
    sc = scores.data_ptr() if scores is not None else None
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in cams]
    structs = [camera_struct(c) for c in cams]
    for cs, e in zip(structs, ev):
        ctx.flush.zero_()
        e[0].record(ctx.stream)
        N.check(ctx.lib.rs_project(ctx.r.handle, C.byref(ds.struct), None, 0, C.byref(cs), C.byref(opt_s),
                                   ctx.sptr))
        e[1].record(ctx.stream)
        N.check(ctx.lib.rs_bin(ctx.r.handle, ctx.sptr))
        e[2].record(ctx.stream)
        N.check(ctx.lib.rs_blend(ctx.r.handle, C.byref(opt_s), *out_ptrs, sc, flags, ctx.sptr))
        e[3].record(ctx.stream)
    torch.cuda.synchronize(ctx.dev)
    st = np.array([[e[i].elapsed_time(e[i + 1]) for i in range(3)] for e in ev])
    check_sticky(ctx)
    return st.mean(axis=0)


def measure_render(ctx, scene, frames, opts, steps, warmup, clocks=True):
    """Timed configs[1]-style frames: checked pre-pass (capacity, E/C/P), per-stage pass, then
    K CUDA-graph replays timed with events (L2 flushed between them, outside the events)."""
    from paper_2403_13806_b200.device import device_scene, precision_of
    torch = ctx.torch
    prec = precision_of(opts)
    ds = device_scene(scene, ctx.dev)
    cam0 = frames(0)
    hw = cam0.width * cam0.height
    out = ctx.r.alloc_outputs(cam0, precision=prec)
    E = C_ = P_ = NV = 0
    for s in range(steps):
        _, st = ctx.r.render(ds, frames(s), opts, out=out, count_evals=True)
        E += st.evals
        C_ += st.composites
        P_ += st.n_pairs
        NV += st.n_visible
    ptrs = [out[k].data_ptr() for k in ("rgb", "alpha", "depth", "count")]
    for s in range(warmup):
        ctx.r.render(ds, frames(s), opts, out=out)
    stages = staged_times(ctx, ds, [frames(s) for s in range(min(steps, 50))], opts, ptrs)
    fg = ctx.r.capture(ds, cam0, opts)
    for s in range(warmup):
        fg.replay(frames(s))
    ctx.barrier()
    ctx.r.read_overflow(reset=True)
    ev = ctx.events(steps)
    clk = ClockSampler(ctx.local) if clocks else None
    if clk:
        clk.__enter__()
    ctx.barrier()
    t0 = time.perf_counter()
    for s in range(steps):
        ctx.flush.zero_()
        ev[s][0].record(ctx.stream)
        fg.replay(frames(s))
        ev[s][1].record(ctx.stream)
    ctx.barrier()
    wall = time.perf_counter() - t0
    if clk:
        clk.__exit__(None, None, None)
    check_sticky(ctx)
    t_max = ctx.max_over_ranks(sum(a.elapsed_time(b) for a, b in ev))  # ms, K frames
    n = steps
    fp32_peak = ctx.fp32_peak()
    flops = 16 * E + 11 * C_
    res = {
        "fps": ctx.world * n / (t_max / 1e3), "ms_per_frame": t_max / n, "wall_fps": ctx.world * n / wall,
        "stages_ms": {"preprocess": float(stages[0]), "sort": float(stages[1]), "blend": float(stages[2])},
        "visible_mean": NV / n, "pairs_mean": P_ / n, "evals_per_px": E / n / hw, "composites_per_px": C_ / n / hw,
        "flops_alg_per_frame": flops / n, "bytes_alg_per_frame": bytes_alg_render(len(scene), NV / n, P_ / n, hw),
        "n_gaussians": len(scene), "frames": n, "clocks": clk.summary() if clk else None,
    }
    res["blend_tflops"] = flops / n / (stages[2] / 1e3) / 1e12
    res["blend_frac_fp32"] = res["blend_tflops"] / fp32_peak
    res["hbm_frac"] = res["bytes_alg_per_frame"] / (res["ms_per_frame"] / 1e3) / 1e9 / ctx.hbm()
    return res


def e2e_render(ctx, scene, cams, opts, frames: int):
    """The drop-in call: render.rasterize() -> RenderOutput with host float64/int64 arrays
    (camera in, image out, every frame)."""
    from paper_2403_13806_b200 import _native as N
    from paper_2403_13806_b200.render import rasterize
    for c in cams[:2]:
        rasterize(scene, c, opts)
    ctx.barrier()
    t0 = time.perf_counter()
    for c in cams[:frames]:
        rasterize(scene, c, opts)
    ctx.barrier()
    te = ctx.max_over_ranks(time.perf_counter() - t0)
    hw = cams[0].width * cams[0].height
    return {"value": ctx.world * frames / te, "unit": "frames/s",
            "h2d_bytes_per_step": C.sizeof(N.RsCamera) + C.sizeof(N.RsOptions),
            "d2h_bytes_per_step": hw * (24 + 8 + 8),
            "api": "paper_2403_13806_b200.render.rasterize (scene resident in HBM after the first call)"}


def measure_score(ctx, scene, cams, opts, steps, warmup, staged_views=6):
    """One scoring pass = every camera's score-only frame max-merged into one vector (views
    split contiguously over the ranks), then one all_reduce(MAX) (NCCL). Device time of the
    whole pass with events, max over ranks."""
    from paper_2403_13806_b200 import _native as N
    from paper_2403_13806_b200.device import (camera_struct, device_scene, options_struct, precision_of,
                                              value_dtype)
    from paper_2403_13806_b200.dist import all_reduce_max, shard_range
    torch = ctx.torch
    prec = precision_of(opts)
    ds = device_scene(scene, ctx.dev)
    n = len(cams)
    lo, hi = shard_range(n, ctx.rank, ctx.world)
    mine = cams[lo:hi]
    scores = torch.zeros(len(scene), dtype=value_dtype(prec), device=ctx.dev)
    E = C_ = P_ = NV = 0  # pre-pass over this rank's views: pair capacity and the roofline counts
    sel = mine[::max(1, len(mine) // staged_views)][:staged_views]
    sel_ids = {id(c) for c in sel}
    for c in mine:
        _, st = ctx.r.render(ds, c, opts, color=False, scores=scores, count_evals=id(c) in sel_ids)
        P_ += st.n_pairs
        NV += st.n_visible
        if id(c) in sel_ids:
            E += st.evals
            C_ += st.composites
    opt_s = options_struct(opts)
    structs = [camera_struct(c) for c in mine]
    sc_ptr = scores.data_ptr()

    def one_pass():
        scores.zero_()
        for cs in structs:
            N.check(ctx.lib.rs_render(ctx.r.handle, C.byref(ds.struct), None, 0, C.byref(cs), C.byref(opt_s),
                                      None, None, None, None, sc_ptr, 0, ctx.sptr))
        all_reduce_max(scores)

    for _ in range(warmup):
        one_pass()
    ctx.barrier()
    ctx.r.read_overflow(reset=True)
    ev = ctx.events(steps)
    with ClockSampler(ctx.local) as clk:
        ctx.barrier()
        t0 = time.perf_counter()
        for s in range(steps):
            ctx.flush.zero_()
            ev[s][0].record(ctx.stream)
            one_pass()
            ev[s][1].record(ctx.stream)
        ctx.barrier()
        wall = time.perf_counter() - t0
    check_sticky(ctx)
    t_max = ctx.max_over_ranks(sum(a.elapsed_time(b) for a, b in ev))
    kept = int((scores[:len(scene)] >= 0.01).sum().item())
    stages = staged_times(ctx, ds, sel, opts, [None, None, None, None], scores=scores)
    flops = (16 * E + 5 * C_) / max(len(sel), 1)
    peak = ctx.fp64_peak() if prec == N.RS_F64 else ctx.fp32_peak()
    nv = max(len(mine), 1)
    hw = cams[0].width * cams[0].height
    view_ms = t_max / steps / max(hi - lo, 1)
    res = {
        "views_per_s": steps * n / (t_max / 1e3), "ms_per_pass": t_max / steps, "wall_views_per_s": steps * n / wall,
        "kept_at_0.01": kept, "clocks": clk.summary(), "views": n, "views_this_rank": hi - lo,
        "stages_ms_per_view": {"preprocess": float(stages[0]), "sort": float(stages[1]), "blend": float(stages[2])},
        "visible_mean": NV / nv, "pairs_mean": P_ / nv, "evals_per_px": E / max(len(sel), 1) / hw,
        "composites_per_px": C_ / max(len(sel), 1) / hw,
    }
    blend_t = flops / (stages[2] / 1e3) / 1e12
    byt = bytes_alg_score(len(scene), NV / nv, P_ / nv)
    res["roofline"] = {
        "kernel": "blend64_kernel<0,1,0,1> (score)" if prec == N.RS_F64 else "blend2_kernel<0,1,0,1,0> (score)",
        "bound": "fp64" if prec == N.RS_F64 else "fp32", "achieved": blend_t, "peak": peak, "unit": "TFLOP/s",
        "frac": blend_t / peak,
        "traffic": profiled_traffic("score_fp64" if prec == N.RS_F64 else "score_fp32", "blend2_kernel<0, 1, 0, 1, 0>"),
        "traffic_source": TRAFFIC["score_fp32"] + " (ncu --set full, dram read+write bytes per launch)",
        "algorithmic": "16*E + 5*C flops per view (SURVEY §8d), E/C counted on the staged views",
        "peak_source": "computed: SMs x 64 FP64 lanes x 2 x sm_max_mhz" if prec == N.RS_F64
        else "computed: SMs x 128 FP32 lanes x 2 x sm_max_mhz"}
    res["view_roofline"] = {"bytes_alg_per_view": byt, "achieved_gbs": byt / (view_ms / 1e3) / 1e9,
                            "peak_gbs": ctx.hbm(), "frac": byt / (view_ms / 1e3) / 1e9 / ctx.hbm()}
    return res


def e2e_score(ctx, scene, cams, opts):
    """The drop-in compute_importance (cameras in, float64 host table out), one full pass,
    sharded over the ranks (shard=True: the collective path) when N > 1."""
    from paper_2403_13806_b200 import _native as N
    from paper_2403_13806_b200.dist import shard_range
    from paper_2403_13806_b200.pruning import compute_importance
    compute_importance(scene, cams, opts, shard=ctx.world > 1)
    ctx.barrier()
    t0 = time.perf_counter()
    tab = compute_importance(scene, cams, opts, shard=ctx.world > 1)
    ctx.barrier()
    te = ctx.max_over_ranks(time.perf_counter() - t0)
    lo, hi = shard_range(len(cams), ctx.rank, ctx.world)
    vsz = 8 if getattr(opts, "precision", "fp64") == "fp64" else 4
    return tab, {"value": len(cams) / te, "unit": "views/s",
                 "h2d_bytes_per_step": (hi - lo) * (C.sizeof(N.RsCamera) + C.sizeof(N.RsOptions)),
                 "d2h_bytes_per_step": vsz * len(scene),
                 "api": "paper_2403_13806_b200.pruning.compute_importance (one full pass of all views)"}


def roofline_render(ctx, m, prec_fp64: bool) -> dict:
    kern = "blend64_kernel<1, 0, 0, 1>" if prec_fp64 else "blend2_kernel<1, 0, 0, 1, 0>"
    peak = ctx.fp64_peak() if prec_fp64 else ctx.fp32_peak()
    return {"kernel": kern, "bound": "fp64" if prec_fp64 else "fp32", "achieved": m["blend_tflops"],
            "peak": peak, "unit": "TFLOP/s", "frac": m["blend_tflops"] / peak,
            "traffic": profiled_traffic("render_fp64" if prec_fp64 else "render_fp32", kern),
            "traffic_source": TRAFFIC["render_fp64" if prec_fp64 else "render_fp32"]
            + " (ncu --set full: dram read+write bytes per launch)",
            "algorithmic": "16*E + 11*C flops per frame (SURVEY §8d), E/C counted by the device",
            "peak_source": ("computed: SMs x 64 FP64 lanes x 2 x sm_max_mhz" if prec_fp64 else
                            "computed: SMs x 128 FP32 lanes x 2 x sm_max_mhz")
                           + " (MEASURED_PEAKS.json has no FP32 / FP64 figure; tools/fma_peak.cu measured "
                             "72.2 / 33.6 TFLOP/s of FMA issue on this pool's B200)"}


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------
def run_render(args, ctx):
    from paper_2403_13806_b200 import synth
    scene, cams = make_workload("render", args.n_gaussians)
    frames = lambda s: cams[(s * ctx.world + ctx.rank) % len(cams)]  # noqa: E731
    opts = dict_opts(args.precision)
    m = measure_render(ctx, scene, frames, opts, args.steps, args.warmup)
    W_, H_ = cams[0].width, cams[0].height
    f64 = args.precision == "fp64"
    my_frames = [frames(s) for s in range(min(args.steps, 30))]
    result = {
        "metric": METRIC_RENDER, "value": m["fps"], "unit": "frames/s", "n_gpus": ctx.world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": m["ms_per_frame"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64" if f64 else "f32",
        "data": "synthetic (seeded configs[1]: 500k Gaussians in 32 clusters, SH deg 3; no dataset offline)",
        "config": make_config("render", len(scene), W_, H_, ctx.world),
        "stages_ms": {**m["stages_ms"], "note": "separate pass, three C-ABI stage launches per frame"},
        "wall_fps": m["wall_fps"],
        "workload_stats": {k: m[k] for k in ("visible_mean", "pairs_mean", "evals_per_px", "composites_per_px")},
        "roofline": roofline_render(ctx, m, f64),
        "frame_roofline": {"bytes_alg_per_frame": m["bytes_alg_per_frame"],
                           "achieved_gbs": m["hbm_frac"] * ctx.hbm(), "peak_gbs": ctx.hbm(),
                           "peak_source": ctx.pk["_source"], "frac": m["hbm_frac"]},
        "gpu_launches": args.steps * frame_launches(len(scene), f64),
        "clocks": m["clocks"],
        "e2e": e2e_render(ctx, scene, my_frames, opts, len(my_frames)),
    }
    if ctx.rank == 0 and ctx.world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        sel = [frames(s) for s in range(4)]
        dt, _ = cpu_views(scene, sel, True, threads)
        result["cpu_baseline"] = {"value": len(sel) / dt, "unit": "frames/s", "cores": threads, "kind": "port",
                                  "sample": f"{len(sel)} orbit frames, each on {threads} threads "
                                            f"(oracle/cpu_ref.cpp fp32, tile-parallel), CPU {cpu_model()}"}
    if not args.quick:
        # the reference-arithmetic path on the same frames
        o64 = dict_opts("fp32" if f64 else "fp64")
        m64 = measure_render(ctx, scene, frames, o64, min(args.steps, 100), args.warmup, clocks=False)
        result["fp64" if not f64 else "fp32"] = {
            "fps": m64["fps"], "ms_per_frame": m64["ms_per_frame"], "stages_ms": m64["stages_ms"],
            "e2e_fps": e2e_render(ctx, scene, my_frames, o64, len(my_frames))["value"],
            "roofline": roofline_render(ctx, m64, not f64),
            "note": ("fp64 = the reference's arithmetic (bit-identical to the oracle's Tier C, within ~1e-15 of "
                     "the NumPy reference); the same graph-replay timing") if not f64 else "fp32 contract path"}
        # configs[2] importance scoring (views sharded over the ranks, NCCL MAX all-reduce)
        s2, c2 = synth.config2(0)
        so = dict_opts("fp32")
        sm = measure_score(ctx, s2, c2, so, steps=2, warmup=1)
        _, se2e = e2e_score(ctx, s2, c2, so)
        result["score"] = {"metric": METRIC_SCORE, "value": sm["views_per_s"], "unit": "views/s",
                           "scaling": "strong", "n_gpus": ctx.world, **{k: v for k, v in sm.items()
                                                                         if k != "views_per_s"},
                           "e2e": se2e}
        # FPS vs #Gaussians at 1256x828 (BASELINE metric), configs[1] distributions
        sweep = []
        for n in SWEEP_N:
            sc, cc = synth.config1(0, n=n, n_frames=1000)
            fr = lambda s, cc=cc: cc[(s * ctx.world + ctx.rank) % len(cc)]  # noqa: E731
            ms = measure_render(ctx, sc, fr, opts, 40, 3, clocks=False)
            sweep.append({"n_gaussians": n, "fps": ms["fps"], "ms_per_frame": ms["ms_per_frame"],
                          "stages_ms": ms["stages_ms"], "visible_mean": ms["visible_mean"],
                          "pairs_mean": ms["pairs_mean"], "blend_frac_fp32": ms["blend_frac_fp32"],
                          "hbm_frac": ms["hbm_frac"]})
            del sc
        result["fps_vs_n"] = sweep
    return result


def run_score(args, ctx):
    scene, cams = make_workload("score", args.n_gaussians)
    opts = dict_opts(args.precision)
    sm = measure_score(ctx, scene, cams, opts, args.steps, args.warmup)
    tab, e2e = e2e_score(ctx, scene, cams, opts)
    assert int((tab.values >= 0.01).sum()) == sm["kept_at_0.01"]
    W_, H_ = cams[0].width, cams[0].height
    result = {
        "metric": METRIC_SCORE, "value": sm["views_per_s"], "unit": "views/s", "n_gpus": ctx.world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sm["ms_per_pass"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64" if args.precision == "fp64" else "f32",
        "data": "synthetic (seeded configs[2]: 3M Gaussians, log-scale N(-4,0.6); no dataset offline)",
        "config": make_config("score", len(scene), W_, H_, ctx.world),
        **{k: v for k, v in sm.items() if k not in ("views_per_s", "ms_per_pass")},
        "e2e": e2e,
        "gpu_launches": args.steps * (sm["views_this_rank"] * frame_launches(len(scene), args.precision == "fp64")),
    }
    if ctx.rank == 0 and ctx.world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        sel = cams[:2]
        dt, _ = cpu_views(scene, sel, False, threads)
        result["cpu_baseline"] = {"value": len(sel) / dt, "unit": "views/s", "cores": threads, "kind": "port",
                                  "sample": f"{len(sel)} of the 200 views, each on {threads} threads "
                                            f"(oracle/cpu_ref.cpp fp32 scoring, tile-parallel), CPU {cpu_model()}"}
    return result


def run_trajectory(args, ctx):
    """configs[3] (house: 300-frame trajectory, FPS with vs without visibility filtering,
    bakes at the config's rule, the reference's defaults and a quality-matched threshold) and
    configs[4] (batched multi-view render: 64 frames per GPU per step). Frames split across
    ranks (replicas); each frame timed with CUDA events on the launching stream, L2 flushed
    between frames (outside the events)."""
    from paper_2403_13806_b200 import _native as N
    from paper_2403_13806_b200 import synth
    from paper_2403_13806_b200.device import FrameGraph, camera_struct, device_scene, options_struct
    from paper_2403_13806_b200.visibility import _center, bake_visibility, cluster_cameras
    torch = ctx.torch
    opts = dict_opts(args.precision)
    opt_s = options_struct(opts)
    house = args.workload == "house"
    rank, world = ctx.rank, ctx.world
    if house:
        scene, train_cams, traj = synth.config3(0, n=args.n_gaussians or 6_000_000)
        per_step = 1
        frame_cams = lambda s: [traj[(s * world + rank) % len(traj)]]  # noqa: E731
    else:
        scene, traj = synth.config4(0, n=args.n_gaussians or 1_000_000)
        per_step = 64
        frame_cams = lambda s: [traj[((s * world + rank) * per_step + i) % len(traj)]  # noqa: E731
                                for i in range(per_step)]
    ds = device_scene(scene, ctx.dev)
    W_, H_ = traj[0].width, traj[0].height
    hw = W_ * H_
    T = ((W_ + 15) // 16) * ((H_ + 15) // 16)
    r, lib, sptr = ctx.r, ctx.lib, ctx.sptr
    extra = {}
    tables = {}
    # house bake settings: the config's rule (h >= 0.01 read as the reference's strict
    # h > 0.01, member cameras only), the reference's bake defaults (h > 0.001, 3 jittered
    # auxiliary cameras per member, visibility.py:175-177), and quality-matched thresholds
    # (h > 1e-4 and h > 0: every Gaussian a member camera composites -- the reference's >= 45 dB
    # acceptance bar on the baking views, test_acceptance.py:303-329)
    bakes = (("filtered", 0.01, 0), ("filtered_ref_defaults", 0.001, 3), ("filtered_1e-4", 1e-4, 0),
             ("filtered_0", 0.0, 0)) if house else ()
    if house:
        clustering = cluster_cameras(np.array([_center(c) for c in train_cams]), 64, seed=0)
        ctx.barrier()
        for arm, t_c, aux in bakes:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ctx.stream)
            vt = bake_visibility(scene, clustering, train_cams, t_cluster=t_c, aux_per_camera=aux, seed=0,
                                 options=opts, shard=world > 1)
            e1.record(ctx.stream)
            ctx.barrier()
            counts = vt.active_counts()
            extra.setdefault("bake", {})[arm] = {
                "clusters": 64, "cameras": len(train_cams), "aux_per_camera": aux, "t_cluster": t_c,
                "ms": e0.elapsed_time(e1), "active_mean": float(counts.mean()), "active_min": int(counts.min()),
                "active_max": int(counts.max())}
            tables[arm] = (vt, {j: vt.visible_indices(j, ctx.dev) for j in range(vt.k)})

    def list_for(arm, cam):
        vt, ls = tables[arm]
        return ls[vt.nearest_cluster(_center(cam))]

    out = r.alloc_outputs(traj[0])
    outs = r.outputs_struct(out)
    arms = [(a, True) for a, _, _ in bakes] + [("unfiltered", False)] if house else [("all", False)]
    res_arms = {}
    for arm, filt in arms:
        E = C_ = P_ = NV = NI = 0
        nfr = 0
        for s in range(args.steps):  # checked pre-pass: pair capacity + E/C/P statistics
            for cam in frame_cams(s):
                idx = list_for(arm, cam) if filt else None
                _, st = r.render(ds, cam, opts, out=out, active_idx=idx, count_evals=True)
                E += st.evals
                C_ += st.composites
                P_ += st.n_pairs
                NV += st.n_visible
                NI += st.n_items
                nfr += 1
        plan = [(camera_struct(cam), list_for(arm, cam) if filt else None)
                for s in range(args.steps) for cam in frame_cams(s)]
        # house: one CUDA graph per index list (a filtered frame is otherwise bound by the host
        # launching ~12 kernels); camera uploaded per frame, then one graph launch
        graphs = {}
        if house:
            torch.cuda.synchronize(ctx.dev)
            for _, idx in plan:
                key = None if idx is None else idx.data_ptr()
                if key not in graphs:
                    graphs[key] = FrameGraph(r, ds, traj[0], opts, out, None, idx,
                                             int(idx.numel()) if idx is not None else 0)

        def launch(cs, idx):
            if graphs:
                N.check(lib.rs_set_camera(r.handle, C.byref(cs), sptr))
                graphs[None if idx is None else idx.data_ptr()].graph.replay()
                return
            N.check(lib.rs_render_ex(r.handle, C.byref(ds.struct), idx.data_ptr() if idx is not None else None,
                                     int(idx.numel()) if idx is not None else 0, C.byref(cs), C.byref(opt_s),
                                     C.byref(outs), None, 0, sptr))

        for cs, idx in plan[:max(args.warmup, 1)]:
            launch(cs, idx)
        if graphs:  # every graph launched once before the timed region (first launches upload it)
            seen = set()
            for cs, idx in plan:
                key = None if idx is None else idx.data_ptr()
                if key not in seen:
                    seen.add(key)
                    launch(cs, idx)
        ctx.barrier()
        r.read_overflow(reset=True)
        evs = ctx.events(len(plan))
        with ClockSampler(ctx.local) as clk:
            ctx.barrier()
            for (cs, idx), (a, b) in zip(plan, evs):
                ctx.flush.zero_()
                a.record(ctx.stream)
                launch(cs, idx)
                b.record(ctx.stream)
            ctx.barrier()
        check_sticky(ctx)
        t_max = ctx.max_over_ranks(sum(a.elapsed_time(b) for a, b in evs))
        if os.environ.get("RS_BENCH_DEBUG"):
            ft = np.array([a.elapsed_time(b) for a, b in evs]) * 1e3
            print(f"[debug] {arm}: frame us min {ft.min():.1f} med {np.median(ft):.1f} mean {ft.mean():.1f} "
                  f"max {ft.max():.1f}, graphs {len(graphs)}", file=sys.stderr)
        sel = [c for s in range(args.steps) for c in frame_cams(s)][:6]
        stages = staged_times(ctx, ds, sel, opts, [out[k].data_ptr() for k in ("rgb", "alpha", "depth", "count")]) \
            if not filt else None
        res_arms[arm] = {
            "fps": world * nfr / (t_max / 1e3), "ms_per_frame": t_max / nfr, "clocks": clk.summary(),
            "projected_mean": NI / nfr, "visible_mean": NV / nfr, "pairs_mean": P_ / nfr,
            "pairs_per_tile_mean": P_ / nfr / T, "evals_per_px": E / nfr / hw, "composites_per_px": C_ / nfr / hw,
            "flops_alg_per_frame": (16 * E + 11 * C_) / nfr,
            "bytes_alg_per_frame": bytes_alg_render(NI / nfr, NV / nfr, P_ / nfr, hw),
            "frames": nfr * world}
        if stages is not None:
            res_arms[arm]["stages_ms"] = {"preprocess": float(stages[0]), "sort": float(stages[1]),
                                          "blend": float(stages[2])}
    main_arm = res_arms["filtered" if house else "all"]
    ref_arm = res_arms["unfiltered" if house else "all"]
    if house:
        # quality of each bake vs the full render (the reference's acceptance metric, PSNR,
        # test_acceptance.py:303-329) on baking (training) views and on trajectory frames
        for arm, _, _ in bakes:
            for where, cams_q in (("baking_views", train_cams[::32]), ("trajectory", traj[::19])):
                ps = []
                for cam in cams_q:
                    full, _ = r.render(ds, cam, opts)
                    full = full["rgb"].clone()
                    filt_img, _ = r.render(ds, cam, opts, active_idx=list_for(arm, cam))
                    mse = float(((filt_img["rgb"].double() - full.double()) ** 2).mean().item())
                    ps.append(float("inf") if mse == 0 else 10.0 * np.log10(1.0 / mse))
                res_arms[arm][f"psnr_vs_full_db_{where}"] = {
                    "mean": float(np.mean([p for p in ps if np.isfinite(p)])) if any(np.isfinite(ps)) else "inf",
                    "min": float(np.min(ps)) if np.isfinite(np.min(ps)) else "inf", "frames": len(ps)}
        extra["fps_unfiltered"] = res_arms["unfiltered"]["fps"]
        extra["filtering_speedup"] = res_arms["filtered"]["fps"] / res_arms["unfiltered"]["fps"]
        ok = [a for a, _, _ in bakes
              if res_arms[a]["psnr_vs_full_db_baking_views"]["min"] == "inf"
              or res_arms[a]["psnr_vs_full_db_baking_views"]["min"] >= 45.0]
        best = max(ok, key=lambda a: res_arms[a]["fps"]) if ok else None
        extra["quality_matched"] = {"arm": best, "fps": res_arms[best]["fps"] if best else None,
                                    "speedup_vs_unfiltered": res_arms[best]["fps"] / res_arms["unfiltered"]["fps"]
                                    if best else None,
                                    "bar": ">= 45 dB vs the full render on every sampled baking view "
                                           "(test_acceptance.py:303-329)"}
    # roofline of the dominant kernel (the blend of the unfiltered / batch frames)
    fl, bl = ref_arm["flops_alg_per_frame"], ref_arm["stages_ms"]["blend"]
    ach = fl / (bl / 1e3) / 1e12
    f64 = args.precision == "fp64"
    peak = ctx.fp64_peak() if f64 else ctx.fp32_peak()
    t_frame = main_arm["ms_per_frame"]
    result = {
        "metric": METRICS[args.workload], "value": main_arm["fps"], "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_frame * per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64" if args.precision == "fp64" else "f32",
        "data": f"synthetic (seeded configs[{3 if house else 4}]; no dataset offline)",
        "config": make_config(args.workload, len(scene), W_, H_, world),
        "frames_per_gpu_per_step": per_step,
        "arms": res_arms, "clocks": main_arm["clocks"],
        "gpu_launches": sum(a["frames"] // world for a in res_arms.values())
        * frame_launches(len(scene), args.precision == "fp64"),
        "roofline": {"kernel": ("blend64_kernel<1, 0, 0, 1>" if f64 else "blend2_kernel<1, 0, 0, 1, 0>")
                     + (" (unfiltered frames)" if house else ""),
                     "bound": "fp64" if f64 else "fp32", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                     "frac": ach / peak,
                     "traffic": None if (house or f64) else profiled_traffic("batch_fp32", "blend2_kernel<1, 0, 0, 1, 0>"),
                     "traffic_source": None if (house or f64) else TRAFFIC["batch_fp32"],
                     "algorithmic": "16*E + 11*C flops per frame (SURVEY §8d)",
                     "peak_source": "computed: SMs x %d FP%d lanes x 2 x sm_max_mhz" % ((64, 64) if f64 else (128, 32))},
        "frame_roofline": {"bytes_alg_per_frame": main_arm["bytes_alg_per_frame"],
                           "achieved_gbs": main_arm["bytes_alg_per_frame"] / (t_frame / 1e3) / 1e9,
                           "peak_gbs": ctx.hbm(),
                           "frac": main_arm["bytes_alg_per_frame"] / (t_frame / 1e3) / 1e9 / ctx.hbm()},
        **extra,
    }
    # e2e through the public API (host results every frame)
    from paper_2403_13806_b200.render import rasterize
    from paper_2403_13806_b200.visibility import render_from_viewpoint
    sel = [c for s in range(args.steps) for c in frame_cams(s)][:8]
    vis = tables["filtered"][0] if house else None
    call = (lambda c: render_from_viewpoint(scene, vis, c, opts)) if house else (lambda c: rasterize(scene, c, opts))
    call(sel[0])
    ctx.barrier()
    t0 = time.perf_counter()
    for c in sel:
        call(c)
    ctx.barrier()
    te = ctx.max_over_ranks(time.perf_counter() - t0)
    result["e2e"] = {"value": world * len(sel) / te, "unit": "frames/s",
                     "h2d_bytes_per_step": per_step * (C.sizeof(N.RsCamera) + C.sizeof(N.RsOptions)),
                     "d2h_bytes_per_step": per_step * hw * (24 + 8 + 8),
                     "api": "paper_2403_13806_b200." + ("visibility.render_from_viewpoint" if house
                                                        else "render.rasterize") + f" ({len(sel)} frames)"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        if house:
            cam = frame_cams(0)[0]
            dt, _ = cpu_views(scene, [cam], True, threads)
            result["cpu_baseline"] = {"value": 1.0 / dt, "unit": "frames/s", "cores": threads, "kind": "port",
                                      "sample": f"1 unfiltered trajectory frame on {threads} threads "
                                                f"(oracle/cpu_ref.cpp fp32, tile-parallel), CPU {cpu_model()}"}
        else:
            crop = crop_camera(frame_cams(0)[0], 4)
            dt, _ = cpu_views(scene, [crop], True, threads)
            result["cpu_baseline"] = {"value": 1.0 / (16 * dt), "unit": "frames/s", "cores": threads, "kind": "port",
                                      "sample": f"the central 480x270 window (1/16) of one 1920x1080 view on "
                                                f"{threads} threads, rate scaled to whole frames (oracle/cpu_ref.cpp "
                                                f"fp32, tile-parallel), CPU {cpu_model()}"}
    return result


def run_train(args, ctx):
    """Training step of the backward path: per view the training
    forward (rs_render_ex recording tau / last) and rs_backward for a dense random
    dL/dimage, gradients for every Gaussian parameter; views split across ranks."""
    from paper_2403_13806_b200 import _native as N
    from paper_2403_13806_b200.device import camera_struct, device_scene, options_struct
    torch = ctx.torch
    opts = dict_opts("fp32")
    opt_s = options_struct(opts)
    scene, cams = make_workload("train", args.n_gaussians)
    ds = device_scene(scene, ctx.dev)
    r, dev = ctx.r, ctx.dev
    W_, H_ = cams[0].width, cams[0].height
    frames = lambda s: cams[(s * ctx.world + ctx.rank) % len(cams)]  # noqa: E731
    out = r.alloc_outputs(cams[0])
    out["tau"] = torch.empty((H_, W_), dtype=torch.float32, device=dev)
    out["last"] = torch.empty((H_, W_), dtype=torch.int32, device=dev)
    for s in range(min(args.steps, 50)):  # size the pair capacity (checked renders)
        r.render(ds, frames(s), opts, out=out)
    outs = r.outputs_struct(out)
    n = ds.n
    gimg = torch.randn((H_, W_, 3), dtype=torch.float32, device=dev, generator=torch.Generator(dev).manual_seed(0))
    g = [torch.empty(k, dtype=torch.float32, device=dev) for k in (3 * n, 48 * n, 3 * n, 4 * n, n, n)]
    touched = torch.empty(n, dtype=torch.uint8, device=dev)
    lib, sptr = r.lib, ctx.sptr

    def step(cs, ev):
        ev[0].record(ctx.stream)
        N.check(lib.rs_render_ex(r.handle, C.byref(ds.struct), None, 0, C.byref(cs), C.byref(opt_s),
                                 C.byref(outs), None, 0, sptr))
        ev[1].record(ctx.stream)
        N.check(lib.rs_backward(r.handle, C.byref(ds.struct), None, 0, C.byref(opt_s), gimg.data_ptr(),
                                out["tau"].data_ptr(), out["last"].data_ptr(), *(t.data_ptr() for t in g),
                                touched.data_ptr(), sptr))
        ev[2].record(ctx.stream)

    plan = [camera_struct(frames(s)) for s in range(args.steps)]
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in plan]
    for s in range(args.warmup):
        step(plan[s % len(plan)], ev[0])
    ctx.barrier()
    r.read_overflow(reset=True)
    with ClockSampler(ctx.local) as clk:
        ctx.barrier()
        for cs, e in zip(plan, ev):
            ctx.flush.zero_()
            step(cs, e)
        ctx.barrier()
    check_sticky(ctx)
    fwd = np.array([a.elapsed_time(b) for a, b, _ in ev])
    bwd = np.array([b.elapsed_time(c) for _, b, c in ev])
    t_max = ctx.max_over_ranks(float(fwd.sum() + bwd.sum()))
    # e2e: a device-resident optimizer step through the public training pair --
    # rasterize_cached(device_outputs) -> L2 loss on the device -> rasterize_backward(device)
    # -> in-place SGD on the parameter planes; per step the camera goes up, the loss comes down
    from paper_2403_13806_b200.device import DeviceScene
    from paper_2403_13806_b200.render import rasterize_backward, rasterize_cached
    pl, shp = ds.planes.clone(), ds.sh.clone()
    dsp = DeviceScene.from_tensors(pl, shp, ds.sh_degree, check_finite=False)
    target = torch.zeros((H_, W_, 3), dtype=torch.float32, device=dev)

    def opt_step(cam):
        img, cache = rasterize_cached(dsp, cam, opts, device_outputs=True)
        diff = img["rgb"] - target
        loss = (diff * diff).mean()
        gr = rasterize_backward(dsp, cam, cache, diff * (2.0 / diff.numel()), device=True)
        with torch.no_grad():
            pl[0:3] -= 1e-4 * gr["positions"].T
            pl[3] -= 1e-4 * gr["opacity_logits"]
            pl[4:7] -= 1e-4 * gr["log_scales"].T
            pl[7:11] -= 1e-4 * gr["quaternions"].T
            shp.sub_(1e-4 * gr["sh"].reshape(-1, 48))
        return float(loss.item())

    ke = min(args.steps, 30)
    for s in range(2):
        opt_step(frames(s))
    ctx.barrier()
    t0 = time.perf_counter()
    for s in range(ke):
        opt_step(frames(s))
    ctx.barrier()
    te = ctx.max_over_ranks(time.perf_counter() - t0)
    e2e = {"value": ctx.world * ke / te, "unit": "views/s",
           "h2d_bytes_per_step": C.sizeof(N.RsCamera) + C.sizeof(N.RsOptions), "d2h_bytes_per_step": 4,
           "api": "render.rasterize_cached(device_outputs=True) + rasterize_backward(device=True) + in-place "
                  "SGD on DeviceScene.from_tensors parameters (one optimizer step per view)"}
    return {
        "metric": METRIC_TRAIN, "value": ctx.world * args.steps / (t_max / 1e3), "unit": "views/s",
        "n_gpus": ctx.world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded configs[1], random dL/dimage; no dataset offline)",
        "config": make_config("train", n, W_, H_, ctx.world),
        "stages_ms": {"forward_with_cache": float(fwd.mean()), "backward": float(bwd.mean())},
        "gpu_launches": args.steps * (frame_launches(n, False) + 2), "clocks": clk.summary(),
        "e2e": e2e,
        # the training pair is a widening beyond SURVEY §8's rows: §8d gives no algorithmic
        # flop/byte model for the backward, and oracle/ has no CPU restatement of it (its
        # parity is anchored on the reference's own fp64 gradients, tests/golden/grad.npz)
        "roofline": None,
        "roofline_note": "no SURVEY §8d algorithmic model for the backward; the forward's blend roofline "
                         "is the render line's",
        "cpu_baseline": None,
        "cpu_baseline_note": "no CPU restatement of the backward in oracle/ (parity vs the reference's "
                             "fp64 gradients, tests/golden/grad.npz)",
    }


def main():
    args = parse()
    rc = maybe_spawn(args)
    if rc is not None:
        sys.exit(rc)
    if args.impl == "reference":
        return run_reference(args)
    ctx = Ctx(args)
    fn = {"render": run_render, "score": run_score, "house": run_trajectory, "batch": run_trajectory,
          "train": run_train}[args.workload]
    result = fn(args, ctx)
    if ctx.rank == 0:
        print(json.dumps(result), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
