#!/usr/bin/env python
"""Benchmark: RadSplat render FPS at 1256x828 (BASELINE configs[1]) and
importance-score views/s (configs[2]) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload render|score]
                    [--impl b200|reference] [--no-cpu-baseline]

One JSON line on rank 0 (contract in the task brief):
* render (default): a step = one 500k-Gaussian 1256x828 frame per rank along
  the 1000-frame orbit (rank r renders frame (s*N + r) mod 1000): weak scaling,
  value = frames/s over all ranks; each frame is one CUDA-graph launch
  (rs_render captured once, camera uploaded per frame), timed with CUDA events
  on the launching stream. Per-stage device times (preprocess / sort / blend)
  come from a separate pass with events around the three C-ABI stages. L2 is
  flushed (256 MB memset) between timed steps, outside the events.
* score: a step = one full scoring pass of configs[2] (3M Gaussians, 200
  Fibonacci views, 1256x828): views sharded contiguously across ranks, one
  NCCL MAX all-reduce; strong scaling, value = views/s.
* --impl reference: the CPU oracle port (oracle/cpu_ref.cpp, the restated
  reference algorithm; the reference itself is pure NumPy and cannot travel)
  on all host cores, same metric and config, rank 0 only.
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="default: render 200 frames, score 5 passes, house 300 frames, batch 3 x 64 frames")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", choices=("render", "score", "house", "batch", "train"), default="render")
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--n-gaussians", type=int, default=None, help="override N (debug only)")
    ap.add_argument("--precision", choices=("fp32", "fp64"), default="fp32",
                    help="arithmetic of the timed frames (fp32 = BASELINE configs' dtype)")
    a = ap.parse_args()
    if a.steps is None:
        a.steps = {"render": 200, "score": 5, "house": 300, "batch": 3, "train": 100}[a.workload]
    return a


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ---------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi -lms 200 during the timed region (clocks + throttle reasons)."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index: int):
        self.index = index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-i", str(self.index), "-lms", "200"], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None
        return self

    def __exit__(self, *a):
        self.lines = []
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
        for ln in getattr(self, "lines", []):
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
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "_fallback": True}


# ---------------------------------------------------------------------------
# CPU baseline (oracle port, all host cores)
# ---------------------------------------------------------------------------
def cpu_views(scene, cams, images: bool, threads: int | None = None, precision: str = "fp32"):
    from oracle import oracle as O
    O.build()
    t0 = time.perf_counter()
    r = O.views(scene, cams, dict_opts(precision), np.float32 if precision == "fp32" else np.float64,
                threads=threads, scores=not images, images=images)
    return time.perf_counter() - t0, r


def dict_opts(precision: str = "fp32"):
    from paper_2403_13806_b200.render import RasterizeOptions
    return RasterizeOptions(near_limit=0.2, precision=precision)


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------
def make_workload(kind: str, n_override=None):
    from paper_2403_13806_b200 import synth
    if kind == "house":
        scene, _, traj = synth.config3(0, n=n_override or 6_000_000)
        return scene, traj
    if kind == "batch":
        return synth.config4(0, n=n_override or 1_000_000)
    if kind in ("render", "train"):
        scene, cams = synth.config1(0, n=n_override or 500_000)
        return scene, cams
    scene, cams = synth.config2(0, n=n_override or 3_000_000)
    return scene, cams


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    scene, cams = make_workload(args.workload, args.n_gaussians)
    threads = os.cpu_count() or 1
    images = args.workload != "score"
    # a step = one frame (or view) rendered by all host threads (bounded sample);
    # a wall-clock guard keeps the whole arm within a few minutes on small hosts
    for s in range(args.warmup):
        cpu_views(scene, cams[s:s + 1], images, threads=threads)
    total_t, done, budget = 0.0, 0, float(os.environ.get("RADSPLAT_REF_BUDGET_S", 240))
    for s in range(args.steps):
        dt, _ = cpu_views(scene, [cams[s % len(cams)]], images, threads=threads)
        total_t += dt
        done += 1
        if total_t > budget:
            break
    value = done / total_t
    unit = "frames/s" if images else "views/s"
    line = {
        "metric": METRICS[args.workload], "impl": "reference", "value": value, "unit": unit,
        "n_gpus": world, "steps": args.steps, "steps_completed": done, "warmup": args.warmup,
        "ms_per_step": 1e3 * total_t / done,
        "higher_is_better": True, "scaling": "weak" if images else "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (seeded, BASELINE configs distributions)",
        "config": {"workload": WORKLOADS[args.workload], "n_gaussians": len(scene), "width": cams[0].width,
                   "height": cams[0].height},
        "cpu_baseline": {"value": value, "unit": unit, "cores": threads, "kind": "port",
                         "sample": f"1 {'frame' if images else 'view'} per step on {threads} threads "
                                   f"(oracle/cpu_ref.cpp fp32 restatement, tile-parallel); CPU {cpu_model()}"},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def bytes_alg_render(n_in, n_vis, P, HW):
    """SURVEY §8d per-frame algorithmic bytes."""
    return 236 * n_in + 2 * 48 * n_vis + 2 * 12 * P + 4 * P + 20 * HW


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    from paper_2403_13806_b200 import _native as N
    from paper_2403_13806_b200.device import camera_struct, device_scene, options_struct, renderer
    from paper_2403_13806_b200.dist import all_reduce_max, shard_range

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    opts = dict_opts(args.precision)
    PREC = 1 if args.precision == "fp64" else 0
    r = renderer(dev)
    lib = r.lib
    opt_s = options_struct(opts)
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    pk = peaks()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    if args.workload in ("house", "batch"):
        return run_trajectory(args, rank, world, local, dev, opts, r, opt_s, stream, flush, pk, barrier)
    if args.workload == "train":
        return run_train(args, rank, world, local, dev, opts, r, opt_s, stream, flush, pk, barrier)
    scene, cams = make_workload(args.workload, args.n_gaussians)
    ds = device_scene(scene, dev)
    W_, H_ = cams[0].width, cams[0].height
    result = {}
    if args.workload == "render":
        frames = lambda s: cams[(s * world + rank) % len(cams)]  # noqa: E731
        out = r.alloc_outputs(cams[0], precision=PREC)
        # untimed pre-pass over every frame the timed loop will render: sizes the
        # pair capacity (overflow-checked) and counts E / C for the roofline
        E = C_ = P_ = NV = 0
        for s in range(args.steps):
            _, st = r.render(ds, frames(s), opts, out=out, count_evals=True)
            E += st.evals
            C_ += st.composites
            P_ += st.n_pairs
            NV += st.n_visible
        cam_structs = [camera_struct(frames(s)) for s in range(args.steps)]
        ptr = {k: v.data_ptr() for k, v in out.items()}

        def step(cs, evs):
            evs[0].record(stream)
            N.check(lib.rs_project(r.handle, C.byref(ds.struct), None, 0, C.byref(cs), C.byref(opt_s), sptr))
            evs[1].record(stream)
            N.check(lib.rs_bin(r.handle, sptr))
            evs[2].record(stream)
            N.check(lib.rs_blend(r.handle, C.byref(opt_s), ptr["rgb"], ptr["alpha"], ptr["depth"], ptr["count"],
                                 None, 0, sptr))
            evs[3].record(stream)

        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
        for s in range(args.warmup):
            step(camera_struct(frames(s)), ev[0])
        barrier()
        # (1) per-stage device times: the three C-ABI stages launched one by one
        for s in range(args.steps):
            flush.zero_()
            step(cam_structs[s], ev[s])
        torch.cuda.synchronize(dev)
        stage = np.array([[ev[s][i].elapsed_time(ev[s][i + 1]) for i in range(3)] for s in range(args.steps)])
        # (2) the timed frames: each one CUDA-graph launch (camera upload + memset + 12 kernels)
        fg = r.capture(ds, frames(0), opts)
        gev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for s in range(args.warmup):
            fg.replay(frames(s))
        barrier()
        with ClockSampler(local) as clk:
            barrier()
            t0 = time.perf_counter()
            for s in range(args.steps):
                flush.zero_()
                gev[s][0].record(stream)
                fg.replay(frames(s))
                gev[s][1].record(stream)
            barrier()
            wall = time.perf_counter() - t0
        st = r.stats()
        assert not st.overflow
        t_frames = float(sum(a.elapsed_time(b) for a, b in gev))  # ms, device time of the K frames
        t_staged = float(stage.sum())
        t_local = torch.tensor([t_frames], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
        t_max = float(t_local.item())
        value = world * args.steps / (t_max / 1e3)
        blend_ms = float(stage[:, 2].sum())
        fp32_peak = sms * 128 * 2 * pk.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
        flops = 16 * E + 11 * C_
        achieved = flops / (blend_ms / 1e3) / 1e12
        hw = W_ * H_
        frame_bytes = bytes_alg_render(len(scene), NV / args.steps, P_ / args.steps, hw)
        result.update({
            "metric": METRICS["render"], "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64" if PREC else "f32",
            "data": "synthetic (seeded configs[1]: 500k Gaussians in 32 clusters, SH deg 3; no dataset offline)",
            "config": {"workload": "configs[1] orbit render", "n_gaussians": len(scene), "width": W_, "height": H_,
                       "tile": 16, "frames": args.steps, "l2": "flushed (256 MB memset) between timed steps",
                       "parallelism": f"frames split across {world} GPU(s), no communication"},
            "stages_ms": {"preprocess": float(stage[:, 0].mean()), "sort": float(stage[:, 1].mean()),
                          "blend": float(stage[:, 2].mean()),
                          "note": "separate pass, three C-ABI stage launches per frame"},
            "fps_without_graph": world * args.steps / (t_staged / 1e3) if world == 1 else None,
            "wall_fps": world * args.steps / wall,
            "workload_stats": {"visible_mean": NV / args.steps, "pairs_mean": P_ / args.steps,
                               "evals_per_px": E / args.steps / hw, "composites_per_px": C_ / args.steps / hw},
            "roofline": {"kernel": "blend2_kernel<COLOR>", "bound": "fp32", "achieved": achieved,
                         "peak": fp32_peak, "unit": "TFLOP/s", "frac": achieved / fp32_peak,
                         "traffic": profiled_traffic("blend2_kernel<1, 0, 0, 1, 0>"),
                         "traffic_source": TRAFFIC_FILE + " (ncu --set full, dram read+write bytes per launch)",
                         "algorithmic": "16*E + 11*C flops per frame (SURVEY §8d)",
                         "peak_source": "computed: SMs x 128 FP32 lanes x 2 x sm_max_mhz"},
            "frame_roofline": {"bytes_alg_per_frame": frame_bytes,
                               "achieved_gbs": frame_bytes / (t_max / args.steps / 1e3) / 1e9,
                               "peak_gbs": pk.get("hbm_gbs"),
                               "frac": frame_bytes / (t_max / args.steps / 1e3) / 1e9 / pk.get("hbm_gbs", 6548.8)},
            "gpu_launches": args.steps * frame_launches(W_, H_),
            "clocks": clk.summary(),
        })
        # e2e: the reference-facing call (rasterize -> RenderOutput with host numpy
        # fp64 arrays), camera in, image + alpha + count + depth out, every step
        from paper_2403_13806_b200.render import rasterize
        ke = min(args.steps, 30)
        for s in range(2):
            rasterize(scene, frames(s), opts)
        barrier()
        t0 = time.perf_counter()
        for s in range(ke):
            rasterize(scene, frames(s), opts)
        barrier()
        te = time.perf_counter() - t0
        te_t = torch.tensor([te], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te_t, op=dist.ReduceOp.MAX)
        result["e2e"] = {"value": world * ke / float(te_t.item()), "unit": "frames/s",
                         "h2d_bytes_per_step": C.sizeof(N.RsCamera) + C.sizeof(N.RsOptions),
                         "d2h_bytes_per_step": hw * (24 + 8 + 8),
                         "api": "paper_2403_13806_b200.render.rasterize (scene resident in HBM after first call)"}
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            threads = os.cpu_count() or 1
            sel = [frames(s) for s in range(4)]
            dt, _ = cpu_views(scene, sel, True, threads=threads)
            result["cpu_baseline"] = {"value": len(sel) / dt, "unit": "frames/s", "cores": threads, "kind": "port",
                                      "sample": f"{len(sel)} orbit frames, each on {threads} threads "
                                                f"(oracle/cpu_ref.cpp fp32, tile-parallel), CPU {cpu_model()}"}
    else:
        n = len(cams)
        lo, hi = shard_range(n, rank, world)
        mine = [camera_struct(c) for c in cams[lo:hi]]
        scores = torch.zeros(len(scene), dtype=torch.float64 if PREC else torch.float32, device=dev)
        # pre-pass: overflow-checked capacity sizing over this rank's views
        P_ = 0
        for c in cams[lo:hi]:
            _, st = r.render(ds, c, opts, color=False, scores=scores)
            P_ += st.n_pairs
        sc_ptr = scores.data_ptr()

        def one_pass():
            scores.zero_()
            for cs in mine:
                N.check(lib.rs_render(r.handle, C.byref(ds.struct), None, 0, C.byref(cs), C.byref(opt_s), None, None,
                                      None, None, sc_ptr, 0, sptr))
            all_reduce_max(scores)

        for _ in range(args.warmup):
            one_pass()
        barrier()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        with ClockSampler(local) as clk:
            barrier()
            t0 = time.perf_counter()
            for s in range(args.steps):
                flush.zero_()
                evs[s][0].record(stream)
                one_pass()
                evs[s][1].record(stream)
            barrier()
            wall = time.perf_counter() - t0
        assert not r.stats().overflow
        t_local = torch.tensor([sum(a.elapsed_time(b) for a, b in evs)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
        t_max = float(t_local.item())
        value = args.steps * n / (t_max / 1e3)
        kept = int((scores >= 0.01).sum().item())
        # e2e: the reference-facing compute_importance (cameras in, fp64 host table out)
        from paper_2403_13806_b200.pruning import compute_importance
        compute_importance(scene, cams, opts)
        barrier()
        t0 = time.perf_counter()
        tab = compute_importance(scene, cams, opts)
        barrier()
        te = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        assert int((tab.values >= 0.01).sum()) == kept
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            threads = os.cpu_count() or 1
            sel = cams[:2]
            dt, _ = cpu_views(scene, sel, False, threads=threads)
            result_cpu = {"value": len(sel) / dt, "unit": "views/s", "cores": threads, "kind": "port",
                          "sample": f"{len(sel)} of the 200 views, each on {threads} threads "
                                    f"(oracle/cpu_ref.cpp fp32 scoring, tile-parallel), CPU {cpu_model()}"}
        else:
            result_cpu = None
        e2e = {"value": n / float(te.item()), "unit": "views/s",
               "h2d_bytes_per_step": (hi - lo) * (C.sizeof(N.RsCamera) + C.sizeof(N.RsOptions)),
               "d2h_bytes_per_step": 4 * len(scene),
               "api": "paper_2403_13806_b200.pruning.compute_importance (one full pass of all views)"}
        result.update({
            "metric": METRIC_SCORE, "value": value, "unit": "views/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64" if PREC else "f32",
            "data": "synthetic (seeded configs[2]: 3M Gaussians, log-scale N(-4,0.6); no dataset offline)",
            "config": {"workload": "configs[2] importance scoring", "n_gaussians": len(scene), "views": n,
                       "width": W_, "height": H_, "l2": "flushed (256 MB memset) between timed passes",
                       "parallelism": f"views sharded over {world} GPU(s) + NCCL all_reduce(MAX)"},
            "kept_at_0.01": kept, "wall_views_per_s": args.steps * n / wall,
            "e2e": e2e,
            **({"cpu_baseline": result_cpu} if result_cpu else {}),
            "gpu_launches": args.steps * len(mine) * frame_launches(W_, H_),
            "clocks": clk.summary(),
        })
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_trajectory(args, rank, world, local, dev, opts, r, opt_s, stream, flush, pk, barrier):
    """configs[3] (house: 300-frame trajectory, FPS with vs without visibility
    filtering) and configs[4] (batched multi-view render: 64 frames per GPU per
    step). Frames are split across ranks with no communication (replicas); each
    frame is one rs_render_ex launch sequence timed with CUDA events on the
    launching stream, L2 flushed between frames (outside the events)."""
    import torch
    import torch.distributed as dist

    from paper_2403_13806_b200 import _native as N
    from paper_2403_13806_b200 import synth
    from paper_2403_13806_b200.device import camera_struct, device_scene
    from paper_2403_13806_b200.visibility import _center, bake_visibility, cluster_cameras

    house = args.workload == "house"
    if house:
        scene, train_cams, traj = synth.config3(0, n=args.n_gaussians or 6_000_000)
        per_step = 1
        frame_cams = lambda s: [traj[(s * world + rank) % len(traj)]]  # noqa: E731
    else:
        scene, traj = synth.config4(0, n=args.n_gaussians or 1_000_000)
        per_step = 64
        frame_cams = lambda s: [traj[((s * world + rank) * per_step + i) % len(traj)]  # noqa: E731
                                for i in range(per_step)]
    ds = device_scene(scene, dev)
    W_, H_ = traj[0].width, traj[0].height
    hw = W_ * H_
    T = ((W_ + 15) // 16) * ((H_ + 15) // 16)
    lib = r.lib
    sptr = stream.cuda_stream
    extra = {}
    if house:
        # bake: k-means (k=64) over the 512 training-camera centres, then one importance
        # pass per cluster over its member cameras; list = {h > 0.01} (reference strict >,
        # visibility.py:204; aux cameras 0 = "from that cluster's cameras")
        clustering = cluster_cameras(np.array([_center(c) for c in train_cams]), 64, seed=0)
        barrier()
        tables = {}
        # "filtered": the configs[3] rule (h >= 0.01 read as the reference's strict h > 0.01, member
        # cameras only); "filtered_ref_defaults": the reference's bake defaults (h > 0.001 and 3
        # jittered auxiliary cameras per member, visibility.py:175-177)
        for arm, t_c, aux in (("filtered", 0.01, 0), ("filtered_ref_defaults", 0.001, 3)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            vt = bake_visibility(scene, clustering, train_cams, t_cluster=t_c, aux_per_camera=aux, seed=0,
                                 options=opts)
            e1.record(stream)
            barrier()
            counts = vt.active_counts()
            extra.setdefault("bake", {})[arm] = {
                "clusters": 64, "cameras": len(train_cams), "aux_per_camera": aux, "t_cluster": t_c,
                "ms": e0.elapsed_time(e1), "active_mean": float(counts.mean()), "active_min": int(counts.min()),
                "active_max": int(counts.max())}
            tables[arm] = (vt, {j: vt.visible_indices(j, dev) for j in range(vt.k)})
        vis = tables["filtered"][0]

        def list_for(arm, cam):
            vt, ls = tables[arm]
            return ls[vt.nearest_cluster(_center(cam))]
    out = r.alloc_outputs(traj[0])
    outs = r.outputs_struct(out)

    arms = ([("filtered", True), ("filtered_ref_defaults", True), ("unfiltered", False)] if house
            else [("all", False)])
    res_arms = {}
    for arm, filt in arms:
        # untimed checked pre-pass over every timed frame: pair capacity + E/C/P statistics
        E = C_ = P_ = NV = NI = 0
        nfr = 0
        for s in range(args.steps):
            for cam in frame_cams(s):
                idx = list_for(arm, cam) if filt else None
                _, st = r.render(ds, cam, opts, out=out, active_idx=idx, count_evals=True)
                E += st.evals
                C_ += st.composites
                P_ += st.n_pairs
                NV += st.n_visible
                NI += st.n_items
                nfr += 1
        plan = []
        for s in range(args.steps):
            for cam in frame_cams(s):
                idx = list_for(arm, cam) if filt else None
                plan.append((camera_struct(cam), idx))

        # house: one CUDA graph per index list (64 cluster lists per filtered arm, one unfiltered),
        # captured after the capacity pre-pass; a frame = camera upload + one graph launch (the
        # small filtered frames are otherwise bound by the host launching ~15 kernels)
        graphs = {}
        if house:
            from paper_2403_13806_b200.device import FrameGraph
            torch.cuda.synchronize(dev)
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
        barrier()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in plan]
        with ClockSampler(local) as clk:
            barrier()
            for (cs, idx), (a, b) in zip(plan, evs):
                flush.zero_()
                a.record(stream)
                launch(cs, idx)
                b.record(stream)
            barrier()
        assert not r.stats().overflow
        t_local = torch.tensor([sum(a.elapsed_time(b) for a, b in evs)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
        t_max = float(t_local.item())
        res_arms[arm] = {
            "fps": world * nfr / (t_max / 1e3), "ms_per_frame": t_max / nfr, "clocks": clk.summary(),
            "projected_mean": NI / nfr, "visible_mean": NV / nfr, "pairs_mean": P_ / nfr,
            "pairs_per_tile_mean": P_ / nfr / T, "evals_per_px": E / nfr / hw, "composites_per_px": C_ / nfr / hw,
            "bytes_alg_per_frame": bytes_alg_render(NI / nfr, NV / nfr, P_ / nfr, hw),
            "frames": nfr * world}
    main_arm = res_arms["filtered" if house else "all"]
    t_max = main_arm["ms_per_frame"] * (main_arm["frames"] // world)
    metric = METRICS[args.workload]
    if house:
        extra["fps_unfiltered"] = res_arms["unfiltered"]["fps"]
        extra["fps_ref_defaults"] = res_arms["filtered_ref_defaults"]["fps"]
        extra["filtering_speedup"] = res_arms["filtered"]["fps"] / res_arms["unfiltered"]["fps"]
    value = main_arm["fps"]
    result = {
        "metric": metric, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32",
        "data": f"synthetic (seeded configs[{3 if house else 4}]; no dataset offline)",
        "config": {"workload": WORKLOADS[args.workload],
                   "n_gaussians": len(scene), "width": W_, "height": H_, "tile": 16,
                   "frames_per_gpu_per_step": per_step, "l2": "flushed (256 MB memset) between timed frames",
                   "parallelism": f"frames split across {world} GPU(s), no communication"},
        "arms": res_arms, "clocks": main_arm["clocks"],
        "gpu_launches": sum(a["frames"] // world for a in res_arms.values()) * frame_launches(W_, H_),
        "frame_roofline": {"bytes_alg_per_frame": main_arm["bytes_alg_per_frame"],
                           "achieved_gbs": main_arm["bytes_alg_per_frame"] / (main_arm["ms_per_frame"] / 1e3) / 1e9,
                           "peak_gbs": pk.get("hbm_gbs"),
                           "frac": main_arm["bytes_alg_per_frame"] / (main_arm["ms_per_frame"] / 1e3) / 1e9
                           / pk.get("hbm_gbs", 6548.8)},
        **extra,
    }
    if house:
        # quality of the filtered frames vs the full render (reference acceptance: PSNR,
        # test_acceptance.py:303-329), on a sample of the timed frames
        for arm in ("filtered", "filtered_ref_defaults"):
            ps = []
            for cam in [c for s in range(args.steps) for c in frame_cams(s)][:16]:
                full, _ = r.render(ds, cam, opts)
                full = full["rgb"].clone()
                filt, _ = r.render(ds, cam, opts, active_idx=list_for(arm, cam))
                mse = float(((filt["rgb"] - full) ** 2).mean().item())
                ps.append(99.0 if mse == 0 else 10.0 * np.log10(1.0 / mse))
            res_arms[arm]["psnr_vs_full_db"] = {"mean": float(np.mean(ps)), "min": float(np.min(ps)),
                                                "frames": len(ps)}
    # e2e through the public API (host results every frame)
    from paper_2403_13806_b200.render import rasterize
    from paper_2403_13806_b200.visibility import render_from_viewpoint
    sel = [c for s in range(args.steps) for c in frame_cams(s)][:8]
    call = (lambda c: render_from_viewpoint(scene, vis, c, opts)) if house else (lambda c: rasterize(scene, c, opts))
    call(sel[0])
    barrier()
    t0 = time.perf_counter()
    for c in sel:
        call(c)
    barrier()
    te = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    result["e2e"] = {"value": world * len(sel) / float(te.item()), "unit": "frames/s",
                     "h2d_bytes_per_step": per_step * (C.sizeof(N.RsCamera) + C.sizeof(N.RsOptions)),
                     "d2h_bytes_per_step": per_step * hw * (24 + 8 + 8),
                     "api": "paper_2403_13806_b200." + ("visibility.render_from_viewpoint" if house
                                                        else "render.rasterize") + f" ({len(sel)} frames)"}
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_train(args, rank, world, local, dev, opts, r, opt_s, stream, flush, pk, barrier):
    """Training step of the backward path: per view the training
    forward (rs_render_ex recording tau / last) and rs_backward for a dense random
    dL/dimage, gradients for every Gaussian parameter; views split across ranks."""
    import torch
    import torch.distributed as dist

    from paper_2403_13806_b200 import _native as N
    from paper_2403_13806_b200.device import camera_struct, device_scene

    scene, cams = make_workload("train", args.n_gaussians)
    ds = device_scene(scene, dev)
    W_, H_ = cams[0].width, cams[0].height
    frames = lambda s: cams[(s * world + rank) % len(cams)]  # noqa: E731
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
    lib, sptr = r.lib, stream.cuda_stream

    def step(cs, ev):
        ev[0].record(stream)
        N.check(lib.rs_render_ex(r.handle, C.byref(ds.struct), None, 0, C.byref(cs), C.byref(opt_s),
                                 C.byref(outs), None, 0, sptr))
        ev[1].record(stream)
        N.check(lib.rs_backward(r.handle, C.byref(ds.struct), None, 0, C.byref(opt_s), gimg.data_ptr(),
                                out["tau"].data_ptr(), out["last"].data_ptr(), *(t.data_ptr() for t in g),
                                touched.data_ptr(), sptr))
        ev[2].record(stream)

    plan = [camera_struct(frames(s)) for s in range(args.steps)]
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in plan]
    for s in range(args.warmup):
        step(plan[s % len(plan)], ev[0])
    barrier()
    with ClockSampler(local) as clk:
        barrier()
        for cs, e in zip(plan, ev):
            flush.zero_()
            step(cs, e)
        barrier()
    assert not r.stats().overflow
    fwd = np.array([a.elapsed_time(b) for a, b, _ in ev])
    bwd = np.array([b.elapsed_time(c) for _, b, c in ev])
    t_local = torch.tensor([float(fwd.sum() + bwd.sum())], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    t_max = float(t_local.item())
    result = {
        "metric": METRICS["train"], "value": world * args.steps / (t_max / 1e3), "unit": "views/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded configs[1], random dL/dimage; no dataset offline)",
        "config": {"workload": WORKLOADS["train"], "n_gaussians": n, "width": W_, "height": H_,
                   "l2": "flushed (256 MB memset) between timed steps",
                   "parallelism": f"views split across {world} GPU(s), no communication"},
        "stages_ms": {"forward_with_cache": float(fwd.mean()), "backward": float(bwd.mean())},
        "gpu_launches": args.steps * (frame_launches(W_, H_) + 2), "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.destroy_process_group()


TRAFFIC_FILE = "profiles/round1_ncu_full_configs1_traffic.json"


def profiled_traffic(kernel: str):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full capture (or None)."""
    try:
        return json.loads((ROOT / TRAFFIC_FILE).read_text()).get(kernel)
    except (OSError, ValueError):
        return None


def frame_launches(W, H):
    """Kernels per frame (image size independent): project, depth-key compaction + histograms,
    4 depth passes, segment rows / scan / placement, chunk count, tile chunks, tile scan (ranges
    + blend order), expansion (sparse and dense chunks), blend."""
    return 1 + 1 + 4 + 3 + 1 + 1 + 1 + 2 + 1


if __name__ == "__main__":
    main()
