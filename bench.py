#!/usr/bin/env python
"""Benchmark of the B200-native Faster-GS training step (one JSON line on rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload H] [--impl ours|reference]

A step = one training iteration on one view per GPU (weak scaling: the
view batch grows with N): render -> L1+D-SSIM loss -> backward -> (N>1: NCCL
all-reduce of the flat gradient buffer over NVLink) -> fused Adam.  The views
cycle over an 8-camera ring around the scene (a trainer walking its camera
set); every view's target is rendered from the ground-truth store once.  The default
workload "H" is BASELINE.json's metric point: 3M Gaussians, SH degree 3,
1920x1080 (synthetic scene, random-init parameters; target rendered from the
ground-truth store, trained store = seeded perturbation of it).

`value`  : view-steps/s over all ranks, inputs (targets) resident in HBM.
`e2e`    : the same through the public C-ABI call (ts_train_step) with the
           target copied from pinned host memory every step and the loss read
           back every step.
`roofline`: dominant kernel of the step, algorithmic bytes per
           launch / its CUDA-event duration measured over the timed region.
`cpu_baseline`: the C++ CPU oracle (oracle/, a port of SPEC.md) timed on this
           host's cores on one full step of the same workload (rank 0, N=1).
--impl reference: the CPU oracle alone, K steps on the host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2602_09999_b200 import scene, types as T  # noqa: E402

METRIC = "train steps/s & fwd+bwd Mpix/s at 3M Gaussians 1080p; % HBM roofline"
RASTER_STAGES = ("preprocess", "depth_sort", "scan", "duplicate", "tile_sort", "ranges", "blend", "blend_bwd",
                 "project_bwd")
REASON_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def stage_bytes(st, n, deg, n_tiles):
    """Algorithmic bytes per stage; V, I, Ip, P measured for the view."""
    D = (deg + 1) ** 2
    V, I, Ip, P = st["V"], st["I"], st["Ip"], st["P"]
    return {
        "preprocess": 48 * n + (40 + 12 * D) * V,
        "depth_sort": 0,            # the sort's bytes are charged once (24 I) to the sort as a whole
        "scan": 8 * n,
        "duplicate": 32 * V + 12 * I,
        "tile_sort": 24 * I,
        "ranges": 8 * I + 8 * n_tiles,
        "blend": 8 * n_tiles + 40 * Ip + 20 * P,
        "loss": 36 * P,
        "blend_bwd": 8 * n_tiles + 40 * Ip + 32 * P + 36 * V,
        "project_bwd": (140 + 24 * D) * V,
        "adam": 1652 * n,
        # fused_backward_update: theta, m, v read + written (no gradient buffer), 2D grads, stats
        "project_bwd_adam": 1416 * n + 52 * V,
    }


class ClockSampler:
    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(prefix="clk", suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) != 3:
                    continue
                try:
                    rows.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
                except ValueError:
                    continue
        os.unlink(self.path)
        load = [r for r in rows if not (r[2] & 0x1)] or rows
        reasons = set()
        for r in load:
            for bit, name in REASON_BITS.items():
                if r[2] & bit and bit != 0x1:
                    reasons.add(name)
        return {"sm_mhz": float(np.median([r[0] for r in load])) if load else None,
                "sm_max_mhz": max(r[1] for r in rows) if rows else None,
                "reasons": sorted(reasons), "samples": len(load)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


REF_STEPS = 10  # cap of the reference (CPU) arm's timed steps (~3 s each at workload H)
N_VIEWS = 8  # training cameras cycled one per step (per GPU), as a 3DGS trainer walks its view set


def view_camera(w, j):
    """Camera j of the ring: the headline view (j = 0) rotated by 360/N_VIEWS * j degrees about the
    scene's vertical axis.  Every view sees the whole synthetic cube (same per-view workload)."""
    base = np.array([0.3, -0.8, -3.5])
    a = math.radians(360.0 / N_VIEWS * j)
    R = np.array([[math.cos(a), 0, math.sin(a)], [0, 1, 0], [-math.sin(a), 0, math.cos(a)]])
    return scene.make_camera(w.width, w.height, tuple(R @ base))


def cpu_step_baseline(w, gt, p0, cams, cfg, targets, steps=1, warmup=0):
    """The C++ oracle (port of SPEC.md) on all host cores: full single-view training steps, step i on
    view i mod len(cams)."""
    from oracle import oracle as O
    cores = os.cpu_count() or 1
    O.set_workers(cores)
    n = w.n
    params = p0.copy()
    m = np.zeros_like(params)
    v = np.zeros_like(params)
    acc = np.zeros(n, np.float32)
    vc = np.zeros(n, np.float32)
    times, stages = [], None
    for i in range(warmup + steps):
        adam = T.AdamConfig.make(step=i + 1)
        t0 = time.perf_counter()
        j = i % len(cams)
        _, st = O.train_step(params, m, v, n, cams[j], cfg, targets[j], adam, acc, vc)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
            stages = st
    t = float(np.mean(times))
    return {"value": 1.0 / t, "unit": "steps/s", "cores": cores, "kind": "port",
            "sample": f"{steps} full training step(s) of workload {w.name} ({n} Gaussians, SH{w.sh_degree}, "
                      f"{w.width}x{w.height}, 1 view per step): render+loss+backward+Adam",
            "s_per_step": t,
            "stage_s": dict(zip(("preprocess", "binning", "blend", "loss", "raster_bwd", "project_bwd", "adam"),
                                [round(float(x), 4) for x in stages[:7]])) if stages is not None else None}


def run_reference(args):
    world, rank, local = dist_env()
    if rank != 0:
        return 0
    w = scene.WORKLOADS[args.workload]
    from oracle import oracle as O
    gt = scene.random_params(w.n, w.s0, w.m_o, w.seed)
    # bounded sample: at most REF_STEPS timed steps (+1 warm-up) so the arm ends in about a minute
    steps, warmup = max(1, min(args.steps, REF_STEPS)), min(args.warmup, 1)
    cams = [view_camera(w, j) for j in range(min(N_VIEWS, warmup + steps))]
    cfg = T.RenderConfig.make(sh_degree=w.sh_degree)
    O.set_workers(os.cpu_count() or 1)
    targets = [O.render(gt, w.n, c, cfg)[0] for c in cams]
    p0 = scene.perturb(gt, w.n, w.seed)
    if not args.no_morton:  # same Gaussian order as the GPU arm
        O.morton_reorder(p0, w.n)
    cb = cpu_step_baseline(w, gt, p0, cams, cfg, targets, steps=steps, warmup=warmup)
    val = cb["value"]
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "steps/s", "n_gpus": world,
            "steps": steps, "warmup": warmup, "steps_requested": args.steps, "ms_per_step": 1e3 / val, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded random Gaussians, self-rendered target)",
            "config": {"workload": w.name, "gaussians": w.n, "sh_degree": w.sh_degree,
                       "resolution": f"{w.width}x{w.height}", "views_per_step": 1, "parallelism": "host threads",
                       "views": f"{N_VIEWS}-camera ring, one view per step",
                       "gaussian_order": "random" if args.no_morton else "morton"},
            "cpu_baseline": {"value": val, "unit": "steps/s", "cores": cb["cores"], "kind": "port",
                             "sample": cb["sample"]},
            "e2e": {"value": val, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "stage_s": cb["stage_s"]}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2602_09999_b200.dp import DataParallelStep
    from paper_2602_09999_b200.tilesplat import Engine, PinnedBuffer

    world, rank, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    stream = torch.cuda.current_stream()
    w = scene.WORKLOADS[args.workload]
    n = w.n
    gt = scene.random_params(n, w.s0, w.m_o, w.seed)
    # the view ring: rank r renders views r, r + N, ... (disjoint slices of each step's batch);
    # every view's target is rendered from the GT store and kept in a device slot
    cams = [view_camera(w, j) for j in range(N_VIEWS)]
    cam = cams[rank % N_VIEWS]
    cfg = T.RenderConfig.make(sh_degree=w.sh_degree)
    e = Engine(local, stream=stream.cuda_stream)
    e.set_params(gt, n)
    targets = []
    for j, c in enumerate(cams):
        t, _, _ = e.render(c, cfg)
        e.set_target(j, t)
        targets.append(t)
    target = targets[rank % N_VIEWS]
    p0 = scene.perturb(gt, n, w.seed)
    e.set_params(p0, n)
    if not args.no_morton:
        # steady-state training order: morton_reorder fires every 5000
        # iterations while densifying, so a 3M-Gaussian store is in z-order; rendering is
        # order-invariant (bitwise), the arrays just gain spatial locality
        perm = e.morton_reorder()
        p0 = scene.reorder_params(p0, n, perm)
    dp = DataParallelStep(e, mode=args.dp_mode)
    step = 0

    def view_of(s_):  # this rank's view at training step s_
        return (s_ * world + rank) % N_VIEWS
    # auto = the faster single-GPU mode as measured (profiles/): the separate float4 Adam sweep runs at the
    # HBM roof while the fused kernel is occupancy-bound, so auto picks "fused"
    fused_bwd = args.adam_mode == "fused_backward"
    if args.densify and world > 1:
        raise SystemExit("--densify runs on one GPU (the multi-GPU path needs the statistics all-reduce)")
    if fused_bwd and world > 1:
        raise SystemExit("fused_backward needs the full gradient on one rank (world size 1)")
    mode = T.ADAM_FUSED_BACKWARD if fused_bwd else T.ADAM_FUSED

    def adam_cfg(m=None):
        # the gradient buffer is consumed by this step's optimizer; the next backward
        # overwrites every row (no clear pass).  Sharded mode clears explicitly.
        return T.AdamConfig.make(step=step, extent=1.0, mode=mode if m is None else m,
                                 zero_grads=0 if args.dp_mode == "allreduce" else 1)

    densify_log = []

    def train_step():
        j = view_of(step)
        if world == 1:  # one public C-ABI call: forward, loss, backward, Adam (target slot on the device)
            e.train_step(cams[j], cfg, adam_cfg(), slot=j, want_loss=False)
        else:
            dp.step([(cams[j], cfg, j)], adam_cfg())
        if args.densify and step % 100 == 0:
            # densify / prune on the SPEC interval (every 100 iterations), as in
            # config 3's densification phase; counted in the timed region
            densify_log.append((step,) + e.densify_and_prune(2e-4, 1.0, w.seed, step))

    for _ in range(args.warmup):
        step += 1
        train_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    # per-stage breakdown: a profiled loop (CUDA events around every stage on the
    # context stream) before the timed region, which runs without the stage events
    e.set_profiling(True)
    for _ in range(min(args.steps, 30)):
        step += 1
        train_step()
    torch.cuda.synchronize()
    stimes = e.stage_times()
    e.set_profiling(False)

    # ---- timed region (device-resident targets) ----
    clk = ClockSampler(local)
    clk.start()
    l0 = e.launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(args.steps):
        step += 1
        train_step()
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    launches = e.launch_count() - l0
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    vstats = e.view_stats()
    # fused_backward merges K9 and Adam: the raster-only fwd+bwd split comes from a
    # short profiled loop of the same step with the separate optimizer sweep
    split_times = stimes
    if fused_bwd:
        e.set_profiling(True)
        for _ in range(min(args.steps, 20)):
            step += 1
            j = view_of(step)
            dp.step([(cams[j], cfg, j)], adam_cfg(T.ADAM_FUSED))
        torch.cuda.synchronize()
        split_times = e.stage_times()
        e.set_profiling(False)

    # ---- e2e: public C-ABI call with host (pinned) target and loss read-back each step ----
    pins = []
    for j in sorted({view_of(s_) for s_ in range(N_VIEWS)}):  # the views this rank trains
        pb = PinnedBuffer((w.height, w.width, 3))
        pb.array[...] = targets[j]
        pins.append((j, pb))
    pin_of = dict(pins)
    # this box's pinned host -> device bandwidth for one target (the e2e leg's per-step copy)
    scratch = torch.empty(w.height * w.width * 3, dtype=torch.float32, device=f"cuda:{local}")
    src = torch.from_numpy(pins[0][1].array.reshape(-1))  # pinned (ts_host_alloc)
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    c0.record(stream)
    for _ in range(5):
        scratch.copy_(src, non_blocking=True)
    c1.record(stream)
    torch.cuda.synchronize()
    h2d_ms = c0.elapsed_time(c1) / 5
    del scratch
    e2e_steps = max(3, min(args.steps, 50))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        step += 1
        j = view_of(step)
        if world == 1:
            e.train_step(cams[j], cfg, adam_cfg(), target_ptr=pin_of[j].ptr, want_loss=True)
        else:
            e.render(cams[j], cfg, outputs=False)
            e.training_loss(target=pin_of[j].array, want_value=True)
            e.backward(None)
            dp.exchange_and_step(adam_cfg())
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    for _, pb in pins:
        pb.free()

    # ---- per-stage accounting over the timed region ----
    bytes_ = stage_bytes(vstats, n, w.sh_degree, cam.n_tiles)
    avg = {k: (tot / max(1, c)) for k, (tot, c) in stimes.items()}
    calls = {k: c for k, (tot, c) in stimes.items()}
    if fused_bwd:   # the project_bwd stage ran the fused backward + Adam kernel
        avg["project_bwd_adam"] = avg.pop("project_bwd")
        calls["project_bwd_adam"] = calls.pop("project_bwd")
        avg.pop("adam", None)
        calls.pop("adam", None)
    split = {k: (tot / max(1, c)) for k, (tot, c) in split_times.items()}
    fwd_bwd_ms = sum(split[k] for k in RASTER_STAGES)
    R = sum(bytes_[k] for k in RASTER_STAGES)
    peak, peak_kind = hbm_peak()
    dom = max(avg, key=lambda k: avg[k])
    dom_bytes = bytes_[dom] if dom != "depth_sort" else 0
    if dom in ("depth_sort", "tile_sort"):
        dom, dom_bytes = "sort", bytes_["tile_sort"]
        dom_ms = avg["depth_sort"] + avg["tile_sort"]
    else:
        dom_ms = avg[dom]
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9 if dom_ms > 0 else 0.0
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            with open(tf) as f:
                traffic = json.load(f).get(args.workload, {}).get(dom)
        except Exception:
            traffic = None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_step_baseline(w, gt, p0, cams[:1], cfg, targets[:1], steps=1, warmup=0)

    if rank == 0:
        value = world / (ms * 1e-3)
        P = w.width * w.height
        line = {
            "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded random Gaussians; target self-rendered from the GT store; trained store = "
                    "perturbed GT)",
            "config": {"workload": w.name, "gaussians": n, "sh_degree": w.sh_degree,
                       "resolution": f"{w.width}x{w.height}", "views_per_step": world, "views_per_gpu": 1,
                       "views": f"{N_VIEWS}-camera ring (headline view rotated about the scene axis), "
                                f"rank r trains view (step * N + r) mod {N_VIEWS}",
                       "parallelism": f"dp{world} (views; NCCL {args.dp_mode} of 59N fp32 grads)",
                       "optimizer": "fused_backward (SPEC.md:492-500)" if fused_bwd else "fused (SPEC.md:473-480)",
                       "l2": "no flush: per-step working set ~9 GB >> 126 MB L2",
                       "gaussian_order": "random" if args.no_morton else
                       "morton (SPEC.md:264-272 morton_reorder applied at setup, as the training schedule does)"},
            "e2e": {"value": world / (e2e_ms * 1e-3), "unit": "steps/s",
                    "h2d_bytes_per_step": int(w.height * w.width * 3 * 4 + 104 + 64),
                    "d2h_bytes_per_step": 16, "api": "ts_train_step (C-ABI) with pinned host target",
                    "h2d_ms_per_target": round(h2d_ms, 4),
                    "h2d_gbs": round(w.height * w.width * 3 * 4 / (h2d_ms * 1e-3) / 1e9, 2),
                    "note": "the target upload overlaps the previous step; when it takes longer than a "
                            "device step, the leg is bound by this box's host-to-device bandwidth"},
            "stage_ms_split": {k: round(v, 4) for k, v in split.items()} if fused_bwd else None,
            "gpu_launches": int(launches),
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "algorithmic_bytes_per_launch": int(dom_bytes), "avg_launch_ms": dom_ms,
                         "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                         "note": ("the peak is a 1:1 read:write copy test; this kernel's mix (Adam: 4 reads : 3 "
                                  "writes) streams faster than it, hence frac > 1" if achieved > peak else None)},
            "fwd_bwd": {"ms": fwd_bwd_ms,
                        "source": "profiled loop (stage CUDA events; separate-optimizer steps)" if fused_bwd
                        else "profiled loop (stage CUDA events)", "mpix_s": world * P / (fwd_bwd_ms * 1e-3) / 1e6,
                        "algorithmic_bytes": int(R), "achieved_gbs": R / (fwd_bwd_ms * 1e-3) / 1e9,
                        "roofline_frac": R / (fwd_bwd_ms * 1e-3) / 1e9 / peak},
            "stage_ms": {k: round(v, 4) for k, v in avg.items()},
            "densify": [{"step": d[0], "n_after": d[1], "clones": d[2][0], "splits": d[2][1], "pruned": d[2][2]}
                        for d in densify_log] if args.densify else None,
            "stage_calls": calls,
            "view": vstats,
            "clocks": {k: clocks[k] for k in ("sm_mhz", "sm_max_mhz", "reasons")},
        }
        if cpu is not None:
            line["cpu_baseline"] = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
            line["cpu_baseline"]["stage_s"] = cpu["stage_s"]
        print(json.dumps(line), flush=True)
    e.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--workload", default="H", choices=sorted(scene.WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--dp-mode", default="allreduce", choices=("allreduce", "sharded", "chunked"))
    ap.add_argument("--adam-mode", default="auto", choices=("auto", "fused", "fused_backward"),
                    help="optimizer mode (SPEC.md:525): fused = separate fused-Adam sweep (SPEC.md:473-480); "
                         "fused_backward = Adam inside the backward (SPEC.md:492-500, 1 GPU only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--densify", action="store_true",
                    help="densify_and_prune every 100 iterations inside the timed region (config 3, N=1)")
    ap.add_argument("--no-morton", action="store_true",
                    help="keep the generator's random Gaussian order instead of the z-order training state")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        if args.steps > 20:
            args.steps = 20   # each CPU step is a full multi-second H step; keep the run within minutes
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
