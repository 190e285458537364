#!/usr/bin/env python
"""Benchmark of the B200-native Faster-GS training step (one JSON line on rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload H] [--impl ours|reference]

A step = one training iteration over the step's view batch: per view render -> L1+D-SSIM
loss -> backward (gradients summed over the batch), then (N>1: one NCCL
exchange of the flat 59N gradient buffer over NVLink) -> fused Adam.  The views cycle
over an 8-camera ring around the scene (a trainer walking its camera set); every view's
target is rendered from the ground-truth store once.

Batches (`config.views_per_step`):
  * every workload but c4 trains ONE view per GPU per step (weak scaling: the batch grows
    with N).  The default "H" is BASELINE.json's metric point: 3M Gaussians, SH3, 1920x1080;
  * c4 (6M Gaussians, 1080p) trains a fixed 8-view batch per step, split 8/N views per GPU
    (strong scaling, north_star's 1/2/4/8-GPU config): N=1 accumulates all 8 views, then one Adam.
With --gpus N > 1 and no torchrun environment the script re-launches itself under
torch.distributed.run with N ranks (one per GPU, NCCL); the default exchange for N > 1 is
"sharded" (reduce-scatter -> Adam on 1/N -> all-gather).

`value`  : steps/s x (views per step / views per step at N=1) for weak scaling, i.e. view-steps/s
           over all ranks; steps/s of the fixed batch for strong scaling.  Inputs (targets)
           resident in HBM.
`e2e`    : the same through the public C-ABI (ts_train_step, or forward/loss/backward + the
           exchange for batches) with every step's targets copied from pinned host memory and
           the loss read back; warmed up, then timed in 5 chunks (spread reported).
`roofline`: dominant kernel of the step, algorithmic bytes per launch / its
           CUDA-event duration measured over the timed region.
`compute`: blend kernels' fragment evaluations/s and issue-slot fraction (ncu instruction
           counts in profiles/inst.json over the live duration and SM clock).
`cpu_baseline`: the C++ CPU oracle (oracle/, a port of SPEC.md) timed on this host's cores on
           one full step of the same workload (rank 0, N=1).
--impl reference: the CPU oracle alone, a bounded number of steps on the host cores.
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
    """SM clock and clock-event reasons sampled DURING the timed region.

    An NVML thread (5 ms period) that is confirmed sampling before start() returns, so even a
    short timed region (tens of ms) carries samples; nvidia-smi -lms is the fallback."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = None
        self.thread = None
        self.rows = []
        self.stop_flag = None

    def _nvml_handle(self):
        import pynvml
        import torch
        pynvml.nvmlInit()
        try:
            p = torch.cuda.get_device_properties(self.gpu)
            bus = "%08X:%02X:%02X.0" % (p.pci_domain_id, p.pci_bus_id, p.pci_device_id)
            return pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml.nvmlDeviceGetHandleByIndex(self.gpu)

    def start(self):
        import threading
        try:
            import pynvml
            h = self._nvml_handle()
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.stop_flag = threading.Event()
            first = threading.Event()

            def run():
                while True:
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.rows.append((float(sm), float(mx), int(rs)))
                    except Exception:
                        pass
                    first.set()
                    if self.stop_flag.wait(0.005):
                        return

            self.thread = threading.Thread(target=run, daemon=True)
            self.thread.start()
            first.wait(2.0)
            return
        except Exception:
            self.thread = None
        fd, self.path = tempfile.mkstemp(prefix="clk", suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            t0 = time.time()  # wait for the first sample line so the timed region is covered
            while time.time() - t0 < 5 and os.path.getsize(self.path) == 0:
                time.sleep(0.01)
        except Exception:
            self.proc = None

    def stop(self):
        if self.thread is not None:
            self.stop_flag.set()
            self.thread.join(timeout=2)
            rows = self.rows
        elif self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock sampler (nvml / nvidia-smi)"], "samples": 0}
        else:
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


REF_VIEW_STEPS = 10  # cap of the reference (CPU) arm's timed views (~3 s each at workload H)
N_VIEWS = scene.RING_VIEWS  # training cameras cycled per step, as a 3DGS trainer walks its view set


def view_camera(w, j):
    """Camera j of the benchmark's view ring (scene.ring_camera)."""
    return scene.ring_camera(w, j, N_VIEWS)


def batch_of(w, world):
    """(views per step, scaling): c4 is a fixed 8-view batch split over the GPUs (strong); every
    other workload trains one view per GPU per step (weak)."""
    if w.views > 1:
        if w.views % world:
            raise SystemExit(f"workload {w.name}: {w.views} views per step do not split over {world} GPUs")
        return w.views, "strong"
    return world, "weak"


def step_views(step, batch, world, rank):
    """Ring views of this rank at training step `step` (1-based): the step's batch is the global
    view indices [step*batch, step*batch + batch); rank r takes every world-th one."""
    return [(step * batch + k) % N_VIEWS for k in range(rank, batch, world)]


def bench_config(w, args, world, batch, scaling):
    """The config dict of BOTH arms (identical keys and values for the same workload)."""
    return {"workload": w.name, "gaussians": w.n, "sh_degree": w.sh_degree,
            "resolution": f"{w.width}x{w.height}", "views_per_step": batch if scaling == "strong" else 1,
            "batch_scaling": scaling,
            "views": f"{N_VIEWS}-camera ring (headline view rotated about the scene axis)",
            "optimizer": "fused_backward (SPEC.md:492-500)" if args.adam_mode == "fused_backward"
            else "fused (SPEC.md:473-480)",
            "precision": "fp32",
            "l2": "no flush: per-step working set ~9 GB >> 126 MB L2",
            "gaussian_order": "random" if args.no_morton else
            "morton (SPEC.md:264-272 morton_reorder applied at setup, as the training schedule does)"}


def cpu_step_baseline(w, p0, cams, cfg, targets, views_per_step=1, steps=1, warmup=0):
    """The C++ oracle (port of SPEC.md) on all host cores: full training steps of `views_per_step`
    views each (render, loss, backward summed over the views, then Adam), views cycling over cams."""
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
    k = 0
    for i in range(warmup + steps):
        adam = T.AdamConfig.make(step=i + 1)
        t0 = time.perf_counter()
        if views_per_step == 1:
            _, st = O.train_step(params, m, v, n, cams[k % len(cams)], cfg, targets[k % len(cams)], adam, acc, vc)
            k += 1
        else:
            G = np.zeros_like(params)
            st = None
            for _ in range(views_per_step):
                j = k % len(cams)
                k += 1
                rgb, _, _, _ = O.render(params, n, cams[j], cfg)
                _, dl = O.training_loss(rgb, targets[j])
                g, _, a_, c_ = O.backward(params, n, cams[j], cfg, dl)
                G += g
                acc += a_
                vc += c_
            O.adam_step(params, G, m, v, n, list(adam.lr), adam.beta1, adam.beta2, adam.eps, adam.bc1, adam.bc2,
                        mode=T.ADAM_FUSED)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
            stages = st
    t = float(np.mean(times))
    return {"value": 1.0 / t, "unit": "steps/s", "cores": cores, "kind": "port",
            "sample": f"{steps} full training step(s) of workload {w.name} ({n} Gaussians, SH{w.sh_degree}, "
                      f"{w.width}x{w.height}, {views_per_step} view(s) per step): render+loss+backward+Adam",
            "s_per_step": t,
            "stage_s": dict(zip(("preprocess", "binning", "blend", "loss", "raster_bwd", "project_bwd", "adam"),
                                [round(float(x), 4) for x in stages[:7]])) if stages is not None else None}


def run_reference(args):
    world, rank, local = dist_env()
    if rank != 0:
        return 0
    w = scene.WORKLOADS[args.workload]
    from oracle import oracle as O
    batch, scaling = batch_of(w, world)
    vps = batch if scaling == "strong" else 1
    gt = scene.random_params(w.n, w.s0, w.m_o, w.seed)
    # bounded sample: at most REF_VIEW_STEPS timed views (+1 warm-up step) so the arm ends in minutes
    steps = max(1, min(args.steps, REF_VIEW_STEPS // vps))
    warmup = min(args.warmup, 1)
    cams = [view_camera(w, j) for j in range(min(N_VIEWS, (warmup + steps) * vps))]
    cfg = T.RenderConfig.make(sh_degree=w.sh_degree)
    O.set_workers(os.cpu_count() or 1)
    targets = [O.render(gt, w.n, c, cfg)[0] for c in cams]
    p0 = scene.perturb(gt, w.n, w.seed)
    del gt
    if not args.no_morton:  # same Gaussian order as the GPU arm
        O.morton_reorder(p0, w.n)
    cb = cpu_step_baseline(w, p0, cams, cfg, targets, views_per_step=vps, steps=steps, warmup=warmup)
    # the same unit as our arm: view-steps/s for the weak (one view per GPU) workloads, steps/s of
    # the fixed batch for c4; the CPU arm is one host, so it is compared at its own batch
    val = cb["value"]
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "steps/s", "n_gpus": world,
            "steps": steps, "warmup": warmup, "steps_requested": args.steps, "ms_per_step": 1e3 / val,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded random Gaussians; target self-rendered from the GT store; trained store = "
                    "perturbed GT)",
            "config": bench_config(w, args, 1, vps if scaling == "strong" else 1, scaling),
            "parallelism": f"{cb['cores']} host threads (std::thread pool)",
            "cpu_baseline": {"value": val, "unit": "steps/s", "cores": cb["cores"], "kind": "port",
                             "sample": cb["sample"]},
            "e2e": {"value": val, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "stage_s": cb["stage_s"]}
    print(json.dumps(line), flush=True)
    return 0


def compute_roofline(avg_ms, vstats, clocks, n_tiles, workload):
    """Blend kernels (K6 / K8): fragment evaluations per second (256 pixels x processed list
    positions Ip per pass) and the issue-slot fraction = warp instructions per launch (ncu,
    profiles/inst.json, same workload) / (duration x 148 SMs x 4 schedulers x SM clock)."""
    inst = {}
    f = os.path.join(ROOT, "profiles", "inst.json")
    if os.path.exists(f):
        try:
            with open(f) as fh:
                inst = json.load(fh).get(workload, {})
        except Exception:
            inst = {}
    ceil = {}
    fc = os.path.join(ROOT, "profiles", "issue_ceiling.json")
    if os.path.exists(fc):
        try:
            with open(fc) as fh:
                ceil = json.load(fh).get("dense_inst_per_sm_cycle", {})
        except Exception:
            ceil = {}
    mhz = clocks.get("sm_mhz") or 1965.0
    out = {"fragment_evals_per_pass": 256 * vstats["Ip"], "sm_mhz": mhz,
           "issue_peak_winst_per_s": 148 * 4 * mhz * 1e6}
    for k in ("blend", "blend_bwd", "preprocess", "loss", "project_bwd"):
        if k not in avg_ms or avg_ms[k] <= 0:
            continue
        t = avg_ms[k] * 1e-3
        row = {"ms": round(avg_ms[k], 4)}
        if k in ("blend", "blend_bwd"):
            row["fragment_evals_per_s"] = 256 * vstats["Ip"] / t
        wi = inst.get(k)
        if wi:
            row["warp_inst_per_launch"] = wi
            row["issue_frac"] = wi / (t * out["issue_peak_winst_per_s"])
            # fraction of the kernel's measured issue ceiling: live warp instructions per SM cycle
            # over the rate the same kernel sustains on the dense scene (profiles/issue_ceiling.json)
            dense = ceil.get(k)
            if dense:
                row["inst_per_sm_cycle"] = wi / (t * 148 * mhz * 1e6)
                row["issue_ceiling_inst_per_sm_cycle"] = dense
                row["frac_of_issue_ceiling"] = row["inst_per_sm_cycle"] / dense
        out[k] = row
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2602_09999_b200.dp import DataParallelStep
    from paper_2602_09999_b200.tilesplat import Engine, PinnedBuffer

    world, rank, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    # one explicit stream for the engine, torch's collectives and the timing events (the legacy
    # default stream would not order against the engine's work: handle 0 = "own stream")
    stream = torch.cuda.Stream(device=local)
    torch.cuda.set_stream(stream)
    w = scene.WORKLOADS[args.workload]
    n = w.n
    batch, scaling = batch_of(w, world)
    gt = scene.random_params(n, w.s0, w.m_o, w.seed)
    cams = [view_camera(w, j) for j in range(N_VIEWS)]
    cfg = T.RenderConfig.make(sh_degree=w.sh_degree)
    e = Engine(local, stream=stream.cuda_stream)
    e.set_params(gt, n)
    mine = sorted({j for s_ in range(N_VIEWS) for j in step_views(s_, batch, world, rank)})
    targets = {}
    for j in mine:   # every view this rank trains: target rendered from the GT store, kept in a device slot
        t, _, _ = e.render(cams[j], cfg)
        e.set_target(j, t)
        targets[j] = t
    p0 = scene.perturb(gt, n, w.seed)
    del gt
    e.set_params(p0, n)
    if not args.no_morton:
        # steady-state training order: morton_reorder fires every 5000
        # iterations while densifying, so a 3M-Gaussian store is in z-order; rendering is
        # order-invariant (bitwise), the arrays just gain spatial locality
        perm = e.morton_reorder()
        p0 = scene.reorder_params(p0, n, perm)
    e.set_graph(args.graph)   # CUDA-graph mode of the single-call step (ts_set_graph)
    dp_mode = args.dp_mode or ("sharded" if world > 1 else "allreduce")
    dp = DataParallelStep(e, mode=dp_mode)
    step = 0
    fused_bwd = args.adam_mode == "fused_backward"
    if args.densify and world > 1:
        raise SystemExit("--densify runs on one GPU (the multi-GPU path needs the statistics all-reduce)")
    if fused_bwd and (world > 1 or len(step_views(1, batch, world, rank)) > 1):
        raise SystemExit("fused_backward needs the full single-view gradient on one rank")
    mode = T.ADAM_FUSED_BACKWARD if fused_bwd else T.ADAM_FUSED
    single_call = world == 1 and batch == 1

    def adam_cfg(m=None):
        # the gradient buffer is consumed by this step's optimizer; the next backward
        # overwrites every row (no clear pass)
        return T.AdamConfig.make(step=step, extent=1.0, mode=mode if m is None else m, zero_grads=0)

    densify_log = []

    def train_step():
        vs = step_views(step, batch, world, rank)
        if single_call:  # one public C-ABI call: forward, loss, backward, Adam (target slot on the device)
            e.train_step(cams[vs[0]], cfg, adam_cfg(), slot=vs[0], want_loss=False)
        else:
            dp.step([(cams[j], cfg, j) for j in vs], adam_cfg())
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
    if world > 1:
        dist.barrier()

    # graph mode captures a view's step the second time it is seen (and toggling the stage
    # profiling drops the graphs): two rounds of the view ring right before the timed region, so
    # that no capture lands in it
    if args.graph:
        for _ in range(2 * N_VIEWS + 1):
            step += 1
            train_step()
        args.warmup += 2 * N_VIEWS + 1
        torch.cuda.synchronize()

    # ---- timed region (device-resident targets) ----
    clk = ClockSampler(local)
    clk.start()
    gs0 = e.graph_stats()
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
    e.synchronize()  # settles the graph steps (replays a voided one) after the timed region
    gs1 = e.graph_stats()
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
            dp.step([(cams[j], cfg, j) for j in step_views(step, batch, world, rank)], adam_cfg(T.ADAM_FUSED))
        torch.cuda.synchronize()
        split_times = e.stage_times()
        e.set_profiling(False)

    # ---- e2e: public C-ABI calls with host (pinned) targets and the loss read back each step ----
    P = w.width * w.height
    pins = {}
    for j in mine:
        pb = PinnedBuffer((w.height, w.width, 3))
        pb.array[...] = targets[j]
        pins[j] = pb
    # this box's pinned host -> device bandwidth for one target (the e2e leg's per-step copy)
    scratch = torch.empty(P * 3, dtype=torch.float32, device=f"cuda:{local}")
    src = torch.from_numpy(pins[mine[0]].array.reshape(-1))  # pinned (ts_host_alloc)
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    c0.record(stream)
    for _ in range(5):
        scratch.copy_(src, non_blocking=True)
    c1.record(stream)
    torch.cuda.synchronize()
    h2d_ms = c0.elapsed_time(c1) / 5
    del scratch

    def e2e_step():
        vs = step_views(step, batch, world, rank)
        if single_call:
            e.train_step(cams[vs[0]], cfg, adam_cfg(), target_ptr=pins[vs[0]].ptr, want_loss=True)
            return
        for i, j in enumerate(vs):
            e.render(cams[j], cfg, outputs=False)
            e.training_loss(target=pins[j].array, want_value=(i == len(vs) - 1))
            e.backward(None)
        dp.exchange_and_step(adam_cfg())

    for _ in range(3):            # warm-up: copy stream, staging buffers, pinned loss slot
        step += 1
        e2e_step()
    torch.cuda.synchronize()
    chunks = 5
    per_chunk = max(2, args.steps // chunks)
    chunk_ms = []
    for _ in range(chunks):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(per_chunk):
            step += 1
            e2e_step()
        torch.cuda.synchronize()
        chunk_ms.append((time.perf_counter() - t0) * 1e3 / per_chunk)
    e2e_ms = float(np.mean(chunk_ms))
    if world > 1:
        t = torch.tensor([e2e_ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    for pb in pins.values():
        pb.free()

    # ---- SPEC binning counters: instances per bounding / culling mode and the
    # radix key-bytes metrics of the combined 48-bit vs two-stage sort (PAPER §B.2), view 0 ----
    bcnt = {}
    for name_, bm, cm in (("square", 0, 0), ("rect", 1, 0), ("rect_opacity", 2, 0), ("exact", 2, 1)):
        c_ = T.RenderConfig.make(sh_degree=w.sh_degree, bound_mode=bm, cull_mode=cm)
        e.render(cams[0], c_, outputs=False)
        bcnt["instances_" + name_] = e.view_stats()["I"]
    e.render(cams[0], cfg, outputs=False)
    vs0 = e.view_stats()
    key32 = cams[0].n_tiles >= 65536
    bcnt["sort_key_bytes_combined"] = 6 * vs0["I"]                                  # 48-bit keys over I
    bcnt["sort_key_bytes_two_stage"] = 4 * vs0["V"] + (4 if key32 else 2) * vs0["I"]  # depth over V + tile over I
    bcnt["two_stage_over_combined"] = round(bcnt["sort_key_bytes_two_stage"] / max(1, bcnt["sort_key_bytes_combined"]), 4)

    # ---- per-stage accounting over the profiled loop ----
    bytes_ = stage_bytes(vstats, n, w.sh_degree, cams[0].n_tiles)
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
    # dominant kernel: largest device time per STEP (a batch step runs the raster stages once per view)
    per_step = {k: avg[k] * calls[k] for k in avg}
    dom = max(per_step, key=lambda k: per_step[k])
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
        vps = batch if scaling == "strong" else 1
        cpu = cpu_step_baseline(w, p0, cams[:vps], cfg, [targets[j] for j in range(vps)], views_per_step=vps,
                                steps=1, warmup=0)

    if rank == 0:
        # weak: every rank trains one view per step -> view-steps/s over the job; strong: steps/s
        value = (world if scaling == "weak" else 1) / (ms * 1e-3)
        e2e_value = (world if scaling == "weak" else 1) / (e2e_ms * 1e-3)
        vpr = len(step_views(1, batch, world, rank))
        spread = [round((world if scaling == "weak" else 1) / (x * 1e-3), 2) for x in chunk_ms]
        line = {
            "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded random Gaussians; target self-rendered from the GT store; trained store = "
                    "perturbed GT)",
            "config": bench_config(w, args, world, batch, scaling),
            "parallelism": f"dp{world} (views; NCCL {dp_mode} of the 59N fp32 gradient buffer)" if world > 1
            else "1 GPU",
            "views_per_gpu_per_step": vpr,
            "e2e": {"value": e2e_value, "unit": "steps/s",
                    "h2d_bytes_per_step": int(vpr * (P * 3 * 4) + 104 + 64),
                    "d2h_bytes_per_step": 16,
                    "api": "ts_train_step (C-ABI) with pinned host target" if single_call
                    else "ts_forward + ts_loss(pinned host target) + ts_backward per view, exchange, ts_adam_step",
                    "chunks_steps_s": spread, "warmup_steps": 3, "timed_steps": chunks * per_chunk,
                    "h2d_ms_per_target": round(h2d_ms, 4),
                    "h2d_gbs": round(P * 3 * 4 / (h2d_ms * 1e-3) / 1e9, 2)},
            "stage_ms_split": {k: round(v, 4) for k, v in split.items()} if fused_bwd else None,
            "gpu_launches": int(launches),
            "graph": bool(args.graph and single_call),
            "graph_timed": {k: gs1[k] - gs0[k] for k in ("launches", "captures", "replays")},
            "graph_stats": e.graph_stats(),
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "algorithmic_bytes_per_launch": int(dom_bytes), "avg_launch_ms": dom_ms,
                         "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                         "note": ("the peak is a 1:1 read:write copy test; this kernel's mix (Adam: 4 reads : 3 "
                                  "writes) streams faster than it, hence frac > 1" if achieved > peak else None)},
            "fwd_bwd": {"ms": fwd_bwd_ms,
                        "source": "profiled loop (stage CUDA events; separate-optimizer steps)" if fused_bwd
                        else "profiled loop (stage CUDA events)", "mpix_s": P / (fwd_bwd_ms * 1e-3) / 1e6,
                        "algorithmic_bytes": int(R), "achieved_gbs": R / (fwd_bwd_ms * 1e-3) / 1e9,
                        "roofline_frac": R / (fwd_bwd_ms * 1e-3) / 1e9 / peak},
            "compute": compute_roofline(avg, vstats, clocks, cams[0].n_tiles, w.name),
            "binning_counters": bcnt,
            "stage_ms": {k: round(v, 4) for k, v in avg.items()},
            "densify": [{"step": d[0], "n_after": d[1], "clones": d[2][0], "splits": d[2][1], "pruned": d[2][2]}
                        for d in densify_log] if args.densify else None,
            "stage_calls": calls,
            "view": vstats,
            "clocks": {k: clocks[k] for k in ("sm_mhz", "sm_max_mhz", "reasons", "samples")},
        }
        if cpu is not None:
            line["cpu_baseline"] = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
            line["cpu_baseline"]["stage_s"] = cpu["stage_s"]
        print(json.dumps(line), flush=True)
    e.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def selftest_launcher(args):
    """The multi-rank plumbing without GPU work (CPU test): gloo rendezvous over 127.0.0.1,
    one all-reduce and a max-over-ranks timing reduction, rank 0 prints the JSON line."""
    import torch
    import torch.distributed as dist
    world, rank, _ = dist_env()
    dist.init_process_group("gloo")
    x = torch.ones(4) * (rank + 1)
    dist.all_reduce(x)
    t = torch.tensor([float(rank)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    w = scene.WORKLOADS[args.workload]
    batch, scaling = batch_of(w, world)
    if rank == 0:
        print(json.dumps({"selftest": "launcher", "n_gpus": world, "backend": dist.get_backend(),
                          "allreduce_sum": float(x[0]), "max_rank": float(t[0]), "scaling": scaling,
                          "views_per_step": batch if scaling == "strong" else 1,
                          "views_of_rank0_step1": step_views(1, batch, world, 0)}), flush=True)
    dist.destroy_process_group()
    return 0


def self_launch(args):
    """--gpus N > 1 outside torchrun: re-run this script under torch.distributed.run, one rank per GPU."""
    import socket
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--workload", default="H", choices=sorted(scene.WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--dp-mode", default=None, choices=("allreduce", "sharded", "chunked"),
                    help="gradient exchange for N > 1 (default sharded)")
    ap.add_argument("--adam-mode", default="auto", choices=("auto", "fused", "fused_backward"),
                    help="optimizer mode (SPEC.md:525): fused = separate fused-Adam sweep (SPEC.md:473-480); "
                         "fused_backward = Adam inside the backward (SPEC.md:492-500, 1 GPU only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--densify", action="store_true",
                    help="densify_and_prune every 100 iterations inside the timed region (config 3, N=1)")
    ap.add_argument("--no-morton", action="store_true",
                    help="keep the generator's random Gaussian order instead of the z-order training state")
    ap.add_argument("--graph", dest="graph", action="store_true", default=False,
                    help="CUDA-graph mode of the one-call training step (ts_set_graph)")
    ap.add_argument("--no-graph", dest="graph", action="store_false")
    ap.add_argument("--selftest-launcher", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if args.gpus > 1 and world == 0:
        return self_launch(args)
    if world and world != args.gpus and not args.selftest_launcher:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.selftest_launcher:
        return selftest_launcher(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
