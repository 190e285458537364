"""The train op over the hot path: seeded shuffle-per-epoch
view sampling, render -> loss -> backward -> optimizer step,
then the scheduled densify / opacity reset / Morton / SH-ramp events
(config.events) and a checkpoint every `checkpoint_interval` iterations
(SPEC.md:832, :855).  With antialiasing on the sampling rates
are recomputed every `rate_interval` iterations and after every densification
(new rows), and the clip modes (filter3d_clip, full) apply the 3D-filter clip
after each optimizer step.  Resuming from a checkpoint continues the same schedule
and view order, because both are pure functions of (seed, iteration).

`engine` is the C-ABI Engine (tilesplat.Engine); the tests also drive this
loop with an oracle-backed stand-in to check resume determinism bitwise."""
from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

from . import checkpoint as ckpt
from . import types as T
from .config import TrainConfig, events


@dataclass
class TrainLog:
    losses: list = field(default_factory=list)
    densify: list = field(default_factory=list)   # (iteration, clones, splits, pruned, N_after)
    mortons: list = field(default_factory=list)
    resets: list = field(default_factory=list)
    checkpoints: list = field(default_factory=list)


class Trainer:
    def __init__(self, engine, cameras, targets, cfg: TrainConfig, extent: float | None = None,
                 render_cfg: T.RenderConfig | None = None):
        self.e = engine
        self.cams = list(cameras)
        self.cfg = cfg.validate()
        if extent is None:
            from .scene import scene_extent
            extent = scene_extent(self.cams)
        self.extent = float(extent)
        self.rcfg = render_cfg or T.RenderConfig.make(
            bound_mode=cfg.bound_mode, cull_mode=cfg.cull_mode, aa=cfg.aa_mode, kappa3d=cfg.kappa3d,
            backward_mode=cfg.backward_mode, sigma_cut=cfg.sigma_cut,
            truncation=T.TRUNC_RESPONSE if cfg.truncation == "response" else T.TRUNC_CLASSIC)
        self.aa = T.AA_MODES[cfg.aa_mode]
        self._rates_stale = True
        self.n_views = len(self.cams)
        self._slots = hasattr(engine, "set_target")
        self.targets = targets
        if self._slots:  # targets resident on the device, one slot per view
            for k, t in enumerate(targets):
                engine.set_target(k, t)
        self.log = TrainLog()

    # ---- view sampling: shuffle per epoch, seeded by (seed, epoch) ----
    def _epoch_order(self, epoch: int) -> np.ndarray:
        return np.random.default_rng([self.cfg.seed, epoch]).permutation(self.n_views)

    def views_for(self, it: int):
        """Views of 1-based iteration it (batch_size consecutive draws of the epoch stream)."""
        b = self.cfg.batch_size
        out = []
        for j in range((it - 1) * b, it * b):
            epoch, k = divmod(j, self.n_views)
            out.append(int(self._epoch_order(epoch)[k]))
        return out

    def adam(self, it: int, zero_grads: int = 1) -> T.AdamConfig:
        return T.AdamConfig.make(it, self.extent, mode=self.cfg.optimizer_mode, zero_grads=zero_grads)

    def step(self, it: int) -> float:
        ev = events(it, self.cfg)
        rc = self.rcfg
        rc.sh_degree = ev.sh_degree
        views = self.views_for(it)
        if self.aa != T.AA_OFF and (self._rates_stale or (it - 1) % self.cfg.rate_interval == 0):
            self.e.compute_sampling_rates(self.cams, self.extent)
            self._rates_stale = False
        if len(views) == 1 and hasattr(self.e, "train_step"):
            v = views[0]
            loss = (self.e.train_step(self.cams[v], rc, self.adam(it), slot=v) if self._slots
                    else self.e.train_step(self.cams[v], rc, self.adam(it), target=self.targets[v]))
        else:  # batch: gradients summed over views, one optimizer step
            loss = 0.0
            for v in views:
                self.e.render(self.cams[v], rc, outputs=False)
                loss += (self.e.training_loss(slot=v) if self._slots else self.e.training_loss(self.targets[v]))
                self.e.backward()
            self.e.adam_step(self.adam(it))
        self.log.losses.append(loss)
        if self.aa in (T.AA_FILTER3D_CLIP, T.AA_FULL):  # post-step projection
            self.e.apply_3d_filter_clip(self.cfg.kappa3d)
        if ev.densify:
            s = self.cfg.densify
            n, (c, sp, pr) = self.e.densify_and_prune(s.grad_threshold, self.extent, self.cfg.seed, it)
            self.log.densify.append((it, c, sp, pr, n))
            self._rates_stale = True  # new rows have no sampling rate yet
        if ev.opacity_reset:
            self.e.opacity_reset()
            self.log.resets.append(it)
        if ev.morton:
            self.e.morton_reorder()
            self.log.mortons.append(it)
        if ev.checkpoint and self.cfg.output_dir:
            self.save(it)
        return loss

    def run(self, start: int = 1, stop: int | None = None) -> TrainLog:
        stop = self.cfg.total_iterations if stop is None else stop
        for it in range(start, stop + 1):
            self.step(it)
        return self.log

    # ---- checkpoint / resume ----
    def checkpoint_dir(self, it: int) -> str:
        return os.path.join(self.cfg.output_dir, f"iteration_{it}")

    def save(self, it: int) -> str:
        d = self.checkpoint_dir(it)
        ckpt.save_engine(d, self.e, it, self.cfg)
        self.log.checkpoints.append(it)
        return d

    def resume(self, directory: str) -> int:
        """Load a checkpoint; returns the next iteration to run."""
        ck = ckpt.load_engine(directory, self.e)
        return int(ck["step"]) + 1
