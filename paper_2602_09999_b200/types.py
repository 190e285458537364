"""C-ABI value types shared by the Python host mirror (ctypes layouts of
include/tilesplat_c.h) and the SPEC-level constants.

The field layout mirrors the reference's Camera, the render
feature flags of TrainConfig and the Adam
hyper-parameters / LR schedule.
"""
from __future__ import annotations

import ctypes
import math

import numpy as np

NPARAM = 59          # floats per Gaussian
TILE = 16            # TileGrid tile size

# attribute blocks inside the flat 59*N parameter / gradient / moment buffers
GROUPS = ("means", "log_scales", "quats", "opacity_logits", "sh_dc", "sh_rest")
GROUP_WIDTH = (3, 3, 4, 1, 3, 45)

BOUND_SQUARE, BOUND_RECT, BOUND_RECT_OPACITY = 0, 1, 2
CULL_NONE, CULL_EXACT = 0, 1
BACKWARD_PER_PIXEL, BACKWARD_PER_GAUSSIAN = 0, 1
TRUNC_CLASSIC, TRUNC_RESPONSE = 0, 1  # fragment_alpha modes
ADAM_REFERENCE, ADAM_FUSED, ADAM_SKIP_INVISIBLE, ADAM_FUSED_BACKWARD, ADAM_FUSED_BACKWARD_SKIP = 0, 1, 2, 3, 4
AA_OFF, AA_FILTER3D_ORIGINAL, AA_FILTER3D_CLIP, AA_FULL = 0, 1, 2, 3
AA_MODES = {"off": AA_OFF, "filter3d_original": AA_FILTER3D_ORIGINAL, "filter3d_clip": AA_FILTER3D_CLIP,
            "full": AA_FULL}


class Camera(ctypes.Structure):
    """ts_camera: world->camera row-major 4x4 W, intrinsics, image size."""

    _fields_ = [
        ("W", ctypes.c_float * 16),
        ("fx", ctypes.c_float), ("fy", ctypes.c_float),
        ("cx", ctypes.c_float), ("cy", ctypes.c_float),
        ("near", ctypes.c_float),
        ("width", ctypes.c_int32), ("height", ctypes.c_int32),
    ]

    @classmethod
    def make(cls, W, fx, fy, cx, cy, width, height, near=0.2) -> "Camera":
        c = cls()
        Wf = np.asarray(W, dtype=np.float32).reshape(16)
        for i in range(16):
            c.W[i] = float(Wf[i])
        c.fx, c.fy, c.cx, c.cy, c.near = fx, fy, cx, cy, near
        c.width, c.height = int(width), int(height)
        return c

    @property
    def tiles_x(self) -> int:
        return (self.width + TILE - 1) // TILE

    @property
    def tiles_y(self) -> int:
        return (self.height + TILE - 1) // TILE

    @property
    def n_tiles(self) -> int:
        return self.tiles_x * self.tiles_y

    @property
    def n_pixels(self) -> int:
        return self.width * self.height

    def center(self) -> np.ndarray:
        W = np.array(self.W[:], dtype=np.float64).reshape(4, 4)
        return -W[:3, :3].T @ W[:3, 3]


class RenderConfig(ctypes.Structure):
    """ts_render_config: per-view feature flags."""

    _fields_ = [
        ("sh_degree", ctypes.c_int32),
        ("bound_mode", ctypes.c_int32),
        ("cull_mode", ctypes.c_int32),
        ("truncation", ctypes.c_int32),
        ("early_stop_compat", ctypes.c_int32),
        ("backward_mode", ctypes.c_int32),
        ("tau_alpha", ctypes.c_float),
        ("dilation", ctypes.c_float),
        ("sigma_cut", ctypes.c_float),
        ("bg", ctypes.c_float * 3),
        ("aa_mode", ctypes.c_int32),
        ("kappa3d", ctypes.c_float),
    ]

    @classmethod
    def make(cls, sh_degree=3, bound_mode=BOUND_RECT_OPACITY, cull_mode=CULL_EXACT, early_stop_compat=0,
             backward_mode=BACKWARD_PER_PIXEL, tau_alpha=1.0 / 255.0, dilation=None, sigma_cut=3.33,
             bg=(0.0, 0.0, 0.0), aa="off", kappa3d=0.2, truncation=TRUNC_CLASSIC) -> "RenderConfig":
        """aa: off | filter3d_original | filter3d_clip | full; the 2D dilation defaults to
        0.3 (classic) unless aa == "full", which uses the Mip filter variance 0.1 with compensation."""
        c = cls()
        c.aa_mode = AA_MODES[aa] if isinstance(aa, str) else int(aa)
        c.kappa3d = kappa3d
        if dilation is None:
            dilation = 0.1 if c.aa_mode == AA_FULL else 0.3
        c.sh_degree, c.bound_mode, c.cull_mode = sh_degree, bound_mode, cull_mode
        c.truncation, c.early_stop_compat, c.backward_mode = truncation, early_stop_compat, backward_mode
        c.tau_alpha, c.dilation, c.sigma_cut = tau_alpha, dilation, sigma_cut
        for i in range(3):
            c.bg[i] = bg[i]
        return c


class AdamConfig(ctypes.Structure):
    """ts_adam_config: per-group lr, betas, eps, host bias corrections, mode."""

    _fields_ = [
        ("lr", ctypes.c_float * 6),
        ("beta1", ctypes.c_float), ("beta2", ctypes.c_float), ("eps", ctypes.c_float),
        ("bc1", ctypes.c_float), ("bc2", ctypes.c_float),
        ("mode", ctypes.c_int32),
        ("zero_grads", ctypes.c_int32),
    ]

    @classmethod
    def make(cls, step: int, extent: float = 1.0, mode: int = ADAM_FUSED, zero_grads: int = 1,
             beta1=0.9, beta2=0.999, eps=1e-15, lrs=None) -> "AdamConfig":
        """step is 1-based (bias corrections 1-b^t computed in double on the host, App. A.9)."""
        c = cls()
        if lrs is None:
            lrs = default_lrs(step - 1, extent)
        for i in range(6):
            c.lr[i] = lrs[i]
        c.beta1, c.beta2, c.eps = beta1, beta2, eps
        c.bc1 = 1.0 - math.pow(beta1, step)
        c.bc2 = 1.0 - math.pow(beta2, step)
        c.mode, c.zero_grads = mode, zero_grads
        return c


def mean_lr(step: int, extent: float) -> float:
    """extent * 1.6e-4 * (1e-2)^(step/30000)."""
    return extent * 1.6e-4 * math.pow(1e-2, step / 30000.0)


def default_lrs(step: int, extent: float):
    """LRSchedule: means, scales, rotations, opacity, sh_dc, sh_rest."""
    return (mean_lr(step, extent), 0.005, 0.001, 0.025, 2.5e-3, 1.25e-4)


def sh_active_degree(it: int) -> int:
    """SPEC.md:575-580."""
    return min(3, it // 1000)


def group_slices(n: int):
    """(start, stop) of each attribute block inside a flat 59*N buffer."""
    out, o = [], 0
    for w in GROUP_WIDTH:
        out.append((o, o + w * n))
        o += w * n
    return out


def pack_params(means, log_scales, quats, opacity_logits, sh_dc, sh_rest) -> np.ndarray:
    arrs = [np.ascontiguousarray(a, dtype=np.float32).reshape(-1)
            for a in (means, log_scales, quats, opacity_logits, sh_dc, sh_rest)]
    return np.concatenate(arrs)


def unpack_params(flat: np.ndarray, n: int):
    sl = group_slices(n)
    shapes = ((n, 3), (n, 3), (n, 4), (n,), (n, 3), (n, 15, 3))
    return tuple(flat[a:b].reshape(s) for (a, b), s in zip(sl, shapes))
