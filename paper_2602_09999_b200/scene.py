"""synth_scene and the benchmark workloads.

Seeded random well-conditioned Gaussians in the unit box, cameras on a sphere
looking inward (OpenCV axes: x right, y down, z forward).  Arrays are generated
once on the host (numpy PCG64, bitwise-reproducible for a fixed seed) and
uploaded; the GPU never runs an RNG for scene content.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import types as T
from .types import Camera, pack_params


@dataclass(frozen=True)
class Workload:
    name: str
    n: int
    sh_degree: int
    width: int
    height: int
    s0: float
    m_o: float
    seed: int
    views: int = 1


# SURVEY §8(d) table; "H" is the headline metric point (3M, SH3, 1080p).
WORKLOADS = {
    "c1": Workload("c1", 10_000, 0, 256, 256, 0.02, 0.0, 1),
    "c2": Workload("c2", 1_000_000, 3, 1920, 1080, 0.012, 0.0, 2),
    "H": Workload("H", 3_000_000, 3, 1920, 1080, 0.008, 0.0, 3),
    "c3": Workload("c3", 3_000_000, 3, 1297, 840, 0.008, 0.0, 4),
    "c4": Workload("c4", 6_000_000, 3, 1920, 1080, 0.0065, 0.0, 5, views=8),
    "c5": Workload("c5", 2_500_000, 3, 1332, 876, 0.018, -2.0, 6),
}


def random_params(n: int, s0: float, m_o: float, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    means = rng.uniform(-1.0, 1.0, (n, 3))
    log_scales = math.log(s0) + rng.normal(0.0, 0.3, (n, 3))
    quats = rng.normal(0.0, 1.0, (n, 4))
    logits = rng.normal(m_o, 1.0, n)
    sh_dc = rng.uniform(-1.5, 1.5, (n, 3))
    sh_rest = rng.normal(0.0, 0.05, (n, 15, 3))
    return pack_params(means, log_scales, quats, logits, sh_dc, sh_rest)


def reorder_params(params: np.ndarray, n: int, perm: np.ndarray) -> np.ndarray:
    """Rows of every attribute block of a flat 59*n store in the order perm (new row i = old row perm[i])."""
    out = np.empty_like(params)
    for (a, b), wd in zip(T.group_slices(n), T.GROUP_WIDTH):
        out[a:b] = params[a:b].reshape(n, wd)[perm].ravel()
    return out


def perturb(params: np.ndarray, n: int, seed: int) -> np.ndarray:
    """Training start = GT + seeded perturbation (sigma 0.01 means, 0.1 logits/log-scales)."""
    rng = np.random.default_rng(seed + 1000)
    p = params.copy()
    p[0:3 * n] += rng.normal(0.0, 0.01, 3 * n).astype(np.float32)
    p[3 * n:6 * n] += rng.normal(0.0, 0.1, 3 * n).astype(np.float32)
    p[10 * n:11 * n] += rng.normal(0.0, 0.1, n).astype(np.float32)
    return p


def look_at(eye, target=(0.0, 0.0, 0.0)) -> np.ndarray:
    """World->camera 4x4 (OpenCV axes)."""
    eye = np.asarray(eye, dtype=np.float64)
    z = np.asarray(target, dtype=np.float64) - eye
    z /= np.linalg.norm(z)
    down = np.array([0.0, -1.0, 0.0])
    x = np.cross(down, z)
    if np.linalg.norm(x) < 1e-6:
        x = np.cross(np.array([0.0, 0.0, 1.0]), z)
    x /= np.linalg.norm(x)
    y = np.cross(z, x)
    R = np.stack([x, y, z])
    W = np.eye(4)
    W[:3, :3] = R
    W[:3, 3] = -R @ eye
    return W


def make_camera(width: int, height: int, eye=(0.3, -0.8, -3.5), fov_x_deg: float = 60.0,
                near: float = 0.2) -> Camera:
    f = width / (2.0 * math.tan(math.radians(fov_x_deg) / 2.0))
    return Camera.make(look_at(eye), f, f, width / 2.0, height / 2.0, width, height, near)


def fibonacci_cameras(k: int, width: int, height: int, radius: float = 3.5, fov_x_deg: float = 60.0):
    cams = []
    golden = math.pi * (3.0 - math.sqrt(5.0))
    for i in range(k):
        y = 1.0 - 2.0 * (i + 0.5) / k
        r = math.sqrt(max(0.0, 1.0 - y * y))
        th = golden * i
        eye = (radius * r * math.cos(th), radius * y, radius * r * math.sin(th))
        cams.append(make_camera(width, height, eye, fov_x_deg))
    return cams


def workload_cameras(w: Workload):
    if w.views == 1:
        return [make_camera(w.width, w.height)]
    return fibonacci_cameras(w.views, w.width, w.height)


RING_VIEWS = 8  # training cameras of the benchmark's view ring


def ring_camera(w: Workload, j: int, n_views: int = RING_VIEWS) -> Camera:
    """Camera j of the benchmark's view ring: the headline view (j = 0, eye (0.3, -0.8, -3.5))
    rotated by 360/n_views * j degrees about the scene's vertical axis.  Every view sees the
    whole synthetic cube (same per-view workload)."""
    base = np.array([0.3, -0.8, -3.5])
    a = math.radians(360.0 / n_views * j)
    R = np.array([[math.cos(a), 0, math.sin(a)], [0, 1, 0], [-math.sin(a), 0, math.cos(a)]])
    return make_camera(w.width, w.height, tuple(R @ base))


def scene_extent(cams) -> float:
    """1.1 x radius of the camera-centre bounding sphere; 1.0 for one camera."""
    if len(cams) <= 1:
        return 1.0
    c = np.stack([cam.center() for cam in cams])
    m = c.mean(axis=0)
    return 1.1 * float(np.max(np.linalg.norm(c - m, axis=1)))
