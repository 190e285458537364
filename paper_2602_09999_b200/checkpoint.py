"""Training checkpoint = PLY + config + optimizer-state sidecar,
written every 5000 iterations by train.

Directory layout (identical to include/tilesplat/ply.hpp's save_checkpoint):
  point_cloud.ply   parameters, 3DGS vertex layout (ply.py)
  optimizer.bin     "TSOPT001", int64 N, int64 step, m[59N], v[59N], accum[N], vcount[N]  (float32, LE)
  config.json       the TrainConfig (optional; config.py)
"""
from __future__ import annotations

import os

import numpy as np

from . import ply

MAGIC = b"TSOPT001"


def write_optimizer_state(path, n, step, m, v, accum, vcount):
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(np.array([n, step], "<i8").tobytes())
        for a, size in ((m, 59 * n), (v, 59 * n), (accum, n), (vcount, n)):
            a = np.ascontiguousarray(a, "<f4").reshape(-1)
            if a.size != size:
                raise ValueError("optimizer state size mismatch")
            f.write(a.tobytes())


def read_optimizer_state(path, expect_n=None):
    with open(path, "rb") as f:
        if f.read(8) != MAGIC:
            raise ply.PlyError(f"{path}: bad optimizer sidecar")
        n, step = (int(x) for x in np.frombuffer(f.read(16), "<i8"))
        if expect_n is not None and n != expect_n:
            raise ply.PlyError("sidecar N does not match the PLY")
        out = []
        for size in (59 * n, 59 * n, n, n):
            b = f.read(4 * size)
            if len(b) != 4 * size:
                raise ply.PlyError(f"{path}: truncated sidecar")
            out.append(np.frombuffer(b, "<f4").astype(np.float32))
    return n, step, out[0], out[1], out[2], out[3]


def save(directory, params, n, step, m, v, accum, vcount, config=None, binary=True):
    """Host arrays -> checkpoint directory."""
    os.makedirs(directory, exist_ok=True)
    ply.write_ply(os.path.join(directory, "point_cloud.ply"), params, n, binary=binary)
    write_optimizer_state(os.path.join(directory, "optimizer.bin"), n, step, m, v, accum, vcount)
    if config is not None:
        config.save(os.path.join(directory, "config.json"))


def load(directory):
    """-> dict(params, n, step, m, v, accum, vcount, config or None)."""
    params, n = ply.read_ply(os.path.join(directory, "point_cloud.ply"))
    _, step, m, v, accum, vcount = read_optimizer_state(os.path.join(directory, "optimizer.bin"), n)
    cfg = None
    cpath = os.path.join(directory, "config.json")
    if os.path.exists(cpath):
        from .config import TrainConfig
        cfg = TrainConfig.load(cpath)
    return dict(params=params, n=n, step=step, m=m, v=v, accum=accum, vcount=vcount, config=cfg)


def save_engine(directory, engine, step, config=None):
    """Engine (device state) -> checkpoint."""
    params = engine.get_params()
    _, m, v, accum, vcount = engine.get_state()
    save(directory, params, engine.num_gaussians(), step, m, v, accum, vcount, config)


def load_engine(directory, engine):
    """checkpoint -> Engine; returns the loaded dict (step, config...)."""
    ck = load(directory)
    engine.set_params(ck["params"], ck["n"])
    engine.set_state(m=ck["m"], v=ck["v"], accum=ck["accum"], vcount=ck["vcount"])
    return ck
