"""Fraction of (tile, fragment) pairs the per-warp row cull drops in the blend kernels (workload H)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2602_09999_b200 import scene, types as T
from paper_2602_09999_b200.tilesplat import Engine
w = scene.WORKLOADS["H"]
p = scene.random_params(w.n, w.s0, w.m_o, w.seed)
cam = scene.workload_cameras(w)[0]
cfg = T.RenderConfig.make(sh_degree=3)
e = Engine(0)
e.set_params(p, w.n)
e.render(cam, cfg, outputs=False)
gs, gr, gc, gk = e.debug_preprocess()
keys, vals, ranges = e.debug_instances()
tile = (keys >> np.uint64(32)).astype(np.int64)
ty = tile // cam.tiles_x
my, A, B, C, k2 = gs[vals, 1], gs[vals, 4], gs[vals, 5], gs[vals, 6], gs[vals, 2]
syy = A / (A * C - B * B)
ry = np.sqrt(np.maximum(k2 * syy, 0)) * 1.001 + 0.05
hit = []
for wi in range(2):
    y0 = ty * 16 + wi * 8
    hit.append(~((my + ry < y0) | (my - ry > y0 + 7)))
h0, h1 = hit
print("pairs", len(vals), "warp0 hit", h0.mean(), "warp1 hit", h1.mean(), "both", (h0 & h1).mean(), "none", (~h0 & ~h1).mean())
