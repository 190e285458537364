"""Of the (warp, fragment) pairs that pass the per-warp row cull of the blend kernels, how
many have no pixel with Q <= k2 in the warp (sampled tiles, workload H, ignoring early stop)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2602_09999_b200 import scene, types as T
from paper_2602_09999_b200.tilesplat import Engine
w = scene.WORKLOADS["H"]
p = scene.random_params(w.n, w.s0, w.m_o, w.seed)
cam = scene.workload_cameras(w)[0]
e = Engine(0)
e.set_params(p, w.n)
e.render(cam, T.RenderConfig.make(sh_degree=3), outputs=False)
gs, _, _, _ = e.debug_preprocess()
keys, vals, ranges = e.debug_instances()
rng = np.random.default_rng(0)
tiles = rng.choice(np.flatnonzero(ranges[:, 1] > ranges[:, 0]), 300, replace=False)
tot = passed = anyk = 0
for t in tiles:
    b, en = ranges[t]
    g = vals[b:en]
    mx, my, k2 = gs[g, 0], gs[g, 1], gs[g, 2]
    A, B, C = gs[g, 4], gs[g, 5], gs[g, 6]
    syy = A / (A * C - B * B)
    ry = np.sqrt(np.maximum(k2 * syy, 0)) * 1.001 + 0.05
    tx, ty = t % cam.tiles_x, t // cam.tiles_x
    xs = tx * 16 + np.arange(16)
    for wi in range(2):
        y0 = ty * 16 + wi * 8
        ys = y0 + np.arange(8)
        rc = ~((my + ry < y0) | (my - ry > y0 + 7))
        tot += len(g)
        passed += rc.sum()
        dx = xs[None, None, :] - mx[:, None, None]
        dy = ys[None, :, None] - my[:, None, None]
        Q = dx * (A[:, None, None] * dx + 2 * B[:, None, None] * dy) + dy * (C[:, None, None] * dy)
        k = (Q <= k2[:, None, None]).any(axis=(1, 2))
        anyk += (k & rc).sum()
print(f"pairs {tot}  row-cull pass {passed / tot:.3f}  any-keep among passed {anyk / passed:.3f}")
