"""Per-tile sort bucket occupancy at workload H: expected rank-loop length per element
(sum of squared bucket sizes / list length) for linear-interpolation buckets."""
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
e.morton_reorder()
e.render(cam, T.RenderConfig.make(sh_degree=3), outputs=False)
keys, vals, ranges = e.debug_instances()
dk = (keys & np.uint64(0xFFFFFFFF)).astype(np.int64)
rng = np.random.default_rng(0)
tot_lin = tot_eq = tot_n = 0
for t in rng.choice(np.flatnonzero(ranges[:, 1] - ranges[:, 0] > 64), 400, replace=False):
    b, en = ranges[t]
    k = dk[b:en]
    L = len(k)
    nb = L
    bl = np.minimum(nb - 1, ((k - k.min()) * (nb / (k.max() - k.min() + 1.0))).astype(np.int64))
    c = np.bincount(bl, minlength=nb)
    tot_lin += (c.astype(np.float64) ** 2).sum()
    # equalised: 64 coarse bins, bucket by CDF
    cb = np.minimum(63, ((k - k.min()) * (64 / (k.max() - k.min() + 1.0))).astype(np.int64))
    cc = np.bincount(cb, minlength=64); cdf = np.concatenate([[0], np.cumsum(cc)])
    lo = k.min() + (np.arange(64) * (k.max() - k.min() + 1.0) / 64)
    frac = (k - lo[cb]) / ((k.max() - k.min() + 1.0) / 64)
    be = np.minimum(nb - 1, (cdf[cb] + frac * cc[cb]) * nb / L).astype(np.int64)
    c2 = np.bincount(be, minlength=nb)
    tot_eq += (c2.astype(np.float64) ** 2).sum()
    tot_n += L
print(f"rank-loop length per element: linear {tot_lin / tot_n:.2f}, equalised(64) {tot_eq / tot_n:.2f}")
