"""Per (warp, fragment) work accounting of the blend loops at a workload (CPU, oracle data):
how many warp-fragments pass the per-warp row cull, and how many of those have >= 1 pixel
that keeps the fragment (Q <= k2) while still active (list position < its contributor count)."""
import sys
import numpy as np
sys.path.insert(0, __file__.rsplit("/", 2)[0])
from oracle import oracle as O
from paper_2602_09999_b200 import scene, types as T

wname = sys.argv[1] if len(sys.argv) > 1 else "H"
w = scene.WORKLOADS[wname]
n = w.n
O.set_workers(8)
p = scene.perturb(scene.random_params(n, w.s0, w.m_o, w.seed), n, w.seed)
cam = scene.ring_camera(w, 0)
cfg = T.RenderConfig.make(sh_degree=w.sh_degree)
sp, rect, cnt, dk = O.preprocess(p, n, cam, cfg)
keys, vals, ranges, _ = O.instances(p, n, cam, cfg)
_, _, pc, _ = O.render(p, n, cam, cfg)
rng = np.random.default_rng(0)
tiles = rng.choice(cam.n_tiles, 400, replace=False)
tot = dict(all=0, rowcull=0, kept=0, kept_active=0, half_kept_active=0, px_ka=0, thr_ka=0, pair_work=0)
hist = np.zeros(33, np.int64)
for t in tiles:
    tx, ty = t % cam.tiles_x, t // cam.tiles_x
    b, e = ranges[t]
    ys = np.arange(ty * 16, min(ty * 16 + 16, cam.height))
    xs = np.arange(tx * 16, min(tx * 16 + 16, cam.width))
    cc = np.zeros((16, 16), np.int64)
    cc[:len(ys), :len(xs)] = pc[np.ix_(ys, xs)]
    Lp = int(cc.max())
    if Lp == 0:
        continue
    g = vals[b:b + Lp]
    s = sp[g]
    mx, my, k2 = s[:, 0], s[:, 1], s[:, 2]
    A, B, C = s[:, 4], s[:, 5], s[:, 6]
    det = A.astype(np.float64) * C - B.astype(np.float64) ** 2
    ry = np.sqrt(np.maximum(k2 * A / det, 0)) * 1.001 + 0.05
    PX = (tx * 16 + np.arange(16))[None, None, :]
    PY = (ty * 16 + np.arange(16))[None, :, None]
    dx = PX - mx[:, None, None]
    dy = PY - my[:, None, None]
    Q = dx * (A[:, None, None] * dx + 2 * B[:, None, None] * dy) + dy * (C[:, None, None] * dy)
    keep = Q <= k2[:, None, None]
    active = np.arange(Lp)[:, None, None] < cc[None, :, :]
    for wi in range(2):
        wy0, wy1 = ty * 16 + 8 * wi, ty * 16 + 8 * wi + 7
        rc = ~((my + ry < wy0) | (my - ry > wy1))
        k = keep[:, 8 * wi:8 * wi + 8, :]
        ka = (keep & active)[:, 8 * wi:8 * wi + 8, :]
        tot["all"] += Lp
        tot["rowcull"] += rc.sum()
        tot["kept"] += (rc & k.any(axis=(1, 2))).sum()
        tot["kept_active"] += (rc & ka.any(axis=(1, 2))).sum()
        # half-warps (16 columns x 4 rows each): work if either half needs the fragment
        h0 = ka[:, 0:4, :].any(axis=(1, 2))
        h1 = ka[:, 4:8, :].any(axis=(1, 2))
        tot["half_kept_active"] += (h0.astype(int) + h1.astype(int)).sum() / 2
        sel = rc & ka.any(axis=(1, 2))
        tot["px_ka"] += ka[sel].sum()
        # thread = 1 column x 4 rows: threads with >= 1 kept active pixel
        thr = ka[sel].reshape(-1, 2, 4, 16).any(axis=2)
        tot["thr_ka"] += thr.sum()
        if thr.shape[0]: hist += np.bincount(thr.reshape(thr.shape[0], -1).sum(axis=1), minlength=33)[:33]
        kk = ka[sel]
        p0 = kk[:, [0, 1, 4, 5], :].any(axis=(1, 2))
        p1 = kk[:, [2, 3, 6, 7], :].any(axis=(1, 2))
        tot["pair_work"] += p0.sum() + p1.sum()
print(wname, {k: int(v) for k, v in tot.items()})
print({k: round(v / tot["rowcull"], 3) for k, v in tot.items()})
c = np.cumsum(hist) / hist.sum()
print("active lanes per worked warp-fragment, CDF at 1,2,4,8,16,24,31,32:", [round(float(c[k]), 3) for k in (1, 2, 4, 8, 16, 24, 31, 32)])
print("pixel utilisation in worked warp-fragments:", tot["px_ka"] / (tot["kept_active"] * 128),
      " thread utilisation:", tot["thr_ka"] / (tot["kept_active"] * 32),
      " pairs needed (of 2 per worked warp-fragment):", tot["pair_work"] / (2 * tot["kept_active"]))
