"""Graph-mode vs host-path training at a workload (default H): K steps over the 8-view ring from
the same store; prints per-step losses, max relative param difference and timings."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2602_09999_b200 import scene, types as T
from paper_2602_09999_b200.tilesplat import Engine

name = sys.argv[1] if len(sys.argv) > 1 else "H"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 24
w = scene.WORKLOADS[name]
gt = scene.random_params(w.n, w.s0, w.m_o, w.seed)
cams = [scene.ring_camera(w, j) for j in range(8)]
cfg = T.RenderConfig.make(sh_degree=w.sh_degree)
e = Engine(0)
e.set_params(gt, w.n)
for j, c in enumerate(cams):
    t, _, _ = e.render(c, cfg)
    e.set_target(j, t)
p0 = scene.perturb(gt, w.n, w.seed)
out = {}
for graph in (False, True):
    e.set_params(p0, w.n)
    e.set_graph(graph)
    L = []
    for s in range(1, K + 1):
        L.append(e.train_step(cams[s % 8], cfg, T.AdamConfig.make(step=s), slot=s % 8, want_loss=True))
    e.synchronize()
    t0 = time.perf_counter()
    for s in range(K + 1, K + 41):
        e.train_step(cams[s % 8], cfg, T.AdamConfig.make(step=s), slot=s % 8, want_loss=False)
    e.synchronize()
    dt = (time.perf_counter() - t0) / 40
    out[graph] = (np.array(L), e.get_params(), dt, e.graph_stats())
    e.set_graph(False)
(lh, ph, th, _), (lg, pg, tg, st) = out[False], out[True]
rel = np.abs(pg - ph) / np.maximum(np.abs(ph), 1e-3)
print(json.dumps({"loss_host": lh[:6].tolist(), "loss_graph": lg[:6].tolist(),
                  "loss_max_rel": float(np.max(np.abs(lg - lh) / lh)), "param_max_rel": float(rel.max()),
                  "param_frac_gt_1e-4": float(np.mean(rel > 1e-4)), "ms_host": th * 1e3, "ms_graph": tg * 1e3,
                  "graph_stats": st}))
