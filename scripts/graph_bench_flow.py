"""The bench's exact step sequence (warm-up, profiled host-path loop, timed loop) in graph and
host mode from the same store: timed device ms/step and the end-state difference."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2602_09999_b200 import scene, types as T
from paper_2602_09999_b200.tilesplat import Engine

w = scene.WORKLOADS["H"]
gt = scene.random_params(w.n, w.s0, w.m_o, w.seed)
cams = [scene.ring_camera(w, j) for j in range(8)]
cfg = T.RenderConfig.make(sh_degree=w.sh_degree)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
e = Engine(0, stream=st.cuda_stream)
e.set_params(gt, w.n)
for j, c in enumerate(cams):
    t, _, _ = e.render(c, cfg)
    e.set_target(j, t)
p0 = scene.perturb(gt, w.n, w.seed)
out = {}
for graph in (True, False):
    e.set_params(p0, w.n)
    e.set_graph(graph)
    step = 0
    def one():
        global step
        step += 1
        e.train_step(cams[step % 8], cfg, T.AdamConfig.make(step=step, zero_grads=0), slot=step % 8, want_loss=False)
    for _ in range(10):
        one()
    torch.cuda.synchronize()
    e.set_profiling(True)
    for _ in range(30):
        one()
    torch.cuda.synchronize()
    e.set_profiling(False)
    g0 = e.graph_stats()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(100):
        one()
    b.record(st)
    torch.cuda.synchronize()
    e.synchronize()
    g1 = e.graph_stats()
    out[graph] = (a.elapsed_time(b) / 100, e.get_params(), {k: g1[k] - g0[k] for k in g1})
    e.set_graph(False)
(tg, pg, sg), (th, ph, _) = out[True], out[False]
rel = np.abs(pg - ph) / np.maximum(np.abs(ph), 1e-3)
print(json.dumps({"ms_graph": tg, "ms_host": th, "graph_timed": sg, "param_max_rel": float(rel.max()),
                  "param_frac_gt_1e-3": float(np.mean(rel > 1e-3)), "param_mean_abs_diff": float(np.mean(np.abs(pg - ph)))}))
