"""Device time per training step, graph mode vs host-driven path, bench setup (workload H, 8-view
ring, z-ordered perturbed store, device targets): every view's graph captured first, then K steps
timed with CUDA events on the engine stream (no captures inside the timed region)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_09999_b200 import scene, types as T
from paper_2602_09999_b200.tilesplat import Engine

name = sys.argv[1] if len(sys.argv) > 1 else "H"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 100
w = scene.WORKLOADS[name]
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
e.set_params(p0, w.n)
e.morton_reorder()
res = {}
step = 0
for mode in ("host", "graph", "host", "graph"):
    e.set_graph(mode == "graph")
    for _ in range(24):
        step += 1
        e.train_step(cams[step % 8], cfg, T.AdamConfig.make(step=step, zero_grads=0), slot=step % 8, want_loss=False)
    torch.cuda.synchronize()
    g0 = e.graph_stats()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(K):
        step += 1
        e.train_step(cams[step % 8], cfg, T.AdamConfig.make(step=step, zero_grads=0), slot=step % 8, want_loss=False)
    b.record(st)
    torch.cuda.synchronize()
    g1 = e.graph_stats()
    res.setdefault(mode, []).append(round(a.elapsed_time(b) / K, 4))
    res.setdefault(mode + "_captures_in_timed", []).append(g1["captures"] - g0["captures"])
e.set_graph(False)
res["view"] = e.view_stats()
print(json.dumps(res))
