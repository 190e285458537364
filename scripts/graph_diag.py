"""Per-step device durations of the bench's timed loop in graph mode (after the profiled loop):
which steps are host-path, captured or graph launches, and how long each took on the stream."""
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
e.set_params(scene.perturb(gt, w.n, w.seed), w.n)
e.set_graph(True)
step = 0
def one(loss=False):
    global step
    step += 1
    return e.train_step(cams[step % 8], cfg, T.AdamConfig.make(step=step, zero_grads=0), slot=step % 8, want_loss=loss)
for _ in range(10):
    one()
e.set_profiling(True)
for _ in range(30):
    one()
torch.cuda.synchronize()
e.set_profiling(False)
evs = [torch.cuda.Event(enable_timing=True) for _ in range(41)]
kinds = []
evs[0].record(st)
for i in range(40):
    g0 = e.graph_stats()
    one()
    g1 = e.graph_stats()
    kinds.append("capture" if g1["captures"] > g0["captures"] else "graph" if g1["launches"] > g0["launches"] else "host")
    evs[i + 1].record(st)
torch.cuda.synchronize()
d = [round(evs[i].elapsed_time(evs[i + 1]), 3) for i in range(40)]
print(json.dumps(list(zip(kinds, d))))
# loss of a graph step vs the same step on the host path from the same state
e.synchronize()
p = e.get_params()
_, m, v, _, _ = e.get_state()
l_g = one(loss=True)   # want_loss key: first time -> host path
e.set_graph(False)
print("done", l_g)
