"""Per-stage device times of the training step at a workload (profiling events)."""
import sys, time, json, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2602_09999_b200 import scene, types as T
from paper_2602_09999_b200.tilesplat import Engine

name = sys.argv[1] if len(sys.argv) > 1 else "H"
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 1
w = scene.WORKLOADS[name]
gt = scene.random_params(w.n, w.s0, w.m_o, w.seed)
cam = scene.workload_cameras(w)[0]
cfg = T.RenderConfig.make(sh_degree=w.sh_degree)
e = Engine(0)
e.set_params(gt, w.n)
target, _, _ = e.render(cam, cfg)
e.set_target(0, target)
e.set_params(scene.perturb(gt, w.n, w.seed), w.n)
if os.environ.get("PROBE_MORTON"):
    e.morton_reorder()
if os.environ.get("PROBE_BWD"):
    cfg.backward_mode = int(os.environ["PROBE_BWD"])
for i in range(5):
    e.train_step(cam, cfg, T.AdamConfig.make(step=i + 1, mode=mode), want_loss=False)
e.synchronize()
e.set_profiling(True)
K = 10
for i in range(K):
    e.train_step(cam, cfg, T.AdamConfig.make(step=i + 6, mode=mode), want_loss=False)
tot = {k: v[0] / max(1, v[1]) for k, v in e.stage_times().items()}
e.set_profiling(False)
e.synchronize()
t0 = time.perf_counter()
for i in range(K):
    e.train_step(cam, cfg, T.AdamConfig.make(step=i + 20, mode=mode), want_loss=False)
e.synchronize()
dt = (time.perf_counter() - t0) / K
print(json.dumps({"workload": name, "mode": mode, "stats": e.view_stats(), "stage_ms": {k: round(v, 4) for k, v in tot.items()},
                  "sum_ms": round(sum(tot.values()), 3), "wall_ms_per_step": round(dt * 1e3, 3)}))
