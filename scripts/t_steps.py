import sys, os, time, subprocess
sys.path.insert(0, "/root/repo")
import torch, numpy as np
from paper_2602_09999_b200 import scene, types as T
from paper_2602_09999_b200.tilesplat import Engine
w = scene.WORKLOADS["H"]
gt = scene.random_params(w.n, w.s0, w.m_o, w.seed)
cam = scene.workload_cameras(w)[0]
cfg = T.RenderConfig.make(sh_degree=w.sh_degree)
s = torch.cuda.current_stream()
e = Engine(0, stream=s.cuda_stream)
e.set_params(gt, w.n)
target, _, _ = e.render(cam, cfg)
e.set_target(0, target)
e.set_params(scene.perturb(gt, w.n, w.seed), w.n)
e.morton_reorder()
step = 0
def run(k):
    global step
    ev0 = torch.cuda.Event(enable_timing=True); ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); ev0.record(s); t0 = time.perf_counter()
    for _ in range(k):
        step += 1
        e.train_step(cam, cfg, T.AdamConfig.make(step=step, mode=1, zero_grads=0), slot=0, want_loss=False)
    ev1.record(s); torch.cuda.synchronize()
    return ev0.elapsed_time(ev1) / k, (time.perf_counter() - t0) * 1e3 / k
run(10)
for k in (10, 50, 200):
    print("steps", k, "ms(ev, wall) = %.3f %.3f" % run(k))
p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm", "--format=csv,noheader", "-lms", "100"], stdout=subprocess.DEVNULL)
print("with smi 200", "%.3f %.3f" % run(200))
p.terminate()
e.set_profiling(True); run(20); print({k: round(v[0]/max(1,v[1]),4) for k, v in e.stage_times().items()}); e.set_profiling(False)
print("after 200", "%.3f %.3f" % run(200))
