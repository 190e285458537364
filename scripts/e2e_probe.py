"""Wall-clock per ts_train_step: device-resident target vs pinned host target, with/without loss read-back."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2602_09999_b200 import scene, types as T
from paper_2602_09999_b200.tilesplat import Engine, PinnedBuffer
w = scene.WORKLOADS["H"]
gt = scene.random_params(w.n, w.s0, w.m_o, w.seed)
cam = scene.workload_cameras(w)[0]
cfg = T.RenderConfig.make(sh_degree=3)
e = Engine(0)
e.set_params(gt, w.n)
target, _, _ = e.render(cam, cfg)
e.set_target(0, target)
e.set_params(scene.perturb(gt, w.n, w.seed), w.n)
pin = PinnedBuffer(target.shape)
pin.array[...] = target
step = [0]
def run(kind, k=40):
    for i in range(k + 5):
        if i == 5:
            e.synchronize(); t0 = time.perf_counter()
        step[0] += 1
        a = T.AdamConfig.make(step=step[0], zero_grads=0)
        if kind == "slot":
            e.train_step(cam, cfg, a, slot=0, want_loss=False)
        elif kind == "slot+loss":
            e.train_step(cam, cfg, a, slot=0, want_loss=True)
        elif kind == "pinned":
            e.train_step(cam, cfg, a, target_ptr=pin.ptr, want_loss=False)
        else:
            e.train_step(cam, cfg, a, target_ptr=pin.ptr, want_loss=True)
    e.synchronize()
    return (time.perf_counter() - t0) / k * 1e3
for kind in ("slot", "slot+loss", "pinned", "pinned+loss", "slot"):
    print(kind, round(run(kind), 3), "ms")
