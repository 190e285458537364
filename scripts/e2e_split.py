"""Where the e2e (host target + loss read-back) time goes: device slot vs pinned host target,
with and without the per-step loss read-back (workload H, z-ordered store)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_09999_b200 import scene, types as T
from paper_2602_09999_b200.tilesplat import Engine, PinnedBuffer
w = scene.WORKLOADS["H"]
gt = scene.random_params(w.n, w.s0, w.m_o, w.seed)
cam = scene.workload_cameras(w)[0]
cfg = T.RenderConfig.make(sh_degree=3)
s = torch.cuda.current_stream()
e = Engine(0, stream=s.cuda_stream)
e.set_params(gt, w.n)
tgt, _, _ = e.render(cam, cfg)
e.set_target(0, tgt)
e.set_params(scene.perturb(gt, w.n, w.seed), w.n)
e.morton_reorder()
pin = PinnedBuffer((w.height, w.width, 3))
pin.array[...] = tgt
step = 0
def run(k, host, loss):
    global step
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(k):
        step += 1
        a = T.AdamConfig.make(step=step, mode=1, zero_grads=0)
        if host:
            e.train_step(cam, cfg, a, target_ptr=pin.ptr, want_loss=loss)
        else:
            e.train_step(cam, cfg, a, slot=0, want_loss=loss)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3 / k
run(10, False, False)
for host in (False, True):
    for loss in (False, True):
        print(f"host_target={host} loss={loss}: {run(40, host, loss):.3f} ms/step")
