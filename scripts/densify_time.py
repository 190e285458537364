"""Device time of densify_and_prune and morton_reorder at workload H (3M Gaussians)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_09999_b200 import scene, types as T
from paper_2602_09999_b200.tilesplat import Engine
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
for i in range(20):
    e.train_step(cam, cfg, T.AdamConfig.make(step=i + 1, mode=1, zero_grads=0), slot=0, want_loss=False)
torch.cuda.synchronize()
for name, fn in (("morton_reorder (first: allocates the spare store)", lambda: e.morton_reorder()),
                 ("morton_reorder", lambda: e.morton_reorder()),
                 ("densify_and_prune", lambda: e.densify_and_prune(2e-6, 1.0, 7, 700)),
                 ("densify_and_prune (again)", lambda: e.densify_and_prune(2e-6, 1.0, 8, 800)),
                 ("opacity_reset", lambda: e.opacity_reset())):
    n0 = e.num_gaussians()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); t0 = time.perf_counter(); ev0.record(s)
    r = fn()
    ev1.record(s); torch.cuda.synchronize()
    print(f"{name}: {ev0.elapsed_time(ev1):.3f} ms device, {(time.perf_counter() - t0) * 1e3:.3f} ms wall, N {n0} -> {e.num_gaussians()}")
