"""Toy-scene convergence probe (SPEC acceptance 9/10): train a perturbed store against self-rendered
targets on a ring of training cameras, report the held-out view's PSNR before/after."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2602_09999_b200 import scene, types as T
from paper_2602_09999_b200.tilesplat import Engine

def psnr(a, b):
    return 10 * math.log10(1.0 / max(float(np.mean((a - b) ** 2)), 1e-12))

n, W, H = int(sys.argv[1]) if len(sys.argv) > 1 else 3000, 160, 120
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 600
mode = int(sys.argv[3]) if len(sys.argv) > 3 else T.ADAM_FUSED
gt = scene.random_params(n, 0.04, 0.5, 5)
cams = scene.fibonacci_cameras(9, W, H)
train, held = cams[:8], cams[8]
cfg = T.RenderConfig.make(sh_degree=1)
e = Engine(0)
e.set_params(gt, n)
tg = [e.render(c, cfg)[0].copy() for c in train]
hold = e.render(held, cfg)[0].copy()
rng = np.random.default_rng(1)
p = gt.copy()
p[0:3 * n] += rng.normal(0, 0.03, 3 * n).astype(np.float32)
p[3 * n:6 * n] += rng.normal(0, 0.2, 3 * n).astype(np.float32)
p[10 * n:11 * n] += rng.normal(0, 0.5, n).astype(np.float32)
p[11 * n:14 * n] += rng.normal(0, 0.3, 3 * n).astype(np.float32)
e.set_params(p, n)
for k, t in enumerate(tg):
    e.set_target(k, t)
before = psnr(e.render(held, cfg)[0], hold)
for s in range(1, steps + 1):
    e.train_step(train[s % 8], cfg, T.AdamConfig.make(step=s, extent=3.5, mode=mode), slot=s % 8, want_loss=False)
after = psnr(e.render(held, cfg)[0], hold)
print(f"n={n} steps={steps} mode={mode} held-out PSNR {before:.2f} -> {after:.2f} dB")
np.save("/tmp/toy_params_%d.npy" % mode, e.get_params())
