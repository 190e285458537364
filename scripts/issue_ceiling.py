"""Issue ceiling of the blend kernels (K6 blend_fwd, K8 blend_bwd): the same kernels on a DENSE
scene -- every tile holds ~DEPTH large, faint Gaussians that cover it entirely (o = 0.01, so T stays
above the 1e-4 stop for the whole list), i.e. every pixel keeps every fragment: no row cull, no
lane divergence, no early exit, a long uniform list per tile -- next to the headline workload H.
Under `ncu --metrics smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,
sm__cycles_elapsed.avg,gpu__time_duration.sum -k regex:blend` the dense run gives the issue rate the
kernels' instruction mix sustains when nothing but the mix itself limits it; production over dense
is the kernel's fraction of its measured issue ceiling.

usage: python scripts/issue_ceiling.py [dense|H] [DEPTH]
"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2602_09999_b200 import scene, types as T  # noqa: E402
from paper_2602_09999_b200.tilesplat import Engine  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "dense"
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 600
w = scene.WORKLOADS["H"]
cam = scene.workload_cameras(w)[0]
cfg = T.RenderConfig.make(sh_degree=3)
if which == "dense":
    # world scale 0.3 at o = 0.01 (k2 = -2 ln(tau / o) = 1.87): each splat covers ~8x8 tiles entirely
    # (checked with the oracle: I / tiles ~ 1.3 N / 20); N gives ~depth instances per tile
    n = int(depth * 20 / 1.3 * cam.n_tiles / 8160)
    rng = np.random.default_rng(7)
    means = np.stack([rng.uniform(-1.3, 1.3, n), rng.uniform(-0.8, 0.8, n), rng.uniform(-0.2, 0.2, n)], 1)
    log_scales = np.full((n, 3), math.log(0.3)) + rng.normal(0, 0.05, (n, 3))
    quats = np.tile([1.0, 0.0, 0.0, 0.0], (n, 1)) + rng.normal(0, 0.05, (n, 4))
    logits = np.full(n, math.log(0.01 / 0.99))
    sh_dc = rng.uniform(-1.5, 1.5, (n, 3))
    sh_rest = rng.normal(0.0, 0.05, (n, 15, 3))
    p = T.pack_params(means, log_scales, quats, logits, sh_dc, sh_rest)
else:
    n = w.n
    gt = scene.random_params(w.n, w.s0, w.m_o, w.seed)
    p = scene.perturb(gt, w.n, w.seed)
e = Engine(0)
e.set_params(p, n)
if which != "dense":
    e.morton_reorder()
rgb, Tf, cnt = e.render(cam, cfg)
target = np.clip(rgb + 0.05, 0, 1).astype(np.float32)
for _ in range(3):
    e.render(cam, cfg)
    e.training_loss(target)
    e.backward(None)
e.synchronize()
st = e.view_stats()
print(f"{which}: N={n} I={st['I']} Ip={st['Ip']} mean T={float(Tf.mean()):.3f} "
      f"min count={int(cnt.min())} mean count={float(cnt.mean()):.1f}")
