import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2602_09999_b200 import scene, types as T
from paper_2602_09999_b200.tilesplat import Engine
e = Engine(0)
n = 30_000
gt = scene.random_params(n, 0.02, 0.0, 31)
cam = scene.make_camera(320, 200)
cfg = T.RenderConfig.make(sh_degree=3)
e.set_params(gt, n)
target, _, _ = e.render(cam, cfg)
p0 = scene.perturb(gt, n, 31)
e.set_params(p0, n)
e.render(cam, cfg, outputs=False)
_, _, tc, _ = e.debug_preprocess()
single = tc <= 1
rowmask = {}
outs = []
for m in (1, 3):
    e.set_params(p0, n)
    e.train_step(cam, cfg, T.AdamConfig.make(step=1, mode=m), target=target)
    g, mm, vv, acc, vc = e.get_state()
    outs.append((e.get_params(), mm, vv, acc, vc))
names = ["params", "m", "v", "acc", "vc"]
for nm, a, b in zip(names, *outs):
    if a.size == 59 * n:
        keep = np.concatenate([np.repeat(single, w) for w in T.GROUP_WIDTH])
    else:
        keep = single
    d = np.flatnonzero((a.view(np.uint32) != b.view(np.uint32)) & keep)
    print(nm, "ndiff", d.size, "first", d[:8], "maxabs", np.abs(a - b).max() if a.size else 0)
    if d.size:
        for (s, t), gn in zip(T.group_slices(n), T.GROUPS):
            k = ((d >= s) & (d < t)).sum()
            if k: print("   group", gn, k)
        i = d[0]; print("   a", a[i], "b", b[i])
