import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2602_09999_b200 import scene, types as T
from paper_2602_09999_b200.tilesplat import Engine
for name in ("c5", "H"):
    w = scene.WORKLOADS[name]
    p = scene.random_params(w.n, w.s0, w.m_o, w.seed)
    cam = scene.workload_cameras(w)[0]
    e = Engine(0)
    e.set_params(p, w.n)
    e.render(cam, T.RenderConfig.make(sh_degree=3), outputs=False)
    k, v, r = e.debug_instances()
    L = (r[:, 1] - r[:, 0]).astype(np.int64)
    print(name, e.binning_path(), "I", L.sum(), "max", L.max(), ">16384:", (L > 16384).sum(), "inst in them", L[L > 16384].sum(),
          ">8192:", (L > 8192).sum(), "p50/p90/p99", np.percentile(L, [50, 90, 99]).astype(int))
    e.close()
