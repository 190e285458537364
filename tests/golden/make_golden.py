"""Regenerates tests/golden/*.json: oracle outputs on the seeded BASELINE configs
(c1 full, and a 1080p crop-free subsample) as hashes + summary statistics, so any
drift of the oracle or of the CUDA path is caught against committed values.

usage: python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2602_09999_b200 import scene, types as T  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def golden_case(name, n, s0, m_o, seed, W, H, deg):
    p = scene.random_params(n, s0, m_o, seed)
    cam = scene.make_camera(W, H)
    cfg = T.RenderConfig.make(sh_degree=deg)
    splat, rect, cnt, dkey = O.preprocess(p, n, cam, cfg)
    keys, vals, ranges, _ = O.instances(p, n, cam, cfg)
    rgb, Tf, pc, I = O.render(p, n, cam, cfg)
    return {
        "name": name, "n": n, "s0": s0, "m_o": m_o, "seed": seed, "width": W, "height": H, "sh_degree": deg,
        "instances": int(I), "visible": int((cnt > 0).sum()),
        "sha_tile_count": sha(cnt), "sha_depth_key": sha(dkey), "sha_keys": sha(keys), "sha_vals": sha(vals),
        "sha_ranges": sha(ranges), "sha_contrib": sha(pc),
        "image_mean": [float(x) for x in rgb.reshape(-1, 3).mean(0)], "image_max": float(rgb.max()),
        "T_mean": float(Tf.mean()), "keys_head": [int(k) for k in keys[:8]], "vals_head": [int(v) for v in vals[:8]],
    }


if __name__ == "__main__":
    cases = [golden_case("c1", 10_000, 0.02, 0.0, 1, 256, 256, 0),
             golden_case("c1_sh3_odd", 20_000, 0.015, 0.5, 2, 333, 187, 3)]
    with open(os.path.join(ROOT, "tests", "golden", "oracle_golden.json"), "w") as f:
        json.dump(cases, f, indent=1)
    print("wrote", len(cases), "cases")
