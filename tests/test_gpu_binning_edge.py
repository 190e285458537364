"""Edge cases of the bucketed binning (K1's warp-cooperative exact cull and chunk histograms, the
column scan with its last-CTA range scan, the warp-flattened scatter, the per-tile sort) against
the oracle's stable sort: sorted keys, values and tile ranges bit-exact.

Cases: rects of more than 64 tiles (their per-lane exact-cull path in the scatter) mixed with
small splats, both cull modes; Gaussian counts that leave partial warps, one Gaussian past a
chunk boundary, and a single Gaussian; duplicated rows (equal depth keys: ties on the index).
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2602_09999_b200 import scene, types as T

pytestmark = pytest.mark.gpu


def _scene(n, seed, n_huge=0, dup=0):
    p = scene.random_params(n, 0.03, 0.5, seed)
    rng = np.random.default_rng(seed)
    if n_huge:
        # log-scales of a few Gaussians raised so their tile rects exceed 64 tiles
        idx = rng.choice(n, n_huge, replace=False)
        for k in range(3):
            p[3 * n + 3 * idx + k] = np.float32(np.log(rng.uniform(0.4, 1.2, n_huge)))
    if dup:
        # the first `dup` rows copied over the last ones: identical depth keys, ties broken by index
        for a, b in T.group_slices(n):
            w = (b - a) // n
            blk = p[a:b].reshape(n, w)
            blk[n - dup:] = blk[:dup]
    return p


def _check(engine, p, n, cam, cfg):
    engine.set_params(p, n)
    engine.set_binning(0)
    engine.render(cam, cfg, outputs=False)
    assert engine.binning_path() == "bucket"
    gk, gv, gr = engine.debug_instances()
    ok, ov, orr, _ = O.instances(p, n, cam, cfg, sort="combined")
    assert gk.shape == ok.shape
    assert np.array_equal(gk, ok) and np.array_equal(gv, ov) and np.array_equal(gr, orr)
    return ok.size


@pytest.mark.parametrize("cull", [0, 1])
@pytest.mark.parametrize("bound", [0, 1, 2])
def test_big_rects_mixed_with_small(engine, cull, bound):
    n = 5000
    p = _scene(n, 11 + cull + 3 * bound, n_huge=24)
    cam = scene.make_camera(640, 480, eye=(0.0, 0.0, -3.0), fov_x_deg=60.0)
    cfg = T.RenderConfig.make(sh_degree=1, bound_mode=bound, cull_mode=cull)
    engine.set_params(p, n)
    engine.render(cam, cfg, outputs=False)
    _, rects, _, _ = engine.debug_preprocess()
    # the scene really has rects of more than 64 tiles (rect = tx0, ty0, tx1, ty1; empty: tx0 > tx1)
    area = np.maximum(rects[:, 2] - rects[:, 0] + 1, 0) * np.maximum(rects[:, 3] - rects[:, 1] + 1, 0)
    assert np.any(area > 64)
    assert _check(engine, p, n, cam, cfg) > 0


@pytest.mark.parametrize("n", [1, 31, 33, 6145, 12289])
def test_partial_warps_and_chunk_boundaries(engine, n):
    p = _scene(n, 100 + n)
    cam = scene.make_camera(320, 200, eye=(0.2, -0.1, -3.0), fov_x_deg=55.0)
    cfg = T.RenderConfig.make(sh_degree=0)
    _check(engine, p, n, cam, cfg)


def test_duplicated_rows_tie_on_index(engine):
    n = 4000
    p = _scene(n, 7, n_huge=4, dup=600)
    cam = scene.make_camera(400, 300, eye=(0.0, 0.0, -3.0), fov_x_deg=60.0)
    cfg = T.RenderConfig.make(sh_degree=2)
    _check(engine, p, n, cam, cfg)
