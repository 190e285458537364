"""Antialias module: sampling rates, 3D filter (original and clip),
Mip 2D filter with opacity compensation.

CPU tests pin the oracle to the SPEC examples and to finite differences; GPU tests
(marked) check the CUDA path against the oracle: sampling rates, clip and the
preprocess splat fields bit-exact, images <= 1e-4, gradients within 1e-3.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2602_09999_b200 import scene, types as T


def _cam_at_depth(d, f=100.0, W=64, H=64):
    """camera looking down +z from z = -d (a mean at the origin has depth d)."""
    Wm = np.eye(4)
    Wm[2, 3] = d
    return T.Camera.make(Wm, f, f, W / 2, H / 2, W, H)


def _one(mean=(0.0, 0.0, 0.0), log_scale=0.0, logit=0.0):
    return T.pack_params([mean], [[log_scale] * 3], [[1, 0, 0, 0]], [logit], [[0, 0, 0]], np.zeros((1, 15, 3)))


# ---------------------------------------------------------------- oracle ----
def test_sampling_rate_examples():
    p = _one()
    assert O.compute_sampling_rates(p, 1, [_cam_at_depth(2.0)], 1.0)[0] == np.float32(50.0)
    nu = O.compute_sampling_rates(p, 1, [_cam_at_depth(2.0), _cam_at_depth(4.0)], 1.0)[0]
    assert nu == np.float32(50.0)
    behind = O.compute_sampling_rates(_one(mean=(0.0, 0.0, -5.0)), 1, [_cam_at_depth(2.0)], 2.5)[0]
    assert behind == np.float32(1.0 / 2.5)  # fallback extent^-1


def test_filter3d_original_examples():
    cam = _cam_at_depth(3.0, f=50.0)
    # s = (1,1,1), kappa / nu^2 = 3  ->  s_hat = (2,2,2), o_hat = o / 8
    p = _one(log_scale=0.0, logit=0.0)
    O.set_sampling_rates(np.array([math.sqrt(0.2 / 3.0)], np.float32))
    s1, _, _, _ = O.preprocess(p, 1, cam, T.RenderConfig.make(sh_degree=0, aa="filter3d_original"))
    s2, _, _, _ = O.preprocess(_one(log_scale=math.log(2.0)), 1, cam, T.RenderConfig.make(sh_degree=0))
    assert abs(s1[0, 3] - 0.5 / 8) <= 1e-6
    np.testing.assert_allclose(s1[0, [4, 5, 6, 11]], s2[0, [4, 5, 6, 11]], rtol=1e-5)
    # nu -> infinity: the filter vanishes
    O.set_sampling_rates(np.array([1e15], np.float32))
    s3, _, _, _ = O.preprocess(p, 1, cam, T.RenderConfig.make(sh_degree=0, aa="filter3d_original"))
    s4, _, _, _ = O.preprocess(p, 1, cam, T.RenderConfig.make(sh_degree=0))
    assert np.array_equal(s3, s4)


def test_filter3d_clip_examples():  # SPEC.md:641-644 + idempotence (:660)
    n = 3
    p = T.pack_params([[0, 0, 0]] * n, [[math.log(0.2)] * 3, [math.log(0.01)] * 3, [math.log(0.01), 0.0, -1.0]],
                      [[1, 0, 0, 0]] * n, [0.0] * n, [[0, 0, 0]] * n, np.zeros((n, 15, 3)))
    kappa = 0.2
    nu = np.full(n, math.sqrt(kappa) / 0.05, np.float32)  # floor = 0.05
    q = O.apply_3d_filter_clip(p, n, nu, kappa)
    ls = q[3 * n:6 * n].reshape(n, 3)
    assert np.array_equal(ls[0], p[3 * n:6 * n].reshape(n, 3)[0])  # above the floor: unchanged
    np.testing.assert_allclose(np.exp(ls[1]), 0.05, rtol=1e-6)  # 0.01 -> 0.05
    assert abs(math.exp(ls[2, 0]) - 0.05) < 1e-7 and ls[2, 1] == 0.0 and ls[2, 2] == np.float32(-1.0)
    assert np.array_equal(O.apply_3d_filter_clip(q, n, nu, kappa), q)  # idempotent


def test_mip_compensation_properties():
    rng = np.random.default_rng(7)
    n = 400
    p = scene.random_params(n, 0.01, 0.5, 17)
    cam = scene.make_camera(128, 96)
    off, _, _, _ = O.preprocess(p, n, cam, T.RenderConfig.make(sh_degree=0, dilation=0.1))
    on, _, _, _ = O.preprocess(p, n, cam, T.RenderConfig.make(sh_degree=0, aa="full"))
    vis = off[:, 11] > 0
    assert vis.sum() > 100
    o, oh = off[vis, 3], on[vis, 3]
    assert np.all(oh <= o) and np.all(oh > 0)  # compensation in (0, o]
    # det_post = det(Sigma2D + 0.1 I) (splat field 11); for diagonal-dominant splats det_pre = det_post - 0.1 tr - 0.01
    assert np.array_equal(off[vis][:, 11], on[vis][:, 11])
    # tiny splats fade (ratio well below 1); big splats (det_pre >> dilation) are barely compensated
    assert (oh / o).min() < 0.9
    pb = scene.random_params(n, 0.2, 0.5, 18)
    offb, _, _, _ = O.preprocess(pb, n, cam, T.RenderConfig.make(sh_degree=0, dilation=0.1))
    onb, _, _, _ = O.preprocess(pb, n, cam, T.RenderConfig.make(sh_degree=0, aa="full"))
    big = offb[:, 11] > 1e3
    assert big.sum() > 10 and np.all(onb[big, 3] / offb[big, 3] > 0.99)
    del rng


def _fd_check(aa, classes, seed=3):
    rng = np.random.default_rng(seed)
    n, W, H = 14, 32, 32
    p = scene.random_params(n, 0.12, 1.0, 60 + seed).astype(np.float64)
    p[0:3 * n] *= 0.6
    cam = scene.make_camera(W, H, eye=(0.2, -0.3, -3.0))
    cfg = T.RenderConfig.make(sh_degree=2, bg=(0.1, 0.2, 0.3), aa=aa)
    O.set_sampling_rates(rng.uniform(8.0, 20.0, n).astype(np.float32))
    tgt = rng.uniform(0, 1, (H, W, 3))

    def loss(pp):
        rgb, _, _, _ = O.render(pp, n, cam, cfg, f64=True)
        return np.mean((rgb - tgt) ** 2), rgb

    _, rgb = loss(p)
    G, _, _, _ = O.backward(p, n, cam, cfg, 2 * (rgb - tgt) / rgb.size, f64=True)
    for (a, b), name in zip(T.group_slices(n), T.GROUPS):
        if name not in classes:
            continue
        idx = np.arange(a, b)
        if len(idx) > 40:
            idx = rng.choice(idx, 40, replace=False)
        ok = 0
        for i in idx:
            h = 1e-6 * max(1.0, abs(p[i]))
            pp = p.copy()
            pp[i] += h
            lp, _ = loss(pp)
            pp[i] -= 2 * h
            lm, _ = loss(pp)
            fd = (lp - lm) / (2 * h)
            scale = max(abs(fd), abs(G[i]), 1e-7)
            ok += abs(fd - G[i]) / scale < 1e-3
        assert ok / len(idx) >= 0.95, f"{aa} {name}: {ok}/{len(idx)}"


def test_filter3d_original_gradients_fd():  # full analytic chain through s_hat and the opacity factor
    _fd_check("filter3d_original", set(T.GROUPS))


def test_mip_gradients_fd_opacity_and_colour():
    # the Mip compensation is detached from Sigma2D, so only the opacity and
    # colour classes equal the finite differences of the full function
    _fd_check("full", {"opacity_logits", "sh_dc", "sh_rest"})


# ------------------------------------------------------------------- GPU ----
def _aa_scene():
    n = 30_000
    p = scene.random_params(n, 0.01, 0.3, 23)
    cams = scene.fibonacci_cameras(4, 320, 240)
    return p, n, cams


@pytest.mark.gpu
def test_gpu_sampling_rates_and_clip_bit_exact(engine):
    p, n, cams = _aa_scene()
    engine.set_params(p, n)
    engine.compute_sampling_rates(cams, 1.7)
    nu = engine.get_sampling_rates()
    onu = O.compute_sampling_rates(p, n, cams, 1.7)
    assert np.array_equal(nu.view(np.uint32), onu.view(np.uint32))
    engine.apply_3d_filter_clip(0.2)
    q = engine.get_params()
    oq = O.apply_3d_filter_clip(p, n, onu, 0.2)
    assert np.array_equal(q.view(np.uint32), oq.view(np.uint32))


@pytest.mark.gpu
@pytest.mark.parametrize("aa", ["filter3d_original", "filter3d_clip", "full"])
def test_gpu_antialias_parity(engine, aa):
    p, n, cams = _aa_scene()
    cam = cams[0]
    cfg = T.RenderConfig.make(sh_degree=2, aa=aa)
    engine.set_params(p, n)
    engine.compute_sampling_rates(cams, 1.7)
    onu = O.compute_sampling_rates(p, n, cams, 1.7)
    O.set_sampling_rates(onu)
    # preprocess: tile counts, rects and the exact-op splat fields bitwise
    engine.render(cam, cfg, outputs=False)
    gs, gr, gc, gk = engine.debug_preprocess()
    os_, or_, oc, ok = O.preprocess(p, n, cam, cfg)
    assert np.array_equal(gc, oc) and np.array_equal(gk, ok)
    vis = oc > 0
    exact = [0, 1, 2, 3, 4, 5, 6, 7, 11]
    assert np.array_equal(gs[vis][:, exact].view(np.uint32), os_[vis][:, exact].view(np.uint32))
    keys, vals, ranges = engine.debug_instances()
    okk, ov, orr, _ = O.instances(p, n, cam, cfg, sort="combined")
    assert np.array_equal(keys, okk) and np.array_equal(vals, ov) and np.array_equal(ranges, orr)
    # image and gradients
    rgb, _, _ = engine.render(cam, cfg)
    orgb, _, _, _ = O.render(p, n, cam, cfg)
    assert np.abs(rgb - orgb).max() <= 1e-4
    rng = np.random.default_rng(2)
    dL = rng.normal(0, 1e-3, rgb.shape).astype(np.float32)
    engine.zero_grads()
    engine.backward(dL)
    G, _, _, _, _ = engine.get_state()
    oG, _, _, _ = O.backward(p, n, cam, cfg, dL)
    for (a, b), name in zip(T.group_slices(n), T.GROUPS):
        g, o = G[a:b], oG[a:b]
        floor = 1e-3 * np.sqrt(np.mean(o ** 2)) + 1e-12
        rel = np.abs(g - o) / np.maximum(np.abs(o), floor)
        assert np.mean(rel < 1e-3) >= 0.99, f"{aa} {name}: {np.mean(rel < 1e-3):.4f}"
