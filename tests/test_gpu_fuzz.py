"""Seeded fuzz of the CUDA path against the oracle over the render-configuration space:
Gaussian count, frame size (ragged edge tiles), SH degree, bound mode (square / rect /
opacity-aware rect), cull mode (rect only / exact), early-stop compatibility, opacity
threshold, dilation, background, Mip antialias.  Per case: tile lists, sorted keys and ranges
bit-exact; image and final T within 1e-4; contributor counts equal; parameter gradients
within 1e-3 relative for >= 99% of coordinates per class."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2602_09999_b200 import scene, types as T

pytestmark = pytest.mark.gpu


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(300, 6000))
    W, H = int(rng.integers(24, 300)), int(rng.integers(24, 220))
    p = scene.random_params(n, float(rng.uniform(0.01, 0.08)), float(rng.uniform(-2.0, 1.5)), 500 + seed)
    eye = tuple(rng.uniform(-1.0, 1.0, 3) + np.array([0.0, 0.0, -3.2]))
    cam = scene.make_camera(W, H, eye=eye, fov_x_deg=float(rng.uniform(40.0, 80.0)))
    cfg = T.RenderConfig.make(sh_degree=int(rng.integers(0, 4)), bound_mode=int(rng.integers(0, 3)),
                              cull_mode=int(rng.integers(0, 2)), early_stop_compat=int(rng.integers(0, 2)),
                              tau_alpha=float(rng.choice([1.0 / 255.0, 0.01, 0.05])),
                              dilation=float(rng.choice([0.3, 0.1, 0.0])),
                              bg=tuple(float(x) for x in rng.uniform(0, 1, 3)),
                              aa=str(rng.choice(["off", "off", "full"])))
    return p, n, cam, cfg


@pytest.mark.parametrize("seed", range(40))
def test_fuzz_render_and_gradients(engine, seed):
    p, n, cam, cfg = _case(seed)
    engine.set_params(p, n)
    rgb, Tf, cnt = engine.render(cam, cfg)
    gk, gv, gr = engine.debug_instances()
    ok, ov, orr, _ = O.instances(p, n, cam, cfg, sort="combined")
    assert np.array_equal(gk, ok) and np.array_equal(gv, ov) and np.array_equal(gr, orr)
    orgb, oT, ocnt, _ = O.render(p, n, cam, cfg)
    assert np.abs(rgb - orgb).max() <= 1e-4 and np.abs(Tf - oT).max() <= 1e-4
    assert np.mean(cnt == ocnt) >= 0.999
    dl = np.random.default_rng(seed).normal(0, 1e-2, rgb.shape).astype(np.float32)
    engine.zero_grads()
    engine.backward(dl)
    G, _, _, _, _ = engine.get_state()
    oG, _, _, _ = O.backward(p, n, cam, cfg, dl)
    for (a, b), nm in zip(T.group_slices(n), T.GROUPS):
        g, o = G[a:b].astype(np.float64), oG[a:b].astype(np.float64)
        if not o.any():
            assert not g.any(), nm
            continue
        rms = np.sqrt(np.mean(o * o))
        frac = np.mean(np.abs(g - o) <= 1e-3 * np.maximum(np.abs(o), rms))
        assert frac >= 0.99, f"seed {seed} {nm}: {frac:.4f}"


@pytest.mark.parametrize("seed", range(12))
def test_fuzz_per_gaussian_backward(engine, seed):
    """The per-Gaussian bucket backward (render config backward_mode = 1) over the
    same configuration space (early-stop compat cases excluded: the option requires the standard stop)."""
    p, n, cam, cfg = _case(seed)
    cfg.early_stop_compat = 0
    cfg.backward_mode = T.BACKWARD_PER_GAUSSIAN
    engine.set_params(p, n)
    engine.render(cam, cfg, outputs=False)
    dl = np.random.default_rng(seed).normal(0, 1e-2, (cam.height, cam.width, 3)).astype(np.float32)
    engine.zero_grads()
    engine.backward(dl)
    G, _, _, _, _ = engine.get_state()
    oG, _, _, _ = O.backward(p, n, cam, cfg, dl)
    for (a, b), nm in zip(T.group_slices(n), T.GROUPS):
        g, o = G[a:b].astype(np.float64), oG[a:b].astype(np.float64)
        if not o.any():
            assert not g.any(), nm
            continue
        rms = np.sqrt(np.mean(o * o))
        frac = np.mean(np.abs(g - o) <= 1e-3 * np.maximum(np.abs(o), rms))
        assert frac >= 0.99, f"seed {seed} {nm}: {frac:.4f}"


@pytest.mark.parametrize("seed", range(12))
def test_fuzz_response_truncation(engine, seed):
    """fragment_alpha's response mode (truncation = 1: keep iff G >= exp(-sigma_cut^2/2),
    whatever the opacity) through the whole path: tile lists bit-exact, images, gradients."""
    p, n, cam, cfg = _case(seed)
    cfg.truncation = T.TRUNC_RESPONSE
    cfg.sigma_cut = float(np.random.default_rng(77 + seed).choice([3.33, 2.5, 3.0]))
    engine.set_params(p, n)
    rgb, Tf, cnt = engine.render(cam, cfg)
    gk, gv, gr = engine.debug_instances()
    ok, ov, orr, _ = O.instances(p, n, cam, cfg, sort="combined")
    assert np.array_equal(gk, ok) and np.array_equal(gv, ov) and np.array_equal(gr, orr)
    orgb, oT, ocnt, _ = O.render(p, n, cam, cfg)
    assert np.abs(rgb - orgb).max() <= 1e-4 and np.abs(Tf - oT).max() <= 1e-4
    assert np.mean(cnt == ocnt) >= 0.999
    dl = np.random.default_rng(seed).normal(0, 1e-2, rgb.shape).astype(np.float32)
    engine.zero_grads()
    engine.backward(dl)
    G, _, _, _, _ = engine.get_state()
    oG, _, _, _ = O.backward(p, n, cam, cfg, dl)
    for (a, b), nm in zip(T.group_slices(n), T.GROUPS):
        g, o = G[a:b].astype(np.float64), oG[a:b].astype(np.float64)
        if not o.any():
            assert not g.any(), nm
            continue
        rms = np.sqrt(np.mean(o * o))
        frac = np.mean(np.abs(g - o) <= 1e-3 * np.maximum(np.abs(o), rms))
        assert frac >= 0.99, f"seed {seed} {nm}: {frac:.4f}"


@pytest.mark.parametrize("dilation", [0.3, 0.0])
def test_needles_row_cull_conservative(engine, dilation):
    """High-aspect needles (2D variance up to ~1e5 px^2 along the long axis, sub-pixel across):
    the blend kernels' per-warp row cull bounds each splat by the half-height of its
    alpha >= tau ellipse computed from the rounded conic; it must never drop a fragment
    the exact Q <= k2 test keeps (fp32 cancellation in A C - B^2)."""
    rng = np.random.default_rng(77)
    n = 600
    p = scene.random_params(n, 0.01, 1.0, 78)
    long_axis = np.log(rng.uniform(0.05, 1.5, n))
    ls = np.stack([long_axis, np.full(n, np.log(2e-4)), np.full(n, np.log(2e-4))], 1)
    p[3 * n:6 * n] = ls.astype(np.float32).ravel()
    p[0:3 * n] = rng.uniform(-0.6, 0.6, 3 * n).astype(np.float32)
    cam = scene.make_camera(640, 480, eye=(0.2, -0.3, -3.0))
    cfg = T.RenderConfig.make(sh_degree=1, dilation=dilation)
    engine.set_params(p, n)
    rgb, Tf, cnt = engine.render(cam, cfg)
    orgb, oT, ocnt, _ = O.render(p, n, cam, cfg)
    assert np.abs(rgb - orgb).max() <= 1e-4 and np.abs(Tf - oT).max() <= 1e-4
    assert np.array_equal(cnt, ocnt)
    # the backward replays the same fragments: its colour / opacity 2D gradients (well conditioned,
    # unlike the mean / conic ones of a needle, whose fp32 rounding cancels catastrophically)
    # would lose every fragment a too-tight row cull dropped
    dl = np.random.default_rng(79).normal(0, 1e-2, rgb.shape).astype(np.float32)
    g2 = engine.debug_grad2d(dl)
    _, o2, _, _ = O.backward(p, n, cam, cfg, dl)
    for k, nm in ((5, "do"), (6, "dr"), (7, "dg"), (8, "db")):
        g, o = g2[:, k].astype(np.float64), o2[:, k].astype(np.float64)
        rms = np.sqrt(np.mean(o * o)) + 1e-30
        assert np.mean(np.abs(g - o) <= 1e-3 * np.maximum(np.abs(o), rms)) >= 0.99, nm
