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
