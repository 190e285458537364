"""End-to-end training on a toy scene (SPEC.md acceptance 9 and 10, the GPU path).

A store of 3000 seeded Gaussians renders 8 ring targets and one held-out view; the training store is
the same scene with perturbed means, scales, opacities and colours.  `ts_train_step` (forward, fused
L1 + D-SSIM loss, backward, Adam with the SPEC learning-rate schedule) over the 8 targets must bring
the held-out view to >= 30 dB PSNR (acceptance 9's threshold; the PSNR is computed here in the test,
metrics are not part of the product), and skip-invisible Adam must end elsewhere than the reference
optimizer (acceptance 10: "slightly degrades quality", non-zero divergence)."""
import math

import numpy as np
import pytest

from paper_2602_09999_b200 import scene, types as T

pytestmark = pytest.mark.gpu


def _psnr(a, b):
    return 10.0 * math.log10(1.0 / max(float(np.mean((a - b) ** 2)), 1e-12))


def _toy(engine, mode, steps):
    n, W, H = 3000, 160, 120
    gt = scene.random_params(n, 0.04, 0.5, 5)
    cams = scene.fibonacci_cameras(9, W, H)
    train, held = cams[:8], cams[8]
    cfg = T.RenderConfig.make(sh_degree=1)
    engine.set_params(gt, n)
    targets = [engine.render(c, cfg)[0].copy() for c in train]
    hold = engine.render(held, cfg)[0].copy()
    rng = np.random.default_rng(1)
    p = gt.copy()
    p[0:3 * n] += rng.normal(0, 0.03, 3 * n).astype(np.float32)
    p[3 * n:6 * n] += rng.normal(0, 0.2, 3 * n).astype(np.float32)
    p[10 * n:11 * n] += rng.normal(0, 0.5, n).astype(np.float32)
    p[11 * n:14 * n] += rng.normal(0, 0.3, 3 * n).astype(np.float32)
    engine.set_params(p, n)
    for k, t in enumerate(targets):
        engine.set_target(k, t)
    before = _psnr(engine.render(held, cfg)[0], hold)
    losses = []
    for s in range(1, steps + 1):
        losses.append(engine.train_step(train[s % 8], cfg, T.AdamConfig.make(step=s, extent=3.5, mode=mode),
                                        slot=s % 8))
    after = _psnr(engine.render(held, cfg)[0], hold)
    return before, after, losses, engine.get_params()


def test_toy_scene_reaches_30db_heldout(engine):
    before, after, losses, _ = _toy(engine, T.ADAM_FUSED, 1000)
    assert before < 25.0, before
    assert after >= 30.0, (before, after)
    assert np.mean(losses[-50:]) < 0.5 * np.mean(losses[:50])


def test_skip_invisible_diverges_from_reference(engine):
    _, a_ref, _, p_ref = _toy(engine, T.ADAM_FUSED, 200)
    _, a_skip, _, p_skip = _toy(engine, T.ADAM_SKIP_INVISIBLE, 200)
    assert not np.array_equal(p_ref, p_skip)
    assert np.isfinite(a_skip) and a_skip > 20.0
