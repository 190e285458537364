"""C-ABI error contract on the device path: bad inputs and
out-of-order calls return TS_ERR_VALIDATION with a message (ValidationError in the Python
mirror) and launch nothing; the context stays usable and renders bit-identically after."""
import numpy as np
import pytest

from paper_2602_09999_b200 import scene, types as T
from paper_2602_09999_b200.tilesplat import ValidationError

pytestmark = pytest.mark.gpu


def _small():
    p = scene.random_params(800, 0.05, 0.0, 3)
    return p, 800, scene.make_camera(64, 48), T.RenderConfig.make(sh_degree=1)


def _bad_cfg(**kw):
    cfg = T.RenderConfig.make(sh_degree=1)
    for k, v in kw.items():
        setattr(cfg, k, v)
    return cfg


@pytest.mark.parametrize("field,value", [("sh_degree", 4), ("sh_degree", -1), ("bound_mode", 3), ("cull_mode", 2),
                                         ("truncation", 2), ("backward_mode", 2), ("tau_alpha", 0.0),
                                         ("tau_alpha", 1.0), ("dilation", -0.1), ("aa_mode", 4)])
def test_bad_render_config(engine, field, value):
    p, n, cam, cfg = _small()
    engine.set_params(p, n)
    ref, _, _ = engine.render(cam, cfg)
    l0 = engine.launch_count()
    with pytest.raises(ValidationError):
        engine.render(cam, _bad_cfg(**{field: value}))
    assert engine.launch_count() == l0
    again, _, _ = engine.render(cam, cfg)
    assert np.array_equal(ref, again)


@pytest.mark.parametrize("kw", [dict(truncation=1, sigma_cut=0.0), dict(backward_mode=1, early_stop_compat=1)])
def test_bad_render_config_combinations(engine, kw):
    p, n, cam, cfg = _small()
    engine.set_params(p, n)
    with pytest.raises(ValidationError):
        engine.render(cam, _bad_cfg(**kw))


def test_bad_camera(engine):
    p, n, cam, cfg = _small()
    engine.set_params(p, n)
    bad = scene.make_camera(64, 48)
    bad.fx = 0.0
    with pytest.raises(ValidationError):
        engine.render(bad, cfg)
    huge = scene.make_camera(16 * 4100, 16 * 4100)  # >= 2^24 tiles (beyond the 32-bit key path's limit)
    with pytest.raises(ValidationError):
        engine.render(huge, cfg)


def test_call_order(engine):
    p, n, cam, cfg = _small()
    engine.set_params(p, n)
    with pytest.raises(ValidationError):
        engine.training_loss(np.zeros((48, 64, 3), np.float32))  # no forward yet
    with pytest.raises(ValidationError):
        engine.backward(None)  # no forward / loss
    engine.render(cam, cfg, outputs=False)
    with pytest.raises(ValidationError):
        engine.backward(None)  # forward but no loss: dL/dC unknown
    with pytest.raises(ValidationError):
        engine.training_loss(slot=99)  # no such target slot
    with pytest.raises(ValidationError):
        engine.adam_step(T.AdamConfig.make(step=1, mode=3))  # modes 3/4 run inside the backward
    a = T.AdamConfig.make(step=1)
    a.bc1 = 0.0
    with pytest.raises(ValidationError):
        engine.adam_step(a)
    with pytest.raises(ValidationError):
        engine.adam_step(T.AdamConfig.make(step=1), begin=10, end=59 * n + 1)


def test_antialias_preconditions(engine):
    p, n, cam, cfg = _small()
    engine.set_params(p, n)  # new store: no sampling rates
    with pytest.raises(ValidationError):
        engine.render(cam, T.RenderConfig.make(sh_degree=1, aa="filter3d_original"))
    with pytest.raises(ValidationError):
        engine.apply_3d_filter_clip(0.2)
    with pytest.raises(ValidationError):
        engine.compute_sampling_rates([cam], 0.0)
    engine.compute_sampling_rates([cam], 1.0)
    engine.render(cam, T.RenderConfig.make(sh_degree=1, aa="filter3d_original"), outputs=False)


def test_morton_between_backward_and_step(engine):
    p, n, cam, cfg = _small()
    engine.set_params(p, n)
    engine.render(cam, cfg, outputs=False)
    engine.backward(np.zeros((48, 64, 3), np.float32))
    with pytest.raises(ValidationError):
        engine.morton_reorder()
    engine.adam_step(T.AdamConfig.make(step=1))
    engine.morton_reorder()
