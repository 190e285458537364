"""PLY import/export, checkpoint = PLY + config + optimizer
sidecar, TrainConfig and the train-op
schedule with resume determinism."""
import os
import subprocess

import numpy as np
import pytest

from paper_2602_09999_b200 import checkpoint as ckpt
from paper_2602_09999_b200 import ply, scene, types as T
from paper_2602_09999_b200.config import ConfigError, DensifySchedule, TrainConfig, events

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TS_PLY = os.path.join(ROOT, "tools", "ts_ply")


def _store(n=257, seed=0):
    p = scene.random_params(n, 0.02, 0.0, seed)
    rng = np.random.default_rng(seed)
    p[14 * n:] = rng.normal(0, 0.3, 45 * n).astype(np.float32)   # non-trivial sh_rest
    p[0] = np.float32(1e-38)                                      # subnormal-adjacent value survives ascii
    p[1] = np.float32(-3.4e38)
    return p, n


@pytest.mark.parametrize("binary", [True, False])
def test_ply_roundtrip_bitwise(tmp_path, binary):
    p, n = _store()
    f = tmp_path / "s.ply"
    ply.write_ply(f, p, n, binary=binary)
    q, m = ply.read_ply(f)
    assert m == n and np.array_equal(p.view(np.uint32), q.view(np.uint32))


def test_ply_layout_channel_major(tmp_path):
    n = 3
    p, _ = _store(n)
    rest = np.zeros((n, 15, 3), np.float32)
    for k in range(15):
        for c in range(3):
            rest[:, k, c] = 100 * c + k
    p[14 * n:] = rest.reshape(-1)
    f = tmp_path / "s.ply"
    ply.write_ply(f, p, n)
    data = f.read_bytes()
    header, body = data.split(b"end_header\n", 1)
    names = [l.split()[2].decode() for l in header.splitlines() if l.startswith(b"property")]
    assert names == ply.PROPERTIES and len(names) == 59
    rows = np.frombuffer(body, "<f4").reshape(n, 59)
    for c in range(3):
        for k in range(15):
            assert np.all(rows[:, names.index(f"f_rest_{c * 15 + k}")] == 100 * c + k)
    means, ls, q, op, dc, _ = T.unpack_params(p, n)
    assert np.array_equal(rows[:, 0:3], means) and np.array_equal(rows[:, 51], op)
    assert np.array_equal(rows[:, 52:55], ls) and np.array_equal(rows[:, 55:59], q)
    assert np.array_equal(rows[:, 3:6], dc)


def test_ply_reader_tolerates_extras(tmp_path):
    # 3DGS files carry nx ny nz; types and order may differ; other elements may follow
    p, n = _store(5)
    rows = ply.params_to_rows(p, n)
    order = list(range(59))[::-1]
    props = ["nx", "ny", "nz"] + [ply.PROPERTIES[i] for i in order]
    dt = np.dtype([(nm, "<f8" if nm.startswith("f_rest") else "<f4") for nm in props])
    rec = np.zeros(n, dt)
    for i in order:
        rec[ply.PROPERTIES[i]] = rows[:, i]
    head = ["ply", "format binary_little_endian 1.0", "comment made by test", f"element vertex {n}"]
    head += [f"property {'double' if nm.startswith('f_rest') else 'float'} {nm}" for nm in props]
    head += ["element face 0", "property list uchar int vertex_indices", "end_header"]
    f = tmp_path / "x.ply"
    f.write_bytes(("\n".join(head) + "\n").encode() + rec.tobytes())
    q, m = ply.read_ply(f)
    assert m == n and np.array_equal(p, q)


def test_ply_reader_errors(tmp_path):
    f = tmp_path / "bad.ply"
    f.write_bytes(b"nope\n")
    with pytest.raises(ply.PlyError):
        ply.read_ply(f)
    p, n = _store(4)
    ply.write_ply(f, p, n)
    data = f.read_bytes().replace(b"property float rot_3\n", b"")
    f.write_bytes(data)
    with pytest.raises(ply.PlyError):
        ply.read_ply(f)
    ply.write_ply(f, p, n)
    f.write_bytes(f.read_bytes()[:-10])
    with pytest.raises(ply.PlyError):
        ply.read_ply(f)


@pytest.mark.skipif(not os.path.exists(TS_PLY), reason="tools/ts_ply not built")
@pytest.mark.parametrize("fmt", ["binary", "ascii"])
def test_cpp_codec_matches_python(tmp_path, fmt):
    """include/tilesplat/ply.hpp (C++) and ply.py write the same bytes and read each other."""
    p, n = _store(101)
    a, b, c = tmp_path / "a.ply", tmp_path / "b.ply", tmp_path / "c.ply"
    ply.write_ply(a, p, n, binary=(fmt == "binary"))
    subprocess.run([TS_PLY, str(a), str(b), fmt], check=True, capture_output=True)
    assert a.read_bytes() == b.read_bytes()
    # C++ reads the ascii file and writes binary; Python reads it back bitwise
    subprocess.run([TS_PLY, str(b), str(c), "binary"], check=True, capture_output=True)
    q, m = ply.read_ply(c)
    assert m == n and np.array_equal(p.view(np.uint32), q.view(np.uint32))
    r = subprocess.run([TS_PLY, str(tmp_path / "missing.ply"), str(c)], capture_output=True)
    assert r.returncode == 1


def test_checkpoint_roundtrip(tmp_path):
    p, n = _store(64)
    rng = np.random.default_rng(1)
    m = rng.normal(size=59 * n).astype(np.float32)
    v = np.abs(rng.normal(size=59 * n)).astype(np.float32)
    acc, cnt = rng.random(n).astype(np.float32), rng.integers(0, 9, n).astype(np.float32)
    cfg = TrainConfig(seed=7, total_iterations=1234, densify=DensifySchedule(end=1000))
    ckpt.save(tmp_path / "ck", p, n, 4321, m, v, acc, cnt, config=cfg)
    ck = ckpt.load(tmp_path / "ck")
    assert ck["n"] == n and ck["step"] == 4321 and ck["config"] == cfg
    for k, a in (("params", p), ("m", m), ("v", v), ("accum", acc), ("vcount", cnt)):
        assert np.array_equal(ck[k], a), k
    # sidecar must match the PLY
    ckpt.write_optimizer_state(tmp_path / "ck" / "optimizer.bin", n - 1, 1, m[:59 * (n - 1)], v[:59 * (n - 1)],
                               acc[:-1], cnt[:-1])
    with pytest.raises(ply.PlyError):
        ckpt.load(tmp_path / "ck")


def test_train_config_serialisation():
    c = TrainConfig(seed=3, optimizer_mode=T.ADAM_SKIP_INVISIBLE, morton=False, output_dir="/tmp/x")
    c.densify.grad_threshold = 3e-4
    assert TrainConfig.loads(c.dumps()) == c
    with pytest.raises(ConfigError):
        TrainConfig.from_dict({**c.to_dict(), "bogus": 1})
    with pytest.raises(ConfigError):
        TrainConfig.from_dict({**c.to_dict(), "densify": {"nope": 1}})
    d = c.override(["seed=11", "densify.interval=50", "sort_mode=combined"])
    assert d.seed == 11 and d.densify.interval == 50 and d.sort_mode == "combined"
    with pytest.raises(ConfigError):
        c.override(["densify.bogus=1"])
    with pytest.raises(ConfigError):
        TrainConfig(densify=DensifySchedule(interval=0)).validate()
    with pytest.raises(ConfigError):
        TrainConfig(total_iterations=100).validate()   # densify end 14900 > total


def test_schedule_events():
    c = TrainConfig()
    dens = [it for it in range(1, 30001) if events(it, c).densify]
    assert dens[0] == 600 and dens[-1] == 14900 and len(dens) == (14900 - 600) // 100 + 1
    assert [it for it in range(1, 30001) if events(it, c).opacity_reset] == [3000, 6000, 9000, 12000]
    assert [it for it in range(1, 30001) if events(it, c).morton] == [5000, 10000]
    assert [it for it in range(1, 30001, 5000) if events(it, c).checkpoint] == []
    assert [it for it in range(1, 30001) if events(it, c).checkpoint][:2] == [5000, 10000]
    # rendering degree at iteration it is sh_active_degree(it - 1)
    assert [events(it, c).sh_degree for it in (1, 1000, 1001, 2001, 3001, 29000)] == [0, 0, 1, 2, 3, 3]
    assert not any(events(it, TrainConfig(morton=False)).morton for it in range(1, 15001))


def _toy(n=400, views=4, size=48):
    p = scene.random_params(n, 0.05, 0.5, 5)
    cams = scene.fibonacci_cameras(views, size, size)
    return p, n, cams


def test_trainer_resume_bitwise_cpu(tmp_path):
    """Oracle-backed engine: uninterrupted run == run interrupted at a checkpoint and resumed."""
    from oracle import oracle as O
    from paper_2602_09999_b200.trainer import Trainer
    from tests.cpu_engine import OracleTrainEngine

    p, n, cams = _toy()
    rc = T.RenderConfig.make(sh_degree=0)
    targets = [O.render(scene.perturb(p, n, 9), n, c, rc)[0] for c in cams]
    sched = DensifySchedule(warmup=2, interval=2, end=8, opacity_reset_interval=6, morton_interval=4, sh_ramp=3)

    def cfg(out):
        return TrainConfig(total_iterations=10, seed=5, checkpoint_interval=5, output_dir=str(out), densify=sched)

    a = Trainer(OracleTrainEngine(p, n), cams, targets, cfg(tmp_path / "a"))
    la = a.run()
    assert la.densify and la.mortons == [4, 8] and la.resets == [6] and la.checkpoints == [5, 10]
    b = Trainer(OracleTrainEngine(p, n), cams, targets, cfg(tmp_path / "b"))
    b.run(1, 5)
    c = Trainer(OracleTrainEngine(p[:59], 1), cams, targets, cfg(tmp_path / "c"))
    start = c.resume(b.checkpoint_dir(5))
    assert start == 6
    c.run(start)
    assert a.e.n == c.e.n
    assert np.array_equal(a.e.P, c.e.P) and np.array_equal(a.e.M, c.e.M) and np.array_equal(a.e.V, c.e.V)
    assert la.losses[5:] == c.log.losses


@pytest.mark.gpu
def test_engine_checkpoint_and_trainer_gpu(tmp_path, engine):
    from paper_2602_09999_b200.trainer import Trainer

    p, n, cams = _toy(4000, 6, 96)
    rc = T.RenderConfig.make(sh_degree=3)
    engine.set_params(scene.perturb(p, n, 9), n)
    targets = [engine.render(c, rc)[0] for c in cams]
    engine.set_params(p, n)
    sched = DensifySchedule(warmup=10, interval=10, end=40, opacity_reset_interval=30, morton_interval=20)
    cfg = TrainConfig(total_iterations=60, seed=1, checkpoint_interval=25, output_dir=str(tmp_path), densify=sched)
    tr = Trainer(engine, cams, targets, cfg)
    log = tr.run()
    assert log.checkpoints == [25, 50] and log.mortons == [20, 40] and len(log.densify) == 4
    assert np.mean(log.losses[22:29]) < np.mean(log.losses[:6])
    assert log.resets == [30] and log.losses[30] > log.losses[28]   # opacity reset darkens the next render
    # save -> load restores the device state bitwise
    tr.save(60)
    before = engine.get_params(), engine.get_state()
    engine.set_params(p, n)
    assert tr.resume(tr.checkpoint_dir(60)) == 61
    after = engine.get_params(), engine.get_state()
    assert np.array_equal(before[0], after[0])
    for x, y in zip(before[1][1:], after[1][1:]):
        assert np.array_equal(x, y)


def test_train_config_antialias_modes():
    for m in ("off", "filter3d_original", "filter3d_clip", "full"):
        TrainConfig(aa_mode=m).validate()
    with pytest.raises(ConfigError):
        TrainConfig(aa_mode="mip").validate()
    with pytest.raises(ConfigError):
        TrainConfig(aa_mode="full", kappa3d=0.0).validate()
    c = TrainConfig(aa_mode="full").override(["rate_interval=50"])
    assert c.aa_mode == "full" and c.rate_interval == 50


@pytest.mark.gpu
@pytest.mark.parametrize("aa", ["filter3d_original", "full"])
def test_trainer_antialias_gpu(engine, aa):
    """Training with antialiasing: sampling rates refreshed on the schedule
    and after densification, the clip applied after every optimizer step ("full"); the loss
    falls and, for the clip modes, every scale ends at or above sqrt(kappa)/nu."""
    from paper_2602_09999_b200.trainer import Trainer

    p, n, cams = _toy(4000, 6, 96)
    rc = T.RenderConfig.make(sh_degree=3)
    engine.set_params(scene.perturb(p, n, 9), n)
    targets = [engine.render(c, rc)[0] for c in cams]
    engine.set_params(p, n)
    sched = DensifySchedule(warmup=10, interval=10, end=30, opacity_reset_interval=1000, morton_interval=1000)
    cfg = TrainConfig(total_iterations=40, seed=2, densify=sched, aa_mode=aa, rate_interval=15)
    log = Trainer(engine, cams, targets, cfg).run()
    assert len(log.densify) == 3 and all(np.isfinite(log.losses))
    assert np.mean(log.losses[-6:]) < np.mean(log.losses[:6])
    if aa == "full":
        nu = engine.get_sampling_rates()
        N = engine.num_gaussians()
        s = np.exp(engine.get_params()[3 * N:6 * N].reshape(N, 3).astype(np.float64))
        floor = np.sqrt(cfg.kappa3d) / nu.astype(np.float64)
        assert np.all(s >= floor[:, None] * (1 - 1e-5))
