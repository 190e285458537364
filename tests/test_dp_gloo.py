"""Data-parallel step over views with world_size 2 on CPU (gloo): gradients of the
view batch are summed across ranks and both exchange modes leave
bitwise-identical parameters on every rank, equal to the single-process step."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2602_09999_b200 import scene, types as T

N = 1500
W, H = 64, 48


def _setup():
    p = scene.random_params(N, 0.04, 0.5, 3)
    cams = scene.fibonacci_cameras(2, W, H)
    cfg = T.RenderConfig.make(sh_degree=1)
    targets = [O.render(p, N, c, cfg)[0] for c in cams]
    return scene.perturb(p, N, 3), cams, cfg, targets


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, mode, out_dir):
    import torch.distributed as dist

    from paper_2602_09999_b200.dp import DataParallelStep
    from tests.cpu_engine import CpuEngine

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p0, cams, cfg, targets = _setup()
    e = CpuEngine(p0, N, targets)
    dp = DataParallelStep(e, mode=mode)
    for step in (1, 2):
        views = [(cams[v], cfg, v) for v in dp.my_views(len(cams))]
        dp.step(views, T.AdamConfig.make(step=step))
    dp.reduce_densify_stats()
    np.save(os.path.join(out_dir, f"p{rank}.npy"), e.P[:e.L])
    np.save(os.path.join(out_dir, f"c{rank}.npy"), e.cnt)
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["allreduce", "sharded", "chunked"])
def test_two_rank_step_equals_single_process(tmp_path, mode):
    from tests.cpu_engine import CpuEngine

    mp.spawn(_rank_main, args=(2, _free_port(), mode, str(tmp_path)), nprocs=2, join=True)
    p_r0, p_r1 = np.load(tmp_path / "p0.npy"), np.load(tmp_path / "p1.npy")
    assert np.array_equal(p_r0, p_r1), "replicas diverged"
    # single process: both views accumulated, then the same optimizer steps
    p0, cams, cfg, targets = _setup()
    e = CpuEngine(p0, N, targets)
    for step in (1, 2):
        for v, cam in enumerate(cams):
            e.render(cam, cfg)
            e.training_loss(slot=v)
            e.backward()
        e.adam_step(T.AdamConfig.make(step=step))
    assert np.array_equal(p_r0, e.P[:e.L])
    assert np.array_equal(np.load(tmp_path / "c0.npy"), e.cnt)


def test_shard_bounds_cover_buffer():
    from paper_2602_09999_b200.dp import shard_bounds
    for L in (1, 7, 59 * 1001, 1 << 20):
        for world in (1, 2, 3, 8):
            seen = 0
            for r in range(world):
                b, e, per = shard_bounds(L, world, r)
                assert b == min(L, seen) and per % 4 == 0
                seen = e
            assert seen == L
