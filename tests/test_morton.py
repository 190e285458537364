"""morton_reorder.

CPU: the oracle against SPEC's worked examples and properties.
GPU: ts_morton_reorder's permutation equals the oracle's (bit-exact: codes
are integer work on exact-op quantisation), every per-Gaussian array is
permuted identically, and rendering is bitwise unchanged."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2602_09999_b200 import scene, types as T


def _means_params(means):
    n = len(means)
    p = scene.random_params(n, 0.01, 0.0, 5)
    p[:3 * n] = np.asarray(means, np.float32).reshape(-1)
    return p, n


def test_interleave_examples():
    # 1-bit toy quantisation, (1,1,1) -> 7, x in the LSB
    assert O.morton_interleave(1, 1, 1, 1) == 7
    assert O.morton_interleave(1, 0, 0, 1) == 1
    assert O.morton_interleave(0, 1, 0, 1) == 2
    assert O.morton_interleave(0, 0, 1, 1) == 4
    assert O.morton_interleave(2, 0, 0, 2) == 8
    full = (1 << 21) - 1
    assert O.morton_interleave(full, full, full, 21) == (1 << 63) - 1


def test_unit_cube_origin_first():
    # (0,0,0) in the unit cube -> code 0, first after the sort
    corners = [(x, y, z) for z in (0, 1) for y in (0, 1) for x in (0, 1)]
    rng = np.random.default_rng(0)
    pts = np.concatenate([rng.random((50, 3)), np.array(corners[::-1], np.float64)])
    p, n = _means_params(pts)
    codes = O.morton_codes(p, n)
    i0 = n - 1  # (0,0,0) was appended last
    assert codes[i0] == 0
    perm = O.morton_reorder(p.copy(), n)
    assert perm[0] == i0
    # the max corner stays inside the 21-bit grid (AABB inflated by 1e-6)
    assert codes[n - 8] < (1 << 63)


def test_octant_monotone():
    # codes of a child octant form a contiguous interval -> after
    # sorting, the top 3 bits (first-level octant) are non-decreasing
    rng = np.random.default_rng(1)
    p, n = _means_params(rng.normal(0, 1, (4000, 3)))
    codes = O.morton_codes(p, n)
    perm = O.morton_reorder(p.copy(), n)
    sc = codes[perm]
    assert np.all(np.diff(sc.astype(np.float64)) >= 0)
    for level in (1, 2, 3):
        oct_ = sc >> np.uint64(63 - 3 * level)
        assert np.all(np.diff(oct_.astype(np.int64)) >= 0)


def test_reorder_permutes_every_array():
    rng = np.random.default_rng(2)
    n = 3000
    p = scene.random_params(n, 0.02, 0.0, 3)
    m = rng.normal(size=59 * n).astype(np.float32)
    v = np.abs(rng.normal(size=59 * n)).astype(np.float32)
    acc = rng.random(n).astype(np.float32)
    vc = rng.integers(0, 5, n).astype(np.float32)
    p2, m2, v2, acc2, vc2 = p.copy(), m.copy(), v.copy(), acc.copy(), vc.copy()
    perm = O.morton_reorder(p2, n, m2, v2, acc2, vc2)
    assert np.array_equal(np.sort(perm), np.arange(n))
    for a, b in ((p, p2), (m, m2), (v, v2)):
        for g_old, g_new in zip(T.unpack_params(a, n), T.unpack_params(b, n)):
            assert np.array_equal(g_new, g_old[perm])
    assert np.array_equal(acc2, acc[perm]) and np.array_equal(vc2, vc[perm])


def test_stable_ties():
    # duplicated means keep their original relative order
    pts = np.array([[0.5, 0.5, 0.5]] * 5 + [[0.0, 0.0, 0.0], [1.0, 1.0, 1.0]])
    p, n = _means_params(pts)
    perm = O.morton_reorder(p.copy(), n)
    assert list(perm) == [5, 0, 1, 2, 3, 4, 6]


def _untied_scene(name, sh):
    """SPEC.md:247 breaks exact depth-key ties by Gaussian index, so SPEC.md:878's
    bitwise invariance can only hold for scenes without exact ties (random fp32
    depths collide ~n^2/2^23 times): drop the later member of every tie."""
    w = scene.WORKLOADS[name]
    p = scene.random_params(w.n, w.s0, w.m_o, w.seed)
    cam = scene.workload_cameras(w)[0]
    cfg = T.RenderConfig.make(sh_degree=sh)
    _, _, cnt, dkey = O.preprocess(p, w.n, cam, cfg)
    _, first = np.unique(dkey, return_index=True)
    keep = np.zeros(w.n, bool)
    keep[first] = True
    keep |= cnt == 0
    groups = [g[keep] for g in T.unpack_params(p, w.n)]
    n = int(keep.sum())
    return T.pack_params(*groups), n, cam, cfg


def test_render_invariant_cpu():
    # SPEC.md:878 on the oracle (small scene)
    p, n, cam, cfg = _untied_scene("c1", 0)
    a = O.render(p, n, cam, cfg)
    q = p.copy()
    O.morton_reorder(q, n)
    b = O.render(q, n, cam, cfg)
    assert np.array_equal(a[0], b[0])


@pytest.mark.gpu
def test_morton_gpu_matches_oracle(engine):
    rng = np.random.default_rng(3)
    n = 200_000
    p = scene.random_params(n, 0.01, 0.0, 21)
    m = rng.normal(size=59 * n).astype(np.float32)
    v = np.abs(rng.normal(size=59 * n)).astype(np.float32)
    acc = rng.random(n).astype(np.float32)
    vc = rng.integers(0, 5, n).astype(np.float32)
    engine.set_params(p, n)
    engine.set_state(m=m, v=v, accum=acc, vcount=vc)
    perm = engine.morton_reorder()
    p2, m2, v2, acc2, vc2 = p.copy(), m.copy(), v.copy(), acc.copy(), vc.copy()
    operm = O.morton_reorder(p2, n, m2, v2, acc2, vc2)
    assert np.array_equal(perm, operm)
    assert np.array_equal(engine.get_params(), p2)
    _, gm, gv, gacc, gvc = engine.get_state()
    assert np.array_equal(gm, m2) and np.array_equal(gv, v2)
    assert np.array_equal(gacc, acc2) and np.array_equal(gvc, vc2)


@pytest.mark.gpu
def test_morton_render_bitwise_unchanged(engine):
    p, n, cam, cfg = _untied_scene("c2", 3)
    engine.set_params(p, n)
    rgb0, T0, c0 = engine.render(cam, cfg)
    engine.morton_reorder()
    rgb1, T1, c1 = engine.render(cam, cfg)
    assert np.array_equal(rgb0, rgb1) and np.array_equal(T0, T1) and np.array_equal(c0, c1)
