"""ctypes binding of the CPU oracle (oracle/libtsoracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline leg, never by the product package.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "libtsoracle.so")

f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
vp = ctypes.c_void_p
i64 = ctypes.c_int64


def build():
    subprocess.check_call(["make", "-s", "-C", _HERE])


def _load():
    if not os.path.exists(_LIB):
        build()
    lib = ctypes.CDLL(_LIB)
    sig = {
        "tso_set_workers": (None, [ctypes.c_int]),
        "tso_get_workers": (ctypes.c_int, []),
        "tso_expf": (ctypes.c_float, [ctypes.c_float]),
        "tso_cos2pi": (ctypes.c_float, [ctypes.c_float]),
        "tso_logf": (ctypes.c_float, [ctypes.c_float]),
        "tso_rotation_from_quaternion_f64": (ctypes.c_int, [f64p, f64p]),
        "tso_build_covariance3d_f64": (None, [f64p, f64p, f64p]),
        "tso_eval_sh_f64": (None, [f64p, f64p, ctypes.c_int, f64p]),
        "tso_project_mean_f64": (ctypes.c_int, [vp, f64p, f64p, f64p]),
        "tso_project_covariance_f64": (None, [vp, f64p, f64p, f64p]),
        "tso_invert_cov2d_f64": (ctypes.c_int, [f64p, ctypes.c_double, f64p, ctypes.POINTER(ctypes.c_double)]),
        "tso_preprocess": (None, [i64, f32p, vp, vp, f32p, i32p, u32p, u32p]),
        "tso_build_instances": (i64, [i64, f32p, i32p, u32p, u32p, vp, vp, u64p, u32p]),
        "tso_sort_combined": (None, [i64, u64p, u32p]),
        "tso_sort_two_stage": (i64, [i64, ctypes.c_int, u64p, u32p]),
        "tso_tile_ranges": (None, [i64, u64p, ctypes.c_int32, u32p]),
        "tso_render": (i64, [i64, f32p, vp, vp, f32p, f32p, u32p]),
        "tso_render_f64": (i64, [i64, f64p, vp, vp, f64p, f64p, u32p]),
        "tso_render_weight_sum": (None, [i64, f32p, vp, vp, f64p]),
        "tso_training_loss": (ctypes.c_double, [ctypes.c_int32, ctypes.c_int32, f32p, f32p, f32p]),
        "tso_training_loss_f64": (ctypes.c_double, [ctypes.c_int32, ctypes.c_int32, f64p, f64p, f64p]),
        "tso_backward": (None, [i64, f32p, vp, vp, f32p, f32p, f32p, f32p, f32p]),
        "tso_backward_f64": (None, [i64, f64p, vp, vp, f64p, f64p, f64p, f64p, f64p]),
        "tso_adam_step": (None, [i64, f32p, f32p, f32p, f32p, f32p, ctypes.c_float, ctypes.c_float,
                                 ctypes.c_float, ctypes.c_float, ctypes.c_float, ctypes.c_int32, vp]),
        "tso_adam_step_f64": (None, [i64, f64p, f64p, f64p, f64p, f64p, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_double, ctypes.c_double, ctypes.c_double]),
        "tso_mean_lr": (ctypes.c_double, [i64, ctypes.c_double]),
        "tso_densify_and_prune": (i64, [i64, f32p, f32p, f32p, f32p, f32p, ctypes.c_float, ctypes.c_float,
                                        ctypes.c_uint64, i64, f32p, f32p, f32p, i64p]),
        "tso_opacity_reset": (None, [i64, f32p]),
        "tso_morton_interleave": (ctypes.c_uint64, [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                                    ctypes.c_int]),
        "tso_morton_codes": (None, [i64, f32p, vp]),
        "tso_morton_reorder": (None, [i64, f32p, vp, vp, vp, vp, vp]),
        "tso_train_step": (ctypes.c_double, [i64, f32p, f32p, f32p, vp, vp, f32p, f32p, ctypes.c_float,
                                             ctypes.c_float, ctypes.c_float, ctypes.c_float, ctypes.c_float,
                                             f32p, f32p, f64p]),
        "tso_sh_active_degree": (ctypes.c_int32, [i64]),
        "tso_scene_extent": (ctypes.c_double, [ctypes.c_int32, f64p]),
        "tso_compute_sampling_rates": (None, [i64, f32p, vp, ctypes.c_int32, ctypes.c_float, f32p]),
        "tso_set_sampling_rates": (None, [i64, f32p]),
        "tso_apply_3d_filter_clip": (None, [i64, f32p, f32p, ctypes.c_float]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def _p(s):
    return ctypes.addressof(s)


def set_workers(n: int):
    lib.tso_set_workers(int(n))


def compute_sampling_rates(params, n, cams, extent):
    """compute_sampling_rates."""
    from paper_2602_09999_b200.types import Camera
    arr = (Camera * len(cams))(*cams)
    nu = np.zeros(n, np.float32)
    lib.tso_compute_sampling_rates(n, np.ascontiguousarray(params, np.float32), ctypes.addressof(arr), len(cams),
                                   float(extent), nu)
    return nu


def set_sampling_rates(nu):
    """sampling rates used by preprocess / backward with aa_mode 1 (filter3d_original)."""
    nu = np.ascontiguousarray(nu, np.float32)
    lib.tso_set_sampling_rates(nu.size, nu)


def apply_3d_filter_clip(params, n, nu, kappa3d=0.2):
    """apply_3d_filter_clip on a copy of the flat parameter array."""
    out = np.array(params, np.float32, copy=True)
    lib.tso_apply_3d_filter_clip(n, out, np.ascontiguousarray(nu, np.float32), float(kappa3d))
    return out


def preprocess(params, n, cam, cfg):
    splat = np.zeros(n * 12, np.float32)
    rect = np.zeros(n * 4, np.int32)
    cnt = np.zeros(n, np.uint32)
    dkey = np.zeros(n, np.uint32)
    lib.tso_preprocess(n, params, _p(cam), _p(cfg), splat, rect, cnt, dkey)
    return splat.reshape(n, 12), rect.reshape(n, 4), cnt, dkey


def instances(params, n, cam, cfg, sort="combined"):
    """Gaussian-major instances then sorted (combined 64-bit stable or two-stage); returns keys, vals, ranges."""
    splat, rect, cnt, dkey = preprocess(params, n, cam, cfg)
    I = int(cnt.sum(dtype=np.int64))
    keys = np.zeros(I, np.uint64)
    vals = np.zeros(I, np.uint32)
    got = lib.tso_build_instances(n, splat.reshape(-1), rect.reshape(-1), cnt, dkey, _p(cam), _p(cfg), keys, vals)
    assert got == I
    if sort == "combined":
        lib.tso_sort_combined(I, keys, vals)
    elif sort == "two_stage":
        tb = max(1, int(np.ceil(np.log2(max(2, cam.n_tiles)))))
        lib.tso_sort_two_stage(I, tb, keys, vals)
    ranges = np.zeros(cam.n_tiles * 2, np.uint32)
    lib.tso_tile_ranges(I, keys, cam.n_tiles, ranges)
    return keys, vals, ranges.reshape(-1, 2), cnt


def render(params, n, cam, cfg, f64=False):
    H, W = cam.height, cam.width
    if f64:
        rgb = np.zeros(H * W * 3, np.float64)
        T = np.zeros(H * W, np.float64)
        cnt = np.zeros(H * W, np.uint32)
        I = lib.tso_render_f64(n, np.ascontiguousarray(params, np.float64), _p(cam), _p(cfg), rgb, T, cnt)
    else:
        rgb = np.zeros(H * W * 3, np.float32)
        T = np.zeros(H * W, np.float32)
        cnt = np.zeros(H * W, np.uint32)
        I = lib.tso_render(n, params, _p(cam), _p(cfg), rgb, T, cnt)
    return rgb.reshape(H, W, 3), T.reshape(H, W), cnt.reshape(H, W), int(I)


def weight_sum(params, n, cam, cfg):
    out = np.zeros(cam.height * cam.width, np.float64)
    lib.tso_render_weight_sum(n, params, _p(cam), _p(cfg), out)
    return out.reshape(cam.height, cam.width)


def training_loss(rgb, target, f64=False):
    H, W = rgb.shape[:2]
    dt = np.float64 if f64 else np.float32
    x = np.ascontiguousarray(rgb, dt).reshape(-1)
    y = np.ascontiguousarray(target, dt).reshape(-1)
    d = np.zeros_like(x)
    fn = lib.tso_training_loss_f64 if f64 else lib.tso_training_loss
    loss = fn(H, W, x, y, d)
    return float(loss), d.reshape(H, W, 3)


def backward(params, n, cam, cfg, dLdC, f64=False):
    dt = np.float64 if f64 else np.float32
    G = np.zeros(59 * n, dt)
    g2 = np.zeros(9 * n, dt)
    acc = np.zeros(n, dt)
    vc = np.zeros(n, dt)
    fn = lib.tso_backward_f64 if f64 else lib.tso_backward
    fn(n, np.ascontiguousarray(params, dt), _p(cam), _p(cfg), np.ascontiguousarray(dLdC, dt).reshape(-1),
       G, g2, acc, vc)
    return G, g2.reshape(n, 9), acc, vc


def adam_step(params, grads, m, v, n, lr, beta1, beta2, eps, bc1, bc2, mode=1, visible=None):
    lr = np.asarray(lr, np.float32)
    vis = None if visible is None else visible.ctypes.data_as(ctypes.c_void_p)
    lib.tso_adam_step(n, params, grads, m, v, lr, beta1, beta2, eps, bc1, bc2, mode, vis)


def densify(params, m, v, accum, vcount, n, grad_thresh, extent, seed, it):
    op = np.zeros(59 * 3 * n, np.float32)
    om = np.zeros(59 * 3 * n, np.float32)
    ov = np.zeros(59 * 3 * n, np.float32)
    st = np.zeros(3, np.int64)
    na = lib.tso_densify_and_prune(n, params, m, v, accum, vcount, grad_thresh, extent, seed, it, op, om, ov, st)
    na = int(na)
    # outputs were written with stride na (block layout of the compacted store)
    return op[:59 * na].copy(), om[:59 * na].copy(), ov[:59 * na].copy(), na, st


def morton_interleave(qx, qy, qz, bits=21):
    return int(lib.tso_morton_interleave(qx, qy, qz, bits))


def morton_codes(params, n):
    out = np.zeros(n, np.uint64)
    lib.tso_morton_codes(n, np.ascontiguousarray(params, np.float32), out.ctypes.data)
    return out


def _vp_or_none(a):
    return None if a is None else a.ctypes.data


def morton_reorder(params, n, m=None, v=None, accum=None, vcount=None):
    """In-place permutation of the given float32 arrays; returns perm[new] = old."""
    perm = np.zeros(n, np.uint32)
    lib.tso_morton_reorder(n, params, _vp_or_none(m), _vp_or_none(v), _vp_or_none(accum), _vp_or_none(vcount),
                           perm.ctypes.data)
    return perm


def train_step(params, m, v, n, cam, cfg, target, adam, accum, vcount):
    st = np.zeros(8, np.float64)
    lr = np.array(adam.lr[:], np.float32)
    loss = lib.tso_train_step(n, params, m, v, _p(cam), _p(cfg), np.ascontiguousarray(target, np.float32).reshape(-1),
                              lr, adam.beta1, adam.beta2, adam.eps, adam.bc1, adam.bc2, accum, vcount, st)
    return float(loss), st
