"""Python mirror of the reference `tilesplat` operation set over the C-ABI of
libtilesplat_b200.so (include/tilesplat_c.h).

The reference API is SPEC.md's typed operation list (render, training_loss,
backward, adam_step_*, densify_and_prune, opacity_reset) over a column-oriented
ParameterStore; `Engine` exposes exactly those operations, with the reference's
error behaviour (validation errors raise `ValidationError`, mirroring exit code
1; device failures raise `DeviceError`).  There is no CPU fallback: importing
this module without the built library, or creating an Engine without an sm_100
device, raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from .types import AdamConfig, Camera, RenderConfig, NPARAM

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtilesplat_b200.so")
# experiments only: an alternative in-tree build of the same library (tuning variants)
if os.environ.get("TS_LIB_VARIANT"):
    LIB_PATH = os.path.join(_HERE, f"libtilesplat_b200_{os.environ['TS_LIB_VARIANT']}.so")

TS_OK, TS_ERR_VALIDATION, TS_ERR_CHECK, TS_ERR_CUDA, TS_ERR_OOM, TS_ERR_STATE = range(6)


class TilesplatError(RuntimeError):
    pass


class ValidationError(TilesplatError):
    pass


class DeviceError(TilesplatError):
    pass


# exported C-ABI symbols (kept in sync with include/tilesplat_c.h; tests check it)
_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_f = ctypes.c_float
_SIGS = {
    "ts_create": [_i32, _vp, ctypes.POINTER(_vp)],
    "ts_destroy": [_vp],
    "ts_last_error": [_vp],
    "ts_version": [],
    "ts_synchronize": [_vp],
    "ts_set_params": [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp],
    "ts_set_params_flat": [_vp, _i64, _vp],
    "ts_get_params_flat": [_vp, _vp],
    "ts_num_gaussians": [_vp, ctypes.POINTER(_i64)],
    "ts_forward": [_vp, _vp, _vp, _vp, _vp, _vp],
    "ts_set_target": [_vp, _i32, _i32, _i32, _vp],
    "ts_loss": [_vp, _vp, _i32, _vp],
    "ts_backward": [_vp, _vp],
    "ts_zero_grads": [_vp],
    "ts_mark_grads_consumed": [_vp],
    "ts_grad_buffer": [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_i64)],
    "ts_param_buffer": [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_i64)],
    "ts_stats_buffer": [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp)],
    "ts_reserve_flat": [_vp, _i64],
    "ts_adam_step": [_vp, _vp],
    "ts_adam_step_range": [_vp, _vp, _i64, _i64],
    "ts_train_step": [_vp, _vp, _vp, _vp, _i32, _vp, _vp],
    "ts_backward_adam": [_vp, _vp, _vp],
    "ts_densify": [_vp, _f, _f, ctypes.c_uint64, _i64, _vp, _vp],
    "ts_opacity_reset": [_vp],
    "ts_morton_reorder": [_vp, _vp],
    "ts_set_state": [_vp, _vp, _vp, _vp, _vp, _vp],
    "ts_get_state": [_vp, _vp, _vp, _vp, _vp, _vp],
    "ts_debug_preprocess": [_vp, _vp, _vp, _vp, _vp],
    "ts_debug_instances": [_vp, ctypes.POINTER(_i64), _vp, _vp, _vp],
    "ts_debug_grad2d": [_vp, _vp, _vp],
    "ts_view_stats": [_vp, _vp],
    "ts_set_profiling": [_vp, _i32],
    "ts_stage_times": [_vp, _vp, _vp, _i32],
    "ts_set_binning": [_vp, _i32],
    "ts_compute_sampling_rates": [_vp, _vp, _i32, _f],
    "ts_set_sampling_rates": [_vp, _vp],
    "ts_get_sampling_rates": [_vp, _vp],
    "ts_apply_3d_filter_clip": [_vp, _f],
    "ts_debug_loss_grad": [_vp, _vp],
    "ts_binning_path": [_vp, _vp],
    "ts_launch_count": [_vp, ctypes.POINTER(_i64)],
    "ts_set_graph": [_vp, _i32],
    "ts_graph_stats": [_vp, _vp],
    "ts_host_alloc": [ctypes.c_size_t, ctypes.POINTER(_vp)],
    "ts_host_free": [_vp],
}
EXPORTED_SYMBOLS = tuple(_SIGS)
STAGES = ("preprocess", "depth_sort", "scan", "duplicate", "tile_sort", "ranges", "blend",
          "loss", "blend_bwd", "project_bwd", "adam")


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    if not os.path.exists(path):
        raise ImportError(f"libtilesplat_b200.so not built ({path}); run __graft_entry__.build()")
    lib = ctypes.CDLL(path)
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    lib.ts_last_error.restype = ctypes.c_char_p
    lib.ts_version.restype = ctypes.c_char_p
    return lib


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        _lib = load_library()
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


class Engine:
    """One device context (one GPU, one CUDA stream): the ParameterStore, its
    gradients / Adam moments, and the per-view render state."""

    def __init__(self, device: int = 0, stream: int | None = None):
        self._L = lib()
        h = ctypes.c_void_p()
        st = self._L.ts_create(int(device), ctypes.c_void_p(stream) if stream else None, ctypes.byref(h))
        if st != TS_OK:
            raise DeviceError(f"ts_create(device={device}) failed with status {st}: "
                              "an sm_100 (B200) device is required; there is no CPU fallback")
        self._h = h
        self.device = device
        self.stream = int(stream) if stream else None   # None: the context's own stream
        self.n = 0
        self._cam = None

    # ---- plumbing ----
    def _check(self, st: int, what: str):
        if st == TS_OK:
            return
        msg = self._L.ts_last_error(self._h)
        msg = msg.decode() if msg else ""
        if st == TS_ERR_VALIDATION:
            raise ValidationError(f"{what}: {msg}")
        raise DeviceError(f"{what}: status {st}: {msg}")

    def close(self):
        if getattr(self, "_h", None):
            self._L.ts_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self):
        self._check(self._L.ts_synchronize(self._h), "ts_synchronize")

    # ---- ParameterStore ----
    def set_params(self, flat: np.ndarray, n: int):
        flat = _f32(flat)
        assert flat.size == NPARAM * n
        self._check(self._L.ts_set_params_flat(self._h, n, _ptr(flat)), "ts_set_params_flat")
        self.n = n

    def get_params(self) -> np.ndarray:
        out = np.empty(NPARAM * self.num_gaussians(), np.float32)
        self._check(self._L.ts_get_params_flat(self._h, _ptr(out)), "ts_get_params_flat")
        return out

    def num_gaussians(self) -> int:
        n = ctypes.c_int64()
        self._L.ts_num_gaussians(self._h, ctypes.byref(n))
        self.n = int(n.value)
        return self.n

    # ---- SPEC ops ----
    def render(self, cam: Camera, cfg: RenderConfig, outputs: bool = True):
        """render -> (rgb HxWx3, T HxW, contributor count HxW)."""
        self._cam = cam
        if not outputs:
            self._check(self._L.ts_forward(self._h, ctypes.byref(cam), ctypes.byref(cfg), None, None, None),
                        "ts_forward")
            return None
        H, W = cam.height, cam.width
        rgb = np.empty((H, W, 3), np.float32)
        T = np.empty((H, W), np.float32)
        cnt = np.empty((H, W), np.uint32)
        self._check(self._L.ts_forward(self._h, ctypes.byref(cam), ctypes.byref(cfg), _ptr(rgb), _ptr(T), _ptr(cnt)),
                    "ts_forward")
        return rgb, T, cnt

    def set_target(self, slot: int, target: np.ndarray):
        t = _f32(target)
        H, W = t.shape[:2]
        self._check(self._L.ts_set_target(self._h, slot, W, H, _ptr(t)), "ts_set_target")

    def training_loss(self, target: np.ndarray | None = None, slot: int = 0, want_value: bool = True):
        """training_loss on the last render; dL/dC stays on the device."""
        t = None if target is None else _f32(target)
        out = ctypes.c_float()
        self._check(self._L.ts_loss(self._h, _ptr(t), slot, ctypes.byref(out) if want_value else None), "ts_loss")
        return float(out.value) if want_value else None

    def backward(self, dL_dC: np.ndarray | None = None):
        """backward: accumulates parameter gradients and densify stats."""
        d = None if dL_dC is None else _f32(dL_dC)
        self._check(self._L.ts_backward(self._h, _ptr(d)), "ts_backward")

    def backward_adam(self, adam: AdamConfig, dL_dC: np.ndarray | None = None):
        """fused_backward_update: backward + in-place Adam (modes 3/4)."""
        d = None if dL_dC is None else _f32(dL_dC)
        self._check(self._L.ts_backward_adam(self._h, _ptr(d), ctypes.byref(adam)), "ts_backward_adam")

    def zero_grads(self):
        self._check(self._L.ts_zero_grads(self._h), "ts_zero_grads")

    def mark_grads_consumed(self):
        """The next backward overwrites the gradient buffer (sharded data-parallel optimizer)."""
        self._check(self._L.ts_mark_grads_consumed(self._h), "ts_mark_grads_consumed")

    def adam_step(self, cfg: AdamConfig, begin: int | None = None, end: int | None = None):
        if begin is None:
            self._check(self._L.ts_adam_step(self._h, ctypes.byref(cfg)), "ts_adam_step")
        else:
            self._check(self._L.ts_adam_step_range(self._h, ctypes.byref(cfg), begin, end), "ts_adam_step_range")

    def train_step(self, cam: Camera, cfg: RenderConfig, adam: AdamConfig, target: np.ndarray | None = None,
                   slot: int = 0, want_loss: bool = True, target_ptr: int | None = None):
        out = ctypes.c_float()
        if target_ptr is not None:
            tp = ctypes.c_void_p(target_ptr)
        else:
            tp = None if target is None else _ptr(_f32(target))
        self._check(self._L.ts_train_step(self._h, ctypes.byref(cam), ctypes.byref(cfg), tp, slot,
                                          ctypes.byref(adam), ctypes.byref(out) if want_loss else None),
                    "ts_train_step")
        return float(out.value) if want_loss else None

    def set_graph(self, on: bool):
        """CUDA-graph mode of train_step (ts_set_graph): the step of each view is captured once and
        relaunched; results equal the host-driven path (voided steps are replayed)."""
        self._check(self._L.ts_set_graph(self._h, 1 if on else 0), "ts_set_graph")

    def graph_stats(self):
        out = np.zeros(4, np.int64)
        self._check(self._L.ts_graph_stats(self._h, _ptr(out)), "ts_graph_stats")
        return dict(launches=int(out[0]), captures=int(out[1]), replays=int(out[2]), graphs=int(out[3]))

    def densify_and_prune(self, grad_thresh: float, extent: float, seed: int, it: int):
        na = ctypes.c_int64()
        st = (ctypes.c_int64 * 3)()
        self._check(self._L.ts_densify(self._h, grad_thresh, extent, seed, it, ctypes.byref(na), st), "ts_densify")
        self.n = int(na.value)
        return self.n, (int(st[0]), int(st[1]), int(st[2]))

    def opacity_reset(self):
        self._check(self._L.ts_opacity_reset(self._h), "ts_opacity_reset")

    def morton_reorder(self):
        """morton_reorder; returns perm (old index of each new row)."""
        perm = np.empty(self.num_gaussians(), np.uint32)
        self._check(self._L.ts_morton_reorder(self._h, _ptr(perm)), "ts_morton_reorder")
        return perm

    # ---- state ----
    def set_state(self, grads=None, m=None, v=None, accum=None, vcount=None):
        arrs = [None if a is None else _f32(a) for a in (grads, m, v, accum, vcount)]
        self._check(self._L.ts_set_state(self._h, *[_ptr(a) for a in arrs]), "ts_set_state")

    def get_state(self):
        n = self.num_gaussians()
        g = np.empty(NPARAM * n, np.float32)
        m = np.empty(NPARAM * n, np.float32)
        v = np.empty(NPARAM * n, np.float32)
        acc = np.empty(n, np.float32)
        cnt = np.empty(n, np.float32)
        self._check(self._L.ts_get_state(self._h, _ptr(g), _ptr(m), _ptr(v), _ptr(acc), _ptr(cnt)), "ts_get_state")
        return g, m, v, acc, cnt

    def grad_buffer(self):
        p = ctypes.c_void_p()
        n = ctypes.c_int64()
        self._check(self._L.ts_grad_buffer(self._h, ctypes.byref(p), ctypes.byref(n)), "ts_grad_buffer")
        return int(p.value or 0), int(n.value)

    def param_buffer(self):
        p = ctypes.c_void_p()
        n = ctypes.c_int64()
        self._check(self._L.ts_param_buffer(self._h, ctypes.byref(p), ctypes.byref(n)), "ts_param_buffer")
        return int(p.value or 0), int(n.value)

    def stats_buffer(self):
        a = ctypes.c_void_p()
        c = ctypes.c_void_p()
        self._check(self._L.ts_stats_buffer(self._h, ctypes.byref(a), ctypes.byref(c)), "ts_stats_buffer")
        return int(a.value or 0), int(c.value or 0)

    # ---- torch views for collectives (zero-copy, same device memory) ----
    def reserve_flat(self, min_len: int):
        self._check(self._L.ts_reserve_flat(self._h, int(min_len)), "ts_reserve_flat")

    def grad_tensor(self, padded_to: int | None = None):
        from .dp import device_tensor
        p, n = self.grad_buffer()
        if padded_to is not None and padded_to > n:
            self.reserve_flat(padded_to)
            p, n = self.grad_buffer()
            n = padded_to
        return device_tensor(p, n, self.device)

    def param_tensor(self, padded_to: int | None = None):
        from .dp import device_tensor
        p, n = self.param_buffer()
        if padded_to is not None and padded_to > n:
            self.reserve_flat(padded_to)
            p, n = self.param_buffer()
            n = padded_to
        return device_tensor(p, n, self.device)

    def stats_tensors(self):
        from .dp import device_tensor
        a, c = self.stats_buffer()
        n = self.num_gaussians()
        return device_tensor(a, n, self.device), device_tensor(c, n, self.device)

    # ---- parity / debug ----
    def debug_preprocess(self):
        n = self.num_gaussians()
        splat = np.empty((n, 12), np.float32)
        rect = np.empty((n, 4), np.int32)
        cnt = np.empty(n, np.uint32)
        dk = np.empty(n, np.uint32)
        self._check(self._L.ts_debug_preprocess(self._h, _ptr(splat), _ptr(rect), _ptr(cnt), _ptr(dk)),
                    "ts_debug_preprocess")
        return splat, rect, cnt, dk

    def debug_instances(self):
        I = ctypes.c_int64()
        self._check(self._L.ts_debug_instances(self._h, ctypes.byref(I), None, None, None), "ts_debug_instances")
        I = int(I.value)
        keys = np.empty(I, np.uint64)
        vals = np.empty(I, np.uint32)
        Tn = self._cam.n_tiles
        ranges = np.empty((Tn, 2), np.uint32)
        n = ctypes.c_int64()
        self._check(self._L.ts_debug_instances(self._h, ctypes.byref(n), _ptr(keys), _ptr(vals), _ptr(ranges)),
                    "ts_debug_instances")
        return keys, vals, ranges

    def debug_grad2d(self, dL_dC: np.ndarray):
        n = self.num_gaussians()
        out = np.empty((n, 9), np.float32)
        self._check(self._L.ts_debug_grad2d(self._h, _ptr(_f32(dL_dC)), _ptr(out)), "ts_debug_grad2d")
        return out

    def view_stats(self):
        out = np.zeros(4, np.int64)
        self._check(self._L.ts_view_stats(self._h, _ptr(out)), "ts_view_stats")
        return dict(V=int(out[0]), I=int(out[1]), Ip=int(out[2]), P=int(out[3]))

    def set_profiling(self, on: bool):
        self._check(self._L.ts_set_profiling(self._h, 1 if on else 0), "ts_set_profiling")

    def stage_times(self):
        """{stage: (total_ms, calls)} summed since set_profiling(True)."""
        out = np.zeros(len(STAGES), np.float32)
        cnt = np.zeros(len(STAGES), np.int32)
        self._check(self._L.ts_stage_times(self._h, _ptr(out), _ptr(cnt), len(STAGES)), "ts_stage_times")
        return {k: (float(a), int(b)) for k, a, b in zip(STAGES, out, cnt)}

    # ---- antialias ----
    def compute_sampling_rates(self, cams, extent: float):
        """compute_sampling_rates over the training cameras (stored on the device)."""
        arr = (Camera * len(cams))(*cams)
        self._check(self._L.ts_compute_sampling_rates(self._h, arr, len(cams), extent), "ts_compute_sampling_rates")

    def set_sampling_rates(self, nu: np.ndarray):
        self._check(self._L.ts_set_sampling_rates(self._h, _ptr(_f32(nu))), "ts_set_sampling_rates")

    def get_sampling_rates(self) -> np.ndarray:
        out = np.empty(self.num_gaussians(), np.float32)
        self._check(self._L.ts_get_sampling_rates(self._h, _ptr(out)), "ts_get_sampling_rates")
        return out

    def apply_3d_filter_clip(self, kappa3d: float = 0.2):
        self._check(self._L.ts_apply_3d_filter_clip(self._h, kappa3d), "ts_apply_3d_filter_clip")

    def debug_loss_grad(self):
        """dL/dC (H x W x 3) of the last training_loss, read back from the device."""
        H, W = self._cam.height, self._cam.width
        out = np.empty((H, W, 3), np.float32)
        self._check(self._L.ts_debug_loss_grad(self._h, _ptr(out)), "ts_debug_loss_grad")
        return out

    def set_binning(self, mode: int):
        """0 auto (bucketed binning + per-tile sort), 1 force the two-stage radix sort."""
        self._check(self._L.ts_set_binning(self._h, mode), "ts_set_binning")

    def binning_path(self) -> str:
        r = ctypes.c_int32()
        self._check(self._L.ts_binning_path(self._h, ctypes.byref(r)), "ts_binning_path")
        return "radix" if r.value else "bucket"

    def launch_count(self) -> int:
        n = ctypes.c_int64()
        self._check(self._L.ts_launch_count(self._h, ctypes.byref(n)), "ts_launch_count")
        return int(n.value)


class PinnedBuffer:
    """Page-locked host buffer (ts_host_alloc) exposed as a numpy array."""

    def __init__(self, shape, dtype=np.float32):
        L = lib()
        nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        p = ctypes.c_void_p()
        if L.ts_host_alloc(nbytes, ctypes.byref(p)) != TS_OK:
            raise DeviceError("ts_host_alloc failed")
        self._p = p
        buf = (ctypes.c_byte * nbytes).from_address(p.value)
        self.array = np.frombuffer(buf, dtype=dtype).reshape(shape)
        self.ptr = int(p.value)

    def free(self):
        if self._p:
            lib().ts_host_free(self._p)
            self._p = None
