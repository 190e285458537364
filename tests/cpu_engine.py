"""CPU stand-in of the Engine surface used by paper_2602_09999_b200.dp, backed by
the oracle.  TEST INFRASTRUCTURE: lets the data-parallel collective logic run
under gloo on CPU (world_size 2) without a GPU."""
import numpy as np
import torch

from oracle import oracle as O


class CpuEngine:
    def __init__(self, params, n, targets):
        self.n = n
        self.L = 59 * n
        self.cap = self.L + 64
        self.P = np.zeros(self.cap, np.float32)
        self.P[:self.L] = params
        self.G = np.zeros(self.cap, np.float32)
        self.M = np.zeros(self.L, np.float32)
        self.V = np.zeros(self.L, np.float32)
        self.acc = np.zeros(n, np.float32)
        self.cnt = np.zeros(n, np.float32)
        self.targets = targets
        self._view = None

    def render(self, cam, cfg, outputs=False):
        self._view = (cam, cfg)
        rgb, _, _, _ = O.render(self.P[:self.L], self.n, cam, cfg)
        self._rgb = rgb

    def training_loss(self, target=None, slot=0, want_value=True):
        t = self.targets[slot] if target is None else target
        loss, self._dl = O.training_loss(self._rgb, t)
        return loss if want_value else None

    def backward(self, dl=None):
        if getattr(self, "_stale", False):  # consumed buffer: overwrite instead of accumulating
            self.G[:] = 0.0
            self._stale = False
        cam, cfg = self._view
        G, _, a, c = O.backward(self.P[:self.L], self.n, cam, cfg, self._dl if dl is None else dl)
        self.G[:self.L] += G
        self.acc += a
        self.cnt += c

    def adam_step(self, adam, begin=None, end=None):
        b = 0 if begin is None else begin
        e = self.L if end is None else end
        P = self.P[:self.L].copy()
        G = self.G[:self.L].copy()
        M, V = self.M.copy(), self.V.copy()
        O.adam_step(P, G, M, V, self.n, list(adam.lr), adam.beta1, adam.beta2, adam.eps, adam.bc1, adam.bc2,
                    mode=adam.mode)
        self.P[b:e], self.M[b:e], self.V[b:e] = P[b:e], M[b:e], V[b:e]
        if adam.zero_grads:
            self.G[b:e] = 0.0

    def zero_grads(self):
        self.G[:] = 0.0

    def mark_grads_consumed(self):
        self._stale = True

    def reserve_flat(self, min_len):
        assert min_len <= self.cap

    def grad_tensor(self, padded_to=None):
        return torch.from_numpy(self.G[: (padded_to or self.L)])

    def param_tensor(self, padded_to=None):
        return torch.from_numpy(self.P[: (padded_to or self.L)])

    def stats_tensors(self):
        return torch.from_numpy(self.acc), torch.from_numpy(self.cnt)


class OracleTrainEngine:
    """Oracle-backed stand-in of the Engine surface the Trainer drives
    (train_step, densify_and_prune, opacity_reset, morton_reorder, state I/O).
    TEST INFRASTRUCTURE: deterministic, so checkpoint/resume is checked bitwise."""

    def __init__(self, params, n):
        self.set_params(params, n)

    def set_params(self, params, n):
        self.n = n
        self.P = np.array(params, np.float32)
        self.M = np.zeros(59 * n, np.float32)
        self.V = np.zeros(59 * n, np.float32)
        self.acc = np.zeros(n, np.float32)
        self.cnt = np.zeros(n, np.float32)

    def num_gaussians(self):
        return self.n

    def get_params(self):
        return self.P.copy()

    def get_state(self):
        return np.zeros(59 * self.n, np.float32), self.M.copy(), self.V.copy(), self.acc.copy(), self.cnt.copy()

    def set_state(self, grads=None, m=None, v=None, accum=None, vcount=None):
        for name, a in (("M", m), ("V", v), ("acc", accum), ("cnt", vcount)):
            if a is not None:
                setattr(self, name, np.array(a, np.float32))

    def train_step(self, cam, cfg, adam, target=None, slot=0, want_loss=True):
        loss, _ = O.train_step(self.P, self.M, self.V, self.n, cam, cfg, target, adam, self.acc, self.cnt)
        return loss

    def densify_and_prune(self, grad_thresh, extent, seed, it):
        P, M, V, na, st = O.densify(self.P, self.M, self.V, self.acc, self.cnt, self.n, grad_thresh, extent, seed, it)
        self.n, self.P, self.M, self.V = na, P, M, V
        self.acc = np.zeros(na, np.float32)
        self.cnt = np.zeros(na, np.float32)
        return na, (int(st[0]), int(st[1]), int(st[2]))

    def opacity_reset(self):
        O.lib.tso_opacity_reset(self.n, self.P)

    def morton_reorder(self):
        return O.morton_reorder(self.P, self.n, self.M, self.V, self.acc, self.cnt)
