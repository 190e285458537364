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

    def grad_tensor(self, padded_to=None):
        return torch.from_numpy(self.G[: (padded_to or self.L)])

    def param_tensor(self, padded_to=None):
        return torch.from_numpy(self.P[: (padded_to or self.L)])

    def stats_tensors(self):
        return torch.from_numpy(self.acc), torch.from_numpy(self.cnt)
