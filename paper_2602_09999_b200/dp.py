"""Data-parallel training step over views.

Gaussians, Adam moments and densification state are replicated on every rank;
rank r renders its own slice of the view batch and accumulates gradients in
its flat 59*N buffer; one collective over that buffer (NCCL over NVLink on the
B200 nodes, gloo in the CPU tests) sums them (batch gradient = sum
of per-view gradients), then every rank applies the same optimizer update, so
parameters stay bitwise identical across ranks.

Three exchange modes:
  * "allreduce": all_reduce(grads) + replicated fused Adam (rung 1);
  * "sharded":   all_reduce(grads) is replaced by reduce_scatter(grads) ->
                 Adam on this rank's 1/G slice -> all_gather(params) (rung 2),
                 so each rank runs 1/G of the 28 B/element Adam sweep;
  * "chunked":   the all-reduce is issued as K asynchronous chunks of the flat
                 buffer, and the replicated Adam sweeps chunk k as soon as its
                 sum has landed, so the optimizer of chunk k overlaps the
                 transfer of chunk k+1 (rung 3; the stream waits, not the host).

The engine is anything exposing the Engine surface used below (the CUDA
Engine in production; the tests pass a CPU stand-in to exercise the
collective logic with gloo).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


class _CudaArray:
    """Zero-copy __cuda_array_interface__ view of a device fp32 buffer."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3,
                                         "strides": None, "stream": None}


def device_tensor(ptr: int, n: int, device: int) -> torch.Tensor:
    with torch.cuda.device(device):
        return torch.as_tensor(_CudaArray(ptr, n), device=f"cuda:{device}")


def shard_bounds(length: int, world: int, rank: int, align: int = 4):
    """[begin, end) of rank's slice of a flat buffer, 16-byte aligned slices."""
    per = -(-length // world)
    per = -(-per // align) * align
    b = min(length, rank * per)
    e = min(length, b + per)
    return b, e, per


class DataParallelStep:
    """One data-parallel training step over a view batch (module docstring).

    Stream contract: the collectives are issued on torch's current stream, so the
    engine must run on that same stream (Engine(device, stream=torch.cuda.current_stream().cuda_stream)),
    which orders backward -> collective -> optimizer without host waits; a different
    engine stream is rejected.  The skip-invisible optimizer modes use each rank's
    local visibility mask and are rejected for world > 1 (replicas would diverge)."""

    def __init__(self, engine, mode: str = "allreduce", group=None, chunks: int = 8):
        assert mode in ("allreduce", "sharded", "chunked")
        self.e = engine
        self.mode = mode
        self.chunks = chunks
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if self.world > 1 else 0
        self._nccl = self.world > 1 and dist.get_backend(group) == "nccl"
        self._padded_for = None   # N the padded flat buffers were reserved for (sharded mode)
        es = getattr(engine, "stream", None)
        if self.world > 1 and es is not None and torch.cuda.is_available():
            cur = torch.cuda.current_stream(engine.device).cuda_stream
            if int(es) != int(cur):
                raise ValueError("DataParallelStep: the engine must run on torch's current stream "
                                 "(collectives are ordered against it)")

    def my_views(self, n_views: int):
        """Views {r, r+G, ...} of an n_views batch (disjoint slices)."""
        return list(range(self.rank, n_views, self.world))

    def accumulate(self, views):
        """views: iterable of (camera, render_config, target_slot) rendered by THIS rank."""
        for cam, cfg, slot in views:
            self.e.render(cam, cfg, outputs=False)
            self.e.training_loss(slot=slot, want_value=False)
            self.e.backward(None)

    def _reserve_padded(self, per: int):
        """Pad the flat parameter / gradient buffers to world * per once per store size
        (one allocation + tail clear, not per step)."""
        n = self.e.num_gaussians() if hasattr(self.e, "num_gaussians") else None
        if self._padded_for != (n, per):
            self.e.reserve_flat(per * self.world)
            self._padded_for = (n, per)

    def exchange_and_step(self, adam):
        if self.world > 1 and adam.mode in (2, 4):
            raise ValueError("skip-invisible Adam uses the rank-local visibility mask: world size 1 only")
        if self.world == 1:
            self.e.adam_step(adam)
            return
        g = self.e.grad_tensor()
        if self.mode == "allreduce":
            dist.all_reduce(g, op=dist.ReduceOp.SUM, group=self.group)
            self.e.adam_step(adam)
            return
        if self.mode == "chunked":
            L = g.numel()
            bounds = [shard_bounds(L, self.chunks, k)[:2] for k in range(self.chunks)]
            bounds = [(b, e) for b, e in bounds if e > b]
            works = [dist.all_reduce(g[b:e], op=dist.ReduceOp.SUM, group=self.group, async_op=True)
                     for b, e in bounds]
            for (b, e), w in zip(bounds, works):  # in order: the last sweep marks the buffer consumed
                w.wait()
                self.e.adam_step(adam, begin=b, end=e)
            return
        # sharded: reduce-scatter -> Adam on this rank's slice -> all-gather of the parameters.
        # With NCCL both collectives run in place (the rank's slot of the padded buffer is the
        # send / receive buffer); gloo gets a separate staging tensor.
        L = g.numel()
        b, e, per = shard_bounds(L, self.world, self.rank)
        self._reserve_padded(per)
        padded = self.e.grad_tensor(padded_to=per * self.world)
        mine = padded[self.rank * per:(self.rank + 1) * per]
        if self._nccl:
            dist.reduce_scatter_tensor(mine, padded, op=dist.ReduceOp.SUM, group=self.group)
        else:
            out = torch.empty(per, dtype=padded.dtype, device=padded.device)
            dist.reduce_scatter_tensor(out, padded, op=dist.ReduceOp.SUM, group=self.group)
            mine.copy_(out)
        a = type(adam).from_buffer_copy(adam) if hasattr(type(adam), "from_buffer_copy") else adam
        a.zero_grads = 0
        self.e.adam_step(a, begin=b, end=e)
        p = self.e.param_tensor(padded_to=per * self.world)
        pm = p[self.rank * per:(self.rank + 1) * per]
        dist.all_gather_into_tensor(p, pm if self._nccl else pm.clone(), group=self.group)
        # the other ranks' slices still hold this rank's un-reduced gradients: the buffer is
        # consumed, and the next backward overwrites every row instead of accumulating
        self.e.mark_grads_consumed()

    def step(self, views, adam):
        self.accumulate(views)
        self.exchange_and_step(adam)

    def reduce_densify_stats(self):
        """Sum (accum, count) across ranks before a densify event (replicas stay identical)."""
        if self.world == 1:
            return
        a, c = self.e.stats_tensors()
        dist.all_reduce(a, group=self.group)
        dist.all_reduce(c, group=self.group)
