"""The C++ multi-GPU host path (tools/ts_train_dp.cpp: one host thread per GPU, ncclCommInitAll,
the exchange on each context's stream) in its three exchange modes.  On a 1-GPU box the
communicator has one rank (loopback).  Every step, the exchange + optimizer must leave the
parameters and Adam moments bit for bit where a single-context ts_adam_step over the whole
buffer does, given the same pre-step state and the batch gradient (views accumulated in the
flat buffer; snapshotted, since the rendering gradients use fp32 atomics).  With 2 GPUs the
same holds for the 2-rank sum, and every replica must equal rank 0 bit for bit."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tools", "ts_train_dp")


def _gpus():
    import torch
    return torch.cuda.device_count()


def _run(g, mode, views=4):
    out = subprocess.run([EXE, str(g), mode, "20000", "4", str(views), "--check"], capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr + out.stdout
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("mode", ["allreduce", "sharded", "chunked"])
def test_cpp_dp_loopback_bitwise(mode):
    r = _run(1, mode)
    assert r["gpus"] == 1 and r["replicas_bitwise_equal"] and r["check_mismatches"] == 0 and r["iters"] == 4


@pytest.mark.parametrize("mode", ["allreduce", "sharded", "chunked"])
def test_cpp_dp_two_gpus(mode):
    if _gpus() < 2:
        pytest.skip("needs 2 GPUs")
    r = _run(2, mode)
    assert r["gpus"] == 2 and r["replicas_bitwise_equal"] and r["check_mismatches"] == 0
