"""bench.py's multi-rank plumbing on CPU: `--gpus 2` outside torchrun re-launches itself
with 2 ranks (rendezvous on 127.0.0.1), and c4's fixed 8-view batch splits 4 + 4."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])


def test_self_launch_two_ranks_strong_c4():
    r = _run(["--gpus", "2", "--workload", "c4", "--selftest-launcher"])
    assert r["n_gpus"] == 2 and r["allreduce_sum"] == 3.0 and r["max_rank"] == 1.0
    assert r["scaling"] == "strong" and r["views_per_step"] == 8 and r["views_of_rank0_step1"] == [0, 2, 4, 6]


def test_self_launch_weak_default():
    r = _run(["--gpus", "2", "--selftest-launcher"])
    assert r["n_gpus"] == 2 and r["scaling"] == "weak" and r["views_per_step"] == 1


def test_step_views_partition_the_batch():
    sys.path.insert(0, ROOT)
    import bench
    for world in (1, 2, 4, 8):
        for step in (1, 2, 7):
            seen = sorted(j for r in range(world) for j in bench.step_views(step, 8, world, r))
            assert seen == list(range(8))   # c4: every ring view once per step
        weak = [bench.step_views(step, world, world, r)[0] for r in range(world) for step in (3,)]
        assert len(set(weak)) == world      # weak: distinct views per rank
