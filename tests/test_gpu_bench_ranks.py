"""bench.py's multi-rank path (the one the driver's N=2,4,8 scaling run
takes) on a one-GPU box: two torchrun ranks share cuda:0 and talk over gloo
(LT_BENCH_SHARED_GPU, a test mode; the real run is one rank per GPU over
NCCL). Checks the sharding, the all-gather inside the step and the
max-over-ranks / sum-over-ranks reduction of the line:

  * C3 (strong scaling): two shards simulate exactly the iterations of the
    whole set on one rank;
  * C2 (weak scaling): two replica grids, the line counts both;
  * C4: conditions sharded by cost, the sweep line over all of them.
"""
import json
import os
import socket
import subprocess
import sys

import pytest

from tests.conftest import ROOT

pytestmark = pytest.mark.gpu


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def bench(workload, ranks, *extra):
    env = dict(os.environ, LT_BENCH_SHARED_GPU="1")
    base = ["bench.py", "--gpus", str(ranks), "--workload", workload, "--steps", "1", "--warmup", "1",
            "--no-cpu-baseline", "--no-e2e", "--no-sweeps", *extra]
    if ranks > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={ranks}",
               "--master-addr", "127.0.0.1", "--master-port", str(free_port())] + base
    else:
        env.pop("WORLD_SIZE", None)
        cmd = [sys.executable] + base
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    lines = [json.loads(l) for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout  # rank 0 alone prints
    return lines[0]


def test_c3_two_shards_simulate_the_whole_set():
    one = bench("c3", 1)
    two = bench("c3", 2)
    assert two["n_gpus"] == 2 and two["scaling"] == "strong"
    assert two["config"]["engine_iterations_per_step"] == one["config"]["engine_iterations_per_step"]
    assert two["config"]["failed_scenarios"] == 0
    assert "test mode" in two["config"]["parallelism"]


def test_c2_two_replicas_count_both():
    one = bench("c2", 1)
    two = bench("c2", 2)
    assert two["n_gpus"] == 2 and two["scaling"] == "weak"
    it1, it2 = one["config"]["engine_iterations_per_step"], two["config"]["engine_iterations_per_step"]
    assert it1 < it2 < 3 * it1  # rank 1's grid has its own seeds


def test_c4_sharded_conditions():
    two = bench("c4", 2, "--warmup", "0")
    assert two["n_gpus"] == 2 and two["unit"] == "conditions/s" and two["value"] > 0
    assert two["config"]["test_mode"].startswith("LT_BENCH_SHARED_GPU")
