"""Multi-rank host logic on CPU (gloo, world_size 2): cost-balanced sharding
and the all-gather exchange reproduce the single-process results exactly.
Each rank runs its shard through the C restatement (the CUDA path needs a
GPU; the sharding/gather code is the same)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2508_08343_b200 import distributed as D


def test_balanced_shards_partition():
    costs = np.random.default_rng(0).pareto(1.5, size=1000)
    shards = D.balanced_shards(costs, 8)
    allidx = np.sort(np.concatenate(shards))
    np.testing.assert_array_equal(allidx, np.arange(1000))
    loads = [costs[s].sum() for s in shards]
    assert max(loads) <= min(loads) + costs.max() + 1e-9  # LPT bound


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import paper_2508_08343_b200 as lt
    from paper_2508_08343_b200.batch import ConditionBatch, sim_options
    from oracle.pyoracle import PortOracle
    from tests import workloads as W

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    port_or = PortOracle(threads=2)
    b = W.c2_batch(duration_s=120.0, stride=23)
    full = D.simulate_sharded(b, port_or, lt.h100_like_config(1), sim_options(None, True))
    conds, cfg, grid, dur, seed, opts = W.sweep_cases()
    pl, fr = D.sweep_sharded(ConditionBatch.from_conditions(conds), port_or, cfg, grid, dur, seed, opts,
                             sim_options())
    if rank == 0:
        q.put((full.tobytes(), pl.tobytes(), fr.tobytes()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gather_matches_single_process():
    import paper_2508_08343_b200 as lt
    from paper_2508_08343_b200 import _abi as A
    from paper_2508_08343_b200.batch import ConditionBatch, sim_options
    from oracle.pyoracle import PortOracle
    from tests import workloads as W

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    full_b, pl_b, fr_b = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    single = PortOracle(threads=2)
    b = W.c2_batch(duration_s=120.0, stride=23)
    ref, _ = single.simulate(b, lt.h100_like_config(1), sim_options(None, True))
    got = np.frombuffer(full_b, dtype=A.SUMMARY_DT)
    np.testing.assert_array_equal(got, ref)
    conds, cfg, grid, dur, seed, opts = W.sweep_cases()
    rp, rf = single.sweep(ConditionBatch.from_conditions(conds), cfg, grid, dur, seed, opts, sim_options())
    np.testing.assert_array_equal(np.frombuffer(pl_b, dtype=A.PLACEMENT_DT), rp)
    np.testing.assert_array_equal(np.frombuffer(fr_b, dtype=A.FRONTIER_DT).reshape(rf.shape), rf)
