"""Multi-GPU sharding of the DT sweep: one process per GPU (torch.distributed,
NCCL on B200s, gloo in the CPU tests), scenarios/conditions sharded with no
data-path collective, and one exchange step -- an all-gather of the
fixed-size per-scenario / per-condition result records.

The reference's only parallelism is run_parallel over independent grid
points / conditions (placement.cpp:65-96, :492-522); here the same
independence is used across ranks, and within a rank the device batch
covers the shard.
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import numpy as np

from . import _abi as A
from .batch import ConditionBatch, WorkloadBatch, frontier_capacity


def balanced_shards(costs: Sequence[float], world: int) -> List[np.ndarray]:
    """Longest-processing-time greedy assignment of items to `world` ranks
    (heavy scenarios dominate the tail). Each shard keeps its items
    in ascending index order; the union is a partition of range(len(costs))."""
    costs = np.asarray(costs, dtype=np.float64)
    order = np.argsort(-costs, kind="stable")
    load = np.zeros(world)
    owner = np.empty(len(costs), dtype=np.int64)
    for i in order:
        r = int(np.argmin(load))
        owner[i] = r
        load[r] += costs[i]
    return [np.nonzero(owner == r)[0] for r in range(world)]


def scenario_costs(batch: WorkloadBatch) -> np.ndarray:
    """Estimated work per scenario: sum over adapters of rate * duration *
    (mean output + 1) for generated scenarios, sum of outputs for scripted."""
    sc = batch.scenarios
    ad = batch.adapters
    lens = batch.lengths
    out = np.zeros(len(sc))
    for i, s in enumerate(sc):
        if s["n_requests"] >= 0:
            r = batch.requests[s["request_offset"]:s["request_offset"] + s["n_requests"]]
            out[i] = float(r["output_tokens"].sum()) + len(r)
            continue
        a = ad[s["adapter_offset"]:s["adapter_offset"] + s["n_adapters"]]
        mo = lens[s["length_index"]]["mean_output"]
        out[i] = float(a["rate"].sum()) * s["duration_s"] * (mo + 1.0)
    return out


def subset(batch: WorkloadBatch, idx: np.ndarray) -> WorkloadBatch:
    """The scenarios `idx` of a batch (adapter/request arrays are shared)."""
    return WorkloadBatch(batch.scenarios[idx].copy(), batch.adapters, batch.lengths, batch.full_lengths,
                         batch.requests)


def condition_subset(cb: ConditionBatch, idx: np.ndarray) -> ConditionBatch:
    return ConditionBatch(cb.conditions[idx].copy(), cb.templates, cb.lengths, cb.full_lengths)


def all_gather_records(records: np.ndarray, idx: np.ndarray, n_total: int, group=None,
                       device=None) -> np.ndarray:
    """All-gather structured records produced by each rank for its `idx`
    shard; every rank returns the full array in global order. The payload is
    moved as one uint8 tensor per rank (padded to the largest shard), on
    `device` (a CUDA device for NCCL) or CPU (gloo)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dt = records.dtype
    n_local = torch.tensor([len(idx)], dtype=torch.int64, device=device)
    sizes = [torch.zeros_like(n_local) for _ in range(world)]
    dist.all_gather(sizes, n_local, group=group)
    sizes = [int(s.item()) for s in sizes]
    width = max(sizes) if sizes else 0
    pay = np.zeros(width, dtype=[("i", np.int64), ("r", dt)])
    pay["i"][:len(idx)] = idx
    pay["r"][:len(idx)] = records[:len(idx)]
    t = torch.from_numpy(pay.view(np.uint8).copy()).to(device) if device is not None else \
        torch.from_numpy(pay.view(np.uint8).copy())
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t, group=group)
    full = np.zeros(n_total, dtype=dt)
    for r, o in enumerate(outs):
        part = o.cpu().numpy().view(pay.dtype)[:sizes[r]]
        full[part["i"]] = part["r"]
    return full


def simulate_sharded(batch: WorkloadBatch, runner, config, options: A.lt_sim_options, group=None,
                     device=None):
    """lt_simulate_batch over all ranks: shard by cost, run the local shard on
    this rank's device (`runner` = Device.runner, or an oracle runner in CPU
    tests), all-gather the per-scenario lt_sim_summary records."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    shards = balanced_shards(scenario_costs(batch), world)
    mine = shards[rank]
    local, _ = runner.simulate(subset(batch, mine), config, options)
    return all_gather_records(local, mine, len(batch.scenarios), group, device)


def sweep_sharded(conds: ConditionBatch, runner, config, grid, duration_s: float, seed: int, options,
                  sim: A.lt_sim_options, group=None, device=None, costs: Optional[Sequence[float]] = None):
    """lt_sweep_batch over all ranks: every grid point of a condition stays on
    one rank (K3's reduction is local); placements and frontiers are
    all-gathered."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = len(conds.conditions)
    if costs is None:
        t = conds.templates
        costs = [float(t[c["mix_offset"]:c["mix_offset"] + c["mix_count"]]["rate"].mean()) for c in conds.conditions]
    shards = balanced_shards(costs, world)
    mine = shards[rank]
    pl, fr = runner.sweep(condition_subset(conds, mine), config, grid, duration_s, seed, options, sim)
    maxf = frontier_capacity(grid)  # the same on every rank, also one with no conditions
    rec_dt = np.dtype([("p", A.PLACEMENT_DT), ("f", A.FRONTIER_DT, (maxf,))])
    rec = np.zeros(len(mine), dtype=rec_dt)
    rec["p"] = pl
    if len(mine):
        rec["f"] = fr.reshape(len(mine), maxf)
    full = all_gather_records(rec, mine, n, group, device)
    return full["p"], full["f"]
