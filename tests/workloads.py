"""Workload builders shared by the tests, tools/make_golden.py and bench.py.

The BASELINE.md configs (C1-C5) are built exactly as SURVEY.md 8(d) specifies;
the *_cases helpers are smaller seeded sets used for parity.
"""
from __future__ import annotations

import numpy as np

import paper_2508_08343_b200 as lt
from paper_2508_08343_b200 import _abi as A
from paper_2508_08343_b200.batch import WorkloadBatch

PAPER_RATES = [3.2, 1.6, 0.8, 0.4, 0.1, 0.05, 0.025, 0.0125, 0.00625, 0.003125]


def fixture_config(fx) -> lt.ServerConfig:
    """ServerConfig of a reference JSON fixture (json_io.cpp:188-235 field names)."""
    c = fx["config"]
    e = c["estimators"]
    mem = e["memory"]
    return lt.ServerConfig(
        slots=c["slots"], loaded_adapter_priority=c.get("loaded_adapter_priority", True),
        iteration_cap=c.get("iteration_cap", 100_000_000), ideal_includes_input=c.get("ideal_includes_input", False),
        latency=lt.LatencyCoefficients(**e["latency"]),
        memory=lt.MemoryModel(total_kv_budget=mem["total_kv_budget"], kv_bytes_per_token=mem.get("kv_bytes_per_token", 0.0),
                              slot_cost_table={int(k): v for k, v in mem.get("slot_cost_tokens", {}).items()},
                              slot_cost_base_rank8=mem.get("slot_cost_base_rank8")),
        load=lt.LoadLatencyTable(cpu_load_seconds={int(k): v for k, v in e["load"]["cpu_load_seconds"].items()},
                                 disk_multiplier=e["load"].get("disk_multiplier", 1.7),
                                 default_source=lt.LoadSource.Disk if e["load"].get("source") == "disk" else lt.LoadSource.Cpu))


def fixture_scripted(fx):
    ads = [lt.AdapterSpec(a["adapter_id"], a["rank"], 1.0) for a in fx["adapters"]]
    reqs = [lt.Request(r["request_id"], r["adapter_id"], r["arrival_time_s"], r["input_tokens"], r["output_tokens"])
            for r in fx["requests"]]
    return ads, reqs


def scripted_workload(adapters, duration_s):
    w = lt.WorkloadSpec(adapters=list(adapters), duration_s=duration_s)
    w.lengths = lt.LengthSpec.mean(1.0, 0.0, 1.0, 0.0)
    return w


def arrival_cases():
    cases = []
    rng = np.random.default_rng(11)
    for i in range(24):
        n = int(rng.choice([1, 3, 8, 17, 40]))
        ids = list(range(1, n + 1))
        if i % 4 == 1:
            ids = [int(x) for x in rng.permutation(np.arange(1000, 1000 + 7 * n, 7))]
        ads = []
        for k, aid in enumerate(ids):
            rank = int(rng.choice([0, 8, 16, 32]))
            rate = float(rng.choice([0.01, 0.1, 0.5, 2.0]))
            ad = lt.AdapterSpec(aid, rank, rate)
            if i % 5 == 2 and k % 3 == 0:
                ad.lengths = lt.LengthSpec.mean(40.0, 30.0, 12.0, 9.0)
            ads.append(ad)
        lengths = [lt.LengthSpec.mean(250, 50, 231, 50), lt.LengthSpec.mean(23, 5, 27, 5),
                   lt.LengthSpec.mean(2048, 512, 1024, 256), lt.LengthSpec.mean(3.0, 4.0, 2.0, 3.0),
                   lt.LengthSpec.mean(64, 0, 128, 0)][i % 5]
        seed = [0, 1, 17, 2 ** 32 + 5, 2 ** 63 + 12345, 987654321][i % 6]
        cases.append(lt.WorkloadSpec(adapters=ads, lengths=lengths, duration_s=float(rng.choice([30.0, 90.0, 200.0])),
                                     seed=seed))
    return cases


def c2_workloads(duration_s: float = 600.0, stride: int = 1):
    """C2: N in {8..256 step 8} x rank mode {8,16,32,mixed} x r in
    {3.2,...,0.0125}; per-adapter rate 8r/N; Mean(250,80,231,80); G=min(N,32);
    seed 1234+i; loop order N, rank, r."""
    rs = [3.2, 1.6, 0.8, 0.4, 0.1, 0.05, 0.025, 0.0125]
    wls, slots = [], []
    i = 0
    for n in range(8, 257, 8):
        for rank_mode in (8, 16, 32, "mixed"):
            for r in rs:
                if i % stride == 0:
                    ads = []
                    for aid in range(1, n + 1):
                        rank = (8, 16, 32)[(aid - 1) % 3] if rank_mode == "mixed" else rank_mode
                        ads.append(lt.AdapterSpec(aid, rank, 8.0 * r / n))
                    wls.append(lt.WorkloadSpec(adapters=ads, lengths=lt.LengthSpec.mean(250, 80, 231, 80),
                                               duration_s=duration_s, seed=1234 + i))
                    slots.append(min(n, 32))
                i += 1
    return wls, slots


def c2_batch(duration_s: float = 600.0, stride: int = 1) -> WorkloadBatch:
    """Vectorised C2 packing (same content as c2_workloads)."""
    rs = np.array([3.2, 1.6, 0.8, 0.4, 0.1, 0.05, 0.025, 0.0125])
    ns, modes, rr, seeds = [], [], [], []
    i = 0
    for n in range(8, 257, 8):
        for m in range(4):
            for r in rs:
                if i % stride == 0:
                    ns.append(n)
                    modes.append(m)
                    rr.append(r)
                    seeds.append(1234 + i)
                i += 1
    ns = np.array(ns)
    scen = np.zeros(len(ns), dtype=A.SCENARIO_DT)
    offs = np.concatenate([[0], np.cumsum(ns)[:-1]])
    scen["adapter_offset"] = offs
    scen["n_adapters"] = ns
    scen["length_index"] = 0
    scen["duration_s"] = duration_s
    scen["seed"] = np.array(seeds, dtype=np.uint64)
    scen["slots"] = np.minimum(ns, 32)
    scen["mode"] = A.MODE_MEAN
    scen["n_requests"] = -1
    ads = np.zeros(int(ns.sum()), dtype=A.ADAPTER_DT)
    ids = np.concatenate([np.arange(1, n + 1) for n in ns])
    mode_rep = np.repeat(np.array(modes), ns)
    ranks = np.where(mode_rep == 3, np.array([8, 16, 32])[(ids - 1) % 3], np.array([8, 16, 32, 0])[mode_rep])
    ads["adapter_id"] = ids
    ads["rank"] = ranks
    ads["rate"] = np.repeat(8.0 * np.array(rr) / ns, ns)
    ads["length_index"] = -1
    lens = np.zeros(1, dtype=A.LENGTH_DT)
    lens[0] = (A.MODE_MEAN, 0, 250.0, 80.0, 231.0, 80.0, 0, 0)
    return WorkloadBatch(scen, ads, lens, np.zeros(2, dtype=np.int32), np.zeros(0, dtype=A.REQUEST_DT))


def summary_cases():
    """~60 seeded engines spanning idle, saturated, slot-starved, KV-starved
    (preemption) and oversized-request regimes, on h100_like."""
    wls, slots = [], []
    rng = np.random.default_rng(5)
    for i in range(60):
        n = int(rng.choice([1, 4, 8, 24, 64, 130]))
        rank_mode = int(rng.integers(0, 4))
        agg = float(rng.choice([0.05, 0.4, 2.0, 6.0, 12.0]))
        lengths = [lt.LengthSpec.mean(250, 80, 231, 80), lt.LengthSpec.mean(2048, 512, 1024, 256),
                   lt.LengthSpec.mean(23, 5, 27, 5), lt.LengthSpec.mean(9000, 4000, 300, 100)][i % 4]
        ads = []
        for aid in range(1, n + 1):
            rank = (8, 16, 32)[(aid - 1) % 3] if rank_mode == 3 else (8, 16, 32)[rank_mode]
            if i % 7 == 3 and aid % 5 == 0:
                rank = 0
            ads.append(lt.AdapterSpec(aid, rank, agg / n))
        wls.append(lt.WorkloadSpec(adapters=ads, lengths=lengths, duration_s=float(rng.choice([60.0, 180.0])),
                                   seed=int(rng.integers(0, 2 ** 40))))
        slots.append(int(min(n, rng.choice([1, 2, 8, 32]))))
    return WorkloadBatch.from_workloads(wls, slots=slots), lt.h100_like_config(8)


def sweep_cases():
    conds = lt.enumerate_conditions([3.2, 0.4, 0.05, 0.0125], [8, 16, 32], lt.LengthSpec.mean(250, 50, 231, 50),
                                    triple_size=3, condition_stride=9)
    grid = lt.SweepGrid(n_values=[1, 2, 4, 8, 16, 32, 64], g_mode=lt.GMode.Geometric)
    return conds, lt.h100_like_config(1), grid, 120.0, 5, lt.SweepOptions(early_exit=True, early_exit_k=2)


def scripted_fuzz(seed: int, n_requests: int = 60, n_adapters: int = 5, tight: bool = True):
    """AC2-style randomized scripted scenario (acceptance.cpp:212-318)."""
    rng = np.random.default_rng(seed)
    ads = [lt.AdapterSpec(k + 1, int(rng.choice([0, 8, 16])), 1.0) for k in range(n_adapters)]
    t = np.sort(rng.uniform(0.0, 8.0, size=n_requests))
    if seed % 3 == 0:
        t = np.round(t, 1)  # ties in arrival time
    reqs = [lt.Request(i, int(rng.integers(1, n_adapters + 1)), float(t[i]), int(rng.integers(1, 40)),
                       int(rng.integers(1, 30))) for i in range(n_requests)]
    cfg = lt.ServerConfig(
        slots=int(rng.integers(1, 4)),
        latency=lt.LatencyCoefficients(1e-3, 2e-4, 5e-4, 2e-3, 0.02, 0.01, 1.1),
        memory=lt.MemoryModel(total_kv_budget=int(rng.integers(150, 600)) if tight else 100000,
                              slot_cost_table={8: 10, 16: 20}),
        load=lt.LoadLatencyTable(cpu_load_seconds={8: 0.05, 16: 0.09}),
        loaded_adapter_priority=bool(seed % 2 == 0))
    return ads, reqs, cfg


def full_mode_cases():
    """Full-mode length decks (sample_lengths, workload.cpp:149-161): deck sizes
    from 1 to beyond the device's shared-memory deck (8192), per-adapter lists,
    reshuffles on wrap, shared seeds."""
    rng = np.random.default_rng(77)
    wls = []
    for i in range(18):
        D = [1, 2, 7, 50, 300, 9000][i % 6]
        pairs = [(int(rng.integers(1, 400)), int(rng.integers(1, 300))) for _ in range(D)]
        n = [1, 5, 12, 40][i % 4]
        ads = [lt.AdapterSpec(k + 1, (8, 16, 32)[k % 3], float(rng.choice([0.05, 0.3, 2.0]))) for k in range(n)]
        if i % 3 == 1:
            own = [(int(rng.integers(1, 900)), int(rng.integers(1, 90))) for _ in range(int(rng.integers(1, 40)))]
            for a in ads[::2]:
                a.lengths = lt.LengthSpec.full(own)
        if i % 5 == 2:
            ads[0].lengths = lt.LengthSpec.mean(100.0, 20.0, 60.0, 10.0)
        wls.append(lt.WorkloadSpec(adapters=ads, lengths=lt.LengthSpec.full(pairs), duration_s=150.0,
                                   seed=100 + i // 2))
    return WorkloadBatch.from_workloads(wls, mode=lt.LengthMode.Full), lt.h100_like_config(8)


def _flat_batch(ns, ranks_per_adapter, rates_per_adapter, seeds, slots, lens_row, duration_s):
    """WorkloadBatch of generated scenarios with adapter ids 1..N each."""
    ns = np.asarray(ns, dtype=np.int64)
    scen = np.zeros(len(ns), dtype=A.SCENARIO_DT)
    scen["adapter_offset"] = np.concatenate([[0], np.cumsum(ns)[:-1]])
    scen["n_adapters"] = ns
    scen["length_index"] = 0
    scen["duration_s"] = duration_s
    scen["seed"] = np.asarray(seeds, dtype=np.uint64)
    scen["slots"] = slots
    scen["mode"] = A.MODE_MEAN
    scen["n_requests"] = -1
    ads = np.zeros(int(ns.sum()), dtype=A.ADAPTER_DT)
    ads["adapter_id"] = np.concatenate([np.arange(1, n + 1) for n in ns])
    ads["rank"] = ranks_per_adapter
    ads["rate"] = rates_per_adapter
    ads["length_index"] = -1
    lens = np.zeros(1, dtype=A.LENGTH_DT)
    lens[0] = lens_row
    return WorkloadBatch(scen, ads, lens, np.zeros(2, dtype=np.int32), np.zeros(0, dtype=A.REQUEST_DT))


def c3_batch(n_conditions: int = 2048, duration_s: float = 600.0) -> WorkloadBatch:
    """C3: the first 2,048 conditions of enumerate_conditions over the
    paper's rates x ranks {8,16,32}, triple size 3, each instantiated
    (placement.cpp:139-157) at N in {3, 6, ..., 96} with G = min(N, 16):
    65,536 scenarios, Mean(250,80,231,80), 600 s, one shared seed 7."""
    conds = lt.enumerate_conditions(PAPER_RATES, [8, 16, 32], lt.LengthSpec.mean(250, 80, 231, 80))[:n_conditions]
    n_list = np.arange(3, 97, 3)
    ns, rk, rt = [], [], []
    for c in conds:
        mr = np.array([leg.rank for leg in c.mix])
        mt = np.array([leg.rate for leg in c.mix])
        for n in n_list:
            ids = np.arange(n) % len(c.mix)
            ns.append(n)
            rk.append(mr[ids])
            rt.append(mt[ids])
    ns = np.array(ns)
    return _flat_batch(ns, np.concatenate(rk), np.concatenate(rt), np.full(len(ns), 7, dtype=np.uint64),
                       np.minimum(ns, 16), (A.MODE_MEAN, 0, 250.0, 80.0, 231.0, 80.0, 0, 0), duration_s)


def c5_batch(start: int = 0, count: int = 524_288, duration_s: float = 600.0) -> WorkloadBatch:
    """C5, scenarios [start, start + count) of 524,288: N = 8(1 + i mod 32),
    rank {8,16,32}[(i/32) mod 3], aggregate rate {0.5,1,2,4}[(i/96) mod 4] req/s
    split over the N adapters, Mean(2048,512,1024,256), 600 s, G = min(N, 32),
    seed 2^32 + i (per-scenario keys). Run under the llama31_8b / qwen25_7b profiles."""
    return c5_batch_at(np.arange(start, start + count, dtype=np.int64), duration_s)


def c5_batch_at(i, duration_s: float = 600.0) -> WorkloadBatch:
    """The C5 scenarios of the given indices (see c5_batch)."""
    i = np.asarray(i, dtype=np.int64)
    ns = 8 * (1 + i % 32)
    rank = np.array([8, 16, 32])[(i // 32) % 3]
    lam = np.array([0.5, 1.0, 2.0, 4.0])[(i // 96) % 4]
    return _flat_batch(ns, np.repeat(rank, ns), np.repeat(lam / ns, ns), (2 ** 32 + i).astype(np.uint64),
                       np.minimum(ns, 32), (A.MODE_MEAN, 0, 2048.0, 512.0, 1024.0, 256.0, 0, 0), duration_s)


C4_LENGTHS = [(23, 5, 27, 5), (250, 50, 231, 50), (423, 80, 358, 80), (128, 32, 231, 64), (512, 128, 256, 64),
              (1024, 256, 512, 128), (64, 0, 128, 0), (2048, 512, 1024, 256)]


def c4_conditions(count: int = 16_384):
    """C4: the 2,200 rate x rank triples (paper rates, ranks
    {8,16,32}, triple size 3, canonical enumerate_conditions order) under each
    of the 8 length settings, first `count` in (length setting, condition) order."""
    conds = []
    for L in C4_LENGTHS:
        conds += lt.enumerate_conditions(PAPER_RATES, [8, 16, 32], lt.LengthSpec.mean(*L))
        if len(conds) >= count:
            break
    return conds[:count]


def c4_grid():
    """C4's grid: N {1, 2, 4, ..., 256}, explicit G {2, ..., 64}; early exit k = 3; 600 s; seed 5."""
    grid = lt.SweepGrid(n_values=[1, 2, 4, 8, 16, 32, 64, 128, 256], g_mode=lt.GMode.Explicit,
                        g_values=[2, 4, 8, 16, 32, 64])
    return grid, lt.SweepOptions(early_exit=True, early_exit_k=3), 600.0, 5


def c4_sample_indices():
    """Sampled C4 conditions for the parity fixtures: 6 per length setting
    (the last setting only has C4's first 984 conditions), spread over the
    2,200 triples in canonical order (heavy 3.2 req/s mixes first, the
    lightest last)."""
    idx = []
    for s in range(len(C4_LENGTHS)):
        avail = min(2200, 16_384 - 2200 * s)
        for j in (0, 331, 662, 983, 1460, 2199):
            if j < avail:
                idx.append(2200 * s + j)
    return idx


C5_SAMPLE_STRIDE = 1021  # prime: every (N, rank, rate) combination of the 384-periodic grid is hit
