"""Python mirror of the reference's public types (proj/core/include/loratwin/*.hpp).

Field names, defaults and meanings follow the reference so callers and tests
read like the reference's own (server_config.hpp:26-43, estimators.hpp:33-71,
workload.hpp:26-99, engine.hpp:29-64, metrics.hpp:27-40, placement.hpp:32-95).
"""
from __future__ import annotations

import enum
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple


class LoratwinError(Exception):
    """Base of the reference's exception taxonomy (errors.hpp:25-54)."""


class ValidationError(LoratwinError):
    """Bad user input (errors.hpp:25-29)."""


class ConfigError(LoratwinError):
    """Incomplete or infeasible server configuration (errors.hpp:31-36)."""


class FitError(LoratwinError):
    """Least-squares fitting failure (errors.hpp:38-42); off the hot path."""


class SimulationError(LoratwinError):
    """A simulation that cannot make progress (errors.hpp:44-49)."""


class InternalError(LoratwinError):
    """Broken internal invariant (errors.hpp:51-54)."""


class UnsupportedError(LoratwinError):
    """Input outside what the B200 device path implements."""


class DeviceError(LoratwinError):
    """CUDA failure or no usable B200."""


ERROR_CLASSES = {1: ValidationError, 2: ConfigError, 3: SimulationError, 4: InternalError,
                 5: UnsupportedError, 6: DeviceError}


class LengthMode(enum.IntEnum):  # workload.hpp:26
    Full = 0
    Mean = 1


class LoadSource(enum.IntEnum):  # estimators.hpp:29
    Cpu = 0
    Disk = 1


class Phase(enum.IntEnum):  # kv_scheduler.hpp:28
    Waiting = 0
    Running = 1
    Preempted = 2
    Finished = 3
    Rejected = 4


@dataclass
class LatencyCoefficients:  # estimators.hpp:33-43
    k1: float = 0.0
    k2: float = 0.0
    k3: float = 0.0
    k4: float = 0.0
    k5: float = 0.0
    k6: float = 0.0
    k7: float = 1.0


@dataclass
class MemoryModel:  # estimators.hpp:45-58
    total_kv_budget: int = 0
    kv_bytes_per_token: float = 0.0
    slot_cost_table: Dict[int, int] = field(default_factory=dict)
    slot_cost_base_rank8: Optional[float] = None


@dataclass
class LoadLatencyTable:  # estimators.hpp:60-67
    cpu_load_seconds: Dict[int, float] = field(default_factory=dict)
    disk_multiplier: float = 1.7
    default_source: LoadSource = LoadSource.Cpu


@dataclass
class ServerConfig:  # server_config.hpp:26-43
    slots: int = 1
    latency: LatencyCoefficients = field(default_factory=LatencyCoefficients)
    memory: MemoryModel = field(default_factory=MemoryModel)
    load: LoadLatencyTable = field(default_factory=LoadLatencyTable)
    loaded_adapter_priority: bool = True
    iteration_cap: int = 100_000_000
    ideal_includes_input: bool = False


def h100_like_config(slots: int) -> ServerConfig:
    """The reference's only preset (server_config.cpp:30-51; configs/h100_like.json)."""
    return ServerConfig(
        slots=slots,
        latency=LatencyCoefficients(1e-5, 2e-6, 2e-5, 3.5e-4, 0.022, 0.015, 1.15),
        memory=MemoryModel(total_kv_budget=320_000, kv_bytes_per_token=160.0 * 1024.0,
                           slot_cost_base_rank8=800.0),
        load=LoadLatencyTable(cpu_load_seconds={8: 0.04, 16: 0.07, 32: 0.12, 64: 0.22, 128: 0.40},
                              disk_multiplier=1.7, default_source=LoadSource.Cpu))


def config_from_json(d: dict, slots: int = None) -> ServerConfig:
    """ServerConfig from the reference's JSON schema (json_io.cpp:188-235)."""
    lat, mem, load = d["latency"], d["memory"], d["load"]
    return ServerConfig(
        slots=d.get("slots", 1) if slots is None else slots,
        loaded_adapter_priority=d.get("loaded_adapter_priority", True),
        iteration_cap=d.get("iteration_cap", 100_000_000), ideal_includes_input=d.get("ideal_includes_input", False),
        latency=LatencyCoefficients(*(lat[k] for k in ("k1", "k2", "k3", "k4", "k5", "k6", "k7"))),
        memory=MemoryModel(total_kv_budget=mem["total_kv_budget"], kv_bytes_per_token=mem.get("kv_bytes_per_token", 0.0),
                           slot_cost_table={int(k): v for k, v in mem.get("slot_cost_tokens", {}).items()},
                           slot_cost_base_rank8=mem.get("slot_cost_base_rank8")),
        load=LoadLatencyTable(cpu_load_seconds={int(k): v for k, v in load["cpu_load_seconds"].items()},
                              disk_multiplier=load.get("disk_multiplier", 1.7),
                              default_source=LoadSource.Disk if load.get("default_source") == "disk" else LoadSource.Cpu))


def profile_config(name: str, slots: int) -> ServerConfig:
    """A packaged profile: h100_like (the reference preset), llama31_8b or
    qwen25_7b (synthetic, configs/README.md)."""
    import json
    import os
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "configs", name + ".json")
    with open(path) as f:
        return config_from_json(json.load(f), slots)


@dataclass
class LengthSpec:  # workload.hpp:31-65
    mode: LengthMode = LengthMode.Mean
    full_lengths: List[Tuple[int, int]] = field(default_factory=list)
    mean_input: float = 0.0
    std_input: float = 0.0
    mean_output: float = 0.0
    std_output: float = 0.0

    @staticmethod
    def full(pairs) -> "LengthSpec":
        return LengthSpec(mode=LengthMode.Full, full_lengths=[(int(a), int(b)) for a, b in pairs])

    @staticmethod
    def mean(mean_in: float, std_in: float, mean_out: float, std_out: float) -> "LengthSpec":
        return LengthSpec(mode=LengthMode.Mean, mean_input=mean_in, std_input=std_in,
                          mean_output=mean_out, std_output=std_out)

    def key(self):
        return (int(self.mode), tuple(self.full_lengths), self.mean_input, self.std_input,
                self.mean_output, self.std_output)


@dataclass
class AdapterSpec:  # workload.hpp:71-76
    adapter_id: int = 0
    rank: int = 8
    rate: float = 0.0
    lengths: Optional[LengthSpec] = None


@dataclass
class WorkloadSpec:  # workload.hpp:78-89
    adapters: List[AdapterSpec] = field(default_factory=list)
    lengths: LengthSpec = field(default_factory=LengthSpec)
    duration_s: float = 0.0
    seed: int = 0


@dataclass
class Request:  # workload.hpp:91-99
    request_id: int = 0
    adapter_id: int = 0
    arrival_time_s: float = 0.0
    input_tokens: int = 1
    output_tokens: int = 1


@dataclass
class SimOptions:  # engine.hpp:29-35
    check_invariants: bool = False
    record_iteration_trace: bool = False
    iteration_cap_override: Optional[int] = None


@dataclass
class RequestState:  # kv_scheduler.hpp:30-41
    request: Request
    phase: Phase
    tokens_generated: int
    first_token_time_s: Optional[float]
    completion_time_s: float
    preemption_count: int
    # filled by the report call (run_simulation / run_scripted / simulate_report)
    token_emit_times_s: List[float] = field(default_factory=list)


@dataclass
class LoadEvent:  # adapter_cache.hpp:28-34
    time_s: float
    adapter_id: int
    rank: int
    source: "LoadSource"
    latency_s: float


@dataclass
class IterationTraceRow:  # engine.hpp:37-45
    time_s: float
    iteration: int
    r_running: int
    r_waiting: int
    a_running: int
    lat_step_s: float
    loads: int


@dataclass
class MetricsSummary:  # metrics.hpp:27-40
    throughput_tok_s: float = 0.0
    itl_mean_s: float = 0.0
    itl_p50_s: float = 0.0
    itl_p99_s: float = 0.0
    ttft_mean_s: float = 0.0
    ttft_p50_s: float = 0.0
    ttft_p99_s: float = 0.0
    ideal_throughput_tok_s: float = 0.0
    starved: bool = False
    finished_count: int = 0
    rejected_count: int = 0
    degenerate: bool = False


@dataclass
class SimulationResult:  # engine.hpp:47-64
    requests: List[RequestState]
    iterations: int
    final_clock_s: float
    duration_s: float
    truncated: bool
    slots: int
    served_adapters: int
    kv_capacity_tokens: int
    load_events: int
    preemptions: int
    tokens_in_window: int
    digest: int
    metrics: MetricsSummary
    # SimulationResult.load_events / iteration_trace of the reference (the
    # count above keeps the name load_events); filled by the report call,
    # iteration_trace only with SimOptions.record_iteration_trace
    load_event_list: List[LoadEvent] = field(default_factory=list)
    iteration_trace: List[IterationTraceRow] = field(default_factory=list)


@dataclass
class AdapterTemplate:  # placement.hpp:32-35
    rank: int = 8
    rate: float = 0.0


@dataclass
class Condition:  # placement.hpp:37-40
    mix: List[AdapterTemplate] = field(default_factory=list)
    lengths: LengthSpec = field(default_factory=LengthSpec)


class GMode(enum.IntEnum):
    Geometric = 0
    Explicit = 1


@dataclass
class SweepGrid:  # placement.hpp:77-88
    n_values: List[int] = field(default_factory=list)
    g_mode: GMode = GMode.Geometric
    g_values: List[int] = field(default_factory=list)

    def g_candidates(self, n: int) -> List[int]:  # placement.cpp:159-167
        gs = [8, n // 4, n // 2, n] if self.g_mode == GMode.Geometric else list(self.g_values)
        return sorted({min(max(g, 1), n) for g in gs})


@dataclass
class SweepOptions:  # placement.hpp:90-95
    early_exit: bool = True
    early_exit_k: int = 3
    jobs: int = 1
    mode: LengthMode = LengthMode.Mean


@dataclass
class FrontierPoint:  # placement.hpp:60-66
    n: int = 0
    g: int = 0
    throughput_tok_s: float = 0.0
    starved: bool = False
    skipped: bool = False


@dataclass
class PlacementResult:  # placement.hpp:68-75
    max_throughput_tok_s: float = 0.0
    n_star: int = 0
    g_star: int = 0
    frontier: List[FrontierPoint] = field(default_factory=list)
    all_starved: bool = False
    frontier_open: bool = False


def instantiate_condition(condition: Condition, served_adapters: int, duration_s: float,
                          seed: int) -> WorkloadSpec:
    """placement.cpp:139-157: adapter ids 1..N, (rank, rate) round-robin over the mix."""
    if not condition.mix:
        raise ValidationError("condition.mix: must be non-empty")
    if served_adapters < 1:
        raise ValidationError("served_adapters: must be >= 1")
    adapters = []
    for i in range(served_adapters):
        leg = condition.mix[i % len(condition.mix)]
        adapters.append(AdapterSpec(adapter_id=i + 1, rank=leg.rank, rate=leg.rate))
    return WorkloadSpec(adapters=adapters, lengths=condition.lengths, duration_s=duration_s, seed=seed)


@dataclass
class DatasetSpec:  # placement.hpp:126-137
    rates: List[float] = field(default_factory=list)
    ranks: List[int] = field(default_factory=list)
    triple_size: int = 3
    condition_stride: int = 1
    lengths: LengthSpec = field(default_factory=LengthSpec)
    duration_s: float = 600.0
    seed: int = 0
    grid: SweepGrid = field(default_factory=SweepGrid)
    sweep: SweepOptions = field(default_factory=SweepOptions)


@dataclass
class DatasetProgress:  # placement.hpp:143-147
    total_conditions: int = 0
    completed: int = 0
    failed: int = 0


FEATURE_NAMES = ["rate_max", "rate_min", "rate_mean", "rate_std", "rank_max", "rank_min", "rank_mean", "rank_std",
                 "input_len_max", "input_len_min", "input_len_mean", "input_len_std", "output_len_max",
                 "output_len_min", "output_len_mean", "output_len_std"]  # placement.cpp:100-107


def enumerate_conditions(rates, ranks, lengths: LengthSpec, triple_size: int = 3,
                         condition_stride: int = 1) -> List[Condition]:
    """placement.cpp:298-340: non-decreasing index tuples of rates x ranks, lexicographic."""
    if triple_size < 1:
        raise ValidationError("dataset.triple_size: must be >= 1")
    if not rates:
        raise ValidationError("dataset.rates: must be non-empty")
    if not ranks:
        raise ValidationError("dataset.ranks: must be non-empty")
    if condition_stride < 1:
        raise ValidationError("dataset.condition_stride: must be >= 1")

    def combos(n):
        out = []
        idx = [0] * triple_size
        while True:
            out.append(list(idx))
            pos = triple_size - 1
            while pos >= 0 and idx[pos] == n - 1:
                pos -= 1
            if pos < 0:
                break
            idx[pos] += 1
            for j in range(pos + 1, triple_size):
                idx[j] = idx[pos]
        return out

    conds = []
    counter = 0
    for rt in combos(len(rates)):
        for kt in combos(len(ranks)):
            keep = counter % condition_stride == 0
            counter += 1
            if not keep:
                continue
            conds.append(Condition(mix=[AdapterTemplate(rank=ranks[kt[l]], rate=rates[rt[l]])
                                        for l in range(triple_size)], lengths=lengths))
    return conds
