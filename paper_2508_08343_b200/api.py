"""Public API: the reference's hot-path functions, executed on a B200.

Mirrors run_simulation / run_scripted (engine.hpp:70-78), compute_metrics
(metrics.hpp:49-50), generate_arrivals (workload.hpp:111-113) and
sweep_optimal (placement.hpp:100-102), plus their batched forms, which are the
product: one call simulates thousands of independent engines. Everything runs
through libloratwin_gpu.so (include/loratwin_gpu.h); there is no CPU path —
without the built library or a B200 these calls raise.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from typing import List, Optional, Sequence

import numpy as np

from . import _abi as A
from .batch import (ConditionBatch, PackedConfig, PackedGrid, Runner, WorkloadBatch, sim_options)
from .types import (AdapterSpec, Condition, DatasetProgress, DatasetSpec, DeviceError, ERROR_CLASSES, FrontierPoint, LengthMode, LengthSpec,
                    IterationTraceRow, LoadEvent, LoadSource, LoratwinError, MetricsSummary, Phase, PlacementResult,
                    Request, RequestState,
                    ServerConfig, SimOptions, SimulationResult, SweepGrid, SweepOptions, WorkloadSpec)

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LT_GPU_LIB") or os.path.join(PKG_DIR, "lib", "libloratwin_gpu.so")

_lib: Optional[A.Lib] = None
_devices = {}


def load_library() -> A.Lib:
    """Loads the in-tree CUDA library; raises if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        _lib = A.Lib(LIB_PATH, "lt_")
        if _lib.abi_version() != A.ABI_VERSION:
            raise DeviceError("libloratwin_gpu.so ABI version mismatch")
    return _lib


class Device:
    """One lt_ctx: one B200 (lt_create), or several (lt_create_devices: the
    batch calls shard scenarios / conditions across them and gather the
    sweeps' placements to the first device)."""

    def __init__(self, index: int = 0, devices: Optional[Sequence[int]] = None):
        self.lib = load_library()
        st = A.lt_status()
        if devices is None:
            self.ctx = self.lib.create(index, C.byref(st))
        else:
            arr = (C.c_int32 * len(devices))(*devices)
            self.ctx = self.lib.create_devices(arr, len(devices), C.byref(st))
        if not self.ctx:
            raise DeviceError(st.message.decode())
        self.index = index if devices is None else devices[0]
        self.devices = [index] if devices is None else list(devices)
        self.runner = Runner(self.lib, self.ctx, self.message)

    def device_count(self) -> int:
        return self.lib.device_count(self.ctx)

    def gather_transport(self) -> str:
        return {A.GATHER_NONE: "none", A.GATHER_NCCL: "nccl", A.GATHER_PEER: "peer"}[
            self.lib.gather_transport(self.ctx)]

    def message(self, i: int) -> str:
        buf = C.create_string_buffer(512)
        self.lib.last_message(self.ctx, i, buf, 512)
        return buf.value.decode()

    def stream(self) -> int:
        return self.lib.stream(self.ctx) or 0

    def timing(self) -> dict:
        t = A.lt_timing()
        self.lib.last_timing(self.ctx, C.byref(t))
        return {name: getattr(t, name) for name, _ in A.lt_timing._fields_}

    def close(self):
        if self.ctx:
            self.lib.destroy(self.ctx)
            self.ctx = None

    # --- batched entry points (the product) -----------------------------------
    def simulate_batch(self, batch: WorkloadBatch, config: ServerConfig, options: Optional[SimOptions] = None,
                       want_states: bool = False, want_digest: bool = False, libm_variant: int = -1,
                       want_percentiles: bool = False):
        """run_simulation / run_scripted + compute_metrics for every scenario. The
        TTFT/ITL percentiles cost a second recording engine pass; they are filled
        only with want_percentiles (sweeps never read them)."""
        return self.runner.simulate(batch, config, sim_options(options, want_digest, libm_variant, want_percentiles),
                                    want_states)

    def simulate_report(self, batch: WorkloadBatch, config: ServerConfig, options: Optional[SimOptions] = None,
                        want_digest: bool = False, libm_variant: int = -1, want_percentiles: bool = False):
        """lt_simulate_report: (summaries, request states, report) where the
        report holds the trace rows, load events and per-request emit times
        (numpy arrays with their per-scenario / per-request offsets)."""
        return self.runner.report(batch, config, sim_options(options, want_digest, libm_variant, want_percentiles,
                                                             report=True))

    def generate_arrivals_batch(self, batch: WorkloadBatch, libm_variant: int = -1):
        return self.runner.generate_arrivals(batch, sim_options(None, False, libm_variant))

    def sweep_batch(self, conds: ConditionBatch, config: ServerConfig, grid: SweepGrid, duration_s: float,
                    seed: int, options: Optional[SweepOptions] = None, libm_variant: int = -1):
        return self.runner.sweep(conds, config, grid, duration_s, seed, options or SweepOptions(),
                                 sim_options(None, False, libm_variant))

    def plan(self, batch: WorkloadBatch, config: ServerConfig, options: Optional[SimOptions] = None,
             want_digest: bool = False) -> "Plan":
        return Plan(self, batch, config, sim_options(options, want_digest))


class Plan:
    """Inputs uploaded once and kept in HBM (lt_plan_*): run() re-simulates
    the whole batch on device; results() copies the summaries back."""

    def __init__(self, dev: Device, batch: WorkloadBatch, config: ServerConfig, opts: A.lt_sim_options):
        self.dev = dev
        self._keep = (batch, PackedConfig(config), opts)
        self.n = len(batch.scenarios)
        st = A.lt_status()
        cb = batch.c_struct()
        self.h = dev.lib.plan_simulate(dev.ctx, C.byref(cb), C.byref(self._keep[1].c), C.byref(opts), C.byref(st))
        if not self.h:
            raise DeviceError(st.message.decode())

    def run(self):
        st = A.lt_status()
        if self.dev.lib.plan_run(self.h, C.byref(st)) != A.LT_OK:
            raise DeviceError(st.message.decode())

    def results(self) -> np.ndarray:
        out = np.zeros(max(self.n, 1), dtype=A.SUMMARY_DT)
        st = A.lt_status()
        self.dev.lib.plan_results(self.h, out.ctypes.data, None, C.byref(st))
        if st.code == A.LT_ERR_DEVICE:
            raise DeviceError(st.message.decode())
        return out[:self.n]

    def trim(self):
        """lt_plan_trim: release the regenerated buffers until the next run."""
        self.dev.lib.plan_trim(self.h)

    def device_summaries(self):
        """(device pointer, bytes) of the lt_sim_summary array this plan writes."""
        p = C.c_void_p()
        n = C.c_int64()
        self.dev.lib.plan_summaries_device(self.h, C.byref(p), C.byref(n))
        return p.value or 0, n.value

    def close(self):
        if self.h:
            self.dev.lib.plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def device_group(devices: Sequence[int]) -> Device:
    """A multi-device context over `devices` (a device may repeat)."""
    return Device(devices=devices)


def device(index: int = 0) -> Device:
    if index not in _devices:
        _devices[index] = Device(index)
    return _devices[index]


# --- conversions ----------------------------------------------------------------

def raise_for(row, message: str):
    code = int(row["status"])
    if code != A.LT_OK:
        raise ERROR_CLASSES.get(code, LoratwinError)(message)


def metrics_of(row) -> MetricsSummary:
    return MetricsSummary(throughput_tok_s=float(row["throughput_tok_s"]), itl_mean_s=float(row["itl_mean_s"]),
                          itl_p50_s=float(row["itl_p50_s"]), itl_p99_s=float(row["itl_p99_s"]),
                          ttft_mean_s=float(row["ttft_mean_s"]), ttft_p50_s=float(row["ttft_p50_s"]),
                          ttft_p99_s=float(row["ttft_p99_s"]),
                          ideal_throughput_tok_s=float(row["ideal_throughput_tok_s"]),
                          starved=bool(row["starved"]), finished_count=int(row["finished_count"]),
                          rejected_count=int(row["rejected_count"]), degenerate=bool(row["degenerate"]))


def result_of(row, states, i: int, report=None, want_trace: bool = False) -> SimulationResult:
    reqs: List[RequestState] = []
    loads: List[LoadEvent] = []
    trace: List[IterationTraceRow] = []
    if report is not None:
        lo = int(report["load_offset"][i])
        for e in report["loads"][lo:lo + int(row["load_events"])]:
            loads.append(LoadEvent(time_s=float(e["time_s"]), adapter_id=int(e["adapter_id"]), rank=int(e["rank"]),
                                   source=LoadSource(int(e["source"])), latency_s=float(e["latency_s"])))
        if want_trace:
            to = int(report["trace_offset"][i])
            for t in report["trace"][to:to + int(row["iterations"])]:
                trace.append(IterationTraceRow(time_s=float(t["time_s"]), iteration=int(t["iteration"]),
                                               r_running=int(t["r_running"]), r_waiting=int(t["r_waiting"]),
                                               a_running=int(t["a_running"]), lat_step_s=float(t["lat_step_s"]),
                                               loads=int(t["loads"])))
    if states is not None:
        off = int(states["req_offset"][i])
        for k in range(int(row["n_requests"])):
            j = off + k
            first = float(states["first_token_time_s"][j])
            emits: List[float] = []
            if report is not None:
                eo = int(report["emit_offset"][j])
                emits = report["emit_times"][eo:eo + int(states["tokens_generated"][j])].tolist()
            reqs.append(RequestState(
                request=Request(request_id=k, adapter_id=int(states["adapter_id"][j]),
                                arrival_time_s=float(states["arrival_time_s"][j]),
                                input_tokens=int(states["input_tokens"][j]),
                                output_tokens=int(states["output_tokens"][j])),
                phase=Phase(int(states["phase"][j])), tokens_generated=int(states["tokens_generated"][j]),
                first_token_time_s=None if math.isnan(first) else first,
                completion_time_s=float(states["completion_time_s"][j]),
                preemption_count=int(states["preemption_count"][j]), token_emit_times_s=emits))
    return SimulationResult(requests=reqs, iterations=int(row["iterations"]), final_clock_s=float(row["final_clock_s"]),
                            duration_s=float(row["duration_s"]), truncated=bool(row["truncated"]),
                            slots=int(row["slots"]), served_adapters=int(row["served_adapters"]),
                            kv_capacity_tokens=int(row["kv_capacity_tokens"]), load_events=int(row["load_events"]),
                            preemptions=int(row["preemptions"]), tokens_in_window=int(row["tokens_in_window"]),
                            digest=int(row["digest"]), metrics=metrics_of(row), load_event_list=loads,
                            iteration_trace=trace)


def placement_of(row, frontier_rows) -> PlacementResult:
    fr = [FrontierPoint(n=int(f["n"]), g=int(f["g"]), throughput_tok_s=float(f["throughput_tok_s"]),
                        starved=bool(f["starved"]), skipped=bool(f["skipped"]))
          for f in frontier_rows[:int(row["frontier_count"])]]
    return PlacementResult(max_throughput_tok_s=float(row["max_throughput_tok_s"]), n_star=int(row["n_star"]),
                           g_star=int(row["g_star"]), frontier=fr, all_starved=bool(row["all_starved"]),
                           frontier_open=bool(row["frontier_open"]))


# --- reference-shaped single calls ---------------------------------------------

def run_simulation(workload: WorkloadSpec, config: ServerConfig, mode: LengthMode = LengthMode.Mean,
                   options: Optional[SimOptions] = None, dev: Optional[Device] = None) -> SimulationResult:
    """engine.hpp:70-71 — one engine on the B200 (result + device-computed metrics)."""
    dev = dev or device()
    batch = WorkloadBatch.from_workloads([workload], mode=mode)
    out, states, rep = dev.simulate_report(batch, config, options, want_percentiles=True)
    raise_for(out[0], dev.message(0))
    return result_of(out[0], states, 0, rep, bool(options and options.record_iteration_trace))


def run_scripted(requests: Sequence[Request], adapters: Sequence[AdapterSpec], duration_s: float,
                 config: ServerConfig, options: Optional[SimOptions] = None,
                 dev: Optional[Device] = None) -> SimulationResult:
    """engine.hpp:76-78 — the same loop over an explicit request list."""
    dev = dev or device()
    w = WorkloadSpec(adapters=list(adapters), duration_s=duration_s)
    w.lengths.mean_input = w.lengths.mean_output = 1.0  # unused by scripted runs
    batch = WorkloadBatch.from_workloads([w], scripted=[list(requests)])
    out, states, rep = dev.simulate_report(batch, config, options, want_percentiles=True)
    raise_for(out[0], dev.message(0))
    return result_of(out[0], states, 0, rep, bool(options and options.record_iteration_trace))


def _length_means(spec: LengthSpec):
    """(input mean, output mean) of a LengthSpec (workload.cpp:29-50, :75-89):
    Full mode averages the list in order, Mean mode returns the given means."""
    if spec.mode == LengthMode.Full:
        if not spec.full_lengths:
            return 0.0, 0.0
        s_in = s_out = 0.0
        for a, b in spec.full_lengths:
            s_in += float(a)
            s_out += float(b)
        n = float(len(spec.full_lengths))
        return s_in / n, s_out / n
    return spec.mean_input, spec.mean_output


def ideal_throughput(workload: WorkloadSpec, include_input: bool = False) -> float:
    """metrics.cpp:36-45: Σ over adapters in spec order of rate x mean tokens."""
    total = 0.0
    for ad in workload.adapters:
        mi, mo = _length_means(ad.lengths if ad.lengths is not None else workload.lengths)
        tokens = mo + mi if include_input else mo
        total += ad.rate * tokens
    return total


def compute_metrics(result: SimulationResult, workload: WorkloadSpec,
                    ideal_includes_input: bool = False) -> MetricsSummary:
    """metrics.hpp:49-50. Throughput, TTFT and ITL come from the device epilogue
    (K2, and the percentile pass); the ideal throughput and the starved verdict
    depend on the caller's workload and flag (metrics.cpp:72, :108-111), so they
    are recomputed here from `workload`, `ideal_includes_input` and the
    result's rejected requests, exactly as the reference does."""
    m = result.metrics
    ideal = ideal_throughput(workload, ideal_includes_input)
    if not result.requests and m.degenerate:
        return MetricsSummary(ideal_throughput_tok_s=ideal, degenerate=True)
    if not result.requests:
        raise ValueError("compute_metrics needs the per-request states (run_simulation / run_scripted "
                         "return them; batched summaries carry the device-computed metrics)")
    rejected_demand = 0.0
    for r in result.requests:  # request_id order (metrics.cpp:84-89)
        if r.phase == Phase.Rejected:
            rejected_demand += float(r.request.output_tokens) / result.duration_s
    eff = max(ideal - rejected_demand, 0.0)
    return MetricsSummary(throughput_tok_s=m.throughput_tok_s, itl_mean_s=m.itl_mean_s, itl_p50_s=m.itl_p50_s,
                          itl_p99_s=m.itl_p99_s, ttft_mean_s=m.ttft_mean_s, ttft_p50_s=m.ttft_p50_s,
                          ttft_p99_s=m.ttft_p99_s, ideal_throughput_tok_s=ideal,
                          starved=m.throughput_tok_s < 0.9 * eff, finished_count=m.finished_count,
                          rejected_count=m.rejected_count, degenerate=False)


def generate_arrivals(workload: WorkloadSpec, mode_override: Optional[LengthMode] = None,
                      dev: Optional[Device] = None) -> List[Request]:
    """workload.hpp:111-113 — arrivals generated on device (K0 + merge)."""
    dev = dev or device()
    mode = workload.lengths.mode if mode_override is None else mode_override
    batch = WorkloadBatch.from_workloads([workload], mode=mode)
    reqs, counts = dev.generate_arrivals_batch(batch)
    code, idx, msg = dev.runner.last_arrivals_status
    if code != A.LT_OK:
        raise ERROR_CLASSES.get(code, LoratwinError)(msg)
    return [Request(int(r["request_id"]), int(r["adapter_id"]), float(r["arrival_time_s"]),
                    int(r["input_tokens"]), int(r["output_tokens"])) for r in reqs]


def sweep_optimal(condition: Condition, config: ServerConfig, grid: SweepGrid, duration_s: float, seed: int,
                  options: Optional[SweepOptions] = None, dev: Optional[Device] = None) -> PlacementResult:
    """placement.hpp:100-102 — every grid point simulated on device, reduced on device (K3)."""
    dev = dev or device()
    out, fr = dev.sweep_batch(ConditionBatch.from_conditions([condition]), config, grid, duration_s, seed, options)
    raise_for(out[0], dev.message(0))
    return placement_of(out[0], fr[0])


def sweep_conditions(conditions: Sequence[Condition], config: ServerConfig, grid: SweepGrid, duration_s: float,
                     seed: int, options: Optional[SweepOptions] = None,
                     dev: Optional[Device] = None) -> List[PlacementResult]:
    """Batched sweep_optimal (generate_dataset's loop, placement.cpp:492-522).
    Failed conditions are returned as the exception object, like
    generate_dataset records failures and continues."""
    dev = dev or device()
    out, fr = dev.sweep_batch(ConditionBatch.from_conditions(conditions), config, grid, duration_s, seed, options)
    res = []
    for i in range(len(conditions)):
        if int(out[i]["status"]) != A.LT_OK:
            res.append(ERROR_CLASSES.get(int(out[i]["status"]), LoratwinError)(dev.message(i)))
        else:
            res.append(placement_of(out[i], fr[i]))
    return res


# --- dataset generation (placement.hpp:104-158) -------------------------------------------------

class _PackedDataset:
    """lt_dataset_spec plus the arrays its pointers reference."""

    def __init__(self, spec: DatasetSpec):
        from .batch import _LengthTable
        lt = _LengthTable()
        lt.add(spec.lengths)
        self.lens, self.full = lt.arrays()
        self.rates = np.array(spec.rates if spec.rates else [0.0], dtype=np.float64)
        self.ranks = np.array(spec.ranks if spec.ranks else [0], dtype=np.int32)
        self.grid = PackedGrid(spec.grid)
        c = A.lt_dataset_spec()
        c.rates = self.rates.ctypes.data_as(C.POINTER(C.c_double))
        c.n_rates = len(spec.rates)
        c.triple_size = spec.triple_size
        c.ranks = self.ranks.ctypes.data_as(C.POINTER(C.c_int32))
        c.n_ranks = len(spec.ranks)
        c.condition_stride = spec.condition_stride
        c.lengths = A.lt_length_spec.from_buffer_copy(self.lens[0].tobytes())
        c.full_lengths = self.full.ctypes.data_as(C.POINTER(C.c_int32))
        c.n_full_pairs = len(self.full) // 2
        c.duration_s = spec.duration_s
        c.seed = spec.seed
        c.grid = self.grid.c
        o = A.lt_sweep_options()
        o.early_exit, o.early_exit_k = int(spec.sweep.early_exit), spec.sweep.early_exit_k
        o.jobs, o.mode = spec.sweep.jobs, int(spec.sweep.mode)
        c.sweep = o
        self.c = c


def run_generate_dataset(lib: A.Lib, ctx, spec: DatasetSpec, config: ServerConfig, out_csv: str,
                         on_error=None) -> DatasetProgress:
    """Calls lib.generate_dataset (the GPU library or an oracle with the same ABI)."""
    pd = _PackedDataset(spec)
    pc = PackedConfig(config)
    msgs: List[str] = []

    def cb(msg, _user):
        msgs.append(msg.decode())

    fn = A.ERROR_FN(cb)
    prog = A.lt_dataset_progress()
    st = A.lt_status()
    rc = lib.generate_dataset(ctx, C.byref(pd.c), C.byref(pc.c), os.fsencode(out_csv), fn, None, C.byref(prog),
                              C.byref(st))
    if rc != A.LT_OK:
        raise ERROR_CLASSES.get(rc, LoratwinError)(st.message.decode())
    if on_error:
        for m in msgs:
            on_error(m)
    return DatasetProgress(prog.total_conditions, prog.completed, prog.failed)


def generate_dataset(spec: DatasetSpec, config: ServerConfig, out_csv: str, on_error=None,
                     dev: Optional[Device] = None) -> DatasetProgress:
    """placement.hpp:151-153 — every pending condition of the spec swept on the
    B200 in batched lt_sweep_batch calls; rows appended in canonical order,
    resumable by condition hash. Same CSV bytes as the reference."""
    dev = dev or device()
    return run_generate_dataset(dev.lib, dev.ctx, spec, config, out_csv, on_error)


def _condition_args(condition: Condition):
    from .batch import _LengthTable
    lt = _LengthTable()
    lt.add(condition.lengths)
    lens, full = lt.arrays()
    mix = (A.lt_template * max(len(condition.mix), 1))()
    for i, leg in enumerate(condition.mix):
        mix[i].rank, mix[i].rate = leg.rank, leg.rate
    return mix, A.lt_length_spec.from_buffer_copy(lens[0].tobytes()), full


def condition_hash(condition: Condition, duration_s: float, seed: int, grid: SweepGrid, lib=None) -> int:
    """placement.cpp:266-296 (host code of the library; no device needed)."""
    lib = lib or load_library()
    mix, ls, full = _condition_args(condition)
    pg = PackedGrid(grid)
    return int(lib.condition_hash(mix, len(condition.mix), C.byref(ls), full.ctypes.data_as(C.POINTER(C.c_int32)),
                                  duration_s, seed, C.byref(pg.c)))


def encode_workload(condition: Condition, lib=None) -> List[float]:
    """placement.cpp:117-137: the 16 WorkloadFeatures values (FEATURE_NAMES order)."""
    lib = lib or load_library()
    mix, ls, full = _condition_args(condition)
    out = (C.c_double * 16)()
    st = A.lt_status()
    rc = lib.encode_workload(mix, len(condition.mix), C.byref(ls), full.ctypes.data_as(C.POINTER(C.c_int32)), out,
                             C.byref(st))
    if rc != A.LT_OK:
        raise ERROR_CLASSES.get(rc, LoratwinError)(st.message.decode())
    return list(out)
