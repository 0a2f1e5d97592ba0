"""Packing of reference-typed inputs into the C-ABI's POD arrays, and a runner
that drives any library exporting the loratwin_gpu.h entry points."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Callable, Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _abi as A
from .types import (ERROR_CLASSES, Condition, LengthMode, LengthSpec, LoratwinError, ServerConfig, UnsupportedError,
                    SweepGrid, SweepOptions, SimOptions, WorkloadSpec, Request)


class PackedConfig:
    """lt_server_config plus the arrays its pointers reference."""

    def __init__(self, cfg: ServerConfig):
        self.cfg = cfg
        sc = sorted(cfg.memory.slot_cost_table.items())
        ld = sorted(cfg.load.cpu_load_seconds.items())
        self.sc_rank = np.array([r for r, _ in sc], dtype=np.int32)
        self.sc_tok = np.array([t for _, t in sc], dtype=np.int64)
        self.ld_rank = np.array([r for r, _ in ld], dtype=np.int32)
        self.ld_sec = np.array([s for _, s in ld], dtype=np.float64)
        c = A.lt_server_config()
        c.slots = cfg.slots
        c.loaded_adapter_priority = int(bool(cfg.loaded_adapter_priority))
        c.iteration_cap = int(cfg.iteration_cap)
        c.ideal_includes_input = int(bool(cfg.ideal_includes_input))
        c.load_source = int(cfg.load.default_source)
        L = cfg.latency
        c.k1, c.k2, c.k3, c.k4, c.k5, c.k6, c.k7 = L.k1, L.k2, L.k3, L.k4, L.k5, L.k6, L.k7
        c.total_kv_budget = int(cfg.memory.total_kv_budget)
        c.kv_bytes_per_token = float(cfg.memory.kv_bytes_per_token)
        c.has_slot_cost_base_rank8 = int(cfg.memory.slot_cost_base_rank8 is not None)
        c.slot_cost_base_rank8 = float(cfg.memory.slot_cost_base_rank8 or 0.0)
        c.n_slot_cost = len(sc)
        c.slot_cost_rank = self.sc_rank.ctypes.data_as(C.POINTER(C.c_int32)) if len(sc) else None
        c.slot_cost_tokens = self.sc_tok.ctypes.data_as(C.POINTER(C.c_int64)) if len(sc) else None
        c.n_load = len(ld)
        c.load_rank = self.ld_rank.ctypes.data_as(C.POINTER(C.c_int32)) if len(ld) else None
        c.load_seconds = self.ld_sec.ctypes.data_as(C.POINTER(C.c_double)) if len(ld) else None
        c.disk_multiplier = float(cfg.load.disk_multiplier)
        self.c = c


class _LengthTable:
    def __init__(self):
        self.rows: List[tuple] = []
        self.full: List[int] = []
        self.index: Dict[tuple, int] = {}

    def add(self, spec: LengthSpec) -> int:
        k = spec.key()
        if k in self.index:
            return self.index[k]
        off = len(self.full) // 2
        for a, b in spec.full_lengths:
            self.full += [int(a), int(b)]
        self.rows.append((int(spec.mode), 0, spec.mean_input, spec.std_input, spec.mean_output,
                          spec.std_output, off, len(spec.full_lengths)))
        self.index[k] = len(self.rows) - 1
        return self.index[k]

    def arrays(self):
        lens = np.zeros(max(len(self.rows), 1), dtype=A.LENGTH_DT)
        for i, r in enumerate(self.rows):
            lens[i] = r
        full = np.array(self.full if self.full else [0, 0], dtype=np.int32)
        return lens, full


@dataclass
class WorkloadBatch:
    """Packed lt_workload_batch arrays (numpy, C layout)."""

    scenarios: np.ndarray
    adapters: np.ndarray
    lengths: np.ndarray
    full_lengths: np.ndarray
    requests: np.ndarray

    @staticmethod
    def from_workloads(workloads: Sequence[WorkloadSpec], slots: Optional[Sequence[int]] = None,
                       mode: LengthMode = LengthMode.Mean,
                       scripted: Optional[Sequence[Optional[Sequence[Request]]]] = None) -> "WorkloadBatch":
        lt = _LengthTable()
        n = len(workloads)
        scen = np.zeros(n, dtype=A.SCENARIO_DT)
        n_ad = sum(len(w.adapters) for w in workloads)
        ads = np.zeros(max(n_ad, 1), dtype=A.ADAPTER_DT)
        reqs: List[tuple] = []
        k = 0
        for i, w in enumerate(workloads):
            s = scen[i]
            s["adapter_offset"] = k
            s["n_adapters"] = len(w.adapters)
            s["length_index"] = lt.add(w.lengths)
            s["duration_s"] = w.duration_s
            s["seed"] = w.seed
            s["slots"] = slots[i] if slots is not None else 0
            s["mode"] = int(mode)
            for a in w.adapters:
                ads[k] = (a.adapter_id, a.rank, a.rate, lt.add(a.lengths) if a.lengths is not None else -1, 0)
                k += 1
            rl = scripted[i] if scripted is not None else None
            if rl is None:
                s["request_offset"] = 0
                s["n_requests"] = -1
            else:
                s["request_offset"] = len(reqs)
                s["n_requests"] = len(rl)
                for r in rl:
                    reqs.append((r.request_id, r.adapter_id, r.input_tokens, r.output_tokens, 0,
                                 r.arrival_time_s))
        lens, full = lt.arrays()
        req = np.zeros(max(len(reqs), 1), dtype=A.REQUEST_DT)
        for j, r in enumerate(reqs):
            req[j] = r
        return WorkloadBatch(scen, ads[:max(n_ad, 1)], lens, full, req[:len(reqs)] if reqs else req[:0])

    def c_struct(self) -> A.lt_workload_batch:
        b = A.lt_workload_batch()
        b.scenarios = A.ptr(self.scenarios)
        b.n_scenarios = len(self.scenarios)
        b.adapters = A.ptr(self.adapters)
        b.n_adapters = len(self.adapters)
        b.lengths = A.ptr(self.lengths)
        b.n_lengths = len(self.lengths)
        b.full_lengths = A.ptr(self.full_lengths)
        b.n_full_pairs = len(self.full_lengths) // 2
        b.requests = A.ptr(self.requests)
        b.n_requests = len(self.requests)
        return b


@dataclass
class ConditionBatch:
    conditions: np.ndarray
    templates: np.ndarray
    lengths: np.ndarray
    full_lengths: np.ndarray

    @staticmethod
    def from_conditions(conds: Sequence[Condition]) -> "ConditionBatch":
        lt = _LengthTable()
        cd = np.zeros(len(conds), dtype=A.CONDITION_DT)
        n_t = sum(len(c.mix) for c in conds)
        tp = np.zeros(max(n_t, 1), dtype=A.TEMPLATE_DT)
        k = 0
        for i, c in enumerate(conds):
            cd[i] = (k, len(c.mix), lt.add(c.lengths))
            for leg in c.mix:
                tp[k] = (leg.rank, 0, leg.rate)
                k += 1
        lens, full = lt.arrays()
        return ConditionBatch(cd, tp, lens, full)

    def c_struct(self) -> A.lt_condition_batch:
        b = A.lt_condition_batch()
        b.conditions = A.ptr(self.conditions)
        b.n_conditions = len(self.conditions)
        b.templates = A.ptr(self.templates)
        b.n_templates = len(self.templates)
        b.lengths = A.ptr(self.lengths)
        b.n_lengths = len(self.lengths)
        b.full_lengths = A.ptr(self.full_lengths)
        b.n_full_pairs = len(self.full_lengths) // 2
        return b


def sim_options(opts: Optional[SimOptions] = None, want_digest: bool = False,
                libm_variant: int = -1, want_percentiles: bool = False,
                report: bool = False) -> A.lt_sim_options:
    o = A.lt_sim_options()
    opts = opts or SimOptions()
    if opts.record_iteration_trace and not report:
        raise UnsupportedError("SimOptions.record_iteration_trace: trace rows come from the report call "
                               "(Device.simulate_report / run_simulation), not from simulate_batch")
    o.check_invariants = int(opts.check_invariants)
    o.want_digest = int(want_digest)
    # engine.cpp:75 uses value_or(cap): an override <= 1 truncates after the
    # first iteration, like 1 (the ABI reads <= 0 as "no override").
    ov = opts.iteration_cap_override
    o.iteration_cap_override = 0 if ov is None else max(int(ov), 1)
    o.libm_variant = libm_variant
    o.want_percentiles = int(want_percentiles)
    return o


def frontier_capacity(grid: SweepGrid) -> int:
    """Frontier rows per condition (lt_sweep_frontier_capacity): at most
    max(4, |explicit G|) points per N row."""
    return max(sum(max(4, len(grid.g_values)) for _ in grid.n_values), 1)


class PackedGrid:
    def __init__(self, grid: SweepGrid):
        self.n = np.array(grid.n_values, dtype=np.int32)
        self.g = np.array(grid.g_values if grid.g_values else [0], dtype=np.int32)
        c = A.lt_sweep_grid()
        c.n_values = self.n.ctypes.data_as(C.POINTER(C.c_int32)) if len(self.n) else None
        c.n_count = len(grid.n_values)
        c.g_mode = int(grid.g_mode)
        c.g_values = self.g.ctypes.data_as(C.POINTER(C.c_int32))
        c.g_count = len(grid.g_values)
        self.c = c


REQUEST_STATE_FIELDS = [("phase", np.int8), ("tokens_generated", np.int32), ("first_token_time_s", np.float64),
                        ("completion_time_s", np.float64), ("preemption_count", np.int32),
                        ("adapter_id", np.int32), ("input_tokens", np.int32), ("output_tokens", np.int32),
                        ("arrival_time_s", np.float64)]


class Runner:
    """Calls one backend library's batch entry points.

    `ctx` is the library context (None for the oracle libraries, which take
    and ignore it); `message` returns the reference what() text of item i.
    """

    def __init__(self, lib: A.Lib, ctx, message: Callable[[int], str]):
        self.lib = lib
        self.ctx = ctx
        self.message = message

    def _raise(self, code: int, index: int, msg: str):
        cls = ERROR_CLASSES.get(code, LoratwinError)
        err = cls(msg)
        err.index = index
        raise err

    def simulate(self, batch: WorkloadBatch, config: ServerConfig, options: A.lt_sim_options,
                 want_states: bool = False):
        pc = PackedConfig(config)
        n = len(batch.scenarios)
        out = np.zeros(max(n, 1), dtype=A.SUMMARY_DT)
        st = A.lt_status()
        states = None
        states_c = None
        cb = batch.c_struct()
        if want_states:
            # scripted sizes are known; generated sizes come from a first pass
            cap = self._count_requests(batch, options)
            states = {"req_offset": np.zeros(max(n, 1), dtype=np.int64)}
            for name, dt in REQUEST_STATE_FIELDS:
                states[name] = np.zeros(max(cap, 1), dtype=dt)
            states_c = A.lt_request_states()
            states_c.capacity = cap
            states_c.req_offset = A.ptr(states["req_offset"])
            for name, _ in REQUEST_STATE_FIELDS:
                setattr(states_c, name, A.ptr(states[name]))
        self.lib.simulate_batch(self.ctx, C.byref(cb), C.byref(pc.c), C.byref(options),
                                out.ctypes.data, C.byref(states_c) if states_c is not None else None,
                                C.byref(st))
        if st.code == A.LT_ERR_DEVICE:
            self._raise(st.code, st.index, st.message.decode())
        return out[:n], states

    def report(self, batch: WorkloadBatch, config: ServerConfig, options: A.lt_sim_options):
        """lt_simulate_report: summaries, request states and the full report
        (trace rows, load events, per-request emit times). A first
        lt_simulate_batch call sizes the buffers."""
        out, states = self.simulate(batch, config, options, want_states=True)
        n = len(batch.scenarios)
        ok = out["status"] == A.LT_OK
        n_ld = int(out["load_events"].sum()) if n else 0
        n_em = int(out["tokens_total"][ok].sum()) if n else 0
        cap = len(states["phase"])
        rep = {"trace": np.zeros(max(int(out["iterations"].sum()) if n else 0, 1), dtype=A.TRACE_DT),
               "trace_offset": np.zeros(max(n, 1), dtype=np.int64),
               "loads": np.zeros(max(n_ld, 1), dtype=A.LOAD_EVENT_DT),
               "load_offset": np.zeros(max(n, 1), dtype=np.int64),
               "emit_times": np.zeros(max(n_em, 1), dtype=np.float64),
               "emit_offset": np.zeros(max(cap, 1), dtype=np.int64)}
        rc = A.lt_report()
        rc.trace, rc.trace_capacity, rc.trace_offset = rep["trace"].ctypes.data, len(rep["trace"]), \
            rep["trace_offset"].ctypes.data
        rc.loads, rc.load_capacity, rc.load_offset = rep["loads"].ctypes.data, len(rep["loads"]), \
            rep["load_offset"].ctypes.data
        rc.emit_times, rc.emit_capacity, rc.emit_offset = rep["emit_times"].ctypes.data, len(rep["emit_times"]), \
            rep["emit_offset"].ctypes.data
        states_c = A.lt_request_states()
        states_c.capacity = cap
        states_c.req_offset = A.ptr(states["req_offset"])
        for name, _ in REQUEST_STATE_FIELDS:
            setattr(states_c, name, A.ptr(states[name]))
        pc = PackedConfig(config)
        cb = batch.c_struct()
        st = A.lt_status()
        self.lib.simulate_report(self.ctx, C.byref(cb), C.byref(pc.c), C.byref(options), out.ctypes.data,
                                 C.byref(states_c), C.byref(rc), C.byref(st))
        if st.code == A.LT_ERR_DEVICE:
            self._raise(st.code, st.index, st.message.decode())
        return out[:n], states, rep

    def _count_requests(self, batch: WorkloadBatch, options) -> int:
        sc = batch.scenarios
        if len(sc) and np.all(sc["n_requests"] >= 0):
            return int(sc["n_requests"].sum())
        _, counts = self.generate_arrivals(batch, options, capacity=0)
        return int(counts.sum())

    def generate_arrivals(self, batch: WorkloadBatch, options: A.lt_sim_options, capacity: Optional[int] = None):
        n = len(batch.scenarios)
        offsets = np.zeros(max(n, 1), dtype=np.int64)
        counts = np.zeros(max(n, 1), dtype=np.int64)
        st = A.lt_status()
        cb = batch.c_struct()
        if capacity is None:
            self.lib.generate_arrivals_batch(self.ctx, C.byref(cb), C.byref(options), None, 0,
                                             offsets.ctypes.data, counts.ctypes.data, C.byref(st))
            capacity = int(counts[:n].sum())
        reqs = np.zeros(max(capacity, 1), dtype=A.REQUEST_DT)
        st = A.lt_status()
        self.lib.generate_arrivals_batch(self.ctx, C.byref(cb), C.byref(options), reqs.ctypes.data,
                                         capacity, offsets.ctypes.data, counts.ctypes.data, C.byref(st))
        if st.code == A.LT_ERR_DEVICE:
            self._raise(st.code, st.index, st.message.decode())
        self.last_arrivals_status = (st.code, st.index, st.message.decode())
        return reqs[:capacity] if capacity else reqs[:0], counts[:n]

    def sweep(self, conds: ConditionBatch, config: ServerConfig, grid: SweepGrid, duration_s: float,
              seed: int, options: SweepOptions, sim: A.lt_sim_options):
        pc = PackedConfig(config)
        pg = PackedGrid(grid)
        n = len(conds.conditions)
        maxf = frontier_capacity(grid)
        out = np.zeros(max(n, 1), dtype=A.PLACEMENT_DT)
        fr = np.zeros(max(n * maxf, 1), dtype=A.FRONTIER_DT)
        so = A.lt_sweep_options()
        so.early_exit = int(options.early_exit)
        so.early_exit_k = options.early_exit_k
        so.jobs = options.jobs
        so.mode = int(options.mode)
        st = A.lt_status()
        cb = conds.c_struct()
        self.lib.sweep_batch(self.ctx, C.byref(cb), C.byref(pc.c), C.byref(pg.c), float(duration_s),
                             int(seed), C.byref(so), C.byref(sim), out.ctypes.data, fr.ctypes.data, maxf,
                             C.byref(st))
        if st.code == A.LT_ERR_DEVICE:
            self._raise(st.code, st.index, st.message.decode())
        return out[:n], fr[:n * maxf].reshape(n, maxf)
