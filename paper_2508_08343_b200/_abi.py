"""ctypes mirror of include/loratwin_gpu.h (the C-ABI every backend exports).

The GPU library exports the `lt_*` symbols. The oracle libraries under
oracle/_ref export the same signatures with other prefixes (`ltref_`,
`ltor_`); only tests and bench.py's baseline legs load those.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

ABI_VERSION = 4

# enum lt_code
LT_OK, LT_ERR_VALIDATION, LT_ERR_CONFIG, LT_ERR_SIMULATION, LT_ERR_INTERNAL, LT_ERR_UNSUPPORTED, LT_ERR_DEVICE = range(7)
MODE_FULL, MODE_MEAN = 0, 1
SOURCE_CPU, SOURCE_DISK = 0, 1
G_GEOMETRIC, G_EXPLICIT = 0, 1
GATHER_NONE, GATHER_NCCL, GATHER_PEER = 0, 1, 2


class lt_status(C.Structure):
    _fields_ = [("code", C.c_int32), ("kind", C.c_int32), ("index", C.c_int64),
                ("detail_a", C.c_int64), ("detail_b", C.c_int64), ("message", C.c_char * 320)]


class lt_server_config(C.Structure):
    _fields_ = [("slots", C.c_int32), ("loaded_adapter_priority", C.c_int32),
                ("iteration_cap", C.c_int64), ("ideal_includes_input", C.c_int32),
                ("load_source", C.c_int32),
                ("k1", C.c_double), ("k2", C.c_double), ("k3", C.c_double), ("k4", C.c_double),
                ("k5", C.c_double), ("k6", C.c_double), ("k7", C.c_double),
                ("total_kv_budget", C.c_int64), ("kv_bytes_per_token", C.c_double),
                ("has_slot_cost_base_rank8", C.c_int32), ("slot_cost_base_rank8", C.c_double),
                ("n_slot_cost", C.c_int32), ("slot_cost_rank", C.POINTER(C.c_int32)),
                ("slot_cost_tokens", C.POINTER(C.c_int64)),
                ("n_load", C.c_int32), ("load_rank", C.POINTER(C.c_int32)),
                ("load_seconds", C.POINTER(C.c_double)), ("disk_multiplier", C.c_double)]


class lt_length_spec(C.Structure):
    _fields_ = [("mode", C.c_int32), ("_pad", C.c_int32), ("mean_input", C.c_double),
                ("std_input", C.c_double), ("mean_output", C.c_double), ("std_output", C.c_double),
                ("full_offset", C.c_int64), ("full_count", C.c_int64)]


class lt_adapter(C.Structure):
    _fields_ = [("adapter_id", C.c_int32), ("rank", C.c_int32), ("rate", C.c_double),
                ("length_index", C.c_int32), ("_pad", C.c_int32)]


class lt_request(C.Structure):
    _fields_ = [("request_id", C.c_int64), ("adapter_id", C.c_int32), ("input_tokens", C.c_int32),
                ("output_tokens", C.c_int32), ("_pad", C.c_int32), ("arrival_time_s", C.c_double)]


class lt_scenario(C.Structure):
    _fields_ = [("adapter_offset", C.c_int64), ("n_adapters", C.c_int32), ("length_index", C.c_int32),
                ("duration_s", C.c_double), ("seed", C.c_uint64), ("slots", C.c_int32),
                ("mode", C.c_int32), ("request_offset", C.c_int64), ("n_requests", C.c_int64)]


class lt_workload_batch(C.Structure):
    _fields_ = [("scenarios", C.c_void_p), ("n_scenarios", C.c_int64),
                ("adapters", C.c_void_p), ("n_adapters", C.c_int64),
                ("lengths", C.c_void_p), ("n_lengths", C.c_int64),
                ("full_lengths", C.c_void_p), ("n_full_pairs", C.c_int64),
                ("requests", C.c_void_p), ("n_requests", C.c_int64)]


class lt_sim_options(C.Structure):
    _fields_ = [("check_invariants", C.c_int32), ("want_digest", C.c_int32),
                ("iteration_cap_override", C.c_int64), ("libm_variant", C.c_int32),
                ("want_percentiles", C.c_int32)]


class lt_sim_summary(C.Structure):
    _fields_ = [("status", C.c_int32), ("status_kind", C.c_int32), ("status_a", C.c_int64),
                ("status_b", C.c_int64), ("n_requests", C.c_int64), ("iterations", C.c_int64),
                ("final_clock_s", C.c_double), ("duration_s", C.c_double), ("truncated", C.c_int32),
                ("slots", C.c_int32), ("served_adapters", C.c_int32), ("starved", C.c_int32),
                ("kv_capacity_tokens", C.c_int64), ("finished_count", C.c_int64),
                ("rejected_count", C.c_int64), ("preemptions", C.c_int64), ("load_events", C.c_int64),
                ("tokens_in_window", C.c_int64), ("tokens_total", C.c_int64),
                ("throughput_tok_s", C.c_double), ("ideal_throughput_tok_s", C.c_double),
                ("ttft_mean_s", C.c_double), ("itl_mean_s", C.c_double), ("ttft_p50_s", C.c_double),
                ("ttft_p99_s", C.c_double), ("itl_p50_s", C.c_double), ("itl_p99_s", C.c_double),
                ("degenerate", C.c_int32),
                ("_pad", C.c_int32), ("digest", C.c_uint64), ("sum_running", C.c_int64),
                ("sum_visited", C.c_int64), ("sum_arrivals", C.c_int64), ("sum_moves", C.c_int64),
                ("device_cycles", C.c_int64), ("phase_cycles", C.c_int64 * 6)]


class lt_request_states(C.Structure):
    _fields_ = [("capacity", C.c_int64), ("req_offset", C.c_void_p), ("phase", C.c_void_p),
                ("tokens_generated", C.c_void_p), ("first_token_time_s", C.c_void_p),
                ("completion_time_s", C.c_void_p), ("preemption_count", C.c_void_p),
                ("adapter_id", C.c_void_p), ("input_tokens", C.c_void_p), ("output_tokens", C.c_void_p),
                ("arrival_time_s", C.c_void_p)]


class lt_template(C.Structure):
    _fields_ = [("rank", C.c_int32), ("_pad", C.c_int32), ("rate", C.c_double)]


class lt_condition(C.Structure):
    _fields_ = [("mix_offset", C.c_int64), ("mix_count", C.c_int32), ("length_index", C.c_int32)]


class lt_condition_batch(C.Structure):
    _fields_ = [("conditions", C.c_void_p), ("n_conditions", C.c_int64),
                ("templates", C.c_void_p), ("n_templates", C.c_int64),
                ("lengths", C.c_void_p), ("n_lengths", C.c_int64),
                ("full_lengths", C.c_void_p), ("n_full_pairs", C.c_int64)]


class lt_sweep_grid(C.Structure):
    _fields_ = [("n_values", C.POINTER(C.c_int32)), ("n_count", C.c_int32), ("g_mode", C.c_int32),
                ("g_values", C.POINTER(C.c_int32)), ("g_count", C.c_int32), ("_pad", C.c_int32)]


class lt_sweep_options(C.Structure):
    _fields_ = [("early_exit", C.c_int32), ("early_exit_k", C.c_int32), ("jobs", C.c_int32),
                ("mode", C.c_int32)]


class lt_dataset_spec(C.Structure):
    _fields_ = [("rates", C.POINTER(C.c_double)), ("n_rates", C.c_int32), ("triple_size", C.c_int32),
                ("ranks", C.POINTER(C.c_int32)), ("n_ranks", C.c_int32), ("condition_stride", C.c_int32),
                ("lengths", lt_length_spec), ("full_lengths", C.POINTER(C.c_int32)), ("n_full_pairs", C.c_int64),
                ("duration_s", C.c_double), ("seed", C.c_uint64), ("grid", lt_sweep_grid),
                ("sweep", lt_sweep_options)]


class lt_dataset_progress(C.Structure):
    _fields_ = [("total_conditions", C.c_int64), ("completed", C.c_int64), ("failed", C.c_int64)]


ERROR_FN = C.CFUNCTYPE(None, C.c_char_p, C.c_void_p)


class lt_frontier_point(C.Structure):
    _fields_ = [("n", C.c_int32), ("g", C.c_int32), ("throughput_tok_s", C.c_double),
                ("starved", C.c_int32), ("skipped", C.c_int32)]


class lt_placement(C.Structure):
    _fields_ = [("status", C.c_int32), ("status_kind", C.c_int32), ("status_a", C.c_int64),
                ("status_b", C.c_int64), ("max_throughput_tok_s", C.c_double), ("n_star", C.c_int32),
                ("g_star", C.c_int32), ("all_starved", C.c_int32), ("frontier_open", C.c_int32),
                ("frontier_count", C.c_int32), ("_pad", C.c_int32), ("points_simulated", C.c_int64),
                ("iterations", C.c_int64), ("status_point", C.c_int64)]


class lt_timing(C.Structure):
    _fields_ = [("h2d_ms", C.c_double), ("tables_ms", C.c_double), ("merge_ms", C.c_double),
                ("engine_ms", C.c_double), ("reduce_ms", C.c_double), ("d2h_ms", C.c_double),
                ("total_ms", C.c_double), ("run_ms", C.c_double), ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64),
                ("engine_launches", C.c_int64), ("algorithmic_bytes", C.c_int64), ("plan_ms", C.c_double),
                ("run_wait_ms", C.c_double), ("gather_ms", C.c_double), ("gather_bytes", C.c_int64),
                ("devices", C.c_int32), ("_pad", C.c_int32)]


class lt_trace_row(C.Structure):
    _fields_ = [("time_s", C.c_double), ("iteration", C.c_int64), ("r_running", C.c_int32),
                ("r_waiting", C.c_int32), ("a_running", C.c_int32), ("loads", C.c_int32), ("lat_step_s", C.c_double)]


class lt_load_event(C.Structure):
    _fields_ = [("time_s", C.c_double), ("adapter_id", C.c_int32), ("rank", C.c_int32), ("source", C.c_int32),
                ("_pad", C.c_int32), ("latency_s", C.c_double)]


class lt_report(C.Structure):
    _fields_ = [("trace", C.c_void_p), ("trace_capacity", C.c_int64), ("trace_offset", C.c_void_p),
                ("loads", C.c_void_p), ("load_capacity", C.c_int64), ("load_offset", C.c_void_p),
                ("emit_times", C.c_void_p), ("emit_capacity", C.c_int64), ("emit_offset", C.c_void_p)]


class lt_tree_params(C.Structure):
    _fields_ = [("max_depth", C.c_int32), ("min_leaf", C.c_int32), ("feature_subset", C.c_int32),
                ("_pad", C.c_int32)]


class lt_forest_params(C.Structure):
    _fields_ = [("n_trees", C.c_int32), ("bootstrap", C.c_int32), ("tree", lt_tree_params)]


class lt_tree_node(C.Structure):
    _fields_ = [("feature_index", C.c_int32), ("left", C.c_int32), ("right", C.c_int32), ("_pad", C.c_int32),
                ("threshold", C.c_double), ("value", C.c_double), ("coverage", C.c_int64)]


# numpy views with the exact C layouts (numpy honours ctypes field offsets)
SCENARIO_DT = np.dtype(lt_scenario)
ADAPTER_DT = np.dtype(lt_adapter)
LENGTH_DT = np.dtype(lt_length_spec)
REQUEST_DT = np.dtype(lt_request)
SUMMARY_DT = np.dtype(lt_sim_summary)
TEMPLATE_DT = np.dtype(lt_template)
CONDITION_DT = np.dtype(lt_condition)
FRONTIER_DT = np.dtype(lt_frontier_point)
PLACEMENT_DT = np.dtype(lt_placement)
TRACE_DT = np.dtype(lt_trace_row)
LOAD_EVENT_DT = np.dtype(lt_load_event)
TREE_NODE_DT = np.dtype(lt_tree_node)

assert SCENARIO_DT.itemsize == 56 and ADAPTER_DT.itemsize == 24 and REQUEST_DT.itemsize == 32
assert LENGTH_DT.itemsize == 56


def ptr(a: np.ndarray | None) -> int | None:
    if a is None or a.size == 0:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


# Every symbol the header declares, with (restype, argtypes).
SIGNATURES = {
    "abi_version": (C.c_int32, []),
    "host_libm_variant": (C.c_int32, []),
    "format_status": (None, [C.c_int32, C.c_int32, C.c_int64, C.c_int64, C.c_char_p, C.c_size_t]),
    "create": (C.c_void_p, [C.c_int32, C.POINTER(lt_status)]),
    "create_devices": (C.c_void_p, [C.POINTER(C.c_int32), C.c_int32, C.POINTER(lt_status)]),
    "create_mask": (C.c_void_p, [C.c_uint64, C.POINTER(lt_status)]),
    "device_count": (C.c_int32, [C.c_void_p]),
    "gather_transport": (C.c_int32, [C.c_void_p]),
    "destroy": (None, [C.c_void_p]),
    "stream": (C.c_void_p, [C.c_void_p]),
    "last_timing": (C.c_int32, [C.c_void_p, C.POINTER(lt_timing)]),
    "last_message": (C.c_int32, [C.c_void_p, C.c_int64, C.c_char_p, C.c_size_t]),
    "generate_arrivals_batch": (C.c_int32, [C.c_void_p, C.POINTER(lt_workload_batch),
                                            C.POINTER(lt_sim_options), C.c_void_p, C.c_int64,
                                            C.c_void_p, C.c_void_p, C.POINTER(lt_status)]),
    "simulate_batch": (C.c_int32, [C.c_void_p, C.POINTER(lt_workload_batch),
                                   C.POINTER(lt_server_config), C.POINTER(lt_sim_options),
                                   C.c_void_p, C.POINTER(lt_request_states), C.POINTER(lt_status)]),
    "simulate_report": (C.c_int32, [C.c_void_p, C.POINTER(lt_workload_batch), C.POINTER(lt_server_config),
                                    C.POINTER(lt_sim_options), C.c_void_p, C.POINTER(lt_request_states),
                                    C.POINTER(lt_report), C.POINTER(lt_status)]),
    "train_tree": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.POINTER(lt_tree_params), C.c_uint64,
                               C.c_uint64, C.c_void_p, C.c_int64, C.c_void_p, C.POINTER(lt_status)]),
    "train_forests": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int32,
                                  C.POINTER(lt_forest_params), C.c_uint64, C.c_void_p, C.c_int64, C.c_void_p,
                                  C.c_void_p, C.POINTER(lt_status)]),
    "predict_forests": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32,
                                    C.c_void_p, C.c_int64, C.c_void_p, C.POINTER(lt_status)]),
    "sweep_frontier_capacity": (C.c_int32, [C.POINTER(lt_sweep_grid)]),
    "sweep_batch": (C.c_int32, [C.c_void_p, C.POINTER(lt_condition_batch), C.POINTER(lt_server_config),
                                C.POINTER(lt_sweep_grid), C.c_double, C.c_uint64,
                                C.POINTER(lt_sweep_options), C.POINTER(lt_sim_options), C.c_void_p,
                                C.c_void_p, C.c_int32, C.POINTER(lt_status)]),
    "generate_dataset": (C.c_int32, [C.c_void_p, C.POINTER(lt_dataset_spec), C.POINTER(lt_server_config),
                                     C.c_char_p, ERROR_FN, C.c_void_p, C.POINTER(lt_dataset_progress),
                                     C.POINTER(lt_status)]),
    "condition_hash": (C.c_uint64, [C.POINTER(lt_template), C.c_int32, C.POINTER(lt_length_spec),
                                    C.POINTER(C.c_int32), C.c_double, C.c_uint64, C.POINTER(lt_sweep_grid)]),
    "encode_workload": (C.c_int32, [C.POINTER(lt_template), C.c_int32, C.POINTER(lt_length_spec),
                                    C.POINTER(C.c_int32), C.POINTER(C.c_double), C.POINTER(lt_status)]),
    "plan_simulate": (C.c_void_p, [C.c_void_p, C.POINTER(lt_workload_batch), C.POINTER(lt_server_config),
                                   C.POINTER(lt_sim_options), C.POINTER(lt_status)]),
    "plan_run": (C.c_int32, [C.c_void_p, C.POINTER(lt_status)]),
    "plan_results": (C.c_int32, [C.c_void_p, C.c_void_p, C.POINTER(lt_request_states), C.POINTER(lt_status)]),
    "plan_destroy": (None, [C.c_void_p]),
    "plan_summaries_device": (C.c_int32, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]),
    "plan_trim": (C.c_int32, [C.c_void_p]),
}

# Symbols the oracle libraries must export (same meaning, other prefix).
ORACLE_SYMBOLS = ["generate_arrivals_batch", "simulate_batch", "sweep_batch"]
# ... and the dataset entry points (the compiled reference only)
DATASET_SYMBOLS = ["generate_dataset", "condition_hash", "encode_workload"]
# ... and the predictor entry points (the compiled reference only)
PREDICTOR_SYMBOLS = ["train_tree", "train_forests", "predict_forests"]


class Lib:
    """A loaded backend library with its symbol prefix."""

    def __init__(self, path: str, prefix: str, symbols=None):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.path = path
        self.prefix = prefix
        self.dll = C.CDLL(path, mode=os.RTLD_LOCAL | os.RTLD_NOW)
        names = symbols if symbols is not None else list(SIGNATURES)
        for name in names:
            fn = getattr(self.dll, prefix + name)
            if name in SIGNATURES:
                res, args = SIGNATURES[name]
                if prefix != "lt_" and args and args[0] is C.c_void_p:
                    pass  # oracle entry points take a (ignored) context pointer too
                fn.restype = res
                fn.argtypes = args
            setattr(self, name, fn)
