"""Throughput on the other BASELINE configs on one B200,
with a CPU-reference parity spot check on a sample of each.

    python tools/bench_configs.py [c3] [c4] [c5] [--c5-count N] [--c4-conditions N] [--no-ref]

C3: 65,536 scenarios (heterogeneous ranks, mixed rates, shared seed 7).
C5: a contiguous chunk of the 524,288-scenario sweep per profile
    (llama31_8b, qwen25_7b; long I/O; per-scenario seeds).
C4: full placement searches (explicit G {2..64}, N {1..256 x2}, early exit k=3).
Each line: device-resident plan timing (CUDA events) and the e2e call.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402

import paper_2508_08343_b200 as lt  # noqa: E402
from paper_2508_08343_b200.batch import ConditionBatch, WorkloadBatch, sim_options  # noqa: E402
from paper_2508_08343_b200.types import profile_config  # noqa: E402
from tests import workloads as W  # noqa: E402

FIELDS = ["status", "iterations", "finished_count", "rejected_count", "preemptions", "load_events",
          "tokens_in_window", "starved", "final_clock_s", "throughput_tok_s", "ttft_mean_s"]


def ref_oracle():
    from oracle.pyoracle import RefOracle, available
    return RefOracle(threads=os.cpu_count() or 1) if available("ref") else None


def sub(b, idx):
    return WorkloadBatch(b.scenarios[idx].copy(), b.adapters, b.lengths, b.full_lengths, b.requests)


def run_sim(name, b, cfg, stride, ref):
    """lt_simulate_batch end to end (chunked by the library when large); the
    device time is the sum of the chunks' pipeline times (CUDA events)."""
    dev = lt.device()
    dev.simulate_batch(b, cfg)  # warm (allocator, module)
    t0 = time.perf_counter()
    out, _ = dev.simulate_batch(b, cfg)
    e2e_s = time.perf_counter() - t0
    t = dev.timing()
    iters = int(out["iterations"].sum())
    line = {"config": name, "scenarios": len(b.scenarios), "engine_iterations": iters,
            "requests": int(out["n_requests"].sum()), "device_ms": t["run_ms"],
            "device_iter_per_s": iters / (t["run_ms"] / 1e3), "engine_ms": t["engine_ms"],
            "e2e_s": e2e_s, "e2e_iter_per_s": iters / e2e_s, "failed": int((out["status"] != 0).sum()),
            "starved": int(out["starved"].sum())}
    if ref is not None and stride:
        idx = np.arange(0, len(b.scenarios), stride)
        t0 = time.perf_counter()
        r, _ = ref.simulate(sub(b, idx), cfg, sim_options())
        cpu_s = time.perf_counter() - t0
        g = out[idx]
        line["cpu_sample"] = {"scenarios": len(idx), "iter_per_s": float(r["iterations"].sum()) / cpu_s,
                              "threads": os.cpu_count(), "seconds": cpu_s,
                              "mismatches": int(sum(int(np.sum(g[f] != r[f])) for f in FIELDS))}
    print(json.dumps(line), flush=True)


def run_c4(n_cond, ref):
    dev = lt.device()
    conds = []
    for L in (lt.LengthSpec.mean(23, 5, 27, 5), lt.LengthSpec.mean(250, 50, 231, 50), lt.LengthSpec.mean(423, 80, 358, 80)):
        conds += lt.enumerate_conditions(W.PAPER_RATES, [8, 16, 32], L)
    conds = conds[:n_cond]
    grid = lt.SweepGrid(n_values=[1, 2, 4, 8, 16, 32, 64, 128, 256], g_mode=lt.GMode.Explicit,
                        g_values=[2, 4, 8, 16, 32, 64])
    cfg = lt.h100_like_config(1)
    opts = lt.SweepOptions(early_exit=True, early_exit_k=3)
    cb = ConditionBatch.from_conditions(conds)
    t0 = time.perf_counter()
    pl, fr = dev.sweep_batch(cb, cfg, grid, 600.0, 5, opts)
    wall = time.perf_counter() - t0
    line = {"config": "C4 placement search", "conditions": len(conds), "wall_s": wall,
            "conditions_per_s": len(conds) / wall, "points_simulated": int(pl["points_simulated"].sum()),
            "engine_iterations": int(pl["iterations"].sum())}
    if ref is not None:
        k = max(1, len(conds) // 16)
        idx = np.arange(0, len(conds), k)
        cbs = ConditionBatch.from_conditions([conds[i] for i in idx])
        t0 = time.perf_counter()
        rp, _ = ref.sweep(cbs, cfg, grid, 600.0, 5, opts, sim_options())
        cpu_s = time.perf_counter() - t0
        gp = pl[idx]
        mism = sum(int(np.sum(gp[f] != rp[f])) for f in ("status", "n_star", "g_star", "all_starved",
                                                          "frontier_open", "max_throughput_tok_s"))
        line["cpu_sample"] = {"conditions": len(idx), "conditions_per_s": len(idx) / cpu_s, "seconds": cpu_s,
                              "threads": os.cpu_count(), "mismatches": mism}
    print(json.dumps(line), flush=True)


def main():
    args = sys.argv[1:]
    which = [a for a in args if not a.startswith("--") and not a.isdigit()] or ["c3", "c4", "c5"]
    c5_count = int(args[args.index("--c5-count") + 1]) if "--c5-count" in args else 32768
    c4_n = int(args[args.index("--c4-conditions") + 1]) if "--c4-conditions" in args else 512
    ref = None if "--no-ref" in args else ref_oracle()
    if "c3" in which:
        run_sim("C3 65,536 scenarios (shared seed 7, G=min(N,16))", W.c3_batch(), lt.h100_like_config(1), 61, ref)
    if "c5" in which:
        for prof in ("llama31_8b", "qwen25_7b"):
            run_sim(f"C5 {prof} scenarios [0, {c5_count}) of 524,288", W.c5_batch(0, c5_count),
                    profile_config(prof, 1), 257, ref)
    if "c4" in which:
        run_c4(c4_n, ref)


if __name__ == "__main__":
    main()
