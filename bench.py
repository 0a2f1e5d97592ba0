#!/usr/bin/env python
"""Benchmark of the batched Digital-Twin sweep (BASELINE.json metric:
simulated engine-iterations/sec, + placement sweeps/sec) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl gpu|reference]

Workload (BASELINE configs[1], SURVEY 8d "C2"): 1,024 scenarios = N in
{8..256 step 8} x rank mode {8,16,32,mixed} x r in {3.2..0.0125}; per-adapter
rate 8r/N; Mean(250,80,231,80) lengths; 600 s simulated; G = min(N,32); seed
1234+i; h100_like server. Synthetic (the reference's own generator, on device).

A step = the whole device pipeline over the batch with inputs resident in HBM:
K0 RNG tables -> arrival counts -> device scan -> merge -> engine (K1) +
metrics epilogue (K2). `e2e` = the same metric through the public C-ABI call
lt_simulate_batch with pinned host buffers (H2D + everything + D2H).
For N>1 (torchrun, one rank per GPU, NCCL) each rank runs its own replica of
the grid (seeds shifted by 1024*rank: weak scaling) and the per-scenario
summaries are all-gathered over NCCL inside the timed step (the path's one
exchange).
`--impl reference` times the reference's own CPU implementation
(oracle/_ref: the unmodified reference TUs) over a bounded sample of the same
grid on all host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "simulated engine-iterations/sec + placement sweeps/sec at 1/2/4/8 B200 vs host CPU"
UNIT = "engine-iterations/s"
WORKLOAD = ("C2: 1,024-scenario grid, N=8..256 step 8 x rank {8,16,32,mixed} x r {3.2..0.0125}, "
            "per-adapter rate 8r/N, Mean(250,80,231,80), 600 s simulated, G=min(N,32), seed 1234+i, h100_like")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled during the timed
    region: NVML every few milliseconds (nvidia-ml-py), else nvidia-smi."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.rows = []  # (sm_mhz, max_mhz, {reason names})
        self.proc = None
        self.nvml = None
        self.stop_flag = threading.Event()
        self.source = None

    def start(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            bits = [pynvml.nvmlClocksThrottleReasonHwSlowdown, pynvml.nvmlClocksThrottleReasonHwThermalSlowdown,
                    pynvml.nvmlClocksThrottleReasonSwThermalSlowdown, pynvml.nvmlClocksThrottleReasonSwPowerCap]
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def loop():
                while not self.stop_flag.is_set():
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                    self.rows.append((float(sm), float(mx), {n for n, b in zip(self.NAMES, bits) if r & b}))
                    time.sleep(0.005)

            self.nvml = pynvml
            self.source = "nvml, 5 ms"
            self.t = threading.Thread(target=loop, daemon=True)
            self.t.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.source = "nvidia-smi, 100 ms"
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7 and parts[0].replace(".", "").isdigit():
                reasons = {self.NAMES[i] for i in range(4) if "Active" in parts[3 + i] and "Not" not in parts[3 + i]}
                mx = float(parts[1]) if parts[1].replace(".", "").isdigit() else None
                self.rows.append((float(parts[0]), mx, reasons))

    def stop(self):
        self.stop_flag.set()
        if self.nvml is not None:
            self.t.join(timeout=2)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        rows = list(self.rows)
        sm = [r[0] for r in rows]
        mx = [r[1] for r in rows if r[1] is not None]
        reasons = sorted(set().union(*[r[2] for r in rows])) if rows else []
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm), "source": self.source}


def measured_peaks():
    for p in (os.path.join(ROOT, "MEASURED_PEAKS.json"),):
        if os.path.exists(p):
            with open(p) as f:
                d = json.load(f)
            return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def ncu_traffic():
    """dram bytes per engine launch from the latest committed ncu --set full
    summary (profiles/r<NN>_engine_ncu.json), if present."""
    import glob

    paths = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_engine_ncu.json")))
    if not paths:
        return None, None
    with open(paths[-1]) as f:
        d = json.load(f)
    m = d.get("metrics", {})
    brief = {"file": os.path.relpath(paths[-1], ROOT), "workload": d.get("workload"),
             "kernel_ms": m.get("gpu__time_duration.sum", [None])[0],
             "issue_active_pct_of_peak": m.get("smsp__issue_active.avg.pct_of_peak_sustained_active", [None])[0],
             "warp_latency_per_inst": m.get("smsp__average_warp_latency_per_inst_issued.ratio", [None])[0]}
    return d.get("dram_bytes_per_launch"), brief


def c2_batch_for_rank(rank: int, duration: float, stride: int = 1):
    from tests import workloads as W

    b = W.c2_batch(duration_s=duration, stride=stride)
    b.scenarios["seed"] = b.scenarios["seed"] + np.uint64(1024 * rank)
    return b


def pinned_copy(batch):
    """The batch's arrays copied into page-locked host memory (for e2e H2D)."""
    import torch

    from paper_2508_08343_b200.batch import WorkloadBatch

    def pin(a):
        t = torch.empty(max(a.nbytes, 1), dtype=torch.uint8, pin_memory=True)
        v = t.numpy()[:a.nbytes].view(a.dtype)
        v[...] = a
        pin.keep.append(t)
        return v
    pin.keep = []
    pb = WorkloadBatch(pin(batch.scenarios), pin(batch.adapters), pin(batch.lengths), pin(batch.full_lengths),
                       pin(batch.requests) if len(batch.requests) else batch.requests)
    return pb, pin.keep


def cpu_reference_run(sample_stride: int, duration: float, threads: int):
    """The reference's own CPU implementation over a bounded sample."""
    import paper_2508_08343_b200 as lt
    from oracle import pyoracle
    from paper_2508_08343_b200.batch import sim_options

    kind = "reference" if pyoracle.available("ref") else "port"
    orc = pyoracle.RefOracle(threads=threads) if kind == "reference" else pyoracle.PortOracle(threads=threads)
    b = c2_batch_for_rank(0, duration, stride=sample_stride)
    t0 = time.perf_counter()
    out, _ = orc.simulate(b, lt.h100_like_config(1), sim_options())
    wall = time.perf_counter() - t0
    iters = int(out["iterations"].sum())
    return {"value": iters / wall, "unit": UNIT, "cores": threads, "kind": kind,
            "wall_s": wall,
            "sample": (("the whole C2 grid" if sample_stride == 1 else f"every {sample_stride}-th C2 scenario")
                       + f" ({len(out)} of 1024 scenarios), run_simulation + compute_metrics (the reference's own "
                       f"TUs, {threads} host threads), {iters} engine-iterations in {wall:.2f} s")}, out, b


def impl_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    vals, walls = [], []
    for i in range(args.warmup + args.steps):
        cb, _, _ = cpu_reference_run(args.ref_stride, args.duration, threads)
        if i >= args.warmup:
            vals.append(cb["value"])
            walls.append(cb["wall_s"])
    v = statistics.mean(vals)
    cb["value"] = v
    line = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * statistics.mean(walls),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "sample_stride": args.ref_stride, "duration_s": args.duration,
                       "step": "one step = the bounded sample (every sample_stride-th C2 scenario)"},
            "cpu_baseline": cb, "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def sweep_secondary(dev, n_cond: int):
    """placement sweeps/sec on a C4-shaped sample (explicit G, early exit k=3, 600 s, seed 5)."""
    import paper_2508_08343_b200 as lt
    from paper_2508_08343_b200.batch import ConditionBatch
    from tests import workloads as W

    conds = lt.enumerate_conditions(W.PAPER_RATES, [8, 16, 32], lt.LengthSpec.mean(250, 50, 231, 50))
    conds = conds[::max(1, len(conds) // n_cond)][:n_cond]
    grid = lt.SweepGrid(n_values=[1, 2, 4, 8, 16, 32, 64, 128, 256], g_mode=lt.GMode.Explicit,
                        g_values=[2, 4, 8, 16, 32, 64])
    cb = ConditionBatch.from_conditions(conds)
    cfg = lt.h100_like_config(1)
    opts = lt.SweepOptions(early_exit=True, early_exit_k=3)
    dev.sweep_batch(cb, cfg, grid, 600.0, 5, opts)  # warm
    t0 = time.perf_counter()
    pl, _ = dev.sweep_batch(cb, cfg, grid, 600.0, 5, opts)
    wall = time.perf_counter() - t0
    return {"metric": "placement sweeps/sec", "value": len(conds) / wall, "unit": "conditions/s",
            "conditions": len(conds), "grid": "N {1..256 x2}, explicit G {2..64}, early exit k=3, 600 s, seed 5",
            "points_simulated": int(pl["points_simulated"].sum()), "wall_s": wall,
            "note": "end to end through lt_sweep_batch (host buffers)"}


def impl_gpu(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2508_08343_b200 as lt

    dev = lt.device(local)
    cfg = lt.h100_like_config(1)
    batch = c2_batch_for_rank(rank, args.duration)
    n_scen = len(batch.scenarios)

    # CPU baseline (rank 0, N=1 only), bounded sample; its results also spot-check parity.
    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu, ref_out, ref_b = cpu_reference_run(args.cpu_stride, args.duration, os.cpu_count() or 1)
        g, _ = dev.simulate_batch(ref_b, cfg)
        fields = ["status", "iterations", "finished_count", "rejected_count", "preemptions", "load_events",
                  "tokens_in_window", "starved", "final_clock_s", "throughput_tok_s", "ttft_mean_s"]
        mism = sum(int(np.sum(g[f] != ref_out[f])) for f in fields)
        parity = {"scenarios": int(len(g)), "fields": fields, "mismatches": mism, "oracle": cpu["kind"]}
        log("cpu baseline", cpu, "parity", parity)

    log(f"[{time.strftime('%X')}] building plan ({n_scen} scenarios)")
    plan = dev.plan(batch, cfg)
    stream = torch.cuda.ExternalStream(dev.stream(), device=torch.device("cuda", local))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")  # > 126 MB L2
    gathered = None
    if world > 1:
        ptr, nbytes = plan.device_summaries()

        class _View:
            __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}
        mine = torch.as_tensor(_View(), device=f"cuda:{local}")
        gathered = [torch.empty_like(mine) for _ in range(world)]

    def step():
        plan.run()
        if world > 1:
            with torch.cuda.stream(stream):
                dist.all_gather(gathered, mine)

    for i in range(args.warmup):
        step()
        torch.cuda.synchronize()
        log(f"[{time.strftime('%X')}] warmup {i} done: {dev.timing()['run_ms']:.1f} ms device pipeline")
    torch.cuda.synchronize()
    res = plan.results()
    iters_rank = int(res["iterations"].sum())
    bad = int(np.sum(res["status"] != 0))
    clocks = ClockSampler(local)
    clocks.start()
    times, eng, algo, launches = [], [], [], 0
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        step()
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
        res_t = plan.results()
        t = dev.timing()
        eng.append(t["engine_ms"])
        algo.append(t["algorithmic_bytes"])
        launches += int(t["engine_launches"])
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    total_ms = sum(times)
    iters_all = iters_rank
    if dist:
        tt = torch.tensor([total_ms], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
        it = torch.tensor([iters_rank], device=f"cuda:{local}", dtype=torch.int64)
        dist.all_reduce(it, op=dist.ReduceOp.SUM)
        iters_all = int(it.item())
    value = iters_all * args.steps / (total_ms / 1000.0)
    ms_per_step = total_ms / args.steps

    log(f"[{time.strftime('%X')}] timed steps: {times}")
    # e2e through the public C-ABI call with pinned host buffers
    e2e = None
    if not args.no_e2e:
        pb, keep = pinned_copy(batch)
        walls, plan_ms, wait_ms = [], [], []
        h2d = d2h = 0
        n_warm = max(1, args.warmup)  # same warm-up as the device-resident leg
        for i in range(max(1, args.e2e_steps) + n_warm):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out, _ = dev.simulate_batch(pb, cfg)
            walls.append(time.perf_counter() - t0)
            tm = dev.timing()
            h2d, d2h = int(tm["h2d_bytes"]), int(tm["d2h_bytes"])
            plan_ms.append(tm["plan_ms"])
            wait_ms.append(tm["run_wait_ms"])
        walls, plan_ms, wait_ms = walls[n_warm:], plan_ms[n_warm:], wait_ms[n_warm:]
        e2e_val = int(out["iterations"].sum()) / statistics.mean(walls)
        if dist:
            tt = torch.tensor([max(walls)], device=f"cuda:{local}", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_val = iters_all / float(tt.item())
        e2e = {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": 1000 * statistics.mean(walls), "call": "lt_simulate_batch (host pinned buffers)",
               "plan_ms": statistics.mean(plan_ms), "run_wait_ms": statistics.mean(wait_ms),
               "warmup_calls": n_warm}
        # The reference's compute_metrics always sorts TTFT/ITL for percentiles
        # (metrics.cpp:101-105); sweeps never read them, so the timed device
        # path skips them. Same call with the percentiles (recording pass +
        # segmented sorts), reported beside it:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev.simulate_batch(pb, cfg, want_percentiles=True)
        e2e["with_percentiles"] = {"value": iters_all / (time.perf_counter() - t0), "unit": UNIT,
                                   "note": "lt_simulate_batch(want_percentiles=1): full compute_metrics incl. "
                                           "TTFT/ITL p50/p99, as the CPU reference computes"}

    log(f"[{time.strftime('%X')}] e2e: {e2e}")
    secondary = None
    if rank == 0 and not args.no_sweeps:
        try:
            secondary = sweep_secondary(dev, args.sweep_conditions)
        except Exception as ex:  # reported, never silently replaced
            secondary = {"error": repr(ex)}

    peak, peak_kind = measured_peaks()
    eng_ms = statistics.mean(eng)
    algo_b = statistics.mean(algo)
    achieved = algo_b / (eng_ms / 1000.0) / 1e9
    traffic, ncu = ncu_traffic()
    if rank != 0:
        return 0
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "scenarios_per_gpu": n_scen, "duration_s": args.duration,
                   "engine_iterations_per_step": iters_all, "failed_scenarios": bad,
                   "l2": "flushed (256 MiB write) before every timed step",
                   "parallelism": f"scenario replicas x{world}, NCCL all-gather of per-scenario records"},
        "e2e": e2e,
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": peak_kind, "kernel": "engine_kernel",
                     "algorithmic_bytes_per_launch": algo_b, "kernel_ms": eng_ms,
                     "note": "B_iter = 20R+16V+24A+16M+64 per engine-iteration (SURVEY 8d); "
                             "engine is latency/issue-bound (one warp per engine), see profiles/"},
        "cpu_baseline": cpu, "parity": parity, "clocks": clk, "secondary": secondary,
        "phase_ms": {k: dev.timing()[k] for k in ("tables_ms", "merge_ms", "engine_ms", "run_ms")},
    }
    if ncu:
        line["roofline"]["ncu"] = ncu
    print(json.dumps(line), flush=True)
    plan.close()
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["gpu", "reference"], default="gpu")
    ap.add_argument("--duration", type=float, default=600.0)
    ap.add_argument("--cpu-stride", type=int, default=1, help="cpu_baseline sample: every k-th C2 scenario")
    ap.add_argument("--ref-stride", type=int, default=3, help="--impl reference sample per step")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--sweep-conditions", type=int, default=64)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sweeps", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return impl_reference(args)
    return impl_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
