#!/usr/bin/env python
"""Benchmark of the batched Digital-Twin sweep (BASELINE.json metric:
simulated engine-iterations/sec + placement sweeps/sec) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl gpu|reference]
                  [--workload c2|c3|c4|c5]

Workloads (synthetic, built by the reference's own generator on
device):
  c1 (BASELINE configs[0]) one Digital Twin run: 8 adapters rank 16 at 0.2 req/s,
     Mean(250,50,231,50), 3600 s, G = 8, seed 1, llama31_8b -- one engine, so
     its time is one warp's latency (reported, not a throughput case).
  c2 (default, BASELINE configs[1]) 1,024 scenarios: N in {8..256 step 8} x
     rank {8,16,32,mixed} x r {3.2..0.0125}; per-adapter rate 8r/N;
     Mean(250,80,231,80); 600 s; G = min(N,32); seed 1234+i; h100_like.
  c3 65,536 scenarios: 2,048 rate x rank conditions x N {3..96}; G = min(N,16);
     shared seed 7.
  c5 1,048,576 scenarios: 524,288 per profile (llama31_8b, qwen25_7b);
     N = 8(1 + i mod 32), long I/O Mean(2048,512,1024,256); seed 2^32 + i.
  c4 16,384 full placement searches (2,200 rate x rank triples x 8 length
     settings; N {1..256}, explicit G {2..64}, early exit k=3, 600 s, seed 5);
     metric: placement sweeps/sec.

A step is one pass of the hot path over the whole workload with its inputs
resident in HBM: K0 RNG tables -> arrival counts -> merge -> engine (K1) +
metrics epilogue (K2), one plan per <= 65,536 scenarios (c3/c5 plans release
their regenerated buffers for the next: lt_plan_trim). `e2e` is the same
metric through the public C-ABI call (lt_simulate_batch / lt_sweep_batch)
from pinned host buffers, host<->device copies inside.

Multi-GPU (one process per GPU, NCCL; `--gpus N` self-launches torchrun when
WORLD_SIZE is unset and refuses to run on fewer GPUs): c2 is weak scaling
(each rank runs its own 1,024-scenario grid, seeds shifted by 1024*rank);
c3/c4/c5 are strong scaling (the fixed scenario / condition set is sharded
by estimated cost, LPT). The fixed-size result records are all-gathered over
NCCL inside the timed step (the path's one exchange).

`--impl reference` times the reference's own CPU implementation
(oracle/_ref: the unmodified reference TUs) on all host cores over the same
workload's reference sample (c2: the whole grid).
"""
from __future__ import annotations

import argparse
import glob
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
SWEEP_UNIT = "conditions/s"
SM_COUNT = 148
PLAN_SCENARIOS = 65_536  # scenarios per device-resident plan (c3/c5)

WORKLOADS = {
    "c1": "C1: single Digital Twin run, llama31_8b profile, 8 LoRA adapters rank 16, 0.2 req/s each (Poisson), "
          "Mean(250,50,231,50), 3600 s simulated, G=8, seed 1 (BASELINE configs[0], latency of one engine)",
    "c2": "C2: 1,024-scenario grid, N=8..256 step 8 x rank {8,16,32,mixed} x r {3.2..0.0125}, per-adapter rate "
          "8r/N, Mean(250,80,231,80), 600 s simulated, G=min(N,32), seed 1234+i, h100_like",
    "c3": "C3: 65,536 scenarios = first 2,048 enumerate_conditions(paper rates x ranks {8,16,32}, triple 3) x "
          "N {3,6..96}, G=min(N,16), Mean(250,80,231,80), 600 s, shared seed 7, h100_like",
    "c5": "C5: 1,048,576 scenarios = 524,288 per profile (llama31_8b, qwen25_7b), N=8(1+i mod 32), rank "
          "{8,16,32}, aggregate {0.5,1,2,4} req/s, Mean(2048,512,1024,256), 600 s, G=min(N,32), seed 2^32+i",
    "c4": "C4: 16,384 placement searches = 2,200 rate x rank triples x 8 length settings (first 16,384), "
          "N {1..256 x2}, explicit G {2..64}, early exit k=3, 600 s, seed 5, h100_like",
}


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


def measured_hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_engine_profile(workload: str):
    """The committed ncu --set full summary of one engine launch of this
    workload (profiles/r<NN>_engine_ncu_<workload>.json, newest round), which
    holds the launch's warp-instruction count, engine-iterations and DRAM bytes."""
    paths = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_engine_ncu_{workload}.json")))
    if not paths:
        return None
    with open(paths[-1]) as f:
        d = json.load(f)
    d["file"] = os.path.relpath(paths[-1], ROOT)
    return d


# --- workloads ---------------------------------------------------------------------------------

def sim_parts(workload: str, rank: int = 0):
    """[(label, WorkloadBatch, ServerConfig)] of a simulate workload."""
    import paper_2508_08343_b200 as lt
    from paper_2508_08343_b200.types import profile_config
    from tests import workloads as W

    if workload == "c1":
        from paper_2508_08343_b200.batch import WorkloadBatch
        from paper_2508_08343_b200.types import profile_config
        wl = lt.WorkloadSpec(adapters=[lt.AdapterSpec(i, 16, 0.2) for i in range(1, 9)],
                             lengths=lt.LengthSpec.mean(250, 50, 231, 50), duration_s=3600.0, seed=1 + 1024 * rank)
        return [("c1", WorkloadBatch.from_workloads([wl], slots=[8]), profile_config("llama31_8b", 8))]
    if workload == "c2":
        b = W.c2_batch(600.0)
        b.scenarios["seed"] = b.scenarios["seed"] + np.uint64(1024 * rank)
        return [("c2", b, lt.h100_like_config(1))]
    if workload == "c3":
        return [("c3", W.c3_batch(), lt.h100_like_config(1))]
    if workload == "c5":
        b = W.c5_batch(0, 524_288)
        return [("c5 llama31_8b", b, profile_config("llama31_8b", 1)), ("c5 qwen25_7b", b, profile_config("qwen25_7b", 1))]
    raise ValueError(workload)


def reference_sample(workload: str):
    """The bounded CPU sample of a workload (the reference arm's step and the
    GPU arm's cpu_baseline): (parts, description)."""
    import paper_2508_08343_b200.distributed as D
    from tests import workloads as W

    if workload == "c1":
        return sim_parts("c1"), "the C1 run itself (1 scenario, one reference thread)"
    if workload == "c2":
        return sim_parts("c2"), "the whole C2 grid (1,024 scenarios)"
    if workload == "c3":
        (lab, b, cfg), = sim_parts("c3")
        idx = np.arange(0, len(b.scenarios), 61)
        return [(lab, D.subset(b, idx), cfg)], f"every 61st C3 scenario ({len(idx)} of 65,536)"
    if workload == "c5":
        from paper_2508_08343_b200.types import profile_config
        idx = np.arange(0, 524_288, 1024)
        out = [(f"c5 {p}", W.c5_batch_at(idx), profile_config(p, 1)) for p in ("llama31_8b", "qwen25_7b")]
        return out, f"every 1024th C5 scenario per profile ({2 * len(idx)} of 1,048,576)"
    if workload == "c4":
        conds = W.c4_conditions()
        idx = [2200 * s + 983 for s in range(8)]
        return [conds[i] for i in idx], "8 C4 conditions (the 984th triple of each length setting, of 16,384)"
    raise ValueError(workload)


def sweep_workload():
    import paper_2508_08343_b200 as lt
    from tests import workloads as W

    grid, opts, dur, seed = W.c4_grid()
    return W.c4_conditions(), lt.h100_like_config(1), grid, opts, dur, seed


def shard(workload: str, parts, rank: int, world: int):
    """This rank's share: c2 replicas (weak), else a cost-balanced shard of
    every part (strong; the same deterministic split on every rank)."""
    import paper_2508_08343_b200.distributed as D

    if world == 1 or workload in ("c1", "c2"):
        return parts
    out = []
    for lab, b, cfg in parts:
        mine = D.balanced_shards(D.scenario_costs(b), world)[rank]
        out.append((lab, D.subset(b, mine), cfg))
    return out


def chunks(batch, max_scenarios: int = PLAN_SCENARIOS, max_requests: float = 2.5e8):
    """Consecutive scenario ranges of at most `max_scenarios` scenarios and
    `max_requests` expected requests (Σ rate x duration) each: one plan each."""
    import paper_2508_08343_b200.distributed as D

    sc, ad = batch.scenarios, batch.adapters
    rate_cum = np.concatenate([[0.0], np.cumsum(ad["rate"])])
    lo, hi = sc["adapter_offset"], sc["adapter_offset"] + sc["n_adapters"]
    req = (rate_cum[hi] - rate_cum[lo]) * sc["duration_s"]
    cuts, acc, cnt = [0], 0.0, 0
    for i, r in enumerate(req):
        if cnt and (cnt >= max_scenarios or acc + r > max_requests):
            cuts.append(i)
            acc, cnt = 0.0, 0
        acc += r
        cnt += 1
    cuts.append(len(sc))
    if len(cuts) == 2:
        return [batch]
    return [D.subset(batch, np.arange(a, b)) for a, b in zip(cuts[:-1], cuts[1:])]


# --- reference arm -----------------------------------------------------------------------------

def run_reference(workload: str, threads: int):
    """The reference's own TUs (oracle/_ref) over the workload's bounded
    sample: run_simulation + compute_metrics (or sweep_optimal for c4) on
    `threads` host threads. Returns (cpu_baseline dict, outputs)."""
    import paper_2508_08343_b200 as lt  # noqa: F401
    from oracle import pyoracle
    from paper_2508_08343_b200.batch import ConditionBatch, sim_options

    kind = "reference" if pyoracle.available("ref") else "port"
    orc = pyoracle.RefOracle(threads=threads) if kind == "reference" else pyoracle.PortOracle(threads=threads)
    sample, desc = reference_sample(workload)
    if workload == "c4":
        _, cfg, grid, opts, dur, seed = sweep_workload()
        t0 = time.perf_counter()
        pl, fr = orc.sweep(ConditionBatch.from_conditions(sample), cfg, grid, dur, seed, opts, sim_options())
        wall = time.perf_counter() - t0
        return {"value": len(sample) / wall, "unit": SWEEP_UNIT, "cores": threads, "kind": kind, "wall_s": wall,
                "sample": f"{desc}: sweep_optimal (the reference's own TUs, {threads} host threads)"}, [(pl, fr)]
    outs, iters, wall = [], 0, 0.0
    for lab, b, cfg in sample:
        t0 = time.perf_counter()
        out, _ = orc.simulate(b, cfg, sim_options())
        wall += time.perf_counter() - t0
        iters += int(out["iterations"].sum())
        outs.append(out)
    return {"value": iters / wall, "unit": UNIT, "cores": threads, "kind": kind, "wall_s": wall,
            "sample": f"{desc}: run_simulation + compute_metrics (the reference's own TUs, {threads} host "
                      f"threads), {iters} engine-iterations in {wall:.2f} s"}, outs


def impl_reference(args):
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    threads = os.cpu_count() or 1
    vals, walls = [], []
    for i in range(args.warmup + args.steps):
        cb, _ = run_reference(args.workload, threads)
        log(f"[{time.strftime('%X')}] reference step {i}: {cb['value']:.4g} {cb['unit']} ({cb['wall_s']:.1f} s)")
        if i >= args.warmup:
            vals.append(cb["value"])
            walls.append(cb["wall_s"])
    v = statistics.mean(vals)
    cb["value"] = v
    _, desc = reference_sample(args.workload)
    line = {"metric": METRIC, "value": v, "unit": cb["unit"], "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * statistics.mean(walls),
            "higher_is_better": True, "scaling": "weak" if args.workload in ("c1", "c2") else "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOADS[args.workload], "sample": desc,
                       "same_config": args.workload in ("c1", "c2"),
                       "step": "one step = the reference sample, on all host cores (rank 0 only)"},
            "cpu_baseline": cb, "e2e": {"value": v, "unit": cb["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --- GPU arm -------------------------------------------------------------------------------------

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


def device_view(ptr: int, nbytes: int, local: int):
    import torch

    class _View:
        __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}
    return torch.as_tensor(_View(), device=f"cuda:{local}")


def parity_against(cpu_outs, dev, workload: str, sample_parts):
    """GPU results on the reference sample vs the reference's outputs."""
    fields = ["status", "iterations", "finished_count", "rejected_count", "preemptions", "load_events",
              "tokens_in_window", "starved", "final_clock_s", "throughput_tok_s", "ttft_mean_s"]
    mism, n = 0, 0
    for (lab, b, cfg), ref_out in zip(sample_parts, cpu_outs):
        g, _ = dev.simulate_batch(b, cfg)
        mism += sum(int(np.sum(g[f] != ref_out[f])) for f in fields)
        n += len(g)
    return {"scenarios": n, "fields": fields, "mismatches": mism}


def issue_roofline(prof, iters_step: int, engine_ms: float, sm_mhz, algo_bytes: float, hbm_peak, hbm_src,
                   longest_cycles: int, launches_engine: int):
    """Binding roofline of the engine kernel: issue slots. achieved = warp
    instructions per engine-iteration (ncu, same workload and build) x this
    step's iterations / the live engine time; peak = 148 SMs x 4 schedulers x
    1 warp-instruction per cycle at the sampled SM clock. HBM is reported
    beside it (SURVEY 8d algorithmic bytes vs the measured peak, and ncu's
    DRAM bytes)."""
    clk = (sm_mhz or 1965.0) * 1e6
    peak = SM_COUNT * 4 * clk
    r = {"bound": "issue", "unit": "warp-inst/s", "peak": peak, "kernel": "engine_kernel", "achieved": None,
         "frac": None, "traffic": None, "engine_ms_per_step": engine_ms, "engine_launches_per_step": launches_engine,
         "peak_note": "148 SMs x 4 SMSPs x 1 issue/cycle at the median sampled SM clock"}
    if prof:
        m = prof.get("metrics", {})
        inst = m.get("smsp__inst_executed.sum", [None])[0]
        its = prof.get("engine_iterations")
        if inst and its:
            per_iter = inst / its
            r["achieved"] = per_iter * iters_step / (engine_ms / 1e3)
            r["frac"] = r["achieved"] / peak
            r["inst_per_iteration"] = per_iter
        r["traffic"] = prof.get("dram_bytes_per_launch")
        r["ncu"] = {"file": prof["file"], "workload": prof.get("workload"),
                    "launch_ms": m.get("gpu__time_duration.sum", [None])[0],
                    "launch_engine_iterations": its, "launch_warp_instructions": inst,
                    "issue_active_pct_of_elapsed": m.get("sm__issue_active.avg.pct_of_peak_sustained_elapsed", [None])[0],
                    "smsp_issue_active_pct_while_resident": m.get("smsp__issue_active.avg.pct_of_peak_sustained_active",
                                                                  [None])[0],
                    "warps_active_pct": m.get("sm__warps_active.avg.pct_of_peak_sustained_active", [None])[0],
                    "cycles_per_issue": m.get("smsp__average_warp_latency_per_inst_issued.ratio", [None])[0]}
    ach = algo_bytes / (engine_ms / 1e3) / 1e9
    r["hbm"] = {"achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak, "peak_source": hbm_src,
                "algorithmic_bytes_per_step": algo_bytes,
                "note": "B_iter = 20R+16V+24A+16M+64 per engine-iteration (SURVEY 8d); the event-driven engine never "
                        "moves these bytes (see traffic)"}
    if r["traffic"] and launches_engine == 1:
        r["hbm"]["measured_dram_gbs"] = r["traffic"] / (engine_ms / 1e3) / 1e9
    # critical path: the longest single engine (one warp, dependent decisions)
    longest_ms = longest_cycles / clk * 1e3
    r["critical_path"] = {"longest_engine_ms": longest_ms, "engine_ms": engine_ms,
                          "ratio": longest_ms / engine_ms if engine_ms else None,
                          "note": "max over engines of device_cycles / SM clock vs the engine kernel time per "
                                  "step: ~1 means the step is one engine's latency, not throughput"}
    return r


COLL_DEV = "cpu"  # the device of collective tensors: cuda:LOCAL_RANK under NCCL
SHARED = bool(os.environ.get("LT_BENCH_SHARED_GPU")) and int(os.environ.get("WORLD_SIZE", "1")) > 1


def impl_gpu(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    global COLL_DEV
    dist = None
    if world > 1:
        import torch.distributed as dist
        if os.environ.get("LT_BENCH_SHARED_GPU"):
            # test mode of the multi-rank path on a one-GPU box: every rank on
            # cuda:0, collectives over gloo on host tensors (never a bench line)
            local = 0
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
            COLL_DEV = "cpu"
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            COLL_DEV = f"cuda:{local}"
    import paper_2508_08343_b200 as lt

    dev = lt.device(local)
    if args.workload == "c4":
        return impl_gpu_sweeps(args, dev, dist, world, rank, local)
    parts = shard(args.workload, sim_parts(args.workload, rank), rank, world)

    # CPU baseline (rank 0, N=1 only), bounded sample; its results also check parity.
    cpu = parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu, cpu_outs = run_reference(args.workload, os.cpu_count() or 1)
        sample_parts, _ = reference_sample(args.workload)
        parity = parity_against(cpu_outs, dev, args.workload, sample_parts)
        parity["oracle"] = cpu["kind"]
        log("cpu baseline", cpu, "parity", parity)

    log(f"[{time.strftime('%X')}] building plans")
    plans = []
    for lab, b, cfg in parts:
        for c in chunks(b):
            p = dev.plan(c, cfg)
            if args.workload not in ("c1", "c2"):
                p.trim()
            plans.append(p)
    n_scen = sum(p.n for p in plans)
    multi = len(plans) > 1
    stream = torch.cuda.ExternalStream(dev.stream(), device=torch.device("cuda", local))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")  # > 126 MB L2
    gathered = mine = None
    if world > 1:  # padded per-rank record buffer for the all-gather
        nbytes = sum(p.device_summaries()[1] for p in plans)
        t = torch.tensor([nbytes], device=COLL_DEV, dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        mine = torch.zeros(int(t.item()), dtype=torch.uint8, device=f"cuda:{local}")
        gathered = [torch.empty_like(mine, device=COLL_DEV) for _ in range(world)]

    def step():
        for p in plans:
            p.run()
            if multi:
                p.trim()
        if world > 1:
            with torch.cuda.stream(stream):
                o = 0
                for p in plans:
                    ptr, nb = p.device_summaries()
                    mine[o:o + nb].copy_(device_view(ptr, nb, local))
                    o += nb
                dist.all_gather(gathered, mine if COLL_DEV != "cpu" else mine.cpu())

    def collect():
        res = [p.results() for p in plans]
        t = dev.timing()
        return res, t

    for i in range(args.warmup):
        step()
        torch.cuda.synchronize()
        log(f"[{time.strftime('%X')}] warmup {i} done")
    res, _ = collect()
    iters_rank = int(sum(int(r["iterations"].sum()) for r in res))
    longest = int(max(int(r["device_cycles"].max()) for r in res if len(r)))
    bad = int(sum(int(np.sum(r["status"] != 0)) for r in res))
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
        em, ab = 0.0, 0
        for p in plans:  # per-plan device timings of this step (CUDA events)
            p.results()
            t = dev.timing()
            em += t["engine_ms"]
            ab += t["algorithmic_bytes"]
            launches += int(t["engine_launches"])
        eng.append(em)
        algo.append(ab)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    total_ms = sum(times)
    iters_all = iters_rank
    if dist:
        tt = torch.tensor([total_ms], device=COLL_DEV, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
        it = torch.tensor([iters_rank], device=COLL_DEV, dtype=torch.int64)
        dist.all_reduce(it, op=dist.ReduceOp.SUM)
        iters_all = int(it.item())
    value = iters_all * args.steps / (total_ms / 1000.0)
    log(f"[{time.strftime('%X')}] timed steps (ms): {times}")
    for p in plans:
        p.close()

    e2e = None
    if not args.no_e2e:
        e2e = e2e_simulate(args, dev, parts, dist, local, iters_all, world)
        log(f"[{time.strftime('%X')}] e2e: {e2e}")

    hbm_peak, hbm_src = measured_hbm_peak()
    roof = issue_roofline(ncu_engine_profile(args.workload), iters_rank, statistics.mean(eng), clk["sm_mhz"],
                          statistics.mean(algo), hbm_peak, hbm_src, longest,
                          launches_engine=len(plans))
    if rank != 0:
        return 0
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak" if args.workload in ("c1", "c2") else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": WORKLOADS[args.workload], "scenarios_per_gpu": n_scen,
                   "engine_iterations_per_step": iters_all, "failed_scenarios": bad, "plans_per_step": len(plans),
                   "l2": "flushed (256 MiB write) before every timed step",
                   "parallelism": (f"scenario replicas x{world}" if args.workload in ("c1", "c2")
                                   else f"cost-balanced scenario shards over {world} GPU(s)")
                   + (", NCCL all-gather of the per-scenario records inside the step" if world > 1 else "")
                   + (" [LT_BENCH_SHARED_GPU test mode: ranks share cuda:0, gloo]" if SHARED else "")},
        "e2e": e2e, "gpu_launches": launches, "roofline": roof, "cpu_baseline": cpu, "parity": parity,
        "clocks": clk,
    }
    if rank == 0 and args.workload == "c2" and not args.no_sweeps:
        try:
            line["secondary"] = sweep_secondary(dev, args.sweep_conditions)
        except Exception as ex:  # reported, never silently replaced
            line["secondary"] = {"error": repr(ex)}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def e2e_simulate(args, dev, parts, dist, local, iters_all, world):
    """The same metric through lt_simulate_batch from pinned host buffers
    (host preparation + H2D + the device pipeline + D2H), per part, after
    warm-up calls; the CPU-side percentile variant is reported beside it."""
    import torch

    pinned = [(pinned_copy(b), cfg) for _, b, cfg in parts]
    walls, plan_ms, wait_ms = [], [], []
    h2d = d2h = 0
    n_warm = max(1, args.warmup) if args.workload in ("c1", "c2") else 1
    n_steps = max(1, args.e2e_steps) if args.workload in ("c1", "c2") else 1
    iters = 0
    for i in range(n_steps + n_warm):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h2d = d2h = pm = wm = 0
        iters = 0
        for (pb, _keep), cfg in pinned:
            out, _ = dev.simulate_batch(pb, cfg)
            tm = dev.timing()
            h2d += int(tm["h2d_bytes"])
            d2h += int(tm["d2h_bytes"])
            pm += tm["plan_ms"]
            wm += tm["run_wait_ms"]
            iters += int(out["iterations"].sum())
        walls.append(time.perf_counter() - t0)
        plan_ms.append(pm)
        wait_ms.append(wm)
    walls, plan_ms, wait_ms = walls[n_warm:], plan_ms[n_warm:], wait_ms[n_warm:]
    wall = statistics.mean(walls)
    val = iters / wall
    if dist:
        tt = torch.tensor([wall], device=COLL_DEV, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        val = iters_all / float(tt.item())
    e2e = {"value": val, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "ms_per_step": 1000 * wall, "call": "lt_simulate_batch (host pinned buffers)",
           "plan_ms": statistics.mean(plan_ms), "run_wait_ms": statistics.mean(wait_ms), "warmup_calls": n_warm,
           "timed_calls": n_steps}
    if args.workload == "c2":
        # compute_metrics always sorts TTFT/ITL for percentiles (metrics.cpp:101-105),
        # which the CPU reference pays; the same call with them, like for like:
        (pb, _keep), cfg = pinned[0]
        pw = []
        pct_warm = max(1, n_warm)  # (the first two calls size the record pool and its sort buffers)
        for i in range(pct_warm + max(1, args.e2e_steps)):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dev.simulate_batch(pb, cfg, want_percentiles=True)
            pw.append(time.perf_counter() - t0)
        wp = statistics.mean(pw[pct_warm:])
        pv = iters / wp
        if dist:  # whole job: every rank's iterations over the slowest rank's call
            tt = torch.tensor([wp], device=COLL_DEV, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            wp = float(tt.item())
            pv = iters_all / wp
        e2e["with_percentiles"] = {"value": pv, "unit": UNIT, "ms_per_step": 1000 * wp, "warmup_calls": pct_warm,
                                   "timed_calls": len(pw) - pct_warm,
                                   "note": "lt_simulate_batch(want_percentiles=1): the full compute_metrics incl. "
                                           "TTFT/ITL p50/p99, as the CPU reference computes; mean of warmed calls"}
    return e2e


def impl_gpu_sweeps(args, dev, dist, world, rank, local):
    """c4: placement sweeps/sec through lt_sweep_batch (host condition
    records in, placements + frontiers out), conditions sharded by cost."""
    import torch

    import paper_2508_08343_b200.distributed as D
    from paper_2508_08343_b200.batch import ConditionBatch

    conds, cfg, grid, opts, dur, seed = sweep_workload()
    cb = ConditionBatch.from_conditions(conds)
    if world > 1:
        t = cb.templates
        costs = [float(t[c["mix_offset"]:c["mix_offset"] + c["mix_count"]]["rate"].mean()) for c in cb.conditions]
        cb = D.condition_subset(cb, D.balanced_shards(costs, world)[rank])
    cpu = parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu, outs = run_reference("c4", os.cpu_count() or 1)
        sample, _ = reference_sample("c4")
        gp, _ = dev.sweep_batch(ConditionBatch.from_conditions(sample), cfg, grid, dur, seed, opts)
        rp = outs[0][0]
        fields = ("status", "n_star", "g_star", "all_starved", "frontier_open", "max_throughput_tok_s")
        parity = {"conditions": len(sample), "fields": list(fields),
                  "mismatches": int(sum(int(np.sum(gp[f] != rp[f])) for f in fields)), "oracle": cpu["kind"]}
    for i in range(args.warmup):
        dev.sweep_batch(cb, cfg, grid, dur, seed, opts)
        log(f"[{time.strftime('%X')}] warmup {i} done")
    clocks = ClockSampler(local)
    clocks.start()
    walls, launches, pts, iters = [], 0, 0, 0
    for _ in range(args.steps):
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pl, fr = dev.sweep_batch(cb, cfg, grid, dur, seed, opts)
        if dist:
            D.all_gather_records(pl, np.arange(len(pl)), len(pl), device=torch.device(COLL_DEV))
        torch.cuda.synchronize()
        walls.append(time.perf_counter() - t0)
        t = dev.timing()
        launches += int(t["engine_launches"])
        pts, iters = int(pl["points_simulated"].sum()), int(pl["iterations"].sum())
    clk = clocks.stop()
    wall = sum(walls)
    if dist:
        tt = torch.tensor([wall], device=COLL_DEV, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        wall = float(tt.item())
    value = len(conds) * args.steps / wall
    if rank != 0:
        return 0
    line = {"metric": METRIC, "value": value, "unit": SWEEP_UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000 * wall / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOADS["c4"], "conditions": len(conds), "points_simulated_per_gpu": pts,
                       "engine_iterations_per_gpu": iters,
                       **({"test_mode": "LT_BENCH_SHARED_GPU: ranks share cuda:0, gloo"} if SHARED else {}),
                       "timing": "wall time of lt_sweep_batch (the sweep's N-row waves are planned on the host per "
                                 "wave), synchronised; max over ranks"},
            "e2e": {"value": value, "unit": SWEEP_UNIT, "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
                    "note": "the sweep has no device-resident form: value is already end to end"},
            "gpu_launches": launches, "cpu_baseline": cpu, "parity": parity, "clocks": clk}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def sweep_secondary(dev, n_cond: int):
    """placement sweeps/sec on a C4 sample (all 8 length settings; explicit G,
    early exit k=3, 600 s, seed 5), beside the C2 line."""
    from paper_2508_08343_b200.batch import ConditionBatch

    conds, cfg, grid, opts, dur, seed = sweep_workload()
    sel = conds[::max(1, len(conds) // n_cond)][:n_cond]
    cb = ConditionBatch.from_conditions(sel)
    dev.sweep_batch(cb, cfg, grid, dur, seed, opts)  # warm
    t0 = time.perf_counter()
    pl, _ = dev.sweep_batch(cb, cfg, grid, dur, seed, opts)
    wall = time.perf_counter() - t0
    return {"metric": "placement sweeps/sec", "value": len(sel) / wall, "unit": SWEEP_UNIT,
            "conditions": len(sel), "sample": f"every {max(1, len(conds) // n_cond)}th C4 condition",
            "points_simulated": int(pl["points_simulated"].sum()), "wall_s": wall,
            "note": "end to end through lt_sweep_batch (host buffers)"}


def self_launch(args) -> int:
    """--gpus N without torchrun: relaunch as N ranks (one per GPU), or refuse."""
    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} requested but only {have} GPU(s) are visible", file=sys.stderr)
        return 2
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["gpu", "reference"], default="gpu")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c2")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--sweep-conditions", type=int, default=64)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sweeps", action="store_true")
    args = ap.parse_args()
    if args.warmup < 0 or args.steps < 1:
        raise SystemExit("bench.py: --steps >= 1 and --warmup >= 0")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        if args.impl == "reference":  # rank 0 alone runs it
            return impl_reference(args)
        return self_launch(args)
    if args.impl == "reference":
        return impl_reference(args)
    return impl_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
