"""Where the C4 sweep's time goes: wall of lt_sweep_batch vs its device
phases (run with LT_HOST_TIMING=1 for the per-wave lines).

    LT_HOST_TIMING=1 python tools/c4_timing.py
"""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402
import paper_2508_08343_b200 as lt  # noqa: E402
from paper_2508_08343_b200.batch import ConditionBatch  # noqa: E402

dev = lt.device(0)
conds, cfg, grid, opts, dur, seed = bench.sweep_workload()
t0 = time.perf_counter()
cb = ConditionBatch.from_conditions(conds)
print(f"ConditionBatch: {1000 * (time.perf_counter() - t0):.1f} ms", file=sys.stderr)
for rep in range(2):
    t0 = time.perf_counter()
    pl, fr = dev.sweep_batch(cb, cfg, grid, dur, seed, opts)
    wall = time.perf_counter() - t0
    t = dev.timing()
    print(f"rep {rep}: wall {1000 * wall:.1f} ms, library total {t['total_ms']:.1f}, engine {t['engine_ms']:.1f}, "
          f"count+merge {t['merge_ms']:.1f}, run {t['run_ms']:.1f}, tables {t['tables_ms']:.1f}, "
          f"reduce {t['reduce_ms']:.1f}, d2h {t['d2h_ms']:.1f}", file=sys.stderr, flush=True)
