"""Scan counters and cycles of C4's largest engines (N = 256, high-rate short
requests) per G, with the stats build (-DLT_SCAN_STATS)."""
import os, sys
os.environ.setdefault("LT_GPU_LIB", os.path.join(os.getcwd(), "paper_2508_08343_b200/lib/libloratwin_gpu_stats.so"))
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2508_08343_b200 as lt
from paper_2508_08343_b200.batch import WorkloadBatch
cond = lt.Condition(mix=[lt.AdapterTemplate(8, 3.2), lt.AdapterTemplate(16, 3.2), lt.AdapterTemplate(32, 3.2)],
                    lengths=lt.LengthSpec.mean(23, 5, 27, 5))
wls, slots = [], []
for n in (64, 128, 256):
    for g in (16, 32, 64):
        wls.append(lt.instantiate_condition(cond, n, 600.0, 5))
        slots.append(g)
b = WorkloadBatch.from_workloads(wls, slots=slots)
out, _ = lt.device().simulate_batch(b, lt.h100_like_config(1))
names = ["fresh_scans", "stop_hits", "nonlane_scans", "rebuilds", "events", "admissions"]
k = 0
for n in (64, 128, 256):
    for g in (16, 32, 64):
        r = out[k]; it = max(1, int(r["iterations"]))
        print(f"N={n} G={g} iters {it} R/it {int(r['sum_running'] / it)} cyc/it {int(r['device_cycles'] / it)} req {r['n_requests']}",
              {nm: round(float(r["phase_cycles"][j]) / it, 2) for j, nm in enumerate(names)}, flush=True)
        k += 1
