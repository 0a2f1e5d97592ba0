"""Scan counters of the critical-path engines (needs the -DLT_SCAN_STATS build)."""
import os, sys
os.environ.setdefault("LT_GPU_LIB", os.path.join(os.getcwd(), "paper_2508_08343_b200/lib/libloratwin_gpu_stats.so"))
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2508_08343_b200 as lt
from paper_2508_08343_b200.batch import WorkloadBatch
from tests import workloads as W
full = W.c2_batch(600.0)
pick = [i for i in range(len(full.scenarios)) if i % 8 == 0 and full.scenarios[i]["n_adapters"] >= 160]
b = WorkloadBatch(full.scenarios[pick].copy(), full.adapters, full.lengths, full.full_lengths, full.requests)
out, _ = lt.device().simulate_batch(b, lt.h100_like_config(1))
names = ["fresh_scans", "stop_cache_hits", "reconciles", "rebuilds", "events", "admissions"]
st = out["phase_cycles"]
for k in range(4):
    it = int(out["iterations"][k])
    print(pick[k], "iters", it, {n: round(float(st[k][j]) / it, 3) for j, n in enumerate(names)})
tot = st.sum(axis=0); it = out["iterations"].sum()
print("all heavy per iteration:", {n: round(float(tot[j]) / it, 3) for j, n in enumerate(names)})
