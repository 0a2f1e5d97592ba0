"""Per-phase engine cycles of the slowest C2 scenarios (needs the -DLT_PHASE_PROF build)."""
import os, sys
os.environ.setdefault("LT_GPU_LIB", os.path.join(os.getcwd(), "paper_2508_08343_b200/lib/libloratwin_gpu_prof.so"))
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2508_08343_b200 as lt
from tests import workloads as W
dev = lt.device()
b = W.c2_batch(600.0)
out, _ = dev.simulate_batch(b, lt.h100_like_config(1))
print("engine_ms", dev.timing()["engine_ms"])
cyc = out["device_cycles"]
names = ["ingest", "retire", "alloc", "admit_pq", "admit_fresh", "load+emit"]
for i in np.argsort(-cyc)[:8]:
    r = out[i]; it = max(1, int(r["iterations"]))
    ph = r["phase_cycles"]
    print(i, "N", b.scenarios[i]["n_adapters"], "iters", it, "R/it", int(r["sum_running"] / it), "pre", r["preemptions"],
          "cyc/it", int(cyc[i] / it), {n: int(ph[k] / it) for k, n in enumerate(names)})
tot = out["phase_cycles"].sum(axis=0)
print("all scenarios share:", {n: round(float(tot[k] / tot.sum()), 3) for k, n in enumerate(names)})
