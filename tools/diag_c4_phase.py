"""Per-phase engine cycles of C4's largest engines (prof build, -DLT_PHASE_PROF)."""
import os, sys
os.environ.setdefault("LT_GPU_LIB", os.path.join(os.getcwd(), "paper_2508_08343_b200/lib/libloratwin_gpu_prof.so"))
sys.path.insert(0, os.getcwd())
import paper_2508_08343_b200 as lt
from paper_2508_08343_b200.batch import WorkloadBatch
cond = lt.Condition(mix=[lt.AdapterTemplate(8, 3.2), lt.AdapterTemplate(16, 3.2), lt.AdapterTemplate(32, 3.2)],
                    lengths=lt.LengthSpec.mean(23, 5, 27, 5))
cases = [(256, 16), (256, 32), (256, 64), (96, 16)]
b = WorkloadBatch.from_workloads([lt.instantiate_condition(cond, n, 600.0, 5) for n, _ in cases], slots=[g for _, g in cases])
out, _ = lt.device().simulate_batch(b, lt.h100_like_config(1))
names = ["ingest", "retire", "alloc", "admit_pq", "admit_fresh", "load+emit"]
for k, (n, g) in enumerate(cases):
    r = out[k]; it = max(1, int(r["iterations"]))
    print(f"N={n} G={g} iters {it} R/it {int(r['sum_running'] / it)} arrivals/it {r['sum_arrivals'] / it:.0f} cyc/it {int(r['device_cycles'] / it)}",
          {nm: int(r["phase_cycles"][j] / it) for j, nm in enumerate(names)}, flush=True)
