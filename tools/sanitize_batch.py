"""Workload for the compute-sanitizer runs of the engine (memcheck, racecheck,
synccheck; tools/gpu_sanitize.sh): scripted fuzz engines (preemption, slot
churn, sole-survivor failures), the summary cases, a C2 subset, one sweep and
one report call -- every engine variant and the report pass."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2508_08343_b200 as lt  # noqa: E402
from paper_2508_08343_b200.batch import ConditionBatch, WorkloadBatch  # noqa: E402
from tests import workloads as W  # noqa: E402

dev = lt.device(0)
for seed in range(0, 24):
    ads, reqs, cfg = W.scripted_fuzz(seed, n_requests=40 + seed % 50, n_adapters=1 + seed % 6, tight=seed % 5 != 4)
    b = WorkloadBatch.from_workloads([W.scripted_workload(ads, 6.0)], scripted=[reqs])
    dev.simulate_batch(b, cfg, want_states=True, want_digest=True)
batch, cfg = W.summary_cases()
for v in ("1", "3", "2"):
    os.environ["LT_ENGINE_VARIANT"] = v
    dev.simulate_batch(batch, cfg, want_digest=True)
os.environ.pop("LT_ENGINE_VARIANT")
dev.simulate_batch(batch, cfg, want_percentiles=True)
dev.simulate_report(batch, cfg)
dev.simulate_batch(W.c2_batch(duration_s=60.0, stride=64), lt.h100_like_config(32))
conds, cfg, grid, dur, seed, opts = W.sweep_cases()
dev.sweep_batch(ConditionBatch.from_conditions(conds[:6]), cfg, grid, 60.0, seed, opts)
print("sanitize batch done")
