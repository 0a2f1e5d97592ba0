import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2508_08343_b200 as lt
from paper_2508_08343_b200.batch import WorkloadBatch
from tests import workloads as W
full = W.c2_batch(600.0)
dev = lt.device()
cfg = lt.h100_like_config(1)
for _ in range(2):
    out, _ = dev.simulate_batch(full, cfg)
t = dev.timing(); cyc_full = out["device_cycles"].astype(float)
order = np.argsort(-cyc_full)
pick = sorted(order[:60].tolist())
print("full: engine_ms %.2f longest %.2f ms" % (t["engine_ms"], cyc_full.max() / 1.965e6))
for variant in ("1",):
    b = WorkloadBatch(full.scenarios[pick].copy(), full.adapters, full.lengths, full.full_lengths, full.requests)
    for _ in range(2):
        o2, _ = dev.simulate_batch(b, cfg)
    t2 = dev.timing(); c2 = o2["device_cycles"].astype(float)
    r = c2 / cyc_full[pick]
    print("heavy-60 alone: engine_ms %.2f longest %.2f ms; per-engine alone/full ratio min %.3f mean %.3f max %.3f" % (
        t2["engine_ms"], c2.max() / 1.965e6, r.min(), r.mean(), r.max()))
    top = np.argsort(-cyc_full[pick])[:10]
    print("top10 full ms", np.round(cyc_full[pick][top] / 1.965e6, 2), "alone", np.round(c2[top] / 1.965e6, 2))
