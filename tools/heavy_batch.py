"""The critical-path C2 engines (r = 3.2, N >= 160: the starved, slot-bound
ones that set the C2 step time) as their own batch, for focused ncu captures
and per-iteration cost checks.

    python tools/heavy_batch.py [runs]
"""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402

import paper_2508_08343_b200 as lt  # noqa: E402
from paper_2508_08343_b200.batch import WorkloadBatch  # noqa: E402
from tests import workloads as W  # noqa: E402

full = W.c2_batch(600.0)
pick = [i for i in range(len(full.scenarios)) if i % 8 == 0 and full.scenarios[i]["n_adapters"] >= 160]
b = WorkloadBatch(full.scenarios[pick].copy(), full.adapters, full.lengths, full.full_lengths, full.requests)
dev = lt.device()
runs = int(sys.argv[1]) if len(sys.argv) > 1 else 2
for _ in range(runs):
    out, _ = dev.simulate_batch(b, lt.h100_like_config(1))
    t = dev.timing()
    it = out["iterations"]
    cyc = out["device_cycles"]
    print(f"{len(pick)} heavy engines: engine_ms {t['engine_ms']:.2f} tables_ms {t['tables_ms']:.2f} "
          f"merge_ms {t['merge_ms']:.2f} max cyc/iter {int((cyc / np.maximum(it, 1)).max())} "
          f"mean cyc/iter {int(cyc.sum() / it.sum())} iters {int(it.sum())}", flush=True)
