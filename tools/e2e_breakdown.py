"""Host/device breakdown of the C2 e2e call (lt_simulate_batch from host buffers).

    LT_HOST_TIMING=1 python tools/e2e_breakdown.py
"""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import paper_2508_08343_b200 as lt  # noqa: E402
from tests import workloads as W  # noqa: E402

b = W.c2_batch(600.0)
dev = lt.device()
cfg = lt.h100_like_config(1)
for k in range(5):
    t0 = time.perf_counter()
    out, _ = dev.simulate_batch(b, cfg)
    wall = (time.perf_counter() - t0) * 1e3
    t = dev.timing()
    print(f"wall {wall:.2f} ms | " + " ".join(f"{k} {v:.2f}" for k, v in t.items() if isinstance(v, float)), flush=True)
