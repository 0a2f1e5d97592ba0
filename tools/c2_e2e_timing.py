"""Host/device timeline of the C2 end-to-end call (lt_simulate_batch over
pinned host buffers): run with LT_HOST_TIMING=1.

    LT_HOST_TIMING=1 python tools/c2_e2e_timing.py
"""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2508_08343_b200 as lt  # noqa: E402

dev = lt.device(0)
(lab, b, cfg), = bench.sim_parts("c2", 0)
pb, _keep = bench.pinned_copy(b)
for rep in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out, _ = dev.simulate_batch(pb, cfg)
    wall = time.perf_counter() - t0
    t = dev.timing()
    print(f"rep {rep}: wall {1000 * wall:.2f} ms plan_ms {t['plan_ms']:.2f} run_wait_ms {t['run_wait_ms']:.2f} "
          f"tables_ms {t['tables_ms']:.2f} merge_ms {t['merge_ms']:.2f} engine_ms {t['engine_ms']:.2f} "
          f"run_ms {t['run_ms']:.2f} d2h_ms {t['d2h_ms']:.2f}", file=sys.stderr, flush=True)
