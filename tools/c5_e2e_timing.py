"""Host/device timeline of one C5 end-to-end call (lt_simulate_batch over
pinned host buffers, chunked and pipelined): run with LT_HOST_TIMING=1.

    LT_HOST_TIMING=1 python tools/c5_e2e_timing.py [c3|c5]
"""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2508_08343_b200 as lt  # noqa: E402

dev = lt.device(0)
parts = bench.sim_parts(sys.argv[1] if len(sys.argv) > 1 else "c5", 0)
pinned = [(bench.pinned_copy(b), cfg) for _, b, cfg in parts]
for rep in range(2):
    for (pb, _keep), cfg in pinned:
        t0 = time.perf_counter()
        out, _ = dev.simulate_batch(pb, cfg)
        t = dev.timing()
        print(f"rep {rep}: wall {1000 * (time.perf_counter() - t0):.1f} ms plan_ms {t['plan_ms']:.1f} "
              f"engine_ms {t['engine_ms']:.1f} tables_ms {t['tables_ms']:.1f} merge_ms {t['merge_ms']:.1f} "
              f"run_ms {t['run_ms']:.1f} h2d {t['h2d_bytes'] / 1e9:.2f} GB, device memory in use "
              f"{(torch.cuda.mem_get_info()[1] - torch.cuda.mem_get_info()[0]) / 1e9:.1f} GB", file=sys.stderr, flush=True)
