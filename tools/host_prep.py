"""Host-preparation timeline of a workload's first bench chunk through
lt_simulate_batch (LT_HOST_TIMING=1 prints it on stderr): where the e2e
call's host time goes.   LT_HOST_TIMING=1 python tools/host_prep.py [c5|c2]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2508_08343_b200 as lt  # noqa: E402

lab, b, cfg = bench.sim_parts(sys.argv[1] if len(sys.argv) > 1 else "c5")[0]
first = bench.chunks(b)[0]
dev = lt.device(0)
for _ in range(5):
    t0 = time.perf_counter()
    dev.simulate_batch(first, cfg)
    t = dev.timing()
    print(f"{len(first.scenarios)} scenarios: call {1e3 * (time.perf_counter() - t0):.1f} ms, plan {t['plan_ms']:.1f} ms, "
          f"run+wait {t['run_wait_ms']:.1f} ms, device run {t['run_ms']:.1f} ms", flush=True)
