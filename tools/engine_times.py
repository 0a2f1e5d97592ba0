"""Engine-kernel time (CUDA events, best of 3 warm runs) of the first bench
plan of each workload: the quick A/B measurement for engine changes.

  python tools/engine_times.py [c2 c3 c5]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2508_08343_b200 as lt  # noqa: E402

dev = lt.device(0)
for w in sys.argv[1:] or ["c2", "c3", "c5"]:
    lab, b, cfg = bench.sim_parts(w)[0]
    first = bench.chunks(b)[0] if w != "c3" else bench.chunks(b)[-1]
    plan = dev.plan(first, cfg)
    eng, run = [], []
    for _ in range(4):
        plan.run()
        res = plan.results()
        t = dev.timing()
        eng.append(t["engine_ms"])
        run.append(t["run_ms"])
    print(json.dumps({"workload": w, "plan": f"{lab} ({len(first.scenarios)} scenarios)",
                      "iterations": int(res["iterations"].sum()), "engine_ms": min(eng[1:]), "run_ms": min(run[1:]),
                      "longest_engine_ms": float(res["device_cycles"].max()) / 1.965e6}), flush=True)
    plan.close()
