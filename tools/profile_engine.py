"""Target of the engine ncu capture: builds the first device-resident plan of
a bench workload (bench.py's chunking), runs it twice and records the
engine-iterations of one launch, so tools/ncu_summary.py can turn the
capture's warp-instruction count into instructions per engine-iteration (the
bench's issue roofline).

  ncu --set full --clock-control none --import-source on -k regex:engine_kernel -s 1 -c 1 \\
      -o OUT python tools/profile_engine.py c2 ITERS.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2508_08343_b200 as lt  # noqa: E402

workload, out = sys.argv[1], sys.argv[2]
lab, b, cfg = bench.sim_parts(workload)[0]
first = bench.chunks(b)[0]
dev = lt.device(0)
plan = dev.plan(first, cfg)
for _ in range(2):
    plan.run()
    res = plan.results()
json.dump({"workload": workload, "plan": f"{lab}: the first bench plan ({len(first.scenarios)} scenarios)",
           "engine_iterations": int(res["iterations"].sum()), "engine_ms": dev.timing()["engine_ms"]},
          open(out, "w"))
plan.close()
