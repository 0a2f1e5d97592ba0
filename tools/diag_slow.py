"""Per-scenario device cycles on C2: which engines form the critical path."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2508_08343_b200 as lt
from tests import workloads as W
dev = lt.device()
b = W.c2_batch(600.0)
out, _ = dev.simulate_batch(b, lt.h100_like_config(1))
t = dev.timing()
print("timing", {k: round(v, 2) for k, v in t.items() if k.endswith('ms')})
cyc = out["device_cycles"]
order = np.argsort(-cyc)
print("total cycles", cyc.sum(), "max", cyc.max(), "p50", np.median(cyc))
for i in order[:12]:
    sc = b.scenarios[i]
    r = out[i]
    print(i, "N", sc["n_adapters"], "rate", round(float(b.adapters[sc["adapter_offset"]]["rate"]) * sc["n_adapters"] / 8, 4),
          "cyc %.3g" % cyc[i], "iters", r["iterations"], "req", r["n_requests"], "R", r["sum_running"], "V", r["sum_visited"],
          "pre", r["preemptions"], "starved", r["starved"], "cyc/iter", int(cyc[i] / max(1, r["iterations"])))
