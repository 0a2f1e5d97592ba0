"""Whole C2 grid (1,024 scenarios, 600 s) on the GPU vs the reference oracle
(oracle/_ref, all host cores): every integer field and the decision digest
bit-exact, FP64 fields bit-exact (itl within 1e-9 relative).

    python tools/c2_full_parity.py [stride]
"""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402

import paper_2508_08343_b200 as lt  # noqa: E402
from oracle.pyoracle import RefOracle  # noqa: E402
from paper_2508_08343_b200.batch import sim_options  # noqa: E402
from tests import workloads as W  # noqa: E402

stride = int(sys.argv[1]) if len(sys.argv) > 1 else 1
b = W.c2_batch(600.0, stride=stride)
cfg = lt.h100_like_config(1)
t = time.time()
g, _ = lt.device().simulate_batch(b, cfg, want_digest=True)
tg = time.time() - t
t = time.time()
r, _ = RefOracle(threads=os.cpu_count()).simulate(b, cfg, sim_options(None, True))
tr = time.time() - t
exact = ["status", "iterations", "finished_count", "rejected_count", "preemptions", "load_events",
         "tokens_in_window", "tokens_total", "starved", "digest", "final_clock_s", "throughput_tok_s", "ttft_mean_s"]
bad = 0
for f in exact:
    m = np.nonzero(g[f] != r[f])[0]
    if len(m):
        bad += len(m)
        print("MISMATCH", f, [(int(i), g[f][i], r[f][i]) for i in m[:5]])
itl = np.abs(g["itl_mean_s"] - r["itl_mean_s"]) > 1e-9 * np.abs(r["itl_mean_s"])
bad += int(itl.sum())
print(f"c2 parity: {len(g)} scenarios, {int(g['iterations'].sum())} iterations, gpu {tg:.2f}s ref {tr:.2f}s, "
      f"mismatches {bad}")
sys.exit(1 if bad else 0)
