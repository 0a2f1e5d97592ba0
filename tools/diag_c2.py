"""Diagnose C2 on GPU vs the reference in chunks with an iteration cap."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2508_08343_b200 as lt
from paper_2508_08343_b200.batch import WorkloadBatch, sim_options
from tests import workloads as W
from oracle.pyoracle import RefOracle

cap = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
full = W.c2_batch(600.0)
ref = RefOracle(threads=os.cpu_count())
dev = lt.device()
cfg = lt.h100_like_config(1)
opts = lt.SimOptions(iteration_cap_override=cap)
chunk = 128
for c0 in range(0, 1024, chunk):
    sc = full.scenarios[c0:c0 + chunk].copy()
    b = WorkloadBatch(sc, full.adapters, full.lengths, full.full_lengths, full.requests)
    t = time.time()
    g, _ = dev.simulate_batch(b, cfg, options=opts, want_digest=True)
    tg = time.time() - t
    t = time.time()
    r, _ = ref.simulate(b, cfg, sim_options(opts, True))
    tr = time.time() - t
    bad = np.nonzero((g["iterations"] != r["iterations"]) | (g["digest"] != r["digest"]) | (g["status"] != r["status"]))[0]
    print(f"chunk {c0}: gpu {tg:.2f}s ref {tr:.2f}s gpu_iters {g['iterations'].sum()} ref_iters {r['iterations'].sum()} "
          f"max_gpu_it {g['iterations'].max()} trunc {g['truncated'].sum()} bad {len(bad)} {[(c0+int(i), int(g['iterations'][i]), int(r['iterations'][i])) for i in bad[:5]]}",
          flush=True)
