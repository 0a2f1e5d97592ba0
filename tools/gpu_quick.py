"""Quick GPU sanity run: hand-traced fixture, a few fuzz cases, smoke."""
import json, os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2508_08343_b200 as lt
from paper_2508_08343_b200.batch import WorkloadBatch, sim_options
from tests import workloads as W
from oracle.pyoracle import RefOracle

fx = json.load(open('tests/golden/hand_traced_two_adapter.json'))
cfg = W.fixture_config(fx); ads, reqs = W.fixture_scripted(fx)
t = time.time()
r = lt.run_scripted(reqs, ads, fx['duration_s'], cfg)
print('fixture', r.iterations, r.final_clock_s, [q.first_token_time_s for q in r.requests], round(time.time() - t, 3))
ref = RefOracle(threads=8)
bad = 0
for seed in range(40):
    ads, reqs, cfg = W.scripted_fuzz(seed)
    b = WorkloadBatch.from_workloads([W.scripted_workload(ads, 6.0)], scripted=[reqs])
    g, _ = lt.device().simulate_batch(b, cfg, want_digest=True)
    rr, _ = ref.simulate(b, cfg, sim_options(None, True))
    for f in ('status', 'iterations', 'digest', 'finished_count', 'preemptions', 'final_clock_s'):
        if g[0][f] != rr[0][f]:
            bad += 1
            print('fuzz mismatch seed', seed, f, g[0][f], rr[0][f])
            break
print('fuzz bad', bad)
import __graft_entry__ as G
G.smoke()
