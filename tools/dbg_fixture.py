import json, os, sys, time
sys.path.insert(0, os.getcwd())
import paper_2508_08343_b200 as lt
from tests import workloads as W
fx = json.load(open('tests/golden/hand_traced_two_adapter.json'))
cfg = W.fixture_config(fx); ads, reqs = W.fixture_scripted(fx)
t = time.time()
try:
    r = lt.run_scripted(reqs, ads, fx['duration_s'], cfg)
    print('scripted ok', r.iterations, r.final_clock_s, time.time() - t)
except Exception as e:
    print('scripted FAIL', type(e).__name__, e)
