"""Target of an ncu launch list of the C2 call with percentiles
(lt_simulate_batch want_percentiles=1), after one warm call.

    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file X.csv python tools/pct_launches.py
"""
import os
import sys

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402
import paper_2508_08343_b200 as lt  # noqa: E402

dev = lt.device(0)
(lab, b, cfg), = bench.sim_parts("c2", 0)
for _ in range(2):
    dev.simulate_batch(b, cfg, want_percentiles=True)
