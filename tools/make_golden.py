"""Generates tests/golden/*.json from the reference (run in the build
container, where /root/reference and oracle/_ref/libloratwin_ref.so exist).

  hand_traced_two_adapter.json   transcribed reference fixture (proj/tests/fixtures)
  derived_values.json            transcribed reference fixture
  arrivals.json                  generate_arrivals of the compiled reference for
                                 seeded workloads (bit patterns as hex)
  summaries.json                 run_simulation + compute_metrics records
  sweeps.json                    sweep_optimal results
The GPU box has no /root/reference; tests compare against these files there.
"""
import json
import os
import shutil
import struct
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2508_08343_b200 as lt  # noqa: E402
from paper_2508_08343_b200.batch import ConditionBatch, WorkloadBatch, sim_options  # noqa: E402
from oracle.pyoracle import RefOracle  # noqa: E402
from tests import workloads as W  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
FIX = "/root/reference/proj/tests/fixtures"


def hexf(x):
    return struct.pack("<d", float(x)).hex()


def main():
    os.makedirs(OUT, exist_ok=True)
    for name in ("hand_traced_two_adapter.json", "derived_values.json", "metrics_manual_oracle.json"):
        shutil.copy(os.path.join(FIX, name), os.path.join(OUT, name))
    ref = RefOracle(threads=8)
    # arrivals
    wls = W.arrival_cases()
    batch = WorkloadBatch.from_workloads(wls, mode=lt.LengthMode.Mean)
    reqs, counts = ref.generate_arrivals(batch, sim_options())
    offs = np.concatenate([[0], np.cumsum(counts)])
    cases = []
    for i, w in enumerate(wls):
        rr = reqs[offs[i]:offs[i + 1]]
        cases.append({"case": i, "n": int(counts[i]),
                      "adapter_id": rr["adapter_id"].tolist(), "input_tokens": rr["input_tokens"].tolist(),
                      "output_tokens": rr["output_tokens"].tolist(),
                      "arrival_hex": [hexf(x) for x in rr["arrival_time_s"]]})
    json.dump({"libm_variant": "fma" if lt_variant() else "generic", "cases": cases},
              open(os.path.join(OUT, "arrivals.json"), "w"))
    # summaries
    batch, cfg = W.summary_cases()
    out, _ = ref.simulate(batch, cfg, sim_options(None, True))
    recs = []
    for i in range(len(out)):
        r = out[i]
        recs.append({k: (hexf(r[k]) if out.dtype[k].kind == "f" else int(r[k])) for k in out.dtype.names
                     if not k.startswith("_") and not k.startswith("sum_")})
    json.dump({"records": recs}, open(os.path.join(OUT, "summaries.json"), "w"))
    # sweeps
    conds, cfg, grid, dur, seed, opts = W.sweep_cases()
    pl, fr = ref.sweep(ConditionBatch.from_conditions(conds), cfg, grid, dur, seed, opts, sim_options())
    recs = []
    for i in range(len(conds)):
        p = pl[i]
        recs.append({"status": int(p["status"]), "message": ref.message(i),
                     "n_star": int(p["n_star"]), "g_star": int(p["g_star"]),
                     "max_throughput_hex": hexf(p["max_throughput_tok_s"]), "all_starved": int(p["all_starved"]),
                     "frontier_open": int(p["frontier_open"]),
                     "frontier": [[int(f["n"]), int(f["g"]), hexf(f["throughput_tok_s"]), int(f["starved"]),
                                   int(f["skipped"])] for f in fr[i][:int(p["frontier_count"])]]})
    json.dump({"records": recs}, open(os.path.join(OUT, "sweeps.json"), "w"))
    print("golden written:", sorted(os.listdir(OUT)))


def lt_variant():
    import ctypes
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2508_08343_b200", "lib", "libloratwin_gpu.so"))
    return lib.lt_host_libm_variant()


if __name__ == "__main__":
    main()
