"""Golden vectors for the north-star configs C4 and C5, generated
from the compiled reference (oracle/_ref/libloratwin_ref.so) in the build
container; the -m gpu tests compare the B200 path against them on the box,
which has no /root/reference.

  c5_sample.json  run_simulation + compute_metrics of every 1021st C5
                  scenario (seed 2^32 + i, Mean(2048,512,1024,256), 600 s),
                  under both profiles (llama31_8b, qwen25_7b), with the
                  per-iteration decision digest
  c4_sample.json  sweep_optimal of 46 C4 conditions drawn from all 8 length
                  settings (explicit G {2..64}, N {1..256}, early exit k=3,
                  600 s, seed 5)

  python tools/make_golden_configs.py [c5] [c4]
"""
import json
import os
import struct
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2508_08343_b200.batch import ConditionBatch, sim_options  # noqa: E402
from paper_2508_08343_b200.types import profile_config  # noqa: E402
from oracle.pyoracle import RefOracle  # noqa: E402
from tests import workloads as W  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def hexf(x):
    return struct.pack("<d", float(x)).hex()


def summary_records(out):
    return [{k: (hexf(r[k]) if out.dtype[k].kind == "f" else int(r[k])) for k in out.dtype.names
             if not k.startswith("_") and not k.startswith("sum_") and k not in ("device_cycles", "phase_cycles")}
            for r in out]


def make_c5(ref):
    idx = np.arange(0, 524_288, W.C5_SAMPLE_STRIDE)
    doc = {"indices": idx.tolist(), "profiles": {}}
    for prof in ("llama31_8b", "qwen25_7b"):
        t0 = time.time()
        out, _ = ref.simulate(W.c5_batch_at(idx), profile_config(prof, 1), sim_options(None, True))
        doc["profiles"][prof] = summary_records(out)
        print(f"c5 {prof}: {len(idx)} scenarios, {int(out['iterations'].sum())} iterations, "
              f"{time.time() - t0:.1f} s", flush=True)
    json.dump(doc, open(os.path.join(OUT, "c5_sample.json"), "w"))


def make_c4(ref):
    conds = W.c4_conditions()
    idx = W.c4_sample_indices()
    grid, opts, dur, seed = W.c4_grid()
    t0 = time.time()
    pl, fr = ref.sweep(ConditionBatch.from_conditions([conds[i] for i in idx]), profile_config("h100_like", 1),
                       grid, dur, seed, opts, sim_options())
    recs = []
    for k, i in enumerate(idx):
        p = pl[k]
        recs.append({"condition": i, "status": int(p["status"]), "message": ref.message(k),
                     "n_star": int(p["n_star"]), "g_star": int(p["g_star"]),
                     "max_throughput_hex": hexf(p["max_throughput_tok_s"]), "all_starved": int(p["all_starved"]),
                     "frontier_open": int(p["frontier_open"]), "points_simulated": int(p["points_simulated"]),
                     "iterations": int(p["iterations"]),
                     "frontier": [[int(f["n"]), int(f["g"]), hexf(f["throughput_tok_s"]), int(f["starved"]),
                                   int(f["skipped"])] for f in fr[k][:int(p["frontier_count"])]]})
    print(f"c4: {len(idx)} conditions, {time.time() - t0:.1f} s", flush=True)
    json.dump({"records": recs}, open(os.path.join(OUT, "c4_sample.json"), "w"))


def main():
    which = sys.argv[1:] or ["c5", "c4"]
    ref = RefOracle(threads=os.cpu_count() or 1)
    if "c5" in which:
        make_c5(ref)
    if "c4" in which:
        make_c4(ref)


if __name__ == "__main__":
    main()
