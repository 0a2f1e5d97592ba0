"""Placement-model training on one B200 vs the reference's own training on
the host: train_placement_model (3 forests x 10 trees,
depth 5, bootstrap) over dataset-shaped rows -- the 16 encode_workload
features of the C4 conditions with synthetic targets (tests/test_gpu_predictor.py
shapes) -- at 16,384 and 65,536 rows, plus feature_subset = 6. Prints one
JSON line per case: GPU wall time (median of 3 warm calls), reference wall
time (one call; the reference trains on one thread), and whether every tree
matches node for node.

  python tools/bench_predictor.py > profiles/r2_predictor.jsonl
"""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2508_08343_b200 as lt  # noqa: E402
from oracle import pyoracle  # noqa: E402
from paper_2508_08343_b200 import predictor as P  # noqa: E402
from tests import workloads as W  # noqa: E402


def rows_of(n_rows: int, seed: int = 3):
    conds = W.c4_conditions()
    x = np.asarray([lt.encode_workload(c) for c in conds])
    reps = -(-n_rows // len(x))
    x = np.tile(x, (reps, 1))[:n_rows]
    rng = np.random.default_rng(seed)
    tput = 400.0 * x[:, 2] / (1.0 + 0.01 * x[:, 4]) + rng.normal(0.0, 5.0, size=len(x))
    n_star = np.clip(np.round(64.0 / (1.0 + x[:, 0]) + rng.integers(0, 3, size=len(x))), 1, 256)
    g_star = np.clip(np.round(np.log2(1.0 + x[:, 6])), 1, 64)
    return [P.DatasetRow(features=list(x[i]), max_throughput_tok_s=float(tput[i]), n_star=int(n_star[i]),
                         g_star=int(g_star[i])) for i in range(len(x))]


def same(a, b):
    for name in ("throughput", "n_star", "g_star"):
        for ta, tb in zip(getattr(a, name).trees, getattr(b, name).trees):
            if len(ta.nodes) != len(tb.nodes):
                return False
            for u, v in zip(ta.nodes, tb.nodes):
                if (u.feature_index, u.left, u.right, u.coverage) != (v.feature_index, v.left, v.right, v.coverage):
                    return False
                if np.float64(u.threshold).tobytes() != np.float64(v.threshold).tobytes():
                    return False
                if np.float64(u.value).tobytes() != np.float64(v.value).tobytes():
                    return False
    return True


def main():
    dev = lt.device(0)
    ref = pyoracle.RefOracle(threads=1)
    for n_rows, subset in ((16_384, 16), (65_536, 16), (16_384, 6)):
        rows = rows_of(n_rows)
        fp = P.ForestParams(n_trees=10, tree=P.TreeParams(max_depth=5, min_leaf=2, feature_subset=subset))
        P.train_placement_model(rows, fp, seed=42, dev=dev)  # warm-up
        walls = []
        for _ in range(3):
            t0 = time.perf_counter()
            a = P.train_placement_model(rows, fp, seed=42, dev=dev)
            walls.append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        b = P.train_placement_model(rows, fp, seed=42, lib=ref.lib, ctx=None)
        ref_s = time.perf_counter() - t0
        gpu_s = statistics.median(walls)
        print(json.dumps({"case": f"train_placement_model, {n_rows} rows, 3 x 10 trees, depth 5, "
                                  f"feature_subset {subset}", "gpu_s": gpu_s, "device_ms": dev.timing()["engine_ms"],
                          "reference_s": ref_s, "reference_threads": 1, "speedup": ref_s / gpu_s,
                          "trees_identical": same(a, b)}), flush=True)


if __name__ == "__main__":
    main()
