"""ncu target: one train_placement_model call (65,536 rows, 3 x 10 trees) after a warm-up."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_08343_b200 as lt  # noqa: E402
from paper_2508_08343_b200 import predictor as P  # noqa: E402
from tools.bench_predictor import rows_of  # noqa: E402

rows = rows_of(int(sys.argv[1]) if len(sys.argv) > 1 else 65_536)
fp = P.ForestParams(n_trees=10, tree=P.TreeParams(max_depth=5, min_leaf=2))
dev = lt.device(0)
P.train_placement_model(rows, fp, seed=42, dev=dev)
P.train_placement_model(rows, fp, seed=42, dev=dev)
