"""Placement-model training on the device: train_tree,
train_forest and train_placement_model grow the reference's CART trees
node for node -- same preorder node vectors, split features, thresholds,
leaf values and coverages, bit-exact -- and ForestModel / PlacementModel
predictions match the reference's (predictor.cpp:202-269), against the
compiled reference (oracle/_ref)."""
import numpy as np
import pytest

import paper_2508_08343_b200 as lt
from paper_2508_08343_b200 import predictor as P
from paper_2508_08343_b200.types import ValidationError
from tests import workloads as W

pytestmark = pytest.mark.gpu


def dataset(n_conditions: int = 3000, seed: int = 3):
    """Dataset-shaped rows: the 16 encode_workload features of C4 conditions
    (many tied feature values: ranks, rates, length settings) and targets
    with ties (n*, g* are small integers)."""
    conds = W.c4_conditions()
    rng = np.random.default_rng(seed)
    pick = rng.choice(len(conds), size=n_conditions, replace=False)
    x = np.asarray([lt.encode_workload(conds[i]) for i in pick])
    tput = 400.0 * x[:, 2] / (1.0 + 0.01 * x[:, 4]) + rng.normal(0.0, 5.0, size=len(x))
    n_star = np.clip(np.round(64.0 / (1.0 + x[:, 0])), 1, 256)
    g_star = np.clip(np.round(np.log2(1.0 + x[:, 6])), 1, 64)
    rows = [P.DatasetRow(features=list(x[i]), max_throughput_tok_s=float(tput[i]), n_star=int(n_star[i]),
                         g_star=int(g_star[i]), all_starved=bool(i % 17 == 0)) for i in range(len(x))]
    return x, tput, n_star, g_star, rows


def same_tree(a: P.DecisionTree, b: P.DecisionTree, where=""):
    assert len(a.nodes) == len(b.nodes), where
    for k, (u, v) in enumerate(zip(a.nodes, b.nodes)):
        assert (u.feature_index, u.left, u.right, u.coverage) == (v.feature_index, v.left, v.right, v.coverage), \
            (where, k, u, v)
        # bit patterns: an empty child (all rows on one side of a threshold
        # that rounds onto the upper value) has the reference's NaN mean
        assert np.float64(u.threshold).tobytes() == np.float64(v.threshold).tobytes(), (where, k, u, v)
        assert np.float64(u.value).tobytes() == np.float64(v.value).tobytes(), (where, k, u, v)


@pytest.mark.parametrize("params", [P.TreeParams(), P.TreeParams(max_depth=8, min_leaf=1),
                                    P.TreeParams(max_depth=3, min_leaf=40), P.TreeParams(feature_subset=5),
                                    P.TreeParams(max_depth=0)])
def test_train_tree_matches_reference(dev, ref, params):
    x, tput, n_star, _, _ = dataset()
    for y, tag in ((tput, 7), (n_star, 1000003)):
        a = P.train_tree(x, y, params, seed=11, tree_tag=tag, dev=dev)
        b = P.train_tree(x, y, params, seed=11, tree_tag=tag, lib=ref.lib, ctx=None)
        same_tree(a, b, f"{params} tag {tag}")


@pytest.mark.parametrize("subset", [16, 6])
def test_train_placement_model_matches_reference(dev, ref, subset):
    x, _, _, _, rows = dataset(6000)
    fp = P.ForestParams(n_trees=10, tree=P.TreeParams(max_depth=5, min_leaf=2, feature_subset=subset))
    a = P.train_placement_model(rows, fp, seed=42, dev=dev)
    b = P.train_placement_model(rows, fp, seed=42, lib=ref.lib, ctx=None)
    for name in ("throughput", "n_star", "g_star"):
        fa, fb = getattr(a, name), getattr(b, name)
        assert len(fa.trees) == len(fb.trees) == 10
        for t, (ta, tb) in enumerate(zip(fa.trees, fb.trees)):
            same_tree(ta, tb, f"{name} tree {t}")
    pa = a.predict_batch(x, dev=dev)
    pb = P._predict([t for f in (b.throughput, b.n_star, b.g_star) for t in f.trees], [0, 1, 2], x,
                    lib=ref.lib, ctx=None)
    np.testing.assert_array_equal(pa, pb)  # (NaN leaves predict NaN on both sides)
    one = a.predict(x[5], dev=dev)
    assert (one.throughput_tok_s, one.n_star, one.g_star) == (pa[0, 5], int(pa[1, 5]), int(pa[2, 5]))


def test_train_forest_without_bootstrap_and_raw_predictions(dev, ref):
    x, tput, _, _, _ = dataset(2000)
    fp = P.ForestParams(n_trees=3, bootstrap=False)
    a = P.train_forest(x, tput, P.PredictTarget.Throughput, fp, seed=9, dev=dev)
    b = P.train_forest(x, tput, P.PredictTarget.Throughput, fp, seed=9, lib=ref.lib, ctx=None)
    for ta, tb in zip(a.trees, b.trees):
        same_tree(ta, tb)
    raw = a.predict_batch(x, raw=True, dev=dev)
    np.testing.assert_array_equal(raw, P._predict(b.trees, [-1], x, lib=ref.lib, ctx=None)[0])


def test_training_errors_match_reference(dev, ref):
    x, tput, _, _, _ = dataset(50)
    for params, msg in ((P.TreeParams(max_depth=-1), "tree.max_depth: must be >= 0"),
                        (P.TreeParams(min_leaf=0), "tree.min_leaf: must be >= 1"),
                        (P.TreeParams(feature_subset=17), "tree.feature_subset: must be in [1, 16]")):
        for kw in ({"dev": dev}, {"lib": ref.lib, "ctx": None}):
            with pytest.raises(ValidationError, match=msg.replace("[", r"\[").replace("]", r"\]")):
                P.train_tree(x, tput, params, **kw)
    for kw in ({"dev": dev}, {"lib": ref.lib, "ctx": None}):
        with pytest.raises(ValidationError, match="forest.n_trees: must be >= 1"):
            P.train_forest(x, tput, P.PredictTarget.Throughput, P.ForestParams(n_trees=0), **kw)
        with pytest.raises(ValidationError, match="training set is empty"):
            P.train_tree(np.zeros((0, 16)), [], **kw)
