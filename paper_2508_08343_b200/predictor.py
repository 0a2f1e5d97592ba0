"""Placement-model training and inference on the B200.

Mirrors predictor.hpp (PredictTarget, TreeNode, DecisionTree, TreeParams,
ForestParams, ForestModel, PlacementModel, train_tree, train_forest,
train_placement_model): the trees are grown by lt_train_tree /
lt_train_forests and evaluated by lt_predict_forests
(include/loratwin_gpu.h); the models are the reference's node vectors,
bit-identical to its own training (tests/test_gpu_predictor.py).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _abi as A
from .types import ERROR_CLASSES, FEATURE_NAMES, DeviceError, LoratwinError, ValidationError

NUM_FEATURES = 16  # placement.hpp:43


class PredictTarget(enum.IntEnum):  # predictor.hpp:29
    Throughput = 0
    NStar = 1
    GStar = 2


@dataclass
class TreeNode:  # predictor.hpp:40-47
    feature_index: int = -1
    threshold: float = 0.0
    left: int = -1
    right: int = -1
    value: float = 0.0
    coverage: int = 0


@dataclass
class DecisionTree:  # predictor.hpp:49-53
    nodes: List[TreeNode] = field(default_factory=list)

    def predict(self, x: Sequence[float], dev=None) -> float:
        return float(_predict([self], [-1], np.asarray([x], dtype=np.float64), dev)[0, 0])


@dataclass
class TreeParams:  # predictor.hpp:55-62
    max_depth: int = 5
    min_leaf: int = 2
    feature_subset: int = NUM_FEATURES


@dataclass
class ForestParams:  # predictor.hpp:72-76
    n_trees: int = 10
    tree: TreeParams = field(default_factory=TreeParams)
    bootstrap: bool = True


@dataclass
class ForestModel:  # predictor.hpp:78-96
    target: PredictTarget = PredictTarget.Throughput
    params: ForestParams = field(default_factory=ForestParams)
    trees: List[DecisionTree] = field(default_factory=list)
    seed: int = 0
    trained_rows: int = 0
    feature_names: List[str] = field(default_factory=lambda: list(FEATURE_NAMES))

    def predict_raw(self, features: Sequence[float], dev=None) -> float:
        return float(self.predict_batch(np.asarray([features], dtype=np.float64), raw=True, dev=dev)[0])

    def predict(self, features: Sequence[float], dev=None) -> float:
        return float(self.predict_batch(np.asarray([features], dtype=np.float64), dev=dev)[0])

    def predict_batch(self, x: np.ndarray, raw: bool = False, dev=None) -> np.ndarray:
        """predict (or predict_raw) for every row of x (n x 16) in one device call."""
        if not self.trees:
            raise ERROR_CLASSES[A.LT_ERR_INTERNAL]("forest has no trees")
        return _predict(self.trees, [-1 if raw else int(self.target)], x, dev)[0]


@dataclass
class DatasetRow:  # placement.hpp:112-120 (the fields training reads)
    features: List[float] = field(default_factory=lambda: [0.0] * NUM_FEATURES)
    max_throughput_tok_s: float = 0.0
    n_star: int = 0
    g_star: int = 0
    all_starved: bool = False
    condition_hash: int = 0
    duration_s: float = 0.0
    seed: int = 0


@dataclass
class Prediction:  # predictor.hpp:108-112
    throughput_tok_s: float = 0.0
    n_star: int = 0
    g_star: int = 0


@dataclass
class PlacementModel:  # predictor.hpp:104-114
    throughput: ForestModel = field(default_factory=ForestModel)
    n_star: ForestModel = field(default_factory=lambda: ForestModel(target=PredictTarget.NStar))
    g_star: ForestModel = field(default_factory=lambda: ForestModel(target=PredictTarget.GStar))

    def predict(self, features: Sequence[float], dev=None) -> Prediction:
        t, n, g = self.predict_batch(np.asarray([features], dtype=np.float64), dev)[:, 0]
        return Prediction(float(t), int(n), int(g))

    def predict_batch(self, x: np.ndarray, dev=None) -> np.ndarray:
        """(3, n) array: throughput, n*, g* for every row of x, one device call."""
        forests = (self.throughput, self.n_star, self.g_star)
        if len({len(f.trees) for f in forests}) != 1:
            return np.stack([f.predict_batch(x, dev=dev) for f in forests])
        return _predict([t for f in forests for t in f.trees], [int(f.target) for f in forests], x, dev)


# --- device calls -----------------------------------------------------------------

def _dev(dev):
    from .api import device

    return dev or device()


def _check(st: A.lt_status):
    if st.code != A.LT_OK:
        if st.code == A.LT_ERR_DEVICE:
            raise DeviceError(st.message.decode())
        raise ERROR_CLASSES.get(st.code, LoratwinError)(st.message.decode())


def _x(x) -> np.ndarray:
    arr = np.ascontiguousarray(np.asarray([getattr(r, "values", r) for r in x], dtype=np.float64))
    if arr.size == 0:
        return arr.reshape(0, NUM_FEATURES)
    if arr.ndim != 2 or arr.shape[1] != NUM_FEATURES:
        raise ValidationError(f"features: expected rows of {NUM_FEATURES} values")
    return arr


def _tree_params(p: TreeParams) -> A.lt_tree_params:
    t = A.lt_tree_params()
    t.max_depth, t.min_leaf, t.feature_subset = p.max_depth, p.min_leaf, p.feature_subset
    return t


def _trees_of(nodes: np.ndarray, offsets, counts) -> List[DecisionTree]:
    out = []
    for o, c in zip(offsets, counts):
        out.append(DecisionTree([TreeNode(int(n["feature_index"]), float(n["threshold"]), int(n["left"]),
                                          int(n["right"]), float(n["value"]), int(n["coverage"]))
                                 for n in nodes[int(o):int(o) + int(c)]]))
    return out


def _pack_trees(trees: Sequence[DecisionTree]):
    counts = [len(t.nodes) for t in trees]
    offsets = np.zeros(len(trees), dtype=np.int64)
    offsets[1:] = np.cumsum(counts)[:-1]
    nodes = np.zeros(max(sum(counts), 1), dtype=A.TREE_NODE_DT)
    k = 0
    for t in trees:
        for n in t.nodes:
            nodes[k] = (n.feature_index, n.left, n.right, 0, n.threshold, n.value, n.coverage)
            k += 1
    return nodes, offsets


def _predict(trees: Sequence[DecisionTree], tags: Sequence[int], x, dev=None, lib=None, ctx=None) -> np.ndarray:
    if lib is None:
        d = _dev(dev)
        lib, ctx = d.lib, d.ctx
    xs = _x(x)
    nodes, offsets = _pack_trees(trees)
    tg = np.asarray(tags, dtype=np.int32)
    out = np.zeros(max(len(xs) * len(tg), 1), dtype=np.float64)
    st = A.lt_status()
    lib.predict_forests(ctx, nodes.ctypes.data, len(nodes), offsets.ctypes.data, len(trees) // len(tg),
                        tg.ctypes.data, len(tg), xs.ctypes.data if len(xs) else None, len(xs), out.ctypes.data,
                        C.byref(st))
    _check(st)
    return out[:len(xs) * len(tg)].reshape(len(tg), len(xs))


def _node_capacity(n_rows: int, max_depth: int) -> int:
    return max(1, min(2 * n_rows - 1, (1 << min(max_depth + 1, 40)) - 1))


def train_tree(x, y, params: Optional[TreeParams] = None, seed: int = 0, tree_tag: int = 0, dev=None,
               lib=None, ctx=None) -> DecisionTree:
    """predictor.hpp:64-70 (CART regression on the device)."""
    params = params or TreeParams()
    xs = _x(x)
    ys = np.ascontiguousarray(np.asarray(y, dtype=np.float64))
    if len(xs) != len(ys):  # validate_training_input (predictor.cpp:191-197)
        if len(xs) == 0:
            raise ValidationError("training set is empty")
        raise ValidationError(f"training features and targets differ in length ({len(xs)} vs {len(ys)})")
    if lib is None:
        d = _dev(dev)
        lib, ctx = d.lib, d.ctx
    cap = _node_capacity(len(xs), params.max_depth)
    nodes = np.zeros(cap, dtype=A.TREE_NODE_DT)
    cnt = np.zeros(1, dtype=np.int32)
    st = A.lt_status()
    lib.train_tree(ctx, xs.ctypes.data if len(xs) else None, len(xs), ys.ctypes.data if len(ys) else None,
                   C.byref(_tree_params(params)), seed, tree_tag, nodes.ctypes.data, cap, cnt.ctypes.data,
                   C.byref(st))
    _check(st)
    return _trees_of(nodes, [0], cnt)[0]


def _train_forests(xs: np.ndarray, ys: List[np.ndarray], targets: List[PredictTarget], params: ForestParams,
                   seed: int, dev=None, lib=None, ctx=None) -> List[ForestModel]:
    if lib is None:
        d = _dev(dev)
        lib, ctx = d.lib, d.ctx
    y = np.ascontiguousarray(np.stack(ys)) if len(xs) else np.zeros((len(ys), 0))
    tags = np.asarray([int(t) for t in targets], dtype=np.int32)
    n_trees = max(params.n_trees, 0)
    cap = max(1, len(targets) * n_trees * _node_capacity(len(xs), params.tree.max_depth))
    nodes = np.zeros(cap, dtype=A.TREE_NODE_DT)
    off = np.zeros(max(len(targets) * n_trees, 1), dtype=np.int64)
    cnt = np.zeros(max(len(targets) * n_trees, 1), dtype=np.int32)
    fp = A.lt_forest_params()
    fp.n_trees, fp.bootstrap, fp.tree = params.n_trees, int(params.bootstrap), _tree_params(params.tree)
    st = A.lt_status()
    lib.train_forests(ctx, xs.ctypes.data if len(xs) else None, len(xs), y.ctypes.data if len(xs) else None,
                      tags.ctypes.data, len(tags), C.byref(fp), seed, nodes.ctypes.data, cap, off.ctypes.data,
                      cnt.ctypes.data, C.byref(st))
    _check(st)
    trees = _trees_of(nodes, off, cnt)
    return [ForestModel(target=t, params=params, trees=trees[g * n_trees:(g + 1) * n_trees], seed=seed,
                        trained_rows=len(xs)) for g, t in enumerate(targets)]


def train_forest(x, y, target: PredictTarget, params: Optional[ForestParams] = None, seed: int = 0,
                 dev=None, lib=None, ctx=None) -> ForestModel:
    """predictor.hpp:98-99."""
    params = params or ForestParams()
    xs = _x(x)
    ys = np.asarray(y, dtype=np.float64)
    if len(xs) != len(ys) and len(xs):
        raise ValidationError(f"training features and targets differ in length ({len(xs)} vs {len(ys)})")
    return _train_forests(xs, [ys], [PredictTarget(target)], params, seed, dev, lib, ctx)[0]


def train_placement_model(rows, params: Optional[ForestParams] = None, seed: int = 0,
                          exclude_starved: bool = True, dev=None, lib=None, ctx=None) -> PlacementModel:
    """predictor.hpp:116-118 / predictor.cpp:250-269: three forests (throughput,
    n*, g*) over the same rows, grown together in one device call. `rows`
    are DatasetRow-like objects (features, max_throughput_tok_s, n_star,
    g_star, all_starved)."""
    params = params or ForestParams()
    keep = [r for r in rows if not (exclude_starved and r.all_starved)]
    if not keep:
        raise ValidationError("no trainable rows (every dataset row is marked all-starved)")
    xs = _x([r.features for r in keep])
    ys = [np.asarray([r.max_throughput_tok_s for r in keep], dtype=np.float64),
          np.asarray([float(r.n_star) for r in keep], dtype=np.float64),
          np.asarray([float(r.g_star) for r in keep], dtype=np.float64)]
    f = _train_forests(xs, ys, [PredictTarget.Throughput, PredictTarget.NStar, PredictTarget.GStar], params, seed,
                       dev, lib, ctx)
    return PlacementModel(throughput=f[0], n_star=f[1], g_star=f[2])
