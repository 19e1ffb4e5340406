"""Importers for trained tree ensembles -> blob v1 (include/tp.h), the input of tp_gbdt_load.

The paper's performance model M is "a Gradient Boosted Decision Tree" in the XGBoost family
(§4.3.1) over [engine size, batch, KV usage, GPU frequency].  Its trained
weights are not published, so these importers let a user bring their own model:

* ``from_xgboost_json``  -- an XGBoost ``Booster.save_model("*.json")`` document (reg:squarederror):
  split ``x < split_condition`` -> left (the blob's rule), leaf value = ``split_conditions[leaf]``,
  prediction = ``base_score`` + sum of leaves.
* ``from_sklearn``       -- scikit-learn ``GradientBoostingRegressor`` /
  ``HistGradientBoostingRegressor``.  scikit-learn splits ``x <= threshold`` (x cast to float32);
  for every float32 x that is ``x < t'`` with t' = the float32 successor of the largest float32
  <= threshold, so thresholds are converted exactly.  Leaf values become float32 (scikit-learn sums
  in float64, so predictions agree to ~1e-7 relative, not bit for bit).

Feature order must be [tp, batch, kv_blocks, freq_mhz] (the blob's fixed order).  Host-side model
plumbing only: nothing here evaluates a model.
"""
from __future__ import annotations

import json

import numpy as np

from .workload import Ensemble, Node, write_blob

N_FEATURES = 4


def _depth(nodes, i=0):
    nd = nodes[i]
    return 0 if nd.feature == -1 else 1 + max(_depth(nodes, nd.left), _depth(nodes, nd.right))


def _ensemble(trees, base):
    return Ensemble(trees, float(np.float32(base)), max([_depth(t) for t in trees], default=0))


def _f32(x) -> float:
    v = np.float32(x)
    if not np.isfinite(v):
        raise ValueError(f"non-finite value {x!r}")
    return float(v)


def _le_to_lt(t: float) -> float:
    """float32 t' with (x < t') == (x <= t) for every float32 x (t a float64 threshold)."""
    f = np.float32(t)
    if float(f) > t:
        f = np.nextafter(f, np.float32(-np.inf))
    return float(np.nextafter(f, np.float32(np.inf)))


def _parse_base_score(v) -> float:
    if isinstance(v, (int, float)):
        return float(v)
    s = str(v).strip().strip("[]")
    return float(s.split(",")[0])


def from_xgboost_json(doc) -> Ensemble:
    """``doc``: a path, a JSON string or the parsed dict of an XGBoost JSON model."""
    if isinstance(doc, (bytes, str)) and not str(doc).lstrip().startswith("{"):
        with open(doc) as f:
            doc = json.load(f)
    elif isinstance(doc, (bytes, str)):
        doc = json.loads(doc)
    learner = doc["learner"]
    obj = learner.get("objective", {}).get("name", "reg:squarederror")
    if obj not in ("reg:squarederror", "reg:linear"):
        raise ValueError(f"unsupported objective {obj!r} (identity link required)")
    nf = int(learner["learner_model_param"].get("num_feature", N_FEATURES))
    if nf != N_FEATURES:
        raise ValueError(f"model has {nf} features, expected {N_FEATURES} [tp, batch, kv, freq]")
    base = _parse_base_score(learner["learner_model_param"].get("base_score", 0.5))
    gb = learner["gradient_booster"]
    model = gb["model"] if "model" in gb else gb["gbtree"]["model"]
    trees = []
    for t in model["trees"]:
        left, right = t["left_children"], t["right_children"]
        feat, cond = t["split_indices"], t["split_conditions"]
        nodes = []
        for i in range(len(left)):
            if left[i] == -1:
                nodes.append(Node(-1, leaf=_f32(cond[i])))
            else:
                if int(feat[i]) >= N_FEATURES:
                    raise ValueError("split on a feature index >= 4")
                nodes.append(Node(int(feat[i]), _f32(cond[i]), int(left[i]), int(right[i])))
        trees.append(nodes)
    return _ensemble(trees, base)


def from_sklearn(est) -> Ensemble:
    """GradientBoostingRegressor (squared error) or HistGradientBoostingRegressor."""
    name = type(est).__name__
    if name == "GradientBoostingRegressor":
        if est.init_ is None or not hasattr(est.init_, "constant_"):
            raise ValueError("needs the default mean init estimator")
        base = float(np.asarray(est.init_.constant_).ravel()[0])
        lr = float(est.learning_rate)
        trees = []
        for row in est.estimators_:
            tr = row[0].tree_
            nodes = []
            for i in range(tr.node_count):
                if tr.children_left[i] == -1:
                    nodes.append(Node(-1, leaf=_f32(lr * float(tr.value[i].ravel()[0]))))
                else:
                    nodes.append(Node(int(tr.feature[i]), _le_to_lt(float(tr.threshold[i])),
                                      int(tr.children_left[i]), int(tr.children_right[i])))
            trees.append(nodes)
        return _ensemble(trees, base)
    if name == "HistGradientBoostingRegressor":
        base = float(np.asarray(est._baseline_prediction).ravel()[0])
        trees = []
        for group in est._predictors:
            pred = group[0]
            nd = pred.nodes
            nodes = []
            for i in range(len(nd)):
                if nd["is_leaf"][i]:
                    nodes.append(Node(-1, leaf=_f32(nd["value"][i])))
                else:
                    if nd["is_categorical"][i]:
                        raise ValueError("categorical splits are not supported")
                    nodes.append(Node(int(nd["feature_idx"][i]), _le_to_lt(float(nd["num_threshold"][i])),
                                      int(nd["left"][i]), int(nd["right"][i])))
            trees.append(nodes)
        return _ensemble(trees, base)
    raise TypeError(f"unsupported estimator {name}")


def to_blob(ens: Ensemble) -> bytes:
    return write_blob(ens)
