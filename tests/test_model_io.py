"""Model importers: XGBoost JSON and scikit-learn ensembles -> blob v1.
CPU: the oracle evaluates the imported blob; it must reproduce the source model's predictions."""
from __future__ import annotations

import json

import numpy as np
import pytest

from paper_2408_05235_b200 import model_io, workload as W

XGB_DOC = {
    "learner": {
        "learner_model_param": {"base_score": "5E-1", "num_feature": "4", "num_class": "0"},
        "objective": {"name": "reg:squarederror"},
        "gradient_booster": {"name": "gbtree", "model": {"trees": [
            {"left_children": [1, -1, -1], "right_children": [2, -1, -1], "split_indices": [3, 0, 0],
             "split_conditions": [1000.0, 10.0, 20.0]},
            {"left_children": [1, 3, -1, -1, -1], "right_children": [2, 4, -1, -1, -1],
             "split_indices": [1, 2, 0, 0, 0], "split_conditions": [8.0, 100.5, 1.25, 0.5, 2.0]},
        ]}}}}


def test_xgboost_json_import(oracle_mod):
    ens = model_io.from_xgboost_json(json.dumps(XGB_DOC))
    assert ens.max_depth == 2 and len(ens.trees) == 2 and ens.base == 0.5
    m = oracle_mod.Model(model_io.to_blob(ens))
    # tree 1: f < 1000 -> 10 else 20; tree 2: B < 8 ? (KV < 100.5 ? 0.5 : 2.0) : 1.25
    assert m.predict_raw(1, 4, 50, 900) == np.float32(0.5 + 10 + 0.5)
    assert m.predict_raw(1, 4, 101, 1000) == np.float32(0.5 + 20 + 2.0)   # f == 1000 goes right
    assert m.predict_raw(1, 8, 0, 999) == np.float32(0.5 + 10 + 1.25)     # B == 8 goes right


def test_xgboost_rejects_other_objectives():
    doc = json.loads(json.dumps(XGB_DOC))
    doc["learner"]["objective"]["name"] = "binary:logistic"
    with pytest.raises(ValueError):
        model_io.from_xgboost_json(doc)


def _profiling_data(rng, n):
    """Samples shaped like the paper's profiling sweep: TP level, batch size, KV usage,
    random frequency in 15 MHz steps; IPS from the generator's surrogate with noise."""
    tp = rng.choice([1, 2, 4, 8], n)
    B = rng.integers(1, 65, n)
    KV = (B * rng.uniform(5, 30, n)).astype(int)
    f = rng.choice(np.arange(600, 1966, 15), n)
    X = np.stack([tp, B, KV, f], 1).astype(np.float32)
    y = W.surrogate_ips(tp, B, KV, f) * (1 + 0.03 * rng.standard_normal(n))
    return X, y


@pytest.mark.parametrize("kind", ["gbr", "hgb"])
def test_sklearn_import_matches_predict(oracle_mod, kind):
    from sklearn.ensemble import GradientBoostingRegressor, HistGradientBoostingRegressor
    rng = np.random.default_rng(0)
    X, y = _profiling_data(rng, 3000)
    est = (GradientBoostingRegressor(n_estimators=40, max_depth=4, random_state=0) if kind == "gbr"
           else HistGradientBoostingRegressor(max_iter=40, max_depth=5, random_state=0)).fit(X, y)
    ens = model_io.from_sklearn(est)
    m = oracle_mod.Model(model_io.to_blob(ens))
    Xt, _ = _profiling_data(rng, 400)
    # points exactly on split thresholds exercise the <= -> < conversion
    thr = [nd.threshold for t in ens.trees for nd in t if nd.feature >= 0][:200]
    feats = [nd.feature for t in ens.trees for nd in t if nd.feature >= 0][:200]
    edge = np.repeat(Xt[:1], len(thr), 0)
    for k, (f, t) in enumerate(zip(feats, thr)):
        edge[k, f] = np.nextafter(np.float32(t), np.float32(-np.inf))   # the largest x <= sklearn threshold
    Xall = np.concatenate([Xt, edge]).astype(np.float32)
    ref = est.predict(Xall)
    got = np.array([m.predict_raw(*x) for x in Xall], dtype=np.float64)
    assert np.allclose(got, ref, rtol=2e-6, atol=1e-5)
