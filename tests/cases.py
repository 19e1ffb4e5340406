"""Hand-built and randomized inputs shared by the oracle pins and the GPU parity tests.

Inputs only (no method arithmetic): instances, requests, deadlines and special ensembles.
"""
from __future__ import annotations

import json
import os

import numpy as np

from paper_2408_05235_b200 import workload as W

HERE = os.path.dirname(os.path.abspath(__file__))


def load_w1():
    with open(os.path.join(HERE, "golden", "w1.json")) as f:
        return json.load(f)


def ensemble_from_nodes(nodes, base=0.0, max_depth=None):
    ns = [W.Node(n["feature"], float(np.float32(n.get("threshold", 0.0))), n.get("left", -1), n.get("right", -1),
                 float(np.float32(n.get("leaf", 0.0)))) for n in nodes]
    if max_depth is None:
        max_depth = _depth(ns)
    return W.Ensemble([ns], float(np.float32(base)), max_depth)


def _depth(nodes, i=0):
    nd = nodes[i]
    return 0 if nd.feature == -1 else 1 + max(_depth(nodes, nd.left), _depth(nodes, nd.right))


def ensemble_depth(ens):
    return max([_depth(t) for t in ens.trees], default=0)


def make_instances(specs, H):
    """specs: list of dict(inst fields..., running=[(a,q,r,flags,dead)], queued=[(q,r,flags,dead)])."""
    inst = np.zeros(len(specs), dtype=W.INST_DTYPE)
    reqs, deads = [], []
    for i, s in enumerate(specs):
        inst[i]["k"] = s.get("k", 1000)
        inst[i]["t_cur"] = s.get("t_cur", 0.0)
        inst[i]["req_begin"] = len(reqs)
        inst[i]["n_run"] = len(s.get("running", []))
        inst[i]["n_queue"] = len(s.get("queued", []))
        inst[i]["N"] = s.get("N", 16)
        inst[i]["kv_cap"] = s.get("kv_cap", 1 << 20)
        inst[i]["max_batch"] = s.get("max_batch", 1 << 20)
        inst[i]["tp"] = s.get("tp", 1)
        for (a, q, r, fl, d) in s.get("running", []):
            reqs.append((a, q, r, fl)); deads.append(d)
        for (q, r, fl, d) in s.get("queued", []):
            reqs.append((0, q, r, fl)); deads.append(d)
    req = np.array(reqs, dtype=W.REQ_DTYPE) if reqs else np.zeros(0, W.REQ_DTYPE)
    return inst, req, np.array(deads, dtype=np.float64)


def w1_inputs(case):
    w = load_w1()
    I = w["instance"]
    lost = set(case.get("lost", []))
    dead = case["dead"]
    running = [(r["a"], r["q"], r["r"], 1 if r["name"] in lost else 0, dead.get(r["name"], 1e9)) for r in w["running"]]
    queued = [(r["q"], r["r"], 1 if r["name"] in lost else 0, dead.get(r["name"], 1e9)) for r in w["queued"]]
    inst, req, td = make_instances([dict(k=I["k"], t_cur=I["t_cur"], N=I["N"], kv_cap=I["kv_cap"],
                                         max_batch=I["max_batch"], tp=I["tp"], running=running, queued=queued)], w["H"])
    ens = ensemble_from_nodes(w["model"]["nodes"], w["model"]["base"], w["model"]["max_depth"])
    return ens, inst, req, td, w["H"], np.array(w["freq"], dtype=np.float32), np.float32(case["tbt"])


def random_tiny_case(rng, H=None, F=None, n_trees=None, depth=None, n_inst=6, allow_bad=True):
    """Small random instances + a small random ensemble (brute-force scale)."""
    H = H or int(rng.integers(1, 9))
    F = F or int(rng.integers(1, 5))
    freq = np.sort(rng.choice(np.arange(40, 140) * 15.0, size=F, replace=False)).astype(np.float32)
    specs = []
    for _ in range(n_inst):
        N = int(rng.choice([1, 2, 3, 16]))
        run = []
        for _ in range(int(rng.integers(0, 5))):
            r = int(rng.integers(1, H + 3))
            a = int(rng.integers(0, r))
            if r - a > H:
                a = r - H
            run.append((a, int(rng.integers(1, 40)), r, int(rng.random() < 0.08), 0.0))
        que = [(int(rng.integers(1, 40)), int(rng.integers(1, H + 1)), 0, 0.0) for _ in range(int(rng.integers(0, 4)))]
        if allow_bad and rng.random() < 0.1 and run:
            a, q, r, fl, d = run[0]
            run[0] = (a, q, r + H + 1, fl, d)        # l > H -> BAD_INPUT
        kv_total = sum(-(-(q + r) // N) for (a, q, r, fl, d) in run)
        specs.append(dict(N=N, tp=int(rng.choice([1, 2, 4, 8])), kv_cap=int(kv_total * rng.uniform(0.6, 1.6)) + 1,
                          max_batch=int(rng.integers(0, 8)), t_cur=float(rng.uniform(0, 100)),
                          running=run, queued=que))
    inst, req, td = make_instances(specs, H)
    ens = W.gen_ensemble(n_trees or int(rng.integers(1, 6)), depth or int(rng.integers(1, 5)),
                         int(rng.integers(1 << 30)), freq, b_max=8, kv_max=60, ragged=True, base=0.25, noise=0.3)
    # deadlines around the surrogate time so that decisions vary
    tau = 1.0 / 40.0
    for i in range(len(inst)):
        b = int(inst[i]["req_begin"])
        for e in range(int(inst[i]["n_run"]) + int(inst[i]["n_queue"])):
            l = int(req[b + e]["r"]) - int(req[b + e]["a"])
            td[b + e] = inst[i]["t_cur"] + l * tau * rng.uniform(0.3, 3.0)
    tbt = np.float32(rng.choice([0.2, 0.05, 0.02, 0.01]))
    return ens, inst, req, td, H, freq, tbt


def subset_inputs(inputs, idx):
    """The instances ``idx`` of a round's inputs as a self-contained round (request rows copied,
    req_begin rebased).  Input plumbing only."""
    inst = inputs["inst"][idx].copy()
    reqs, deads, off = [], [], 0
    for k, i in enumerate(idx):
        b = int(inputs["inst"][i]["req_begin"])
        e = b + int(inputs["inst"][i]["n_run"]) + int(inputs["inst"][i]["n_queue"])
        reqs.append(inputs["req"][b:e])
        deads.append(inputs["t_dead"][b:e])
        inst[k]["req_begin"] = off
        off += e - b
    req = np.concatenate(reqs) if reqs else np.zeros(0, W.REQ_DTYPE)
    td = np.concatenate(deads) if deads else np.zeros(0)
    return dict(inputs, inst=inst, req=req, t_dead=td)
