"""Pins of the oracle's full admission control (PAPER §4.3.2):
checks 1-3 at the maximum frequency for each queued request in FIFO order, "lost" marking when
only the candidate's own deadline fails."""
from __future__ import annotations

import numpy as np
import pytest

import cases
import refimpl
from paper_2408_05235_b200 import workload as W


def w1(oracle_mod, dead, tbt=0.05, lost=()):
    d = {"case": "x", "dead": dead, "tbt": tbt, "lost": list(lost)}
    ens, inst, req, td, H, freq, tbt = cases.w1_inputs(d)
    m = oracle_mod.Model(W.write_blob(ens))
    return oracle_mod.decide(m, inst, req, td, H, freq, tbt, want_grid=False, admission=1)


def test_w1_admitted_normally(oracle_mod):
    """Q1 passes checks 1-3 at 1600 MHz (T_R = [1/64, 2/64, 5/128, 6/128, 7/128] s); Q2 fails check 1."""
    out = w1(oracle_mod, {"R1": 0.2, "R2": 0.2, "Q1": 1.0})
    assert out["n_adm"][0] == 1 and out["adm_lost"][0] == 0
    assert out["level"][0] == 1 and out["status"][0] == refimpl.ST_QUEUE_BLOCKED


def test_w1_admitted_as_lost(oracle_mod):
    """Q1's own deadline 0.03 < T_R[3] = 5/128 at f_max, the others hold: scheduled but "lost"
    (P:529), so the throttle is bypassed to the maximum frequency."""
    out = w1(oracle_mod, {"R1": 0.2, "R2": 0.2, "Q1": 0.03})
    assert out["n_adm"][0] == 1 and out["adm_lost"][0] == 1
    assert out["level"][0] == 1 and out["status"][0] == refimpl.ST_QUEUE_BLOCKED | refimpl.ST_BYPASS_LOST


def test_w1_candidate_would_break_others(oracle_mod):
    """With Q1 R2 would finish at 7/128 = 0.0547 s > 0.05 even at f_max: Q1 is queued (check 3).
    Without Q1 the batch is smaller (B = [2,2,1,1,1] -> 128 IPS at 1600 MHz, T_R[5] = 5/128 < 0.05)."""
    out = w1(oracle_mod, {"R1": 0.2, "R2": 0.05, "Q1": 1.0})
    assert out["n_adm"][0] == 0 and out["status"][0] == refimpl.ST_QUEUE_BLOCKED
    assert out["level"][0] == 1
    # the check-1-only gate (reading A-2) admits Q1 and then nothing passes
    ens, inst, req, td, H, freq, tbt = cases.w1_inputs({"case": "x", "dead": {"R1": 0.2, "R2": 0.05, "Q1": 1.0},
                                                        "tbt": 0.05})
    g = oracle_mod.decide(oracle_mod.Model(W.write_blob(ens)), inst, req, td, H, freq, tbt, want_grid=False)
    assert g["n_adm"][0] == 1 and g["status"][0] & refimpl.ST_INFEASIBLE


def test_w1_tbt_check(oracle_mod):
    """Check 2: mean T' at f_max with Q1 = 7/640 s; a TBT SLO below it queues Q1."""
    out = w1(oracle_mod, {"R1": 0.2, "R2": 0.2, "Q1": 1.0}, tbt=0.0109)
    assert out["n_adm"][0] == 0


def test_admission_brute_force_tiny(oracle_mod):
    rng = np.random.default_rng(17)
    n = 0
    for trial in range(60):
        ens, inst, req, td, H, freq, tbt = cases.random_tiny_case(rng)
        out = oracle_mod.decide(oracle_mod.Model(W.write_blob(ens)), inst, req, td, H, freq, tbt, want_grid=False,
                                admission=1)
        box = refimpl.BoxModel(ens)
        for i in range(len(inst)):
            b = int(inst[i]["req_begin"]); e = b + int(inst[i]["n_run"]) + int(inst[i]["n_queue"])
            ref = refimpl.brute_decide(box, inst[i], req[b:e], td[b:e], H, freq, tbt, admission=1)
            got = dict(level=int(out["level"][i]), status=int(out["status"][i]), n=int(out["n"][i]),
                       n_adm=int(out["n_adm"][i]), adm_lost=int(out["adm_lost"][i]))
            assert got == {k: ref[k] for k in got}, (trial, i)
            n += 1
    assert n >= 300


@pytest.mark.parametrize("name", ["P1", "P2"])
def test_admission_admits_a_prefix_of_the_gate(oracle_mod, name):
    """Checks 2-3 only add conditions to check 1: the admitted prefix never grows."""
    cfg = W.CONFIGS[name]
    blob = W.write_blob(W.config_ensemble(cfg))
    d = W.config_inputs(cfg)
    m = oracle_mod.Model(blob)
    a0 = oracle_mod.decide(m, d["inst"], d["req"], d["t_dead"], d["H"], d["freq"], d["tbt_slo"], want_grid=False)
    a1 = oracle_mod.decide(m, d["inst"], d["req"], d["t_dead"], d["H"], d["freq"], d["tbt_slo"], want_grid=False,
                           admission=1, threads=4)
    assert (a1["n_adm"] <= a0["n_adm"]).all()
    assert (a1["n_adm"] < a0["n_adm"]).any()        # the SLO checks do bind on these workloads
    same = (a1["n_adm"] == a0["n_adm"]) & (a1["adm_lost"] == 0)
    assert np.array_equal(a1["level"][same], a0["level"][same])
