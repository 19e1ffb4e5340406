"""Pins of the CPU oracle against things other than itself (CPU only, no GPU).

Each test names the passage of PAPER.md (P:line) or SPEC.md (S:line) it checks.
"""
from __future__ import annotations

import dataclasses
from fractions import Fraction

import numpy as np
import pytest

import cases
import refimpl
from paper_2408_05235_b200 import workload as W


def run(oracle_mod, ens, inst, req, td, H, freq, tbt, **kw):
    m = oracle_mod.Model(W.write_blob(ens))
    return oracle_mod.decide(m, inst, req, td, H, freq, tbt, **kw)


# ------------------------------------------------------------------ W1 golden example (hand-derived)

def test_w1_projection(oracle_mod):
    w = cases.load_w1()
    ens, inst, req, td, H, freq, tbt = cases.w1_inputs(w["decisions"][0])
    out = run(oracle_mod, ens, inst, req, td, H, freq, tbt, want_tr=True)
    exp = w["expected_projection"]
    assert out["B"][0].tolist() == exp["B"]
    assert out["KV"][0].tolist() == exp["KV"]
    assert int(out["n"][0]) == exp["n"] and int(out["n_adm"][0]) == exp["n_adm"]
    g = w["expected_grid"]
    assert out["ips"][0, 0, :5].tolist() == g["ips_800"]
    assert out["ips"][0, 1, :5].tolist() == g["ips_1600"]
    assert out["tr"][0, 0, :5].tolist() == g["TR_800_ticks"]
    assert [t * 2.0 ** -40 for t in out["tr"][0, 0, :5]] == g["TR_800_s"]
    assert [t * 2.0 ** -40 for t in out["tr"][0, 1, :5]] == g["TR_1600_s"]
    assert out["tr"][0, 0, 4] * 2.0 ** -40 / 5 == g["mean_TBT_800"]


def test_w1_running_only(oracle_mod):
    """Same instance with the queue removed -> the running-only curves (Eq. 2)."""
    w = cases.load_w1()
    ens, inst, req, td, H, freq, tbt = cases.w1_inputs(w["decisions"][0])
    inst = inst.copy()
    inst["n_queue"] = 0
    out = run(oracle_mod, ens, inst, req, td, H, freq, tbt)
    assert out["B"][0].tolist() == w["expected_projection"]["running_only_B"]
    assert out["KV"][0].tolist() == w["expected_projection"]["running_only_KV"]


@pytest.mark.parametrize("case", [d["case"] for d in cases.load_w1()["decisions"]])
def test_w1_decisions(oracle_mod, case):
    d = [x for x in cases.load_w1()["decisions"] if x["case"] == case][0]
    ens, inst, req, td, H, freq, tbt = cases.w1_inputs(d)
    out = run(oracle_mod, ens, inst, req, td, H, freq, tbt, want_grid=False)
    assert int(out["level"][0]) == d["level"]
    assert int(out["status"][0]) == d["status"]


# ------------------------------------------------------------------ SPEC examples (Eq. 1 direct)

def test_spec_per_query_kv(oracle_mod):
    """q=1, r=1024, N=64 -> 1 block at j=s_i, 16 at j=s_i+1023, 0 at s_i+r."""
    ens = cases.ensemble_from_nodes([{"feature": -1, "leaf": 64.0}])
    inst, req, td = cases.make_instances([dict(N=64, running=[(0, 1, 1024, 0, 1e9)])], 1025)
    out = run(oracle_mod, ens, inst, req, td, 1025, np.array([1000.0], np.float32), 1.0, want_grid=False)
    assert out["KV"][0, 0] == 1 and out["KV"][0, 1023] == 16 and out["KV"][0, 1024] == 0
    assert out["B"][0, 1023] == 1 and out["B"][0, 1024] == 0


def test_spec_project_example_rederived(oracle_mod):
    """S:234 (q=1, r=4, N=2, s_i=k) re-derived under reading A-1: B=[1,1,1,1], KV=[1,1,2,2]."""
    ens = cases.ensemble_from_nodes([{"feature": -1, "leaf": 64.0}])
    inst, req, td = cases.make_instances([dict(N=2, running=[(0, 1, 4, 0, 1e9)])], 6)
    out = run(oracle_mod, ens, inst, req, td, 6, np.array([1000.0], np.float32), 1.0, want_grid=False)
    assert out["B"][0].tolist() == [1, 1, 1, 1, 0, 0]
    assert out["KV"][0].tolist() == [1, 1, 2, 2, 0, 0]
    assert out["n"][0] == 4


def test_empty_scoreboard(oracle_mod):
    """empty scoreboard -> n = 0; reading A-15: level 0 + EMPTY."""
    ens = cases.ensemble_from_nodes([{"feature": -1, "leaf": 64.0}])
    inst, req, td = cases.make_instances([dict(N=2)], 4)
    out = run(oracle_mod, ens, inst, req, td, 4, np.array([900.0, 1000.0], np.float32), 1.0)
    assert out["n"][0] == 0 and out["level"][0] == 0 and out["status"][0] == refimpl.ST_EMPTY
    assert out["B"][0].tolist() == [0] * 4


# ------------------------------------------------------------------ token-by-token allocator

def test_projection_equals_token_allocator(oracle_mod, rng):
    """>=1000 random scoreboards, N in {1,2,16,64,128}: Eq. 1-2 == brute-force allocator."""
    ens = cases.ensemble_from_nodes([{"feature": -1, "leaf": 64.0}])
    checked = 0
    for N in [1, 2, 16, 64, 128]:
        specs = []
        H = 40
        for _ in range(220):
            run_ = []
            for _ in range(int(rng.integers(0, 7))):
                r = int(rng.integers(1, 60)); a = int(rng.integers(max(0, r - H), r))
                run_.append((a, int(rng.integers(1, 300)), r, 0, 1e9))
            specs.append(dict(N=N, running=run_))
        inst, req, td = cases.make_instances(specs, H)
        out = run(oracle_mod, ens, inst, req, td, H, np.array([1000.0], np.float32), 16.0, want_grid=False)
        for i, s in enumerate(specs):
            B = np.zeros(H, np.int64); KV = np.zeros(H, np.int64)
            for (a, q, r, fl, d) in s["running"]:
                cur = np.array(refimpl.token_alloc_curve(a, q, r, N, H))
                KV += cur; B += cur > 0
            assert out["B"][i].tolist() == B.tolist()
            assert out["KV"][i].tolist() == KV.tolist()
            checked += 1
    assert checked >= 1000


# ------------------------------------------------------------------ projection invariants

@pytest.mark.parametrize("name", ["P1", "P2"])
def test_projection_invariants(oracle_mod, name):
    cfg = W.CONFIGS[name]
    ens = W.config_ensemble(cfg)
    d = W.config_inputs(cfg)
    out = run(oracle_mod, ens, d["inst"], d["req"], d["t_dead"], d["H"], d["freq"], d["tbt_slo"], want_grid=False, threads=4)
    for i, ins in enumerate(d["inst"]):
        st, n = int(out["status"][i]), int(out["n"][i])
        if st & refimpl.ST_BAD_INPUT:
            continue
        B, KV = out["B"][i].astype(np.int64), out["KV"][i].astype(np.int64)
        assert (np.diff(B) <= 0).all(), "B non-increasing (no arrivals after k)"
        assert (KV >= B).all(), "every active request holds >= 1 block"
        assert (B[n:] == 0).all() and (KV[n:] == 0).all()
        if n > 0:
            assert B[n - 1] >= 1
        if not st & refimpl.ST_KV_OVER:
            assert KV.max(initial=0) <= ins["kv_cap"]
        assert 0 <= out["n_adm"][i] <= ins["n_queue"]
        assert bool(st & refimpl.ST_QUEUE_BLOCKED) == (out["n_adm"][i] < ins["n_queue"])
        assert B[0] == ins["n_run"] + out["n_adm"][i] or n == 0


# ------------------------------------------------------------------ tree ensemble

def test_stump_closed_form(oracle_mod):
    """A single stump on KV: ips = base + (KV < 10.5 ? 7 : 3)."""
    ens = cases.ensemble_from_nodes([{"feature": 2, "threshold": 10.5, "left": 1, "right": 2},
                                     {"feature": -1, "leaf": 7.0}, {"feature": -1, "leaf": 3.0}], base=1.0)
    m = oracle_mod.Model(W.write_blob(ens))
    assert m.predict_raw(1, 1, 10, 900) == np.float32(8.0)
    assert m.predict_raw(1, 1, 11, 900) == np.float32(4.0)


def test_split_is_strict_less(oracle_mod):
    """x < thr goes left, x == thr goes right (XGBoost convention, reading A-7)."""
    ens = cases.ensemble_from_nodes([{"feature": 1, "threshold": 4.0, "left": 1, "right": 2},
                                     {"feature": -1, "leaf": 1.0}, {"feature": -1, "leaf": 2.0}])
    m = oracle_mod.Model(W.write_blob(ens))
    assert m.predict_raw(1, 3, 0, 900) == 1.0
    assert m.predict_raw(1, 4, 0, 900) == 2.0


def _leaf_index_ensemble(rng, n_trees, depth):
    """Trees whose leaves are distinct powers of two: the fp32 sum identifies every leaf hit."""
    trees = []
    p = 0
    for _ in range(n_trees):
        nodes = []

        def build(d):
            nonlocal p
            idx = len(nodes)
            nodes.append(W.Node(-1))
            if d < depth:
                f = int(rng.integers(0, 4))
                thr = [float(rng.choice([1.5, 2, 4, 6])), float(rng.integers(0, 12)) + rng.choice([0, 0.5]),
                       float(rng.integers(0, 50)) + rng.choice([0, 0.5]), float(rng.choice([900, 1000, 1050]))][f]
                nodes[idx] = W.Node(f, float(np.float32(thr)))
                nodes[idx].left = build(d + 1)
                nodes[idx].right = build(d + 1)
            else:
                nodes[idx].leaf = float(2.0 ** (p % 24 - 6)) if n_trees * 2 ** depth <= 24 else float(2.0 ** (p - 6))
                p += 1
            return idx
        build(0)
        trees.append(nodes)
    return W.Ensemble(trees, 0.0, depth)


def test_leaf_index_trees_match_box_membership(oracle_mod, rng):
    ens = _leaf_index_ensemble(rng, 3, 3)       # 24 leaves -> 2^-6 .. 2^17, sums exact in fp32
    m = oracle_mod.Model(W.write_blob(ens))
    box = refimpl.BoxModel(ens)
    X = np.stack([rng.choice([1, 2, 4, 8], 400), rng.integers(0, 13, 400), rng.integers(0, 52, 400),
                  rng.choice([899, 900, 1000, 1050, 1200], 400)], 1).astype(np.float32)
    ref = box.raw(X)
    got = np.array([m.predict_raw(*x) for x in X], dtype=np.float32)
    assert (got == ref).all()


@pytest.mark.parametrize("ragged", [False, True])
def test_random_ensembles_match_box_membership(oracle_mod, rng, ragged):
    """Random ensembles: recursive walk (oracle) == box membership (test), bit-exact fp32 sums."""
    freq = W.freq_levels(8)
    ens = W.gen_ensemble(40, 6, 99 + ragged, freq, b_max=64, kv_max=900, ragged=ragged)
    m = oracle_mod.Model(W.write_blob(ens))
    box = refimpl.BoxModel(ens)
    X = np.stack([rng.choice([1, 2, 4, 8], 300), rng.integers(0, 70, 300), rng.integers(0, 950, 300),
                  rng.choice(freq, 300)], 1).astype(np.float32)
    got = np.array([m.predict_raw(*x) for x in X], dtype=np.float32)
    assert (got == box.raw(X)).all()


def test_constant_ensemble_and_exact_cumsum(oracle_mod):
    """All leaves 0, base 2^5 -> ips = 32 everywhere; T_R[l] = l / 32 exactly (Eq. 3)."""
    ens = W.Ensemble([[W.Node(1, 3.0, 1, 2), W.Node(-1, leaf=0.0), W.Node(-1, leaf=0.0)]] * 3, 32.0, 1)
    inst, req, td = cases.make_instances([dict(N=16, running=[(0, 5, 100, 0, 1e9), (3, 5, 50, 0, 1e9)])], 100)
    out = run(oracle_mod, ens, inst, req, td, 100, np.array([1000.0], np.float32), 1.0, want_tr=True)
    assert (out["ips"][0, 0, :100] == 32.0).all()
    assert out["tr"][0, 0, :100].tolist() == [l * 2 ** 35 for l in range(1, 101)]


def test_cumsum_equals_fraction_sum(oracle_mod):
    """Eq. 3 exactly: the oracle's ticks equal the exact rational sum of fl32(1/ips)."""
    cfg = W.CONFIGS["P1"]
    ens = W.config_ensemble(cfg)
    d = W.config_inputs(cfg, 0, 12)
    out = run(oracle_mod, ens, d["inst"], d["req"], d["t_dead"], d["H"], d["freq"], d["tbt_slo"], want_tr=True)
    checked = 0
    for i in range(12):
        n = int(out["n"][i])
        if out["status"][i] & (refimpl.ST_BAD_INPUT | refimpl.ST_EMPTY | refimpl.ST_BYPASS_LOST):
            continue
        for u in range(len(d["freq"])):
            s = Fraction(0)
            for mm in range(n):
                s += Fraction(float(np.float32(1.0) / out["ips"][i, u, mm]))
                assert s * 2 ** 40 == out["tr"][i, u, mm]
            checked += 1
    assert checked > 10


def test_ips_clamp(oracle_mod):
    """Reading A-8: non-positive / NaN-free out-of-range outputs clamp to [2^-4, 2^17] and flag."""
    ens = cases.ensemble_from_nodes([{"feature": 1, "threshold": 2.0, "left": 1, "right": 2},
                                     {"feature": -1, "leaf": -5.0}, {"feature": -1, "leaf": 1e9}])
    inst, req, td = cases.make_instances([dict(N=16, running=[(0, 5, 3, 0, 1e9), (0, 5, 1, 0, 1e9)])], 4)
    out = run(oracle_mod, ens, inst, req, td, 4, np.array([1000.0], np.float32), 16.0)
    assert out["ips"][0, 0, 0] == 2.0 ** 17     # B = 2 -> right leaf 1e9 -> clamp high
    assert out["ips"][0, 0, 1] == 2.0 ** -4     # B = 1 -> left leaf -5 -> clamp low
    assert out["status"][0] & refimpl.ST_IPS_CLAMPED


# ------------------------------------------------------------------ decisions

def test_all_pass_gives_lowest_and_only_max(oracle_mod):
    """all levels pass -> lowest; only the max passes -> max."""
    ens = cases.ensemble_from_nodes([{"feature": 3, "threshold": 1500.0, "left": 1, "right": 2},
                                     {"feature": -1, "leaf": 8.0}, {"feature": -1, "leaf": 64.0}])
    freq = np.array([1000.0, 1200.0, 1600.0], np.float32)
    inst, req, td = cases.make_instances([dict(N=16, running=[(0, 5, 8, 0, 100.0)]),
                                          dict(N=16, running=[(0, 5, 8, 0, 0.5)])], 8)
    out = run(oracle_mod, ens, inst, req, td, 8, freq, 16.0, want_grid=False)
    assert out["level"].tolist() == [0, 2]      # 8 its at 8 IPS = 1 s >= 0.5 s; at 64 IPS 0.125 s


def test_tbt_tie_passes(oracle_mod):
    """P:513 queues only if the mean TBT *exceeds* the SLO, so mean == SLO passes."""
    ens = cases.ensemble_from_nodes([{"feature": 3, "threshold": 1000.0, "left": 1, "right": 2},
                                     {"feature": -1, "leaf": 32.0}, {"feature": -1, "leaf": 64.0}])
    inst, req, td = cases.make_instances([dict(N=16, running=[(0, 5, 7, 0, 100.0), (2, 5, 6, 0, 100.0)])], 8)
    freq = np.array([900.0, 1100.0], np.float32)
    out = run(oracle_mod, ens, inst, req, td, 8, freq, 1.0 / 32, want_grid=False)
    assert out["level"][0] == 0          # mean T' = 1/32 == SLO -> compliant
    out = run(oracle_mod, ens, inst, req, td, 8, freq, float(np.nextafter(np.float32(1 / 32), np.float32(0))),
              want_grid=False)
    assert out["level"][0] == 1


def test_lost_bypass(oracle_mod):
    """a lost request present -> maximum frequency, search bypassed."""
    ens = cases.ensemble_from_nodes([{"feature": -1, "leaf": 64.0}])
    inst, req, td = cases.make_instances([dict(N=16, running=[(0, 5, 8, 1, 100.0), (0, 5, 3, 0, 100.0)])], 8)
    out = run(oracle_mod, ens, inst, req, td, 8, np.array([900.0, 1000.0, 1100.0], np.float32), 16.0, want_grid=False)
    assert out["level"][0] == 2 and out["status"][0] & refimpl.ST_BYPASS_LOST


def test_lost_entries_ignored_in_e2e_when_not_admitted(oracle_mod):
    """A lost flag on a queued request that is NOT admitted does not bypass."""
    ens = cases.ensemble_from_nodes([{"feature": -1, "leaf": 64.0}])
    inst, req, td = cases.make_instances([dict(N=16, max_batch=1, running=[(0, 5, 8, 0, 100.0)],
                                               queued=[(5, 4, 1, 100.0)])], 8)
    out = run(oracle_mod, ens, inst, req, td, 8, np.array([900.0, 1000.0], np.float32), 16.0, want_grid=False)
    assert out["level"][0] == 0 and out["n_adm"][0] == 0 and not out["status"][0] & refimpl.ST_BYPASS_LOST


def test_bad_input(oracle_mod):
    ens = cases.ensemble_from_nodes([{"feature": -1, "leaf": 64.0}])
    inst, req, td = cases.make_instances([dict(N=16, running=[(0, 5, 9, 0, 100.0)]),   # l = 9 > H
                                          dict(N=16, queued=[(5, 4, 0, 100.0)]),
                                          dict(N=0, running=[(0, 5, 3, 0, 100.0)])], 8)
    req = req.copy()
    req[1]["a"] = 1           # queued entry with a != 0
    out = run(oracle_mod, ens, inst, req, td, 8, np.array([900.0, 1000.0], np.float32), 16.0, want_grid=False)
    assert out["status"].tolist() == [refimpl.ST_BAD_INPUT] * 3
    assert out["level"].tolist() == [1, 1, 1]


def test_brute_force_tiny(oracle_mod):
    """Brute force on tiny inputs: independent Fraction/token/box implementation == oracle."""
    rng = np.random.default_rng(7)
    n_cmp = 0
    for trial in range(60):
        ens, inst, req, td, H, freq, tbt = cases.random_tiny_case(rng)
        out = run(oracle_mod, ens, inst, req, td, H, freq, tbt)
        box = refimpl.BoxModel(ens)
        for i in range(len(inst)):
            b = int(inst[i]["req_begin"]); e = b + int(inst[i]["n_run"]) + int(inst[i]["n_queue"])
            ref = refimpl.brute_decide(box, inst[i], req[b:e], td[b:e], H, freq, tbt)
            got = dict(level=int(out["level"][i]), status=int(out["status"][i]), n=int(out["n"][i]),
                       n_adm=int(out["n_adm"][i]))
            assert got == {k: ref[k] for k in got}, (trial, i)
            if not ref["status"] & refimpl.ST_BAD_INPUT:
                assert out["B"][i].tolist() == ref["B"] and out["KV"][i].tolist() == ref["KV"]
            n_cmp += 1
    assert n_cmp >= 300


def test_decision_monotone_in_slack_and_tbt(oracle_mod):
    """More slack (later deadlines) or a looser TBT SLO never raises the chosen level."""
    cfg = W.CONFIGS["P1"]
    ens = W.config_ensemble(cfg)
    d = W.config_inputs(cfg)
    m = oracle_mod.Model(W.write_blob(ens))
    inst, req, td = d["inst"], d["req"], d["t_dead"]
    owner = np.repeat(np.arange(len(inst)), inst["n_run"] + inst["n_queue"])
    slack = td - inst["t_cur"][owner]
    prev = None
    for s in [0.5, 0.8, 1.0, 1.3, 2.0, 4.0]:
        o = oracle_mod.decide(m, inst, req, inst["t_cur"][owner] + slack * s, d["H"], d["freq"], 0.2, want_grid=False)
        if prev is not None:
            assert (o["level"] <= prev).all()
        prev = o["level"]
    prev = None
    for tbt in [0.004, 0.008, 0.012, 0.02, 0.2]:
        o = oracle_mod.decide(m, inst, req, td + 1e6, d["H"], d["freq"], tbt, want_grid=False)
        if prev is not None:
            assert (o["level"] <= prev).all()
        prev = o["level"]
    assert len(set(prev.tolist())) >= 1


def _monotone_in_f_ensemble(rng, freq, n_trees=12):
    """Trees split either only on frequency (leaves increasing with f) or never on it:
    every fp32 partial sum is then non-decreasing in f (rounding is monotone)."""
    trees = []
    for t in range(n_trees):
        if t % 2 == 0:
            cuts = np.sort(rng.uniform(float(freq.min()) - 20, float(freq.max()) + 20, size=3)).astype(np.float32)
            vals = np.sort(rng.uniform(0.5, 8.0, size=4)).astype(np.float32)
            trees.append([W.Node(3, float(cuts[1]), 1, 2), W.Node(3, float(cuts[0]), 3, 4),
                          W.Node(3, float(cuts[2]), 5, 6), W.Node(-1, leaf=float(vals[0])),
                          W.Node(-1, leaf=float(vals[1])), W.Node(-1, leaf=float(vals[2])),
                          W.Node(-1, leaf=float(vals[3]))])
        else:
            v = rng.uniform(1.0, 6.0, size=2).astype(np.float32)
            trees.append([W.Node(1, float(rng.integers(1, 8)) + 0.5, 1, 2), W.Node(-1, leaf=float(v[0])),
                          W.Node(-1, leaf=float(v[1]))])
    return W.Ensemble(trees, 1.0, 2)


def test_binary_search_equals_exhaustive_on_monotone_models(oracle_mod):
    """the paper's binary search == lowest passing level by exhaustive scan
    whenever the model is monotone in frequency.  The binary search is written here."""
    rng = np.random.default_rng(3)
    agree = 0
    for trial in range(40):
        freq = W.freq_levels(int(rng.integers(2, 17)))
        ens = _monotone_in_f_ensemble(rng, freq)
        cfg = dataclasses.replace(W.CONFIGS["P1"], n_inst=24, seed=5000 + trial)
        d = W.config_inputs(cfg)
        m = oracle_mod.Model(W.write_blob(ens))
        full = oracle_mod.decide(m, d["inst"], d["req"], d["t_dead"], d["H"], freq, 0.2, want_grid=False)
        bs = oracle_mod.decide(m, d["inst"], d["req"], d["t_dead"], d["H"], freq, 0.2, want_grid=False,
                               search="binary")
        assert (bs["level"] == full["level"]).all() and (bs["status"] == full["status"]).all()
        for i in range(24):
            st = int(full["status"][i])
            if st & (refimpl.ST_BAD_INPUT | refimpl.ST_EMPTY | refimpl.ST_BYPASS_LOST):
                continue

            def passes(u):
                one = oracle_mod.decide(m, d["inst"][i:i + 1].copy(), d["req"], d["t_dead"], d["H"],
                                        freq[u:u + 1], 0.2, want_grid=False)
                return not one["status"][0] & refimpl.ST_INFEASIBLE
            lo, hi = 0, len(freq) - 1
            if not passes(hi):
                assert st & refimpl.ST_INFEASIBLE and full["level"][i] == len(freq) - 1
                agree += 1
                continue
            while lo < hi:
                mid = (lo + hi) // 2
                if passes(mid):
                    hi = mid
                else:
                    lo = mid + 1
            assert full["level"][i] == lo
            agree += 1
    assert agree >= 200


def test_binary_search_brute_force_tiny(oracle_mod):
    """Reading A-24: the oracle's binary-search mode == the binary search written from
    the paper over exact Fraction pass/fail (refimpl), on non-monotone random ensembles; and it
    differs from the exhaustive answer on some of them (so the mode is really exercised)."""
    rng = np.random.default_rng(24)
    n_cmp = differ = 0
    for trial in range(80):
        ens, inst, req, td, H, freq, tbt = cases.random_tiny_case(rng, F=int(rng.integers(1, 9)))
        out = run(oracle_mod, ens, inst, req, td, H, freq, tbt, search="binary", want_grid=False)
        exh = run(oracle_mod, ens, inst, req, td, H, freq, tbt, want_grid=False)
        box = refimpl.BoxModel(ens)
        for i in range(len(inst)):
            b = int(inst[i]["req_begin"]); e = b + int(inst[i]["n_run"]) + int(inst[i]["n_queue"])
            ref = refimpl.brute_decide(box, inst[i], req[b:e], td[b:e], H, freq, tbt, search="binary")
            got = dict(level=int(out["level"][i]), status=int(out["status"][i]), n=int(out["n"][i]),
                       n_adm=int(out["n_adm"][i]))
            assert got == {k: ref[k] for k in got}, (trial, i)
            differ += int(out["level"][i] != exh["level"][i] or out["status"][i] != exh["status"][i])
            n_cmp += 1
    assert n_cmp >= 400 and differ >= 5


def test_binary_search_order_and_clamp_of_visited_levels(oracle_mod):
    """A-24: the search visits F-1, then mid = (lo + hi) // 2; IPS_CLAMPED covers visited levels
    only.  F = 4, every level passes: visits 3, 1, 0 -> level 0; level 2 (never visited) is the
    only one whose output clamps, so only the exhaustive scan flags it."""
    f = np.array([1000.0, 1200.0, 1400.0, 1600.0], np.float32)
    ens = cases.ensemble_from_nodes([{"feature": 3, "threshold": 1300.0, "left": 1, "right": 2},
                                     {"feature": -1, "leaf": 50.0},
                                     {"feature": 3, "threshold": 1500.0, "left": 3, "right": 4},
                                     {"feature": -1, "leaf": 1e9}, {"feature": -1, "leaf": 50.0}])
    inst, req, td = cases.make_instances([dict(N=16, running=[(0, 5, 4, 0, 1e6)])], 4)
    exh = run(oracle_mod, ens, inst, req, td, 4, f, 16.0)
    bs = run(oracle_mod, ens, inst, req, td, 4, f, 16.0, search="binary")
    assert exh["level"][0] == 0 and bs["level"][0] == 0
    assert exh["status"][0] == refimpl.ST_IPS_CLAMPED and bs["status"][0] == 0
    # the grid holds the visited levels only
    assert (bs["ips"][0, 2] == 0).all() and (bs["ips"][0, [0, 1, 3], :4] == 50.0).all()
    # non-monotone pass pattern: only levels 0 and 3 pass -> the search (3, 1 fails, 2 fails) ends at 3
    ens2 = cases.ensemble_from_nodes([{"feature": 3, "threshold": 1100.0, "left": 1, "right": 2},
                                      {"feature": -1, "leaf": 64.0},
                                      {"feature": 3, "threshold": 1500.0, "left": 3, "right": 4},
                                      {"feature": -1, "leaf": 1.0}, {"feature": -1, "leaf": 64.0}])
    inst, req, td = cases.make_instances([dict(N=16, running=[(0, 5, 8, 0, 1.0)])], 8)
    assert run(oracle_mod, ens2, inst, req, td, 8, f, 16.0)["level"][0] == 0
    assert run(oracle_mod, ens2, inst, req, td, 8, f, 16.0, search="binary")["level"][0] == 3


def test_zero_drift_replay(oracle_mod):
    """replaying the engine iteration by iteration at a fixed frequency, with the
    model as the engine's true speed, completes every scheduled request exactly at T_R[l]."""
    cfg = dataclasses.replace(W.CONFIGS["P1"], n_inst=10, H=120, seed=77)
    ens = W.gen_ensemble(15, 5, 4, W.freq_levels(cfg.F), b_max=40, kv_max=3000, ragged=True)
    d = W.config_inputs(cfg)
    out = run(oracle_mod, ens, d["inst"], d["req"], d["t_dead"], d["H"], d["freq"], 0.2, want_tr=True)
    box = refimpl.BoxModel(ens)
    checked = 0
    for i, ins in enumerate(d["inst"]):
        if out["status"][i] & (refimpl.ST_BAD_INPUT | refimpl.ST_EMPTY):
            continue
        b = int(ins["req_begin"])
        n_sched = int(ins["n_run"]) + int(out["n_adm"][i])
        reqs = d["req"][b:b + n_sched]
        for u in [0, len(d["freq"]) - 1]:
            done = refimpl.replay_completion(box, ins, reqs, n_sched, float(d["freq"][u]), int(ins["N"]))
            for e in range(n_sched):
                l = int(reqs[e]["r"]) - int(reqs[e]["a"])
                assert done[e] * 2 ** 40 == out["tr"][i, u, l - 1]
            checked += 1
    assert checked >= 8


def test_threads_do_not_change_results(oracle_mod):
    cfg = W.CONFIGS["P2"]
    ens = W.config_ensemble(cfg)
    d = W.config_inputs(cfg, 0, 40)
    a = run(oracle_mod, ens, d["inst"], d["req"], d["t_dead"], d["H"], d["freq"], d["tbt_slo"], threads=1)
    b = run(oracle_mod, ens, d["inst"], d["req"], d["t_dead"], d["H"], d["freq"], d["tbt_slo"], threads=7)
    for k in a:
        assert np.array_equal(a[k], b[k])


def test_malformed_blob_rejected(oracle_mod):
    ens = cases.ensemble_from_nodes([{"feature": 1, "threshold": 2.0, "left": 1, "right": 2},
                                     {"feature": -1, "leaf": 1.0}, {"feature": -1, "leaf": 2.0}])
    blob = bytearray(W.write_blob(ens))
    with pytest.raises(ValueError):
        oracle_mod.Model(bytes(blob[:-1]))
    bad = bytearray(blob)
    bad[0:4] = b"XXXX"
    with pytest.raises(ValueError):
        oracle_mod.Model(bytes(bad))
    cyc = W.Ensemble([[W.Node(1, 2.0, 0, 1), W.Node(-1, leaf=1.0)]], 0.0, 1)   # child points at root
    with pytest.raises(ValueError):
        oracle_mod.Model(W.write_blob(cyc))
