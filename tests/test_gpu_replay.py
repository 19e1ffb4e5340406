"""Trace replay (BASELINE configs[3]) on the GPU: every round's decisions equal the
oracle's on the same state, and the on-GPU state advance equals an independent reference."""
from __future__ import annotations

import dataclasses

import numpy as np
import pytest

import refimpl
from paper_2408_05235_b200 import workload as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build_lib()
    from paper_2408_05235_b200 import replay, tp
    return tp, replay


def _check_rounds(gpu, oracle_mod, rc, ens_cfg, rounds, every=1, admission=0, k2_mode=None, threads=16):
    tp, replay = gpu
    data = W.gen_replay(rc)
    blob = W.write_blob(W.config_ensemble(ens_cfg))
    model = tp.Gbdt(blob, 0)
    om = oracle_mod.Model(blob)
    kw = {} if k2_mode is None else dict(k2_mode=getattr(tp, k2_mode))
    rp = replay.Replay(data, model, admission=admission, **kw)
    stats = np.zeros(5, np.int64)
    checked = 0
    for k in range(rounds):
        if k % every:
            rp.round()
            continue
        inst, req, td, arr_next = rp.state()
        dec = oracle_mod.decide(om, inst, req, td, data["H"], data["freq"], data["tbt_slo"], want_grid=False,
                                admission=1 if admission else 0, adm_limit=admission or 32, threads=threads)
        rp.decide()
        torch.cuda.synchronize()
        assert np.array_equal(rp.level.cpu().numpy(), dec["level"]), k
        assert np.array_equal(rp.status.cpu().numpy().view(np.uint32), dec["status"]), k
        if admission:
            assert np.array_equal(rp.adm_lost.cpu().numpy().view(np.uint32), dec["adm_lost"]), k
        s0 = rp.stats.cpu().numpy().copy()
        rp.advance()
        inst2, req2, td2, arr2 = rp.state()
        e_inst, e_req, e_td, e_arr, e_stats = refimpl.replay_advance(inst, req, td, arr_next, data, dec, om,
                                                                     data["freq"], rc.slot_cap,
                                                                     dec.get("adm_lost"))
        assert np.array_equal(inst2, e_inst), k
        assert np.array_equal(arr2, e_arr), k
        for i in range(rc.n_inst):
            c = int(e_inst[i]["n_run"] + e_inst[i]["n_queue"])
            b = i * rc.slot_cap
            assert np.array_equal(req2[b:b + c], e_req[b:b + c]), (k, i)
            assert np.array_equal(td2[b:b + c], e_td[b:b + c]), (k, i)
        assert np.array_equal(rp.stats.cpu().numpy() - s0, e_stats), k
        checked += 1
    return rp, checked


@pytest.mark.parametrize("k2_mode", ["K2_COMPACT", "K2_RUNS"])
def test_replay_matches_oracle_every_round(gpu, oracle_mod, k2_mode):
    """Replay.decide runs tp_decide on the compact path by default (K1c writes only the m = 1
    column of B / KV, which is what tp_replay_advance reads); the fused run/cell path as well."""
    rc = W.ReplayConfig(n_inst=24, n_requests=2400, span_s=2.0, slot_cap=300, seed=11)
    ens = dataclasses.replace(W.CONFIGS["C4"], n_trees=30, depth=6)
    rp, checked = _check_rounds(gpu, oracle_mod, rc, ens, rounds=40, k2_mode=k2_mode)
    assert checked == 40
    st = rp.stats_dict()
    assert st["completed"] > 0 and st["engine_iterations"] > 0


def test_replay_runs_to_completion(gpu, oracle_mod):
    """A small replay drains: every arrival is consumed and every request completes."""
    tp, replay = gpu
    rc = W.ReplayConfig(n_inst=16, n_requests=800, span_s=1.0, slot_cap=400, seed=3)
    data = W.gen_replay(rc)
    model = tp.Gbdt(W.write_blob(W.config_ensemble(dataclasses.replace(W.CONFIGS["C4"], n_trees=20, depth=5))), 0)
    rp = replay.Replay(data, model)
    for _ in range(200):
        for _ in range(50):
            rp.round()
        if rp.finished():
            break
    assert rp.finished()
    st = rp.stats_dict()
    initial = int((data["inst"]["n_run"] + data["inst"]["n_queue"]).sum())
    assert st["completed"] == initial + rc.n_requests - st["dropped_arrivals"]


def test_replay_with_admission_control(gpu, oracle_mod):
    """The paper's full loop: admission control (checks 1-3, lost marks persisted) + throttle each round."""
    rc = W.ReplayConfig(n_inst=24, n_requests=3000, span_s=1.5, slot_cap=300, seed=12)
    ens = dataclasses.replace(W.CONFIGS["C4"], n_trees=30, depth=6)
    rp, checked = _check_rounds(gpu, oracle_mod, rc, ens, rounds=40, admission=8)
    assert checked == 40
    assert rp.stats_dict()["admissions"] > 0


@pytest.mark.parametrize("admission", [0, 8])
def test_replay_512_instances_sampled(gpu, oracle_mod, admission):
    """BASELINE configs[3] shapes at 512 instances (1/8 of the 4,096-instance replay, the same
    request rate per instance: 125,000 arrivals over the 25 s span) with the configs[3] ensemble
    (500 trees, depth 8): the GPU replay runs every round; on every 5th round the oracle decides the
    GPU's current state and an independent advance checks the state transition."""
    rc = W.ReplayConfig(n_inst=512, n_requests=125_000, seed=1004)
    rp, checked = _check_rounds(gpu, oracle_mod, rc, W.CONFIGS["C4"], rounds=11, every=5, admission=admission)
    assert checked == 3
    st = rp.stats_dict()
    assert st["engine_iterations"] > 0
