"""Full admission control on the GPU (tp_decide_admit) vs the oracle's admission=1."""
from __future__ import annotations

import dataclasses

import numpy as np
import pytest

import cases
from paper_2408_05235_b200 import workload as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build_lib()
    from paper_2408_05235_b200 import runner, tp
    return tp, runner


def run_admit(gpu, blob, inputs, q_max=32):
    tp, runner = gpu
    model = tp.Gbdt(blob, 0)
    I, R, H, F = len(inputs["inst"]), len(inputs["req"]), int(inputs["H"]), len(inputs["freq"])
    ctx = tp.Ctx(0, max(I, 1), max(R, 1), H, F, model)
    ctx.enable_admission(q_max)
    r = runner.Round(inputs, "cuda:0", k2_mode="direct")
    n_adm = torch.zeros(max(I, 1), dtype=torch.int32, device="cuda:0")
    lost = torch.zeros(max(I, 1), dtype=torch.int32, device="cuda:0")
    ctx.decide_admit(model, r.inst, I, r.req, R, r.t_dead, inputs["freq"], inputs["tbt_slo"], r.level, r.status,
                     n_adm, lost)
    torch.cuda.synchronize()
    return dict(level=r.level[:I].cpu().numpy(), status=r.status[:I].cpu().numpy().view(np.uint32),
                n_adm=n_adm[:I].cpu().numpy(), adm_lost=lost[:I].cpu().numpy().view(np.uint32))


def check(gpu, oracle_mod, blob, inputs, q_max=32):
    got = run_admit(gpu, blob, inputs, q_max)
    ref = oracle_mod.decide(oracle_mod.Model(blob), inputs["inst"], inputs["req"], inputs["t_dead"], inputs["H"],
                            inputs["freq"], inputs["tbt_slo"], want_grid=False, admission=1, adm_limit=q_max,
                            threads=8)
    for k in ["level", "status", "n_adm", "adm_lost"]:
        assert np.array_equal(got[k].astype(np.int64), ref[k].astype(np.int64)), k
    return ref


@pytest.mark.parametrize("case", [{"R1": 0.2, "R2": 0.2, "Q1": 1.0}, {"R1": 0.2, "R2": 0.2, "Q1": 0.03},
                                  {"R1": 0.2, "R2": 0.05, "Q1": 1.0}])
def test_w1_admission(gpu, oracle_mod, case):
    ens, inst, req, td, H, freq, tbt = cases.w1_inputs({"case": "x", "dead": case, "tbt": 0.05})
    check(gpu, oracle_mod, W.write_blob(ens), dict(inst=inst, req=req, t_dead=td, H=H, freq=freq, tbt_slo=tbt))


def test_tiny_random_admission(gpu, oracle_mod):
    rng = np.random.default_rng(21)
    for trial in range(80):
        ens, inst, req, td, H, freq, tbt = cases.random_tiny_case(rng)
        check(gpu, oracle_mod, W.write_blob(ens), dict(inst=inst, req=req, t_dead=td, H=H, freq=freq, tbt_slo=tbt))


@pytest.mark.parametrize("name,q_max", [("P1", 32), ("P2", 32), ("P1", 3), ("C2", 8)])
def test_config_admission(gpu, oracle_mod, name, q_max):
    cfg = W.CONFIGS[name]
    blob = W.write_blob(W.config_ensemble(cfg))
    inputs = W.config_inputs(cfg)
    ref = check(gpu, oracle_mod, blob, inputs, q_max)
    assert ref["n_adm"].sum() > 0


def test_admission_with_lost_running(gpu, oracle_mod):
    """Instances carrying lost running requests still run the checks (lost deadlines ignored)."""
    cfg = dataclasses.replace(W.CONFIGS["P1"], n_inst=64, seed=31)
    blob = W.write_blob(W.config_ensemble(W.CONFIGS["P1"]))
    inputs = W.config_inputs(cfg)
    req = inputs["req"].copy()
    req["flags"][::7] = 1       # many lost requests (running and queued)
    check(gpu, oracle_mod, blob, dict(inputs, req=req))
