"""GPU parity of the paper's binary-search throttle (reading A-24).

tp_select_freq_binary (K3 over K2's cell LUT, the search unrolled speculatively over 8 warps) vs
the oracle's search="binary" mode, element by element: level, status (IPS_CLAMPED of the visited
levels only), n, n_adm, B, KV.  Non-monotone ensembles are included so that the binary answer
differs from the exhaustive one on part of the instances.
"""
from __future__ import annotations

import dataclasses

import numpy as np
import pytest

import cases
from paper_2408_05235_b200 import workload as W
from test_gpu_parity import _subset, gpu  # noqa: F401  (fixture)

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(params=["fused", "compact"])
def lut_mode(request):
    """Both paths that read the cell LUT: the speculative warp-per-level K3 (fused) and K3c
    (compact: every level at once, the search replayed on the pass bits)."""
    return request.param


def run_gpu_bs(gpu, blob, inputs, idx=None, mode="fused"):  # noqa: F811
    tp, runner = gpu
    model = tp.Gbdt(blob, 0)
    r = runner.Round(inputs, "cuda:0", k2_mode=mode, model=model, search="binary")
    r.run(model)
    out = r.results(idx)
    del r
    model.free()
    return out


def oracle_bs(oracle_mod, blob, inputs, threads=8):
    return oracle_mod.decide(oracle_mod.Model(blob), inputs["inst"], inputs["req"], inputs["t_dead"], inputs["H"],
                             inputs["freq"], inputs["tbt_slo"], want_grid=False, threads=threads, search="binary")


def check(got, ref, idx=None):
    idx = np.arange(len(ref["level"])) if idx is None else idx
    for k in ["level", "n", "n_adm"]:
        assert np.array_equal(got[k][idx].astype(np.int64), ref[k].astype(np.int64)), k
    assert np.array_equal(got["status"][idx].astype(np.uint32), ref["status"].astype(np.uint32)), "status"
    for k in ["B", "KV"]:
        assert np.array_equal(got[k][idx], ref[k]), k


def test_tiny_random_non_monotone(gpu, oracle_mod, lut_mode):  # noqa: F811
    rng = np.random.default_rng(2424)
    differ = 0
    for trial in range(120):
        ens, inst, req, td, H, freq, tbt = cases.random_tiny_case(rng, F=int(rng.integers(1, 33)))
        inputs = dict(inst=inst, req=req, t_dead=td, H=H, freq=freq, tbt_slo=tbt)
        blob = W.write_blob(ens)
        ref = oracle_bs(oracle_mod, blob, inputs, threads=1)
        check(run_gpu_bs(gpu, blob, inputs, mode=lut_mode), ref)
        exh = oracle_mod.decide(oracle_mod.Model(blob), inst, req, td, H, freq, tbt, want_grid=False)
        differ += int((exh["level"] != ref["level"]).sum())
    assert differ >= 5


def test_visited_levels_clamp_and_non_monotone_path(gpu, oracle_mod, lut_mode):  # noqa: F811
    f = np.array([1000.0, 1200.0, 1400.0, 1600.0], np.float32)
    ens = cases.ensemble_from_nodes([{"feature": 3, "threshold": 1300.0, "left": 1, "right": 2},
                                     {"feature": -1, "leaf": 50.0},
                                     {"feature": 3, "threshold": 1500.0, "left": 3, "right": 4},
                                     {"feature": -1, "leaf": 1e9}, {"feature": -1, "leaf": 50.0}])
    inst, req, td = cases.make_instances([dict(N=16, running=[(0, 5, 4, 0, 1e6)])], 4)
    inputs = dict(inst=inst, req=req, t_dead=td, H=4, freq=f, tbt_slo=16.0)
    got = run_gpu_bs(gpu, W.write_blob(ens), inputs, mode=lut_mode)
    assert got["level"][0] == 0 and got["status"][0] == 0      # level 2 clamps but is never visited
    check(got, oracle_bs(oracle_mod, W.write_blob(ens), inputs))
    ens2 = cases.ensemble_from_nodes([{"feature": 3, "threshold": 1100.0, "left": 1, "right": 2},
                                      {"feature": -1, "leaf": 64.0},
                                      {"feature": 3, "threshold": 1500.0, "left": 3, "right": 4},
                                      {"feature": -1, "leaf": 1.0}, {"feature": -1, "leaf": 64.0}])
    inst, req, td = cases.make_instances([dict(N=16, running=[(0, 5, 8, 0, 1.0)])], 8)
    inputs = dict(inst=inst, req=req, t_dead=td, H=8, freq=f, tbt_slo=16.0)
    assert run_gpu_bs(gpu, W.write_blob(ens2), inputs, mode=lut_mode)["level"][0] == 3


@pytest.mark.parametrize("name", ["P1", "P2", "C1"])
def test_configs(gpu, oracle_mod, name, lut_mode):  # noqa: F811
    cfg = W.CONFIGS[name]
    if name == "C1":
        cfg = dataclasses.replace(cfg, n_inst=4096)
    blob = W.write_blob(W.config_ensemble(cfg))
    inputs = W.config_inputs(cfg)
    check(run_gpu_bs(gpu, blob, inputs, mode=lut_mode), oracle_bs(oracle_mod, blob, inputs))


def test_c2_full(gpu, oracle_mod, lut_mode):  # noqa: F811
    cfg = W.CONFIGS["C2"]
    blob = W.write_blob(W.config_ensemble(cfg))
    inputs = W.config_inputs(cfg)
    ref = oracle_bs(oracle_mod, blob, inputs, threads=16)
    check(run_gpu_bs(gpu, blob, inputs, mode=lut_mode), ref)


def test_c3_sampled(gpu, oracle_mod, lut_mode):  # noqa: F811
    """BASELINE configs[2] at full size, 32 levels (2 speculative rounds); stratified sample."""
    cfg = W.CONFIGS["C3"]
    blob = W.write_blob(W.config_ensemble(cfg))
    inputs = W.config_inputs(cfg)
    sub = np.arange(5, cfg.n_inst, 512)
    got = run_gpu_bs(gpu, blob, inputs, idx=sub, mode=lut_mode)
    check(got, oracle_bs(oracle_mod, blob, _subset(inputs, sub)))


def test_ctx_search_modes(gpu, oracle_mod):  # noqa: F811
    """tp_ctx_set_search: tp_decide / tp_decide_host follow the binary order on the fused path;
    without the fused path (K2 direct) the binary order is refused (TP_ENOTIMPL)."""
    tp, runner = gpu
    cfg = W.CONFIGS["P2"]
    blob = W.write_blob(W.config_ensemble(cfg))
    inputs = W.config_inputs(cfg)
    ref = oracle_bs(oracle_mod, blob, inputs)
    model = tp.Gbdt(blob, 0)
    I, R = len(inputs["inst"]), len(inputs["req"])
    ctx = tp.Ctx(0, I, R, inputs["H"], len(inputs["freq"]), model)
    ctx.set_search("binary")
    r = runner.Round(inputs, "cuda:0", k2_mode="direct")
    ctx.decide(model, r.inst, I, r.req, R, r.t_dead, inputs["freq"], inputs["tbt_slo"], r.level, r.status)
    torch.cuda.synchronize()
    assert np.array_equal(r.level.cpu().numpy(), ref["level"])
    assert np.array_equal(r.status.cpu().numpy().view(np.uint32), ref["status"])
    h_level = torch.zeros(I, dtype=torch.int32).pin_memory()
    h_status = torch.zeros(I, dtype=torch.int32).pin_memory()
    ctx.decide_host(model, inputs["inst"], I, inputs["req"], R, inputs["t_dead"], inputs["freq"], inputs["tbt_slo"],
                    h_level, h_status)
    torch.cuda.synchronize()
    assert np.array_equal(h_level.numpy(), ref["level"])
    ctx.set_k2_mode(tp.K2_DIRECT)
    with pytest.raises(tp.TpError) as e:
        ctx.decide(model, r.inst, I, r.req, R, r.t_dead, inputs["freq"], inputs["tbt_slo"], r.level, r.status)
    assert e.value.code == -5 or "not implemented" in str(e.value)
