"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element.

Bar: B, KV, n, n_adm, status, level bit-exact (integer work); ips bit-exact (the
kernel forms the same fp32 sums in the same tree order; north_star's 1e-5 relative tolerance is
therefore met with margin 0); T_R ticks bit-exact (exact integer sums).
"""
from __future__ import annotations

import dataclasses
import os

import numpy as np
import pytest

import cases
from paper_2408_05235_b200 import workload as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SKIP = 64 | 1 | 2   # BAD_INPUT | EMPTY | BYPASS_LOST: no grid evaluated


@pytest.fixture(scope="module")
def gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build_lib()
    from paper_2408_05235_b200 import runner, tp
    return tp, runner


@pytest.fixture(params=["direct", "runs", "cells", "fused", "compact"])
def mode(request):
    """All K2 variants: tp_predict_ips (direct), tp_predict_ips_runs in run and cell mode, cell
    mode fused with K3 (tp_predict_ips_runs without the ips grid + tp_select_freq_ws), and the
    compact path (tp_project_compact -> tp_predict_cells -> tp_select_freq_compact)."""
    return request.param


def run_gpu(gpu, blob, inputs, want_tr=True, idx=None, mode="runs"):
    tp, runner = gpu
    model = tp.Gbdt(blob, 0)
    r = runner.Round(inputs, "cuda:0", want_tr=want_tr and mode != "compact", k2_mode=mode, model=model)
    r.run(model)
    out = r.results(idx)
    assert ("ips" in out) == (mode not in ("fused", "compact"))   # fused / compact: never materialised
    del r
    model.free()
    return out


def run_oracle(oracle_mod, blob, inputs, want_tr=True, threads=8, want_grid=True):
    return oracle_mod.decide(oracle_mod.Model(blob), inputs["inst"], inputs["req"], inputs["t_dead"], inputs["H"],
                             inputs["freq"], inputs["tbt_slo"], want_grid=want_grid, want_tr=want_tr, threads=threads)


def assert_parity(got, ref, idx=None, grid=True, tr=True, compact=False):
    """ref: oracle outputs for instances idx (default all); got: GPU outputs for all instances,
    or (compact) only for idx, in idx order."""
    idx = np.arange(len(ref["level"])) if idx is None or compact else np.asarray(idx)
    for k in ["level", "n", "n_adm"]:
        assert np.array_equal(got[k][idx].astype(np.int64), ref[k].astype(np.int64)), k
    assert np.array_equal(got["status"][idx].astype(np.uint32), ref["status"].astype(np.uint32)), "status"
    for k in ["B", "KV"]:
        if k in ref:
            assert np.array_equal(got[k][idx], ref[k]), k
    if grid and "ips" in ref:
        for j, i in enumerate(idx):
            if ref["status"][j] & SKIP:
                continue
            n = int(ref["n"][j])
            if "ips" in got:
                g, r = got["ips"][i, :, :n], ref["ips"][j, :, :n]
                assert np.array_equal(g.view(np.uint32), r.view(np.uint32)), f"ips instance {i}"
            if tr and "tr" in ref and "tr" in got:
                assert np.array_equal(got["tr"][i, :, :n], ref["tr"][j, :, :n]), f"T_R instance {i}"


# ------------------------------------------------------------------ hand-worked W1

@pytest.mark.parametrize("case", [d["case"] for d in cases.load_w1()["decisions"]])
def test_w1(gpu, oracle_mod, mode, case):
    d = [x for x in cases.load_w1()["decisions"] if x["case"] == case][0]
    ens, inst, req, td, H, freq, tbt = cases.w1_inputs(d)
    inputs = dict(inst=inst, req=req, t_dead=td, H=H, freq=freq, tbt_slo=tbt)
    blob = W.write_blob(ens)
    got = run_gpu(gpu, blob, inputs, mode=mode)
    assert int(got["level"][0]) == d["level"] and int(got["status"][0]) == d["status"]
    assert_parity(got, run_oracle(oracle_mod, blob, inputs))


# ------------------------------------------------------------------ brute-force scale random cases

def test_tiny_random(gpu, oracle_mod, mode):
    rng = np.random.default_rng(11)
    for trial in range(150):
        ens, inst, req, td, H, freq, tbt = cases.random_tiny_case(rng)
        inputs = dict(inst=inst, req=req, t_dead=td, H=H, freq=freq, tbt_slo=tbt)
        blob = W.write_blob(ens)
        assert_parity(run_gpu(gpu, blob, inputs, mode=mode), run_oracle(oracle_mod, blob, inputs, threads=1))


# ------------------------------------------------------------------ parity configs (several tiles + ragged tails)

@pytest.mark.parametrize("name", ["P1", "P2"])
def test_parity_configs(gpu, oracle_mod, mode, name):
    cfg = W.CONFIGS[name]
    blob = W.write_blob(W.config_ensemble(cfg))
    inputs = W.config_inputs(cfg)
    assert_parity(run_gpu(gpu, blob, inputs, mode=mode), run_oracle(oracle_mod, blob, inputs))


def test_c1_sweep_10k(gpu, oracle_mod, mode):
    """BASELINE configs[0] shape, 10^4 instances (one seeded block per 1024)."""
    cfg = dataclasses.replace(W.CONFIGS["C1"], n_inst=10000)
    blob = W.write_blob(W.config_ensemble(cfg))
    inputs = W.config_inputs(cfg)
    got = run_gpu(gpu, blob, inputs, mode=mode)
    ref = run_oracle(oracle_mod, blob, inputs)
    assert_parity(got, ref)
    assert len(np.unique(ref["level"])) >= 4          # decisions spread over levels


def test_c2_full(gpu, oracle_mod, mode):
    """BASELINE configs[1] at full size: every decision; full grids on a stratified eighth."""
    cfg = W.CONFIGS["C2"]
    blob = W.write_blob(W.config_ensemble(cfg))
    inputs = W.config_inputs(cfg)
    got = run_gpu(gpu, blob, inputs, want_tr=False, mode=mode)
    ref = run_oracle(oracle_mod, blob, inputs, want_grid=False, want_tr=False)
    assert_parity(got, ref, grid=False)
    sub = np.arange(0, cfg.n_inst, 8)
    sub_in = _subset(inputs, sub)
    assert_parity(got, run_oracle(oracle_mod, blob, sub_in, want_tr=False), idx=sub, tr=False)


_subset = cases.subset_inputs


@pytest.mark.parametrize("name,stride", [("C3", 1024), ("C4", 256)])
def test_full_size_sampled(gpu, oracle_mod, mode, name, stride):
    """BASELINE configs[2]/[3] at full size on the GPU; the oracle recomputes a stratified sample."""
    cfg = W.CONFIGS[name]
    blob = W.write_blob(W.config_ensemble(cfg))
    inputs = W.config_inputs(cfg)
    sub = np.arange(3, cfg.n_inst, stride)
    got = run_gpu(gpu, blob, inputs, want_tr=False, idx=sub, mode=mode)
    assert_parity(got, run_oracle(oracle_mod, blob, _subset(inputs, sub), want_tr=False), idx=sub, tr=False,
                  compact=True)


# ------------------------------------------------------------------ edge cases

def test_empty_batch(gpu, oracle_mod, mode):
    cfg = W.CONFIGS["P1"]
    blob = W.write_blob(W.config_ensemble(cfg))
    inputs = dict(W.config_inputs(cfg), inst=np.zeros(0, W.INST_DTYPE), req=np.zeros(0, W.REQ_DTYPE),
                  t_dead=np.zeros(0))
    got = run_gpu(gpu, blob, inputs, mode=mode)
    assert got["level"].shape == (0,)


@pytest.mark.parametrize("F,H,N,depth,n_trees", [(1, 1, 1, 0, 3), (32, 37, 1, 3, 9), (3, 300, 2, 12, 4),
                                                 (17, 65, 128, 1, 0), (32, 1024, 64, 8, 33), (2, 33, 3, 5, 120)])
def test_shapes(gpu, oracle_mod, mode, F, H, N, depth, n_trees):
    """Degenerate and maximal shapes: F = 1 / 32, H = 1 (one iteration), N = 1 (a block per
    token), depth 0 (stumps-free constant trees) and 12 (deepest), zero trees, ragged tails."""
    cfg = dataclasses.replace(W.CONFIGS["P1"], n_inst=70, H=H, F=F, N=N, n_trees=n_trees, depth=depth,
                              seed=3000 + F + H)
    ens = W.gen_ensemble(n_trees, depth, 7 + depth, W.freq_levels(F), b_max=40, kv_max=4000, ragged=True)
    blob = W.write_blob(ens)
    inputs = W.config_inputs(cfg)
    assert_parity(run_gpu(gpu, blob, inputs, mode=mode), run_oracle(oracle_mod, blob, inputs))


def test_many_thresholds(gpu, oracle_mod, mode):
    """> 255 distinct thresholds per feature (16-bit ranks) and thresholds equal to feature values."""
    rng = np.random.default_rng(5)
    freq = W.freq_levels(12)
    trees = []
    for t in range(40):
        nodes = []

        def build(d):
            idx = len(nodes)
            nodes.append(W.Node(-1))
            if d < 7:
                f = int(rng.choice([1, 2, 3], p=[0.3, 0.5, 0.2]))
                thr = [0, float(rng.integers(0, 70)), float(rng.integers(0, 6000)) + rng.choice([0, 0.25]),
                       float(rng.choice(freq))][f]
                nodes[idx] = W.Node(f, float(np.float32(thr)))
                nodes[idx].left = build(d + 1)
                nodes[idx].right = build(d + 1)
            else:
                nodes[idx].leaf = float(np.float32(rng.uniform(0.1, 3.0)))
            return idx
        build(0)
        trees.append(nodes)
    ens = W.Ensemble(trees, 1.0, 7)
    blob = W.write_blob(ens)
    tp, _ = gpu
    info = tp.Gbdt(blob, 0).info()
    assert info.n_cuts[2] > 255
    cfg = dataclasses.replace(W.CONFIGS["P2"], n_inst=50, F=12, seed=91)
    inputs = W.config_inputs(cfg)
    assert_parity(run_gpu(gpu, blob, inputs, mode=mode), run_oracle(oracle_mod, blob, inputs))


def test_clamp_and_bad_input(gpu, oracle_mod, mode):
    ens = cases.ensemble_from_nodes([{"feature": 1, "threshold": 2.0, "left": 1, "right": 2},
                                     {"feature": -1, "leaf": -5.0}, {"feature": -1, "leaf": 1e9}])
    inst, req, td = cases.make_instances([dict(N=16, running=[(0, 5, 3, 0, 1e9), (0, 5, 1, 0, 1e9)]),
                                          dict(N=16, running=[(0, 5, 9, 0, 100.0)]),
                                          dict(N=0, running=[(0, 5, 3, 0, 100.0)]),
                                          dict(N=16, queued=[(5, 4, 0, 100.0)]),
                                          dict(N=16)], 4)
    req = req.copy()
    req[4]["a"] = 2          # queued entry with a != 0 -> BAD_INPUT
    inputs = dict(inst=inst, req=req, t_dead=td, H=4, freq=np.array([1000.0, 1200.0], np.float32), tbt_slo=16.0)
    blob = W.write_blob(ens)
    got = run_gpu(gpu, blob, inputs, mode=mode)
    assert_parity(got, run_oracle(oracle_mod, blob, inputs))
    assert got["status"][0] & 32 and got["status"].tolist()[1:] == [64, 64, 64, 1]


@pytest.mark.parametrize("k2,cells", [(0, False), (1, False), (1, True), (2, True)])
def test_decide_entry_points_agree(gpu, oracle_mod, k2, cells):
    """tp_decide (device) and tp_decide_host (host buffers, e2e path) == the oracle, both K2 modes."""
    tp, runner = gpu
    cfg = W.CONFIGS["P2"]
    blob = W.write_blob(W.config_ensemble(cfg))
    inputs = W.config_inputs(cfg)
    ref = run_oracle(oracle_mod, blob, inputs, want_grid=False, want_tr=False)
    model = tp.Gbdt(blob, 0)
    I, R = len(inputs["inst"]), len(inputs["req"])
    ctx = tp.Ctx(0, I, R, inputs["H"], len(inputs["freq"]), model if cells else None)
    ctx.set_k2_mode(k2)
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
    assert np.array_equal(h_status.numpy().view(np.uint32), ref["status"])
    # packed host buffers: [inst | req | t_dead] in, [level | status] out (one copy each way)
    bi, br = inputs["inst"].nbytes, inputs["req"].nbytes
    h_in = torch.empty(bi + br + inputs["t_dead"].nbytes, dtype=torch.uint8).pin_memory()
    h_in[:bi].copy_(torch.from_numpy(inputs["inst"].view(np.uint8)))
    h_in[bi:bi + br].copy_(torch.from_numpy(inputs["req"].view(np.uint8)))
    h_in[bi + br:].copy_(torch.from_numpy(np.ascontiguousarray(inputs["t_dead"]).view(np.uint8)))
    h_out = torch.full((2, I), -7, dtype=torch.int32).pin_memory()
    ctx.decide_host(model, h_in[:bi], I, h_in[bi:bi + br], R, h_in[bi + br:].view(torch.float64), inputs["freq"],
                    inputs["tbt_slo"], h_out[0], h_out[1])
    torch.cuda.synchronize()
    assert np.array_equal(h_out[0].numpy(), ref["level"])
    assert np.array_equal(h_out[1].numpy().view(np.uint32), ref["status"])


def test_runs_are_fewer_than_grid_rows(gpu, oracle_mod):
    """The run compression is real on the C2 workload (and exact, by the parity tests)."""
    tp, runner = gpu
    cfg = W.CONFIGS["C2"]
    model = tp.Gbdt(W.write_blob(W.config_ensemble(cfg)), 0)
    r = runner.Round(W.config_inputs(cfg), "cuda:0", k2_mode="runs", model=model)
    r.run(model)
    torch.cuda.synchronize()
    runs = tp.runs_total(r.work, r.I, r.H)
    rows = int(r.n.cpu().numpy().astype(np.int64)[(r.status.cpu().numpy() & SKIP) == 0].sum())
    assert 0 < runs < rows / 3


def test_concurrent_streams_share_model(gpu, oracle_mod):
    """One immutable model handle used by two rounds on two streams at once."""
    tp, runner = gpu
    cfg = W.CONFIGS["P1"]
    blob = W.write_blob(W.config_ensemble(cfg))
    a_in = W.config_inputs(cfg)
    b_in = W.config_inputs(dataclasses.replace(cfg, seed=4242))
    model = tp.Gbdt(blob, 0)
    ra, rb = runner.Round(a_in, "cuda:0", model=model), runner.Round(b_in, "cuda:0", model=model)
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        ra.run(model, sa)
        rb.run(model, sb)
    torch.cuda.synchronize()
    assert_parity(ra.results(), run_oracle(oracle_mod, blob, a_in), tr=False)
    assert_parity(rb.results(), run_oracle(oracle_mod, blob, b_in), tr=False)


@pytest.mark.parametrize("N", [7, 1000, 1 << 20])
def test_block_sizes(gpu, oracle_mod, mode, N):
    """K1's block arithmetic (division by N, block boundaries) for unusual N."""
    cfg = dataclasses.replace(W.CONFIGS["P1"], n_inst=40, N=N, seed=6000 + N % 97)
    blob = W.write_blob(W.config_ensemble(W.CONFIGS["P1"]))
    inputs = W.config_inputs(cfg)
    assert_parity(run_gpu(gpu, blob, inputs, mode=mode), run_oracle(oracle_mod, blob, inputs))


def test_imported_sklearn_model(gpu, oracle_mod, mode):
    """A trained scikit-learn ensemble imported through model_io (N4) runs the whole path bit-exact."""
    from sklearn.ensemble import HistGradientBoostingRegressor
    from paper_2408_05235_b200 import model_io
    rng = np.random.default_rng(1)
    n = 4000
    tp_ = rng.choice([1, 2, 4, 8], n)
    B = rng.integers(1, 41, n)
    KV = (B * rng.uniform(5, 60, n)).astype(int)
    f = rng.choice(W.freq_levels(5), n)
    X = np.stack([tp_, B, KV, f], 1).astype(np.float32)
    y = W.surrogate_ips(tp_, B, KV, f) * (1 + 0.03 * rng.standard_normal(n))
    est = HistGradientBoostingRegressor(max_iter=60, max_depth=6, random_state=0).fit(X, y)
    blob = model_io.to_blob(model_io.from_sklearn(est))
    inputs = W.config_inputs(dataclasses.replace(W.CONFIGS["P1"], n_inst=48, seed=777))
    assert_parity(run_gpu(gpu, blob, inputs, mode=mode), run_oracle(oracle_mod, blob, inputs))


# ------------------------------------------------------------------ compact-path geometry

@pytest.mark.parametrize("n_inst,H", [(2000, 512), (300, 2000), (40, 8192), (7, 16384), (2500, 200), (2500, 2000)])
def test_compact_geometry(gpu, oracle_mod, n_inst, H):
    """The compact path's launch geometry against the oracle: K3c with W = 2 warps per instance
    (2,000 instances), K1c segments longer than 32 iterations (H = 2,000: S = 64; H = 8,192 / 16,384:
    one warp per CTA, 66 / 132 KB of per-warp histograms), and the packed K1c of large batches
    (2,500 instances) with 8- and 64-iteration segments."""
    cfg = dataclasses.replace(W.CONFIGS["P2"], n_inst=n_inst, H=H, seed=8100 + H)
    blob = W.write_blob(W.config_ensemble(cfg))
    inputs = W.config_inputs(cfg)
    assert_parity(run_gpu(gpu, blob, inputs, want_tr=False, mode="compact"),
                  run_oracle(oracle_mod, blob, inputs, want_tr=False))


def test_ctx_ips_grid_on_demand(gpu, oracle_mod):
    """A context created for a cell-mode model runs the compact path and owns no ips grid until a
    mode that writes it is selected (C5-sized contexts would otherwise hold a 34 GB grid)."""
    tp, runner = gpu
    cfg = W.CONFIGS["P1"]
    blob = W.write_blob(W.config_ensemble(cfg))
    inputs = W.config_inputs(cfg)
    model = tp.Gbdt(blob, 0)
    I, R = len(inputs["inst"]), len(inputs["req"])
    ctx = tp.Ctx(0, I, R, inputs["H"], len(inputs["freq"]), model)
    assert not ctx.buffers()[4]
    ref = run_oracle(oracle_mod, blob, inputs, want_grid=False, want_tr=False)
    for mode in (tp.K2_COMPACT, tp.K2_RUNS, tp.K2_DIRECT, tp.K2_COMPACT):
        ctx.set_k2_mode(mode)
        if mode != tp.K2_COMPACT:
            assert ctx.buffers()[4]
        r = runner.Round(inputs, "cuda:0", k2_mode="direct")
        ctx.decide(model, r.inst, I, r.req, R, r.t_dead, inputs["freq"], inputs["tbt_slo"], r.level, r.status)
        torch.cuda.synchronize()
        assert np.array_equal(r.level.cpu().numpy(), ref["level"])
        assert np.array_equal(r.status.cpu().numpy().view(np.uint32), ref["status"])
    assert ctx.buffers()[4]          # allocated by the first non-compact mode, kept


def test_compact_packed_fallback(gpu, oracle_mod):
    """Large batches run K1c with packed B * 2^16 + KV histograms; instances whose footprint does not
    fit (KV >= 2^16 blocks, or >= 2^15 requests) go through the wide kernel -- both bit-exact."""
    cfg = dataclasses.replace(W.CONFIGS["C1"], n_inst=3000, seed=4321)     # > 2,368: one warp each
    blob = W.write_blob(W.config_ensemble(cfg))
    inputs = W.config_inputs(cfg)
    inst, req = inputs["inst"].copy(), inputs["req"].copy()
    for i in (5, 1234, 2999):                  # N = 1 and 9,000-token prompts: > 65,536 blocks
        b, nr = int(inst[i]["req_begin"]), int(inst[i]["n_run"])
        inst[i]["N"] = 1
        inst[i]["kv_cap"] = 1 << 22
        req["q"][b:b + nr + int(inst[i]["n_queue"])] = 9000
    assert int(req["q"][int(inst[5]["req_begin"]):][:8].sum()) >= 65536
    inputs = dict(inputs, inst=inst, req=req)
    got = run_gpu(gpu, blob, inputs, want_tr=False, mode="compact")
    ref = run_oracle(oracle_mod, blob, inputs, want_tr=False)
    assert_parity(got, ref)
    assert int(got["KV"][5].max()) >= 65536


def test_compact_packed_long_horizon(gpu, oracle_mod):
    """Large batches (one warp per instance, packed histograms) whose horizon exceeds 1,024
    iterations: the lane segments of the piece pass are then longer than 32 iterations, so K1c
    takes its per-iteration piece form instead of the per-lane head masks -- both bit-exact, in
    the same launch (instances with n <= 1,024 keep the mask form)."""
    cfg = dataclasses.replace(W.CONFIGS["P2"], n_inst=2600, H=2048, seed=8777)
    blob = W.write_blob(W.config_ensemble(cfg))
    inputs = W.config_inputs(cfg)
    inst, req = inputs["inst"].copy(), inputs["req"].copy()
    long_ix = np.arange(3, cfg.n_inst, 7)
    for i in long_ix:                          # one running request with l = 1,100 .. 2,048
        b, nr = int(inst[i]["req_begin"]), int(inst[i]["n_run"])
        if nr:
            a = int(req["a"][b])
            req["r"][b] = a + 1100 + (int(i) * 37) % 949
    inputs = dict(inputs, inst=inst, req=req)
    got = run_gpu(gpu, blob, inputs, want_tr=False, mode="compact")
    assert int((got["n"] > 1024).sum()) >= 200
    idx = np.union1d(long_ix[::3], np.arange(0, cfg.n_inst, 11))
    ref = run_oracle(oracle_mod, blob, cases.subset_inputs(inputs, idx), want_tr=False, want_grid=False,
                     threads=os.cpu_count() or 8)
    for k in ["level", "n", "n_adm"]:
        assert np.array_equal(got[k][idx].astype(np.int64), ref[k].astype(np.int64)), k
    assert np.array_equal(got["status"][idx].astype(np.uint32), ref["status"].astype(np.uint32)), "status"
    for k in ["B", "KV"]:
        assert np.array_equal(got[k][idx], ref[k]), k
