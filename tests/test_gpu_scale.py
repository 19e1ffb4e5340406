"""Parity at the scale the throughput numbers are measured on, through the EXACT path bench.py
times (runner.BenchStep): the compact path K1c -> K2 cell phases -> K3c with the B / KV curves kept
on chip, programmatic dependent launch between the kernels, the step captured as one CUDA graph and
replayed.  Every decision compared is element-wise equal to the oracle's (level, status, n, n_adm:
bit-exact; the decision of P:550-557 via Eq. 1-4).

The oracle decides ~100-150 instances/s per host core at C3/C5 shapes (32 levels x ~560 iterations
x 200 trees per decision), so the full-size GPU runs are compared on contiguous blocks plus
stratified samples (sizes in each test), and the sharded runs of the multi-GPU sweep are compared
with the single-GPU run instance by instance.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

import cases
from paper_2408_05235_b200 import shard, workload as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

THREADS = os.cpu_count() or 8


@pytest.fixture(scope="module")
def gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build_lib()
    from paper_2408_05235_b200 import runner, tp
    return tp, runner


def bench_decisions(gpu, blob, inputs, search="exhaustive", replays=2):
    """All decisions of one bench step on cuda:0 (the graph is replayed ``replays`` times: every
    replay re-resets the cell table and must reproduce the same decisions)."""
    tp, runner = gpu
    model = tp.Gbdt(blob, 0)
    step = runner.BenchStep(inputs, "cuda:0", model, search=search)
    outs = []
    for _ in range(replays):
        step.run()
        outs.append(step.decisions())
    for o in outs[1:]:
        for k in o:
            assert np.array_equal(o[k], outs[0][k]), f"graph replay changed {k}"
    del step
    model.free()
    return outs[0]


def oracle_decisions(oracle_mod, blob, inputs, idx, search="exhaustive"):
    sub = cases.subset_inputs(inputs, np.asarray(idx))
    return oracle_mod.decide(oracle_mod.Model(blob), sub["inst"], sub["req"], sub["t_dead"], sub["H"], sub["freq"],
                             sub["tbt_slo"], want_grid=False, want_curves=False, threads=THREADS, search=search)


def assert_same(got, ref, idx, what=""):
    idx = np.asarray(idx)
    for k in ["level", "n", "n_adm"]:
        g, r = got[k][idx].astype(np.int64), ref[k].astype(np.int64)
        bad = np.nonzero(g != r)[0]
        assert len(bad) == 0, f"{what} {k}: {len(bad)} mismatches, first instance {idx[bad[0]]}"
    g, r = got["status"][idx].astype(np.uint32), ref["status"].astype(np.uint32)
    bad = np.nonzero(g != r)[0]
    assert len(bad) == 0, f"{what} status: {len(bad)} mismatches, first instance {idx[bad[0]]}"


def assert_spread(ref, F):
    """The compared sample exercises the whole decision space: many levels, the lost
    bypass, infeasible instances and blocked queues."""
    assert len(np.unique(ref["level"])) >= F // 2
    st = ref["status"].astype(np.uint32)
    for bit in (2, 4, 16):        # BYPASS_LOST, INFEASIBLE, QUEUE_BLOCKED (include/tp.h)
        assert (st & bit).any(), bit


def test_bench_path_c3_contiguous_and_stratified(gpu, oracle_mod):
    """configs[2] (65,536 instances) through the bench step; the oracle decides instances
    [0, 4096) plus a stratified 1/16 of the rest (every 16th, offset 7)."""
    cfg = W.CONFIGS["C3"]
    blob = W.write_blob(W.config_ensemble(cfg))
    inputs = W.config_inputs(cfg)
    got = bench_decisions(gpu, blob, inputs)
    idx = np.union1d(np.arange(4096), np.arange(7, cfg.n_inst, 16))
    ref = oracle_decisions(oracle_mod, blob, inputs, idx)
    assert_same(got, ref, idx, "C3")
    assert_spread(ref, cfg.F)


def test_bench_path_c5_stratified_and_shards(gpu, oracle_mod):
    """configs[4] (262,144 instances) on ONE GPU through the bench step; the oracle decides every
    32nd instance (8,192) plus 16 instances around every shard boundary of the N = 2 / 4 / 8 sweep.
    Then the last shard of each of those sweeps is generated on its own (as bench.py's ranks do)
    and decided through its own bench step: every one of its decisions must equal the single-GPU
    run's for the same global instance."""
    cfg = W.CONFIGS["C5"]
    blob = W.write_blob(W.config_ensemble(cfg))
    inputs = W.config_inputs(cfg)
    got = bench_decisions(gpu, blob, inputs, replays=1)
    bounds = sorted({shard.shard_range(cfg.n_inst, r, N)[0] for N in (2, 4, 8) for r in range(1, N)})
    edge = np.concatenate([np.arange(b - 8, b + 8) for b in bounds] + [np.arange(8), np.arange(cfg.n_inst - 8,
                                                                                               cfg.n_inst)])
    idx = np.union1d(np.arange(5, cfg.n_inst, 32), edge)
    assert len(idx) >= 8192
    ref = oracle_decisions(oracle_mod, blob, inputs, idx)
    assert_same(got, ref, idx, "C5")
    assert_spread(ref, cfg.F)
    for N in (2, 4, 8):
        i0, i1 = shard.shard_range(cfg.n_inst, N - 1, N)
        part = bench_decisions(gpu, blob, W.config_inputs(cfg, i0, i1), replays=1)
        for k in part:
            assert np.array_equal(part[k], got[k][i0:i1]), f"shard {N - 1}/{N} {k}"
    # the engine-grouped shards bench.py's ranks decide at N > 1 (shard.shard_by_engine): the first
    # and last rank of each sweep, every decision equal to the single-GPU run's
    tpv = W.tp_of(cfg)
    for N in (2, 4, 8):
        for r in (0, N - 1):
            ix = shard.shard_by_engine(tpv, r, N)
            part = bench_decisions(gpu, blob, W.select_instances(inputs, ix), replays=1)
            for k in part:
                assert np.array_equal(part[k], got[k][ix]), f"engine shard {r}/{N} {k}"


def test_bench_path_c4_generator(gpu, oracle_mod):
    """configs[3]'s instance generator and 500-tree ensemble (4,096 instances) through the bench
    step; the oracle decides every 4th instance (1,024)."""
    cfg = W.CONFIGS["C4"]
    blob = W.write_blob(W.config_ensemble(cfg))
    inputs = W.config_inputs(cfg)
    got = bench_decisions(gpu, blob, inputs)
    idx = np.arange(1, cfg.n_inst, 4)
    ref = oracle_decisions(oracle_mod, blob, inputs, idx)
    assert_same(got, ref, idx, "C4")
    assert_spread(ref, cfg.F)


def test_bench_path_binary_search_c3_sample(gpu, oracle_mod):
    """The bench step with the paper's binary-search order (--search binary, reading A-24) on a
    2,048-instance C3 slice, all decisions vs the oracle's binary search."""
    cfg = W.CONFIGS["C3"]
    blob = W.write_blob(W.config_ensemble(cfg))
    inputs = W.config_inputs(cfg, 0, 2048)
    got = bench_decisions(gpu, blob, inputs, search="binary")
    idx = np.arange(2048)
    ref = oracle_decisions(oracle_mod, blob, inputs, idx, search="binary")
    assert_same(got, ref, idx, "C3 binary")
