"""Host-side sharding plumbing (no GPU): the engine-grouped strong-scaling shards bench.py's ranks
decide (shard.shard_by_engine), the cheap per-instance tp (workload.tp_of) they are grouped by, and
the instance selection that builds a rank's round (workload.select_instances)."""
from __future__ import annotations

import dataclasses

import numpy as np

import cases
from paper_2408_05235_b200 import shard, workload as W


def small(name="C3", n=3001):
    return dataclasses.replace(W.CONFIGS[name], n_inst=n)


def test_tp_of_matches_the_generator():
    cfg = small()
    inst, _, _ = W.gen_instances(cfg)
    assert np.array_equal(W.tp_of(cfg), inst["tp"])


def test_engine_shards_partition_and_group():
    cfg = small(n=5003)
    tpv = W.tp_of(cfg)
    for N in (1, 2, 3, 4, 8):
        parts = [shard.shard_by_engine(tpv, r, N) for r in range(N)]
        allix = np.concatenate(parts)
        assert np.array_equal(np.sort(allix), np.arange(cfg.n_inst)), N          # each instance once
        assert [len(p) for p in parts] == shard.shard_counts(cfg.n_inst, N)       # equal counts (+-1)
        assert np.all(np.diff(tpv[allix]) >= 0)                                   # grouped by tp
        if N == 4:   # tp is uniform over {1, 2, 4, 8}: four ranks hold (almost) one engine size each
            for p in parts:
                assert np.bincount(tpv[p]).max() >= 0.9 * len(p)


def test_select_instances_equals_a_row_by_row_copy():
    cfg = small(n=700)
    inp = W.config_inputs(cfg)
    rng = np.random.default_rng(5)
    ix = rng.permutation(cfg.n_inst)[:311]
    got, ref = W.select_instances(inp, ix), cases.subset_inputs(inp, ix)
    for k in ("inst", "req", "t_dead"):
        assert np.array_equal(got[k], ref[k]), k
    empty = W.select_instances(inp, np.zeros(0, np.int64))
    assert len(empty["inst"]) == 0 and len(empty["req"]) == 0
