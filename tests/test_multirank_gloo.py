"""N > 1 host logic on CPU (gloo, world size 2): sharding covers every instance once, shards
generate the same bytes as the whole, and the decision gather reassembles the single-rank result.

The per-rank decisions here come from the oracle (test infrastructure standing in for the GPU
kernels, which the single-GPU parity tests cover); what is under test is the sharding and the
gather that bench.py uses around the kernels.
"""
from __future__ import annotations

import dataclasses
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2408_05235_b200 import shard, workload as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_ranges_partition():
    for n in [1, 7, 1024, 262144]:
        for world in [1, 2, 3, 4, 8]:
            rs = [shard.shard_range(n, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1


def test_shard_generation_matches_whole():
    cfg = dataclasses.replace(W.CONFIGS["P1"], n_inst=2500)
    whole = W.gen_instances(cfg)
    for (i0, i1) in [(0, 1000), (1000, 2500), (1023, 1025), (2400, 2500)]:
        inst, req, td = W.gen_instances(cfg, i0, i1)
        assert len(inst) == i1 - i0
        for k in range(i1 - i0):
            a = whole[0][i0 + k]
            b = inst[k]
            for f in ["n_run", "n_queue", "N", "kv_cap", "max_batch", "tp", "t_cur"]:
                assert a[f] == b[f]
            wa = int(a["req_begin"]); wb = int(b["req_begin"]); c = int(a["n_run"] + a["n_queue"])
            assert np.array_equal(whole[1][wa:wa + c], req[wb:wb + c])
            assert np.array_equal(whole[2][wa:wa + c], td[wb:wb + c])


def _worker(rank, world, port, cfg, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle
    blob = W.write_blob(W.config_ensemble(cfg))
    i0, i1 = shard.shard_range(cfg.n_inst, rank, world)
    d = W.config_inputs(cfg, i0, i1)
    out = oracle.decide(oracle.Model(blob), d["inst"], d["req"], d["t_dead"], d["H"], d["freq"], d["tbt_slo"],
                        want_grid=False, want_curves=False)
    dec = torch.from_numpy(np.stack([out["level"], out["status"].view(np.int32)]).astype(np.int32))
    counts = [shard.shard_range(cfg.n_inst, r, world)[1] - shard.shard_range(cfg.n_inst, r, world)[0]
              for r in range(world)]
    allg = shard.gather_decisions(dec, counts)
    if rank == 0:
        ret.put(allg.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_inst", [61, 64])
def test_gloo_world2_gather_equals_single_rank(oracle_mod, n_inst):
    cfg = dataclasses.replace(W.CONFIGS["P1"], n_inst=n_inst)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cfg, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    blob = W.write_blob(W.config_ensemble(cfg))
    d = W.config_inputs(cfg)
    ref = oracle_mod.decide(oracle_mod.Model(blob), d["inst"], d["req"], d["t_dead"], d["H"], d["freq"],
                            d["tbt_slo"], want_grid=False, want_curves=False)
    assert np.array_equal(got[0], ref["level"])
    assert np.array_equal(got[1].view(np.uint32), ref["status"])
