"""The N > 1 bench path on ONE GPU: two ranks of bench.py under torchrun (gloo, TP_BENCH_DIST_TEST=1)
each decide their shard of a configs[4]-generator workload through the exact bench step, the
decisions travel through shard.DecisionGather (the gather bench.py times), and the gathered GPU
decisions must equal the oracle's for every instance.  The instance count is odd, so the shards
differ by one and the gather's padding path runs."""
from __future__ import annotations

import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from paper_2408_05235_b200 import workload as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_ranks_gathered_gpu_decisions_equal_oracle(oracle_mod, tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build_lib()
    n = 2051
    out = tmp_path / "dec.npy"
    env = dict(os.environ, TP_BENCH_DIST_TEST="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--workload", "C5", "--instances", str(n), "--steps", "2", "--warmup", "3",
           "--no-cpu-baseline", "--e2e-steps", "1", "--dump-decisions", str(out)]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    import json
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["config"]["global_instances"] == n and line["dist"]["world_size"] == 2
    got = np.load(out)
    assert got.shape == (2, n)
    cfg = W.CONFIGS["C5"]
    import dataclasses
    d = W.config_inputs(dataclasses.replace(cfg, n_inst=n))
    blob = W.write_blob(W.config_ensemble(cfg))
    ref = oracle_mod.decide(oracle_mod.Model(blob), d["inst"], d["req"], d["t_dead"], d["H"], d["freq"],
                            d["tbt_slo"], want_grid=False, want_curves=False, threads=os.cpu_count() or 8)
    assert np.array_equal(got[0], ref["level"])
    assert np.array_equal(got[1].view(np.uint32), ref["status"])
