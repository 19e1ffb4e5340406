"""Probe: the compact decision step captured in a CUDA graph vs launched eagerly (device time per
step, CUDA events, L2 flushed between steps).  usage: python tools/graph_probe.py [C1|C2|C3]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2408_05235_b200 import runner, tp, workload as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = W.CONFIGS[name]
blob = W.write_blob(W.config_ensemble(cfg))
inputs = W.config_inputs(cfg)
dev = torch.device("cuda", 0)
model = tp.Gbdt(blob, 0)
rnd = runner.Round(inputs, dev, k2_mode="compact", model=model)
rnd.bkv = False
s = torch.cuda.Stream(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def step():
    rnd.project(s)
    rnd.predict(model, s)
    rnd.select(s)


with torch.cuda.stream(s):
    for _ in range(5):
        step()
torch.cuda.synchronize()
ref = rnd.level.clone()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    step()
torch.cuda.synchronize()


def timeit(fn, k=100):
    ts = []
    for _ in range(k):
        with torch.cuda.stream(s):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            fn()
            b.record(s)
        ts.append((a, b))
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ts])) * 1e3


rnd.level.zero_()
e = timeit(step)
gr = timeit(g.replay)
assert torch.equal(rnd.level, ref)
print(f"{name}: eager {e:.1f} us/step, graph {gr:.1f} us/step")
