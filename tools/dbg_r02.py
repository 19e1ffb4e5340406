"""GPU debug aid: run the compact path on a config slice, optionally binary search, report errors."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2408_05235_b200 import runner, tp, workload as W
name, n, search, bkv = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4] == "1"
cfg = W.CONFIGS[name]
blob = W.write_blob(W.config_ensemble(cfg))
inp = W.config_inputs(cfg, 0, n)
m = tp.Gbdt(blob, 0)
print("tick_shift", m.info().tick_shift, flush=True)
r = runner.Round(inp, "cuda:0", k2_mode="compact", model=m, search=search)
r.bkv = bkv
for stage in ["project", "predict", "select"]:
    if stage == "project": r.project()
    elif stage == "predict": r.predict(m)
    else: r.select()
    torch.cuda.synchronize()
    print("ok", stage, flush=True)
print(tp.compact_stats(m, r.work, r.I, r.H, r.F))
