"""One small compact-path round (+ admission + replay-style ctx decide) for compute-sanitizer runs."""
import dataclasses
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2408_05235_b200 import runner, tp, workload as W  # noqa: E402

for name, n_inst in [("P2", 40), ("C2", 24), ("C1", 3)]:
    cfg = dataclasses.replace(W.CONFIGS[name], n_inst=n_inst)
    blob = W.write_blob(W.config_ensemble(cfg))
    inputs = W.config_inputs(cfg)
    model = tp.Gbdt(blob, 0)
    for search in ("exhaustive", "binary"):
        r = runner.Round(inputs, "cuda:0", k2_mode="compact", model=model, search=search)
        r.run(model)
        torch.cuda.synchronize()
    I, R = len(inputs["inst"]), len(inputs["req"])
    ctx = tp.Ctx(0, I, R, inputs["H"], len(inputs["freq"]), model)
    ctx.enable_admission(4)
    ctx.decide_admit(model, r.inst, I, r.req, R, r.t_dead, inputs["freq"], inputs["tbt_slo"], r.level, r.status)
    ctx.decide(model, r.inst, I, r.req, R, r.t_dead, inputs["freq"], inputs["tbt_slo"], r.level, r.status)
    torch.cuda.synchronize()
    print(name, "levels", r.level[:8].cpu().numpy())
# the large-batch K1c (k1_packed: one warp per instance, persistent CTAs) needs > 2 * 148 * 32 / 4
# instances; a C3-shaped round of 2,600 takes it (plus its hand-over kernel)
cfg = dataclasses.replace(W.CONFIGS["C3"], n_inst=2600)
blob = W.write_blob(W.config_ensemble(cfg))
inputs = W.config_inputs(cfg)
model = tp.Gbdt(blob, 0)
r = runner.Round(inputs, "cuda:0", k2_mode="compact", model=model)
r.bkv = False
r.run(model)
torch.cuda.synchronize()
print("C3 packed levels", r.level[:8].cpu().numpy())
print("sanitize probe done")
