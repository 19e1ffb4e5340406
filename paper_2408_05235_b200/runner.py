"""Device-memory plumbing around the C ABI: upload a round's inputs once, run K1 -> K2 -> K3.

torch provides device memory and streams only; all arithmetic happens in libtp's kernels.
"""
from __future__ import annotations

import numpy as np
import torch

from . import tp
from . import workload as W


def to_device_bytes(a: np.ndarray, device) -> torch.Tensor:
    """A structured / plain numpy array as a raw uint8 device tensor (same bytes)."""
    a = np.ascontiguousarray(a)
    t = torch.from_numpy(a.view(np.uint8).reshape(-1)) if a.size else torch.zeros(16, dtype=torch.uint8)
    return t.to(device)


class Round:
    """One decision round's device buffers (inputs + K1/K2/K3 outputs)."""

    def __init__(self, inputs: dict, device="cuda:0", want_tr=False, k2_mode="cells", model=None,
                 search="exhaustive"):
        dev = torch.device(device)
        self.device = dev
        inst, req, t_dead = inputs["inst"], inputs["req"], inputs["t_dead"]
        self.I, self.R, self.H = len(inst), len(req), int(inputs["H"])
        self.freq = np.asarray(inputs["freq"], dtype=np.float32)
        self.F = len(self.freq)
        self.tbt = np.float32(inputs["tbt_slo"])
        assert inst.dtype == W.INST_DTYPE and req.dtype == W.REQ_DTYPE
        self.inst = to_device_bytes(inst, dev)
        self.req = to_device_bytes(req, dev)
        self.t_dead = torch.from_numpy(np.ascontiguousarray(t_dead, np.float64)).to(dev) if self.R else \
            torch.zeros(1, dtype=torch.float64, device=dev)
        I, H, F = max(self.I, 1), self.H, self.F
        self.B = torch.empty((I, H), dtype=torch.int32, device=dev)
        self.KV = torch.empty((I, H), dtype=torch.int32, device=dev)
        self.n = torch.empty(I, dtype=torch.int32, device=dev)
        self.n_adm = torch.empty(I, dtype=torch.int32, device=dev)
        self.status = torch.empty(I, dtype=torch.int32, device=dev)
        self.level = torch.empty(I, dtype=torch.int32, device=dev)
        # the ips grid exists only on the paths that write it (the fused and compact paths keep the
        # values in the workspace's cell LUT)
        self.ips = torch.zeros((I, F, H), dtype=torch.float32, device=dev) \
            if k2_mode in ("direct", "runs", "cells") else None
        self.tr = torch.zeros((I, F, H), dtype=torch.int64, device=dev) if want_tr else None
        assert k2_mode in ("compact", "fused", "cells", "runs", "direct")
        assert k2_mode not in ("cells", "fused", "compact") or model is not None, \
            "cell mode sizes its workspace from the model"
        self.k2_mode = k2_mode
        assert search in ("exhaustive", "binary")
        assert search == "exhaustive" or (k2_mode in ("fused", "compact") and not want_tr), \
            "binary search reads the cell LUT"
        assert not (want_tr and k2_mode == "compact"), "the compact path emits no T_R"
        self.search = search
        self.model = model
        self.bkv = True             # compact mode: K1c writes the full B/KV rows (tests); bench turns it off
        self.work = torch.empty(tp.tp_predict_ips_workspace_size(model if k2_mode in ("cells", "fused", "compact")
                                                                 else None,
                                                                 I, H, F),
                                dtype=torch.uint8, device=dev) if k2_mode != "direct" else None

    def project(self, stream=None):
        if self.k2_mode == "compact":
            # K1c: full B/KV rows too, so results() can compare them (bench.py passes bkv_rows=False)
            tp.tp_project_compact(self.model, self.work, self.inst, self.I, self.req, self.R, self.t_dead, self.H,
                                  self.B if self.bkv else None, self.KV if self.bkv else None, 1, self.n, self.n_adm,
                                  self.status, stream)
            return
        tp.tp_project(self.inst, self.I, self.req, self.R, self.H, self.B, self.KV, self.n, self.n_adm, self.status,
                      stream)

    def predict(self, model, stream=None):
        if self.k2_mode == "compact":
            tp.tp_predict_cells(model, self.work, self.I, self.H, self.freq, stream)
            return
        if self.k2_mode in ("runs", "cells", "fused"):
            # fused: cell mode without the ips grid (values stay in the workspace for K3)
            tp.tp_predict_ips_runs(model, self.inst, self.I, self.B, self.KV, self.n, self.H, self.freq,
                                   None if self.k2_mode == "fused" else self.ips, self.status, self.work, stream)
        else:
            tp.tp_predict_ips(model, self.inst, self.I, self.B, self.KV, self.n, self.H, self.freq, self.ips,
                              self.status, stream)

    def select(self, stream=None):
        if self.k2_mode == "compact":
            tp.tp_select_freq_compact(self.model, self.work, self.I, self.n, self.H, self.F, self.tbt, self.search,
                                      self.level, self.status, stream)
            return
        if self.search == "binary":
            tp.tp_select_freq_binary(self.model, self.work, self.inst, self.I, self.req, self.R, self.t_dead, self.n,
                                     self.n_adm, self.H, self.F, self.tbt, self.level, self.status, stream)
            return
        if self.k2_mode == "fused":
            tp.tp_select_freq_ws(self.model, self.work, self.inst, self.I, self.req, self.R, self.t_dead, self.n,
                                 self.n_adm, self.H, self.F, self.tbt, self.level, self.status, self.tr, stream)
            return
        tp.tp_select_freq(self.inst, self.I, self.req, self.R, self.t_dead, self.n, self.n_adm, self.ips, self.H,
                          self.F, self.tbt, self.level, self.status, self.tr, stream)

    def run(self, model, stream=None):
        self.project(stream)
        self.predict(model, stream)
        self.select(stream)

    def results(self, idx=None) -> dict:
        """Outputs copied to the host; ``idx`` selects instances (all by default, rows in idx order)."""
        torch.cuda.synchronize(self.device)
        I = self.I
        sel = slice(0, I) if idx is None else torch.as_tensor(np.asarray(idx), device=self.device, dtype=torch.long)
        get = lambda t: t[sel].cpu().numpy()   # noqa: E731
        out = dict(B=get(self.B), KV=get(self.KV), n=get(self.n), n_adm=get(self.n_adm),
                   status=get(self.status).view(np.uint32), level=get(self.level))
        if self.ips is not None:
            out["ips"] = get(self.ips)
        if self.tr is not None:
            out["tr"] = get(self.tr)
        return out


class BenchStep:
    """The exact step bench.py times (and the at-scale parity tests and smoke() check): the
    compact path K1c -> K2 cell phases -> K3c with B / KV kept on chip (no B / KV rows written),
    programmatic dependent launch between the kernels, the three launches (+ the cell-table reset)
    captured once as a CUDA graph and replayed every step.  ``level`` / ``status`` may be views
    into a caller buffer (bench.py writes them straight into the decision gather's send rows)."""

    def __init__(self, inputs: dict, device, model, search="exhaustive", graph=True, level=None, status=None):
        self.device = torch.device(device)
        self.rnd = Round(inputs, self.device, k2_mode="compact", model=model, search=search)
        self.rnd.bkv = False
        if level is not None:
            self.rnd.level, self.rnd.status = level, status
        self.model = model
        self.graph = None
        if graph:
            gs = torch.cuda.Stream(self.device)
            with torch.cuda.stream(gs):
                self.kernels(gs)      # warm-up on the capture stream (attributes, lazy module loading)
            torch.cuda.synchronize(self.device)
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph, stream=gs):
                self.kernels(gs)
            torch.cuda.synchronize(self.device)

    def kernels(self, stream):
        self.rnd.project(stream)
        self.rnd.predict(self.model, stream)
        self.rnd.select(stream)

    def run(self, stream=None):
        """One step on ``stream`` (the captured graph when there is one)."""
        if self.graph is not None:
            self.graph.replay()
        else:
            self.kernels(stream)

    def decisions(self, idx=None) -> dict:
        """level / status / n / n_adm on the host (synchronises)."""
        torch.cuda.synchronize(self.device)
        r = self.rnd
        sel = slice(0, r.I) if idx is None else torch.as_tensor(np.asarray(idx), device=self.device,
                                                                  dtype=torch.long)
        get = lambda t: t[:r.I][sel].cpu().numpy()   # noqa: E731
        return dict(level=get(r.level), status=get(r.status).view(np.uint32), n=get(r.n), n_adm=get(r.n_adm))
