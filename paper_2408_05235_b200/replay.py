"""Trace replay driver (BASELINE configs[3]): every round decides ALL instances
(tp_decide: K1 -> K2 -> K3 on the GPU) and advances every instance by one engine iteration at its
chosen frequency (tp_replay_advance, on the GPU).  The state never leaves the device; torch only
provides the buffers.
"""
from __future__ import annotations

import numpy as np
import torch

from . import tp
from . import workload as W


def _pin(a, dtype=None):
    a = np.ascontiguousarray(a if dtype is None else a.astype(dtype))
    t = torch.from_numpy(a.view(np.uint8).reshape(-1) if a.dtype.fields is not None else a)
    return t.pin_memory()


def _dev(a, dev, dtype=None):
    a = np.ascontiguousarray(a)
    if a.dtype.fields is not None:
        return torch.from_numpy(a.view(np.uint8).reshape(-1)).to(dev)
    return torch.from_numpy(a if dtype is None else a.astype(dtype)).to(dev)


class Replay:
    STATS = ("completed", "met_deadline", "dropped_arrivals", "engine_iterations", "admissions")

    def __init__(self, data: dict, model: tp.Gbdt, device="cuda:0", k2_mode=tp.K2_COMPACT, admission: int = 0,
                 search: str = "exhaustive"):
        """admission = q_max > 0: each round runs the paper's full admission control (tp_decide_admit)
        on at most q_max queued requests per instance before the throttle."""
        dev = torch.device(device)
        # pinned host copies of the initial state and the arrival stream (reset() uploads them)
        self.host = {k: _pin(data[k], np.float64 if k in ("t_dead", "arr_t", "arr_dead") else
                             np.int64 if k == "arr_off" else None)
                     for k in ("inst", "req", "t_dead", "arr_t", "arr_req", "arr_dead", "arr_off")}
        self.dev, self.model = dev, model
        self.I = len(data["inst"])
        self.cap = int(data["slot_cap"])
        self.H = int(data["H"])
        self.freq = np.asarray(data["freq"], np.float32)
        self.F = len(self.freq)
        self.tbt = np.float32(data["tbt_slo"])
        self.inst = _dev(data["inst"], dev)
        self.req = [_dev(data["req"], dev), torch.empty_like(_dev(data["req"], dev))]
        self.t_dead = [_dev(data["t_dead"], dev), torch.empty_like(_dev(data["t_dead"], dev))]
        self.arr_t = _dev(data["arr_t"], dev, np.float64)
        self.arr_req = _dev(data["arr_req"], dev)
        self.arr_dead = _dev(data["arr_dead"], dev, np.float64)
        self.arr_off = _dev(data["arr_off"], dev, np.int64)
        self.arr_next = self.arr_off[:-1].clone()
        self.stats = torch.zeros(5, dtype=torch.int64, device=dev)
        self.level = torch.empty(self.I, dtype=torch.int32, device=dev)
        self.status = torch.empty(self.I, dtype=torch.int32, device=dev)
        self.ctx = tp.Ctx(dev.index or 0, self.I, self.I * self.cap, self.H, self.F, model)
        self.ctx.set_k2_mode(k2_mode)
        self.ctx.set_search(search)
        self.B, self.KV, self.n, self.n_adm, _ = self.ctx.buffers()
        self.admission = int(admission)
        self.adm_lost = None
        if self.admission:
            self.ctx.enable_admission(self.admission)
            self.adm_lost = torch.zeros(self.I, dtype=torch.int32, device=dev)
        self.cur = 0
        self.rounds = 0

    def reset(self, stream=None):
        """Back to the initial state: host -> device copies of the state and the arrival stream
        (pinned, asynchronous on ``stream``), counters cleared."""
        st = stream if stream is not None else torch.cuda.current_stream(self.dev)
        with torch.cuda.stream(st):
            self.inst.copy_(self.host["inst"], non_blocking=True)
            self.req[0].copy_(self.host["req"], non_blocking=True)
            self.t_dead[0].copy_(self.host["t_dead"], non_blocking=True)
            self.arr_t.copy_(self.host["arr_t"], non_blocking=True)
            self.arr_req.copy_(self.host["arr_req"], non_blocking=True)
            self.arr_dead.copy_(self.host["arr_dead"], non_blocking=True)
            self.arr_off.copy_(self.host["arr_off"], non_blocking=True)
            self.arr_next.copy_(self.arr_off[:-1])
            self.stats.zero_()
            if self.adm_lost is not None:
                self.adm_lost.zero_()
        self.cur = 0
        self.rounds = 0

    def host_bytes(self) -> int:
        """Bytes reset() copies host -> device."""
        return int(sum(t.numel() * t.element_size() for t in self.host.values()))

    def decide(self, stream=None):
        if self.admission:
            self.ctx.decide_admit(self.model, self.inst, self.I, self.req[self.cur], self.I * self.cap,
                                  self.t_dead[self.cur], self.freq, self.tbt, self.level, self.status, None,
                                  self.adm_lost, stream)
            return
        self.ctx.decide(self.model, self.inst, self.I, self.req[self.cur], self.I * self.cap, self.t_dead[self.cur],
                        self.freq, self.tbt, self.level, self.status, stream)

    def advance(self, stream=None):
        c, o = self.cur, 1 - self.cur
        tp.tp_replay_advance(self.model, self.inst, self.I, self.req[c], self.t_dead[c], self.req[o], self.t_dead[o],
                             self.cap, self.H, self.B, self.KV, self.n, self.n_adm, self.status, self.level, self.freq,
                             self.arr_t, self.arr_req, self.arr_dead, self.arr_off, self.arr_next, self.stats,
                             self.adm_lost, stream)
        self.cur = o
        self.rounds += 1

    def round(self, stream=None):
        self.decide(stream)
        self.advance(stream)

    def state(self):
        """Host copies of the current state (synchronises)."""
        inst = self.inst.cpu().numpy().view(W.INST_DTYPE).copy()
        req = self.req[self.cur].cpu().numpy().view(W.REQ_DTYPE).copy()
        return inst, req, self.t_dead[self.cur].cpu().numpy().copy(), self.arr_next.cpu().numpy().copy()

    def finished(self) -> bool:
        inst = self.inst.cpu().numpy().view(W.INST_DTYPE)
        return bool((inst["n_run"] + inst["n_queue"]).sum() == 0 and
                    torch.equal(self.arr_next, self.arr_off[1:]))

    def arrivals_consumed(self) -> bool:
        return bool(torch.equal(self.arr_next, self.arr_off[1:]))

    def running(self) -> int:
        """Running requests over all instances (synchronises)."""
        inst = self.inst.cpu().numpy().view(W.INST_DTYPE)
        return int(inst["n_run"].astype(np.int64).sum())

    def in_flight(self) -> int:
        """Requests running or queued over all instances (synchronises)."""
        inst = self.inst.cpu().numpy().view(W.INST_DTYPE)
        return int((inst["n_run"].astype(np.int64) + inst["n_queue"]).sum())

    def stats_dict(self):
        return dict(zip(self.STATS, (int(x) for x in self.stats.cpu().numpy())))
