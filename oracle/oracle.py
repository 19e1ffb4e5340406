"""ORACLE -- TEST INFRASTRUCTURE ONLY (ctypes wrapper of oracle/oracle.c).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  The product path
(paper_2408_05235_b200) never imports it and shares no code with it.

``build()`` compiles oracle.c with plain gcc (no -ffast-math, no FMA
contraction) into oracle/liboracle.so.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

ST_EMPTY, ST_BYPASS_LOST, ST_INFEASIBLE, ST_KV_OVER = 1, 2, 4, 8
ST_QUEUE_BLOCKED, ST_IPS_CLAMPED, ST_BAD_INPUT = 16, 32, 64


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off",
                               "-fno-fast-math", "-Wall", "-o", LIB, SRC, "-lpthread", "-lm"])
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        L.oracle_model_parse.argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(vp)]
        L.oracle_model_parse.restype = ctypes.c_int
        L.oracle_model_free.argtypes = [vp]
        L.oracle_predict_raw.argtypes = [vp, vp]
        L.oracle_predict_raw.restype = ctypes.c_float
        L.oracle_decide.argtypes = [vp, vp, i64, vp, i64, vp, i32, vp, i32, ctypes.c_float,
                                    vp, vp, vp, vp, vp, vp, vp, vp, ctypes.c_int, ctypes.c_int, vp, ctypes.c_int,
                                    ctypes.c_int]
        L.oracle_decide.restype = ctypes.c_int
        _lib = L
    return _lib


class Model:
    """A parsed ensemble (blob v1)."""

    def __init__(self, blob: bytes):
        h = ctypes.c_void_p()
        rc = lib().oracle_model_parse(blob, len(blob), ctypes.byref(h))
        if rc != 0:
            raise ValueError(f"oracle: malformed model blob (rc={rc})")
        self._h = h
        self._blob = blob

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.oracle_model_free(self._h)
            self._h = None

    def predict_raw(self, tp, B, KV, f) -> np.float32:
        x = np.array([tp, B, KV, f], dtype=np.float32)
        return np.float32(lib().oracle_predict_raw(self._h, x.ctypes.data))


def _p(a):
    return None if a is None else a.ctypes.data


def decide(model: Model, inst, req, t_dead, H, freq, tbt_slo, *, want_grid=True, want_tr=False,
           threads: int = 1, want_curves=True, admission: int = 0, adm_limit: int = 32,
           search: str = "exhaustive"):
    """Run O0..O9 on every instance.  Returns a dict of numpy arrays:
    B, KV [I,H] int32; n, n_adm, level [I] int32; status [I] uint32;
    ips [I,F,H] fp32 (if want_grid); tr [I,F,H] int64 ticks of 2^-40 s (if want_tr).
    Grid entries are defined for m <= n only (others stay 0).
    admission=1: the paper's full admission control (checks 1-3 at f_max, lost marking);
    out["adm_lost"] bit c = queued candidate c admitted as lost.
    search="exhaustive": every level is evaluated, answer = lowest passing (reading A-13);
    search="binary": the paper's binary search (reading A-24) -- the grid then holds only
    the levels the search visited."""
    inst = np.ascontiguousarray(inst)
    req = np.ascontiguousarray(req)
    t_dead = np.ascontiguousarray(t_dead, dtype=np.float64)
    freq = np.ascontiguousarray(freq, dtype=np.float32)
    I, F = len(inst), len(freq)
    out = dict(n=np.zeros(I, np.int32), n_adm=np.zeros(I, np.int32),
               level=np.zeros(I, np.int32), status=np.zeros(I, np.uint32))
    if want_curves:
        out["B"] = np.zeros((I, H), np.int32)
        out["KV"] = np.zeros((I, H), np.int32)
    if want_grid:
        out["ips"] = np.zeros((I, F, H), np.float32)
    if want_tr:
        out["tr"] = np.zeros((I, F, H), np.int64)
    if admission:
        out["adm_lost"] = np.zeros(I, np.uint32)
    rc = lib().oracle_decide(model._h, _p(inst), I, _p(req), len(req), _p(t_dead), int(H), _p(freq), F,
                             float(np.float32(tbt_slo)), _p(out.get("B")), _p(out.get("KV")), _p(out["n"]),
                             _p(out["n_adm"]), _p(out.get("ips")), _p(out.get("tr")), _p(out["level"]),
                             _p(out["status"]), int(threads), int(admission), _p(out.get("adm_lost")),
                             int(adm_limit), {"exhaustive": 0, "binary": 1}[search])
    if rc != 0:
        raise ValueError(f"oracle: invalid arguments (rc={rc})")
    return out
