"""Thin Python binding of libtp (include/tp.h) -- argument marshalling only.

Every step of the path runs in libtp's sm_100a kernels; this module only turns torch tensors
(device memory, allocated by the caller) and numpy arrays into pointers and checks return
codes.  It never computes any part of the method and has no CPU fallback: if libtp.so is
missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# TP_LIB_PATH: an alternative in-tree build (tuning variants, tools/build_variant.py)
LIB_PATH = os.environ.get("TP_LIB_PATH") or os.path.join(HERE, "libtp.so")

TP_OK, TP_EINVAL, TP_ENOMEM, TP_ECUDA, TP_EFORMAT, TP_ENOTIMPL = 0, -1, -2, -3, -4, -5
ST_EMPTY, ST_BYPASS_LOST, ST_INFEASIBLE, ST_KV_OVER = 1, 2, 4, 8
ST_QUEUE_BLOCKED, ST_IPS_CLAMPED, ST_BAD_INPUT = 16, 32, 64

# every symbol include/tp.h declares
EXPORTS = ["tp_gbdt_load", "tp_gbdt_free", "tp_gbdt_get_info", "tp_project", "tp_predict_ips",
           "tp_predict_ips_workspace_size", "tp_predict_ips_runs", "tp_runs_total", "tp_cells_total", "tp_select_freq", "tp_select_freq_ws", "tp_ctx_create", "tp_ctx_free",
           "tp_decide", "tp_decide_host", "tp_replay_advance", "tp_ctx_enable_admission", "tp_decide_admit", "tp_ctx_set_k2_mode", "tp_ctx_buffers",
           "tp_select_freq_binary", "tp_ctx_set_search", "tp_project_compact", "tp_predict_cells",
           "tp_select_freq_compact", "tp_compact_stats", "tp_strerror", "tp_abi_version"]
K2_DIRECT, K2_RUNS, K2_COMPACT = 0, 1, 2
SEARCH_EXHAUSTIVE, SEARCH_BINARY = 0, 1

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libtp.so not built ({LIB_PATH}); run __graft_entry__.build()")
_L = ctypes.CDLL(LIB_PATH)

_vp, _i32, _i64, _f32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float


class GbdtInfo(ctypes.Structure):
    _fields_ = [("n_trees", ctypes.c_int32), ("depth", ctypes.c_int32), ("n_cuts", ctypes.c_int32 * 4),
                ("base_score", ctypes.c_float), ("tick_shift", ctypes.c_int32), ("device_bytes", ctypes.c_int64),
                ("node_bytes", ctypes.c_int64)]


_L.tp_gbdt_load.argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.c_int, ctypes.POINTER(_vp)]
_L.tp_gbdt_free.argtypes = [_vp]
_L.tp_gbdt_get_info.argtypes = [_vp, ctypes.POINTER(GbdtInfo)]
_L.tp_project.argtypes = [_vp, _i32, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp]
_L.tp_predict_ips.argtypes = [_vp, _vp, _i32, _vp, _vp, _vp, _i32, _vp, _i32, _vp, _vp, _vp]
_L.tp_predict_ips_workspace_size.argtypes = [_vp, _i32, _i32, _i32]
_L.tp_predict_ips_runs.argtypes = [_vp, _vp, _i32, _vp, _vp, _vp, _i32, _vp, _i32, _vp, _vp, _vp, ctypes.c_size_t, _vp]
_L.tp_ctx_set_k2_mode.argtypes = [_vp, ctypes.c_int]
_L.tp_runs_total.argtypes = [_vp, _i32, _i32, ctypes.POINTER(_i64)]
_L.tp_cells_total.argtypes = [_vp, _vp, _i32, _i32, _i32, ctypes.POINTER(_i64)]
_L.tp_select_freq.argtypes = [_vp, _i32, _vp, _i32, _vp, _vp, _vp, _vp, _i32, _i32, _f32, _vp, _vp, _vp, _vp]
_L.tp_select_freq_ws.argtypes = [_vp, _vp, _vp, _i32, _vp, _i32, _vp, _vp, _vp, _i32, _i32, _f32, _vp, _vp, _vp, _vp]
_L.tp_select_freq_binary.argtypes = [_vp, _vp, _vp, _i32, _vp, _i32, _vp, _vp, _vp, _i32, _i32, _f32, _vp, _vp, _vp]
_L.tp_ctx_set_search.argtypes = [_vp, ctypes.c_int]
_L.tp_project_compact.argtypes = [_vp, _vp, ctypes.c_size_t, _vp, _i32, _vp, _i32, _vp, _i32, _vp, _vp, _i32, _vp,
                                  _vp, _vp, _vp]
_L.tp_predict_cells.argtypes = [_vp, _vp, ctypes.c_size_t, _i32, _i32, _vp, _i32, _vp]
_L.tp_select_freq_compact.argtypes = [_vp, _vp, ctypes.c_size_t, _i32, _vp, _i32, _i32, _f32, _i32, _vp, _vp, _vp]
_L.tp_compact_stats.argtypes = [_vp, _vp, ctypes.c_size_t, _i32, _i32, _i32, _vp]
_L.tp_replay_advance.argtypes = [_vp, _vp, _i32, _vp, _vp, _vp, _vp, _i32, _i32] + [_vp] * 6 + [_vp, _i32] + [_vp] * 8
_L.tp_ctx_enable_admission.argtypes = [_vp, _i32]
_L.tp_decide_admit.argtypes = [_vp, _vp, _vp, _i32, _vp, _i32, _vp, _vp, _i32, _f32, _vp, _vp, _vp, _vp, _vp]
_L.tp_ctx_create.argtypes = [ctypes.c_int, _vp, _i32, _i32, _i32, _i32, ctypes.POINTER(_vp)]
_L.tp_ctx_free.argtypes = [_vp]
_L.tp_decide.argtypes = [_vp, _vp, _vp, _i32, _vp, _i32, _vp, _vp, _i32, _f32, _vp, _vp, _vp]
_L.tp_decide_host.argtypes = [_vp, _vp, _vp, _i32, _vp, _i32, _vp, _vp, _i32, _f32, _vp, _vp, _vp]
_L.tp_ctx_buffers.argtypes = [_vp] + [ctypes.POINTER(_vp)] * 5
_L.tp_strerror.argtypes = [ctypes.c_int]
_L.tp_strerror.restype = ctypes.c_char_p
for _f in EXPORTS:
    if _f != "tp_strerror":
        getattr(_L, _f).restype = ctypes.c_int
_L.tp_predict_ips_workspace_size.restype = ctypes.c_size_t


class TpError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"{what}: {_L.tp_strerror(code).decode()} ({code})")
        self.code = code


def _check(rc, what):
    if rc != TP_OK:
        raise TpError(rc, what)


def _dp(t):
    """Device pointer of a torch tensor (or None)."""
    if t is None:
        return None
    if isinstance(t, int):       # a raw device pointer (e.g. from Ctx.buffers())
        return t
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return t.data_ptr()


def _hp(a):
    """Host pointer of a numpy array or CPU torch tensor."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("expected a C-contiguous array")
        return a.ctypes.data
    if a.is_cuda or not a.is_contiguous():
        raise ValueError("expected a contiguous host tensor")
    return a.data_ptr()


def _stream(stream):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _freq(freq):
    f = np.ascontiguousarray(np.asarray(freq, dtype=np.float32))
    return f, len(f)


def abi_version() -> int:
    return _L.tp_abi_version()


class Gbdt:
    """tp_gbdt_load / tp_gbdt_free: an immutable model on one device."""

    def __init__(self, blob: bytes, device: int = 0):
        h = _vp()
        _check(_L.tp_gbdt_load(blob, len(blob), int(device), ctypes.byref(h)), "tp_gbdt_load")
        self.handle = h
        self.device = device

    def info(self) -> GbdtInfo:
        i = GbdtInfo()
        _check(_L.tp_gbdt_get_info(self.handle, ctypes.byref(i)), "tp_gbdt_get_info")
        return i

    def free(self):
        if self.handle:
            _L.tp_gbdt_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def tp_gbdt_load(blob: bytes, device: int = 0) -> Gbdt:
    return Gbdt(blob, device)


def tp_project(inst, n_inst, req, n_req, H, B, KV, n, n_adm, status, stream=None):
    _check(_L.tp_project(_dp(inst), int(n_inst), _dp(req), int(n_req), int(H), _dp(B), _dp(KV), _dp(n),
                         _dp(n_adm), _dp(status), _stream(stream)), "tp_project")


def tp_predict_ips(model: Gbdt, inst, n_inst, B, KV, n, H, freq, ips, status, stream=None):
    f, F = _freq(freq)
    _check(_L.tp_predict_ips(model.handle, _dp(inst), int(n_inst), _dp(B), _dp(KV), _dp(n), int(H), f.ctypes.data,
                             F, _dp(ips), _dp(status), _stream(stream)), "tp_predict_ips")


def tp_predict_ips_workspace_size(model, n_inst, H, F) -> int:
    """model=None sizes run mode; a Gbdt sizes its cell mode."""
    return int(_L.tp_predict_ips_workspace_size(model.handle if model is not None else None, int(n_inst), int(H),
                                                int(F)))


def tp_predict_ips_runs(model: Gbdt, inst, n_inst, B, KV, n, H, freq, ips, status, workspace, stream=None):
    """workspace: a uint8 CUDA tensor of at least tp_predict_ips_workspace_size(n_inst, H) bytes."""
    f, F = _freq(freq)
    _check(_L.tp_predict_ips_runs(model.handle, _dp(inst), int(n_inst), _dp(B), _dp(KV), _dp(n), int(H),
                                  f.ctypes.data, F, _dp(ips), _dp(status), _dp(workspace), workspace.numel(),
                                  _stream(stream)), "tp_predict_ips_runs")


def runs_total(workspace, n_inst, H) -> int:
    """Runs evaluated by the last tp_predict_ips_runs on ``workspace`` (synchronous diagnostic)."""
    t = _i64()
    _check(_L.tp_runs_total(_dp(workspace), int(n_inst), int(H), ctypes.byref(t)), "tp_runs_total")
    return int(t.value)


def cells_total(workspace, model, n_inst, H, F) -> int:
    """Distinct cells evaluated by the last cell-mode tp_predict_ips_runs (synchronous diagnostic)."""
    t = _i64()
    _check(_L.tp_cells_total(model.handle, _dp(workspace), int(n_inst), int(H), int(F), ctypes.byref(t)),
           "tp_cells_total")
    return int(t.value)


def compact_stats(model: Gbdt, workspace, n_inst, H, F) -> dict:
    """Pieces, end positions and distinct cells of the last tp_project_compact (synchronous)."""
    out = np.zeros(3, np.int64)
    _check(_L.tp_compact_stats(model.handle, _dp(workspace), workspace.numel(), int(n_inst), int(H), int(F),
                               out.ctypes.data), "tp_compact_stats")
    return dict(pieces=int(out[0]), ends=int(out[1]), cells=int(out[2]))


def tp_select_freq(inst, n_inst, req, n_req, t_dead, n, n_adm, ips, H, F, tbt_slo, level, status, tr_ticks=None,
                   stream=None):
    _check(_L.tp_select_freq(_dp(inst), int(n_inst), _dp(req), int(n_req), _dp(t_dead), _dp(n), _dp(n_adm),
                             _dp(ips), int(H), int(F), float(np.float32(tbt_slo)), _dp(level), _dp(status),
                             _dp(tr_ticks), _stream(stream)), "tp_select_freq")


def tp_select_freq_ws(model: Gbdt, workspace, inst, n_inst, req, n_req, t_dead, n, n_adm, H, F, tbt_slo, level, status,
                      tr_ticks=None, stream=None):
    _check(_L.tp_select_freq_ws(model.handle, _dp(workspace), _dp(inst), int(n_inst), _dp(req), int(n_req),
                                _dp(t_dead), _dp(n), _dp(n_adm), int(H), int(F), float(np.float32(tbt_slo)),
                                _dp(level), _dp(status), _dp(tr_ticks), _stream(stream)), "tp_select_freq_ws")


def tp_select_freq_binary(model: Gbdt, workspace, inst, n_inst, req, n_req, t_dead, n, n_adm, H, F, tbt_slo, level,
                          status, stream=None):
    _check(_L.tp_select_freq_binary(model.handle, _dp(workspace), _dp(inst), int(n_inst), _dp(req), int(n_req),
                                    _dp(t_dead), _dp(n), _dp(n_adm), int(H), int(F), float(np.float32(tbt_slo)),
                                    _dp(level), _dp(status), _stream(stream)), "tp_select_freq_binary")


def tp_project_compact(model: Gbdt, workspace, inst, n_inst, req, n_req, t_dead, H, B, KV, bkv_rows, n, n_adm,
                       status, stream=None):
    """K1c: projection + gate + runs / cell claims + deadline list (B, KV may be None)."""
    _check(_L.tp_project_compact(model.handle, _dp(workspace), workspace.numel(), _dp(inst), int(n_inst), _dp(req),
                                 int(n_req), _dp(t_dead), int(H), _dp(B), _dp(KV), int(bkv_rows), _dp(n),
                                 _dp(n_adm), _dp(status), _stream(stream)), "tp_project_compact")


def tp_predict_cells(model: Gbdt, workspace, n_inst, H, freq, stream=None):
    """K2 on the cells tp_project_compact claimed (LUT in the workspace)."""
    f, F = _freq(freq)
    _check(_L.tp_predict_cells(model.handle, _dp(workspace), workspace.numel(), int(n_inst), int(H), f.ctypes.data,
                               F, _stream(stream)), "tp_predict_cells")


def tp_select_freq_compact(model: Gbdt, workspace, n_inst, n, H, F, tbt_slo, search, level, status, stream=None):
    """K3c: one warp per instance, lane = level; search 0 exhaustive (A-13) / 1 binary (A-24)."""
    if isinstance(search, str):
        search = {"exhaustive": SEARCH_EXHAUSTIVE, "binary": SEARCH_BINARY}[search]
    _check(_L.tp_select_freq_compact(model.handle, _dp(workspace), workspace.numel(), int(n_inst), _dp(n), int(H),
                                     int(F), float(np.float32(tbt_slo)), int(search), _dp(level), _dp(status),
                                     _stream(stream)), "tp_select_freq_compact")


def tp_replay_advance(model: Gbdt, inst, n_inst, req, t_dead, req_out, t_dead_out, slot_cap, H, B, KV, n, n_adm,
                      status, level, freq, arr_t, arr_req, arr_dead, arr_off, arr_next, stats, adm_lost=None,
                      stream=None):
    f, F = _freq(freq)
    _check(_L.tp_replay_advance(model.handle, _dp(inst), int(n_inst), _dp(req), _dp(t_dead), _dp(req_out),
                                _dp(t_dead_out), int(slot_cap), int(H), _dp(B), _dp(KV), _dp(n), _dp(n_adm),
                                _dp(status), _dp(level), f.ctypes.data, F, _dp(arr_t), _dp(arr_req), _dp(arr_dead),
                                _dp(arr_off), _dp(arr_next), _dp(stats), _dp(adm_lost), _stream(stream)),
           "tp_replay_advance")


class Ctx:
    """tp_ctx_create / tp_decide / tp_decide_host."""

    def __init__(self, device, n_inst_max, n_req_max, H, F_max, model=None):
        h = _vp()
        _check(_L.tp_ctx_create(int(device), model.handle if model is not None else None, int(n_inst_max),
                                int(n_req_max), int(H), int(F_max), ctypes.byref(h)), "tp_ctx_create")
        self.handle = h
        self.H = H

    def decide(self, model: Gbdt, inst, n_inst, req, n_req, t_dead, freq, tbt_slo, level, status, stream=None):
        f, F = _freq(freq)
        _check(_L.tp_decide(self.handle, model.handle, _dp(inst), int(n_inst), _dp(req), int(n_req), _dp(t_dead),
                            f.ctypes.data, F, float(np.float32(tbt_slo)), _dp(level), _dp(status), _stream(stream)),
               "tp_decide")

    def decide_host(self, model: Gbdt, inst, n_inst, req, n_req, t_dead, freq, tbt_slo, level, status, stream=None):
        f, F = _freq(freq)
        _check(_L.tp_decide_host(self.handle, model.handle, _hp(inst), int(n_inst), _hp(req), int(n_req),
                                 _hp(t_dead), f.ctypes.data, F, float(np.float32(tbt_slo)), _hp(level), _hp(status),
                                 _stream(stream)), "tp_decide_host")

    def enable_admission(self, q_max=32):
        _check(_L.tp_ctx_enable_admission(self.handle, int(q_max)), "tp_ctx_enable_admission")

    def decide_admit(self, model: Gbdt, inst, n_inst, req, n_req, t_dead, freq, tbt_slo, level, status,
                     n_adm=None, adm_lost=None, stream=None):
        f, F = _freq(freq)
        _check(_L.tp_decide_admit(self.handle, model.handle, _dp(inst), int(n_inst), _dp(req), int(n_req),
                                  _dp(t_dead), f.ctypes.data, F, float(np.float32(tbt_slo)), _dp(level), _dp(status),
                                  _dp(n_adm), _dp(adm_lost), _stream(stream)), "tp_decide_admit")

    def set_k2_mode(self, mode):
        _check(_L.tp_ctx_set_k2_mode(self.handle, int(mode)), "tp_ctx_set_k2_mode")

    def set_search(self, search):
        """search: SEARCH_EXHAUSTIVE (reading A-13) or SEARCH_BINARY (the paper's P:555, A-24)."""
        if isinstance(search, str):
            search = {"exhaustive": SEARCH_EXHAUSTIVE, "binary": SEARCH_BINARY}[search]
        _check(_L.tp_ctx_set_search(self.handle, int(search)), "tp_ctx_set_search")

    def buffers(self):
        ptrs = [_vp() for _ in range(5)]
        _check(_L.tp_ctx_buffers(self.handle, *[ctypes.byref(p) for p in ptrs]), "tp_ctx_buffers")
        return [p.value for p in ptrs]

    def free(self):
        if self.handle:
            _L.tp_ctx_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def tp_ctx_create(device, model, n_inst_max, n_req_max, H, F_max) -> Ctx:
    return Ctx(device, n_inst_max, n_req_max, H, F_max, model)
