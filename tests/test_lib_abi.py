"""The C ABI library loads, exports every symbol include/tp.h declares, and rejects bad
arguments on the host before touching the GPU (CPU-only; no compute calls)."""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

import __graft_entry__
from paper_2408_05235_b200 import workload as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def tp():
    __graft_entry__.build_lib()
    from paper_2408_05235_b200 import tp as mod
    return mod


def declared_functions():
    src = open(os.path.join(ROOT, "include", "tp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(tp_\w+)\s*\(", src, flags=re.M)))


def test_header_symbols_exported(tp):
    names = declared_functions()
    assert len(names) >= 12
    lib = ctypes.CDLL(tp.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(tp.EXPORTS) == names


def test_abi_version(tp):
    assert tp.abi_version() == 1


def test_sm100a_code_present(tp):
    import subprocess
    out = subprocess.run(["cuobjdump", "-lelf", tp.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", tp.LIB_PATH], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass            # TMA bulk copy (cp.async.bulk) in K2
    assert "SYNCS" in sass             # mbarrier


def test_host_argument_validation(tp):
    L = tp._L
    vp = ctypes.c_void_p(1)
    # H out of range, negative counts, NULL pointers -> EINVAL without any CUDA call
    assert L.tp_project(vp, 1, vp, 1, 0, vp, vp, vp, vp, vp, None) == tp.TP_EINVAL
    assert L.tp_project(vp, 1, vp, 1, 16385, vp, vp, vp, vp, vp, None) == tp.TP_EINVAL
    assert L.tp_project(vp, -1, vp, 1, 8, vp, vp, vp, vp, vp, None) == tp.TP_EINVAL
    assert L.tp_project(None, 1, vp, 1, 8, vp, vp, vp, vp, vp, None) == tp.TP_EINVAL
    f = np.array([900.0, 800.0], np.float32)        # not ascending
    assert L.tp_predict_ips(vp, vp, 1, vp, vp, vp, 8, f.ctypes.data, 2, vp, vp, None) == tp.TP_EINVAL
    f = np.arange(33, dtype=np.float32) + 1          # F > 32
    assert L.tp_predict_ips(vp, vp, 1, vp, vp, vp, 8, f.ctypes.data, 33, vp, vp, None) == tp.TP_EINVAL
    for bad_tbt in [0.0, 2.0 ** -18, 17.0, float("nan")]:
        assert L.tp_select_freq(vp, 1, vp, 1, vp, vp, vp, vp, 8, 2, bad_tbt, vp, vp, None, None) == tp.TP_EINVAL
    assert L.tp_select_freq(vp, 1, vp, 1, vp, vp, vp, vp, 8, 0, 0.2, vp, vp, None, None) == tp.TP_EINVAL


def test_malformed_blobs_rejected(tp):
    ens = W.Ensemble([[W.Node(1, 2.0, 1, 2), W.Node(-1, leaf=1.0), W.Node(-1, leaf=2.0)]], 0.0, 1)
    good = W.write_blob(ens)
    bad = [good[:-1], b"XXXX" + good[4:], W.write_blob(W.Ensemble([[W.Node(1, 2.0, 0, 1), W.Node(-1, leaf=1.0)]], 0.0, 1)),
           W.write_blob(W.Ensemble([[W.Node(5, 2.0, 1, 2), W.Node(-1, leaf=1.0), W.Node(-1, leaf=2.0)]], 0.0, 1)),
           W.write_blob(W.Ensemble([[W.Node(1, float("nan"), 1, 2), W.Node(-1, leaf=1.0), W.Node(-1, leaf=2.0)]], 0, 1)),
           W.write_blob(W.Ensemble([[W.Node(1, 2.0, 1, 2), W.Node(-1, leaf=1.0), W.Node(-1, leaf=2.0)]], 0.0, 0)),
           W.write_blob(W.Ensemble([[W.Node(1, 2.0, 1, 1), W.Node(-1, leaf=1.0), W.Node(-1, leaf=2.0)]], 0.0, 1))]
    for b in bad:
        h = ctypes.c_void_p()
        assert tp._L.tp_gbdt_load(b, len(b), 0, ctypes.byref(h)) == tp.TP_EFORMAT


def test_binding_has_no_cpu_path():
    """The product package never imports the oracle."""
    pkg = os.path.join(ROOT, "paper_2408_05235_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, fn)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle|liboracle|oracle\.", txt, re.M), fn


def test_compact_entry_validation(tp):
    """The compact path's entries reject bad arguments on the host (no CUDA call is made)."""
    L = tp._L
    vp = ctypes.c_void_p(1)
    f = np.array([1000.0, 1200.0], np.float32)
    fd = f.ctypes.data
    # no model, bad H, bad bkv_rows, B without KV
    assert L.tp_project_compact(None, vp, 1 << 20, vp, 1, vp, 1, vp, 8, None, None, 0, vp, vp, vp, None) == tp.TP_EINVAL
    assert L.tp_project_compact(None, vp, 1 << 20, vp, 1, vp, 1, vp, 0, None, None, 0, vp, vp, vp, None) == tp.TP_EINVAL
    assert L.tp_project_compact(None, vp, 1 << 20, vp, 1, vp, 1, vp, 8, vp, None, 0, vp, vp, vp, None) == tp.TP_EINVAL
    assert L.tp_project_compact(None, vp, 1 << 20, vp, 1, vp, 1, vp, 8, vp, vp, 2, vp, vp, vp, None) == tp.TP_EINVAL
    assert L.tp_predict_cells(None, vp, 1 << 20, 1, 8, fd, 2, None) == tp.TP_EINVAL
    # F out of [1, 32], bad search order, tbt_slo out of range
    assert L.tp_select_freq_compact(None, vp, 1 << 20, 1, vp, 8, 0, 0.2, 0, vp, vp, None) == tp.TP_EINVAL
    assert L.tp_select_freq_compact(None, vp, 1 << 20, 1, vp, 8, 33, 0.2, 0, vp, vp, None) == tp.TP_EINVAL
    assert L.tp_select_freq_compact(None, vp, 1 << 20, 1, vp, 8, 2, 0.2, 2, vp, vp, None) == tp.TP_EINVAL
    assert L.tp_select_freq_compact(None, vp, 1 << 20, 1, vp, 8, 2, 100.0, 0, vp, vp, None) == tp.TP_EINVAL
