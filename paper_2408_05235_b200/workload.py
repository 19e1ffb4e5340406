"""Seeded synthetic inputs for the throttLL'eM frequency-selection path.

This module is the ONLY code shared by the CUDA path (through ``bench.py`` /
tests) and the CPU oracle (through tests).  It draws random numbers and lays
them out in the byte formats ``include/tp.h`` documents; it contains none of
the method's arithmetic (no projection, no tree evaluation, no SLO check).

Shapes follow BASELINE.json ``configs`` and SURVEY.md §8(d):

* lengths are "Azure-like" (§3.4): prompts up to 4000
  tokens, most below 1500; generations 10-700 tokens, most 100-400;
* TBT SLO 200 ms (§5.1);
* frequency levels in 15 MHz steps (§4.3.1) on a B200-like
  range 600-1965 MHz (SURVEY.md §8c reading A-19);
* random gradient-boosted ensembles over the paper's features
  ``[engine size (tp), batch, KV blocks, GPU frequency]``
  whose leaves follow a smooth surrogate IPS shape -- the
  paper's trained model is not published.

Every generator is a pure function of (config, seed); instance ``i`` of a
config is generated from the block ``i // BLOCK`` so any contiguous shard can be
generated alone with identical bytes (multi-GPU runs).
"""
from __future__ import annotations

import dataclasses
import math
import struct

import numpy as np

INST_DTYPE = np.dtype([
    ("k", "<i8"), ("t_cur", "<f8"), ("req_begin", "<i4"), ("n_run", "<i4"),
    ("n_queue", "<i4"), ("N", "<i4"), ("kv_cap", "<i4"), ("max_batch", "<i4"),
    ("tp", "<i4"), ("_pad", "<i4")])
REQ_DTYPE = np.dtype([("a", "<i4"), ("q", "<i4"), ("r", "<i4"), ("flags", "<i4")])
assert INST_DTYPE.itemsize == 48 and REQ_DTYPE.itemsize == 16

FLAG_LOST = 1
BLOCK = 1024  # instances per independently seeded generation block

# feature order fixed by the blob format: [tp, batch, kv_blocks, freq_mhz]
F_TP, F_B, F_KV, F_F = 0, 1, 2, 3


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    n_inst: int
    H: int
    F: int
    n_trees: int
    depth: int
    N: int
    max_batch: int
    run_lo: int
    run_hi: int
    q_hi: int            # queued requests ~ U{0..q_hi}
    c1_shape: bool = False   # C1: <=16 KV blocks per request, l <= 64
    ragged: bool = False
    seed: int = 1001
    tbt_slo: float = 0.2
    f_lo: float = 600.0
    f_hi: float = 1965.0


CONFIGS = {
    # BASELINE.json configs[0]: 1 instance, 8 running + 4 queued, 16 KV blocks/req cap,
    # 8 freq levels, 64-iter horizon, 50-tree depth-6
    "C1": Config("C1", 1, 64, 8, 50, 6, 16, 12, 8, 8, 4, c1_shape=True, seed=1001),
    # configs[1]: 1,024 instances, batch <=64, 16 freq levels, 512-iter horizon, 200x depth-8
    "C2": Config("C2", 1024, 512, 16, 200, 8, 64, 64, 1, 60, 4, seed=1002),
    # configs[2]: 65,536 instances, batch <=256, 32 freq levels, 1,024-iter horizon
    # (tree shape not given by BASELINE.json: 200 x depth 8 assumed)
    "C3": Config("C3", 65536, 1024, 32, 200, 8, 64, 256, 1, 248, 8, seed=1003),
    # configs[3]: trace-replay states, 4,096 instances, 500-tree depth-8
    "C4": Config("C4", 4096, 1024, 32, 500, 8, 64, 256, 1, 248, 8, seed=1004),
    # configs[4]: scaling sweep, 262,144 instances (C3 generator)
    "C5": Config("C5", 262144, 1024, 32, 200, 8, 64, 256, 1, 248, 8, seed=1005),
    # small parity configs (not bench lines): ragged trees, several tiles + ragged tails
    "P1": Config("P1", 64, 200, 5, 37, 7, 16, 40, 0, 36, 6, ragged=True, seed=2001),
    "P2": Config("P2", 300, 512, 16, 60, 8, 64, 64, 1, 60, 4, ragged=True, seed=2002),
}


def freq_levels(F: int, lo: float = 600.0, hi: float = 1965.0) -> np.ndarray:
    """F strictly ascending levels rounded to 15 MHz steps (SURVEY A-19)."""
    if F == 1:
        return np.array([hi], dtype=np.float32)
    lv = np.round(np.linspace(lo, hi, F) / 15.0) * 15.0
    lv = np.maximum.accumulate(lv)
    for i in range(1, F):  # keep strictly ascending for large F
        if lv[i] <= lv[i - 1]:
            lv[i] = lv[i - 1] + 15.0
    return lv.astype(np.float32)


def surrogate_ips(tp, B, KV, f, f_max=1965.0):
    """Smooth IPS shape used only to draw leaf values and deadlines:
    rises with frequency, falls with batch and KV usage (PAPER §3.1-3.2 trends)."""
    return 60.0 * np.sqrt(tp) * (np.asarray(f) / f_max) ** 0.7 / (1.0 + 0.01 * np.asarray(B) + 0.0002 * np.asarray(KV))


# ----------------------------------------------------------------------------------------------
# instance states
# ----------------------------------------------------------------------------------------------

def _lognormal_int(rng, median, sigma, lo, hi, size):
    v = np.exp(np.log(median) + sigma * rng.standard_normal(size))
    return np.clip(np.rint(v), lo, hi).astype(np.int64)


def _gen_block(cfg: Config, block: int, n: int):
    rng = np.random.default_rng([cfg.seed, block])
    H = cfg.H
    tp = rng.choice(np.array([1, 2, 4, 8]), size=n)
    n_run = rng.integers(cfg.run_lo, cfg.run_hi + 1, size=n)
    n_q = rng.integers(0, cfg.q_hi + 1, size=n)
    tot = n_run + n_q
    R = int(tot.sum())
    owner = np.repeat(np.arange(n), tot)
    start = np.concatenate([[0], np.cumsum(tot)[:-1]])
    pos = np.arange(R) - start[owner]
    queued = pos >= n_run[owner]
    if cfg.c1_shape:
        r = rng.integers(1, H + 1, size=R)
        # <= 16 KV blocks per request at N=16: q + r - 1 <= 256
        q = 1 + (rng.random(R) * (256 - r)).astype(np.int64)
    else:
        r = _lognormal_int(rng, 250.0, 0.5, min(10, H), min(700, H), R)
        q = _lognormal_int(rng, 600.0, 0.9, 1, 4000, R)
    a = np.where(queued, 0, (rng.random(R) * r).astype(np.int64))   # progress a in [0, r-1]
    flags = np.zeros(R, dtype=np.int64)
    # 1 % of instances carry one lost running request
    lost_inst = (rng.random(n) < 0.01) & (n_run > 0)
    first = start[lost_inst]
    flags[first] = FLAG_LOST
    N = cfg.N
    # KV capacity: a random fraction around the total final footprint of the running set
    # (generator heuristic; sometimes below the projected peak -> KV_OVER path exercised)
    foot = np.bincount(owner, weights=np.where(queued, 0.0, (q + r) / N), minlength=n)
    kv_cap = np.floor(foot * rng.uniform(0.85, 1.3, size=n) + rng.integers(0, 4, size=n) * (256.0 / N)).astype(np.int64)
    # deadlines: slack_j = l_j * tau_i * g_i * U[1, 1.25], tau_i = 1 / surrogate at f_max and the
    # current batch; g_i ~ U[0.7, 2.0] spreads decisions over the levels, 5 % tight (g < 0.6)
    kv_mid = np.bincount(owner, weights=(q + a) / N, minlength=n)
    tau = 1.0 / surrogate_ips(tp, n_run, kv_mid, cfg.f_hi)
    g = np.where(rng.random(n) < 0.05, rng.uniform(0.3, 0.6, size=n), rng.uniform(0.7, 2.0, size=n))
    l = r - a
    slack = l * (tau * g)[owner] * rng.uniform(1.0, 1.25, size=R)
    t_cur = rng.uniform(0.0, 3600.0, size=n)
    t_dead = t_cur[owner] + slack
    inst = np.zeros(n, dtype=INST_DTYPE)
    inst["k"] = rng.integers(0, 1 << 40, size=n)
    inst["t_cur"] = t_cur
    inst["req_begin"] = start
    inst["n_run"] = n_run
    inst["n_queue"] = n_q
    inst["N"] = N
    inst["kv_cap"] = kv_cap
    inst["max_batch"] = cfg.max_batch
    inst["tp"] = tp
    req = np.zeros(R, dtype=REQ_DTYPE)
    req["a"], req["q"], req["r"], req["flags"] = a, q, r, flags
    return inst, req, t_dead.astype(np.float64)


def tp_of(cfg: Config) -> np.ndarray:
    """Engine size (tp) of every instance of ``cfg``, without generating the requests: the first
    draw of each block's generator (as `_gen_block`)."""
    out = np.empty(cfg.n_inst, np.int64)
    for b in range((cfg.n_inst + BLOCK - 1) // BLOCK):
        b0 = b * BLOCK
        nb = min(BLOCK, cfg.n_inst - b0)
        out[b0:b0 + nb] = np.random.default_rng([cfg.seed, b]).choice(np.array([1, 2, 4, 8]), size=nb)
    return out


def select_instances(inputs: dict, idx) -> dict:
    """The instances ``idx`` (in that order) of a round's inputs as a self-contained round: request
    rows gathered, ``req_begin`` rebased.  Input plumbing only."""
    idx = np.asarray(idx, np.int64)
    inst = inputs["inst"][idx].copy()
    cnt = (inst["n_run"] + inst["n_queue"]).astype(np.int64)
    begin = inst["req_begin"].astype(np.int64)
    off = np.concatenate([[0], np.cumsum(cnt)[:-1]]) if len(idx) else np.zeros(0, np.int64)
    rows = np.repeat(begin - off, cnt) + np.arange(int(cnt.sum()))
    inst["req_begin"] = off
    return dict(inputs, inst=inst, req=inputs["req"][rows], t_dead=inputs["t_dead"][rows])


def gen_instances(cfg: Config, i0: int = 0, i1: int | None = None):
    """Instances [i0, i1) of ``cfg`` (default: all) -> (inst, req, t_dead).

    ``req_begin`` is rebased so the returned arrays are self-contained."""
    if i1 is None:
        i1 = cfg.n_inst
    insts, reqs, deads = [], [], []
    off = 0
    for b in range(i0 // BLOCK, (max(i1, i0 + 1) - 1) // BLOCK + 1):
        b0 = b * BLOCK
        nb = min(BLOCK, cfg.n_inst - b0)
        inst, req, td = _gen_block(cfg, b, nb)
        lo, hi = max(i0, b0) - b0, min(i1, b0 + nb) - b0
        if hi <= lo:
            continue
        inst = inst[lo:hi].copy()
        r0 = int(inst["req_begin"][0])
        r1 = int(inst["req_begin"][-1] + inst["n_run"][-1] + inst["n_queue"][-1])
        inst["req_begin"] += off - r0
        insts.append(inst)
        reqs.append(req[r0:r1])
        deads.append(td[r0:r1])
        off += r1 - r0
    if not insts:
        return np.zeros(0, INST_DTYPE), np.zeros(0, REQ_DTYPE), np.zeros(0, np.float64)
    return np.concatenate(insts), np.concatenate(reqs), np.concatenate(deads)


# ----------------------------------------------------------------------------------------------
# tree ensembles and the blob format (include/tp.h "Blob format v1")
# ----------------------------------------------------------------------------------------------

@dataclasses.dataclass
class Node:
    feature: int          # -1 = leaf
    threshold: float = 0.0
    left: int = -1
    right: int = -1
    leaf: float = 0.0


@dataclasses.dataclass
class Ensemble:
    trees: list            # list[list[Node]], root = node 0 of each tree
    base: float = 0.0
    max_depth: int = 0


def write_blob(ens: Ensemble) -> bytes:
    """Serialise to blob v1: "TPGB", u32 version=1, u32 n_features=4, u32 n_trees,
    u32 max_depth, f32 base_score; per tree u32 n_nodes + n_nodes x
    {i32 feature, f32 threshold, i32 left, i32 right, f32 leaf}."""
    out = [b"TPGB", struct.pack("<IIIIf", 1, 4, len(ens.trees), ens.max_depth, ens.base)]
    for t in ens.trees:
        out.append(struct.pack("<I", len(t)))
        for nd in t:
            out.append(struct.pack("<ifiif", nd.feature, nd.threshold, nd.left, nd.right, nd.leaf))
    return b"".join(out)


def _cut_sets(rng, f_levels, b_max, kv_max):
    tp_cuts = np.array([1.5, 2.0, 3.0, 4.0, 6.0, 8.0])
    def mixed(lo, hi, k):
        ints = rng.integers(int(lo), int(hi) + 1, size=k // 2).astype(np.float64)
        halves = rng.integers(int(lo), int(hi) + 1, size=k - k // 2) + 0.5
        return np.unique(np.concatenate([ints, halves]).astype(np.float32))
    b_cuts = mixed(1, b_max, 255)[:255]
    kv_cuts = mixed(1, kv_max, 255)[:255]
    fl = np.asarray(f_levels, dtype=np.float64)
    mids = (fl[1:] + fl[:-1]) / 2 if len(fl) > 1 else fl
    f_cuts = np.unique(np.concatenate([fl, mids, rng.uniform(fl.min() - 30, fl.max() + 30, size=24)]).astype(np.float32))
    return [np.unique(tp_cuts.astype(np.float32)), b_cuts, kv_cuts, f_cuts]


def gen_ensemble(n_trees: int, depth: int, seed: int, f_levels, b_max: float = 64, kv_max: float = 1500,
                 ragged: bool = False, base: float = 0.5, noise: float = 0.05) -> Ensemble:
    """Random ensemble of depth-``depth`` trees.  Splits pick a feature with weights
    tp 0.05 / batch 0.25 / kv 0.35 / freq 0.35 and a threshold from that feature's
    cut set (<=255 values, integers and half-integers, frequency levels themselves
    included so ``x < thr`` ties are exercised).  A leaf holds
    surrogate(centre of its cell) / n_trees * (1 + noise * N(0,1)).  ``ragged``
    turns internal nodes into early leaves with probability 0.1."""
    rng = np.random.default_rng([seed, 77])
    cuts = _cut_sets(rng, f_levels, b_max, kv_max)
    fl = np.asarray(f_levels, dtype=np.float64)
    dom = [(1.0, 8.0), (0.0, float(b_max)), (0.0, float(kv_max)), (float(fl.min()) - 30.0, float(fl.max()) + 30.0)]
    weights = np.array([0.05, 0.25, 0.35, 0.35])
    trees = []
    for _ in range(n_trees):
        nodes: list[Node] = []

        def build(d, box):
            idx = len(nodes)
            nodes.append(Node(-1))
            make_leaf = d == depth or (ragged and d >= 1 and rng.random() < 0.1)
            if not make_leaf:
                order = rng.choice(4, size=4, replace=False, p=weights)
                for feat in order:
                    lo, hi = box[feat]
                    c = cuts[feat]
                    cand = c[(c > lo) & (c < hi)]
                    if len(cand):
                        thr = float(cand[rng.integers(len(cand))])
                        lb = list(box); lb[feat] = (lo, thr)
                        rb = list(box); rb[feat] = (thr, hi)
                        nodes[idx] = Node(int(feat), thr)
                        nodes[idx].left = build(d + 1, lb)
                        nodes[idx].right = build(d + 1, rb)
                        return idx
            ctr = [0.5 * (lo + hi) for lo, hi in box]
            s = float(surrogate_ips(ctr[0], ctr[1], ctr[2], ctr[3]))
            nodes[idx].leaf = float(np.float32(s / n_trees * (1.0 + noise * rng.standard_normal())))
            return idx

        build(0, dom)
        trees.append(nodes)
    return Ensemble(trees, float(np.float32(base)), depth)


def config_ensemble(cfg: Config) -> Ensemble:
    """The ensemble paired with a config (seed = config seed)."""
    kv_max = cfg.run_hi * 1100.0 / cfg.N if not cfg.c1_shape else cfg.run_hi * 17
    return gen_ensemble(cfg.n_trees, cfg.depth, cfg.seed, freq_levels(cfg.F, cfg.f_lo, cfg.f_hi),
                        b_max=cfg.max_batch, kv_max=kv_max, ragged=cfg.ragged)


def config_inputs(cfg: Config, i0: int = 0, i1: int | None = None):
    """Everything one decision round needs for instances [i0, i1) of ``cfg``."""
    inst, req, t_dead = gen_instances(cfg, i0, i1)
    return dict(inst=inst, req=req, t_dead=t_dead, H=cfg.H,
                freq=freq_levels(cfg.F, cfg.f_lo, cfg.f_hi), tbt_slo=np.float32(cfg.tbt_slo))


# ----------------------------------------------------------------------------------------------
# trace replay (BASELINE configs[3]: 1M requests across 4,096 instance states, re-decided every
# iteration).  Inputs only: an initial state in fixed request slots and an arrival stream.
# ----------------------------------------------------------------------------------------------

# E2E SLO per engine size (Table II: p99 at max load, seconds)
E2E_SLO = {1: 37.7, 2: 30.2, 4: 31.3, 8: 44.0}
# relative request rate per 4-minute bin of the 60-minute Azure trace (medians 5-8
# RPS, peak ~16 near the midpoint, never idle)
RPS_PROFILE = np.array([5, 6, 6, 7, 8, 9, 11, 16, 12, 9, 8, 7, 6, 6, 5], dtype=np.float64)


@dataclasses.dataclass(frozen=True)
class ReplayConfig:
    n_inst: int = 4096
    n_requests: int = 1_000_000
    span_s: float = 25.0      # the 60-minute profile time-scaled to this span
    slot_cap: int = 512       # request slots per instance (running + queued)
    base: Config = CONFIGS["C4"]
    seed: int = 1004


def gen_replay(rc: ReplayConfig):
    """-> dict(inst, req[I*cap], t_dead[I*cap], arr_t, arr_req, arr_dead, arr_off[I+1], freq, H, ...).

    Initial instance states come from the configs[3] generator (clipped to the slots); arrivals
    are drawn over the rate profile, sorted, dealt round-robin to instances; each carries its
    prompt length, its (exactly predicted) generation length and deadline = arrival + E2E SLO of
    its engine size."""
    cfg = dataclasses.replace(rc.base, n_inst=rc.n_inst)
    inst0, req0, dead0 = gen_instances(cfg)
    I, cap = rc.n_inst, rc.slot_cap
    inst = inst0.copy()
    req = np.zeros(I * cap, REQ_DTYPE)
    dead = np.zeros(I * cap, np.float64)
    for i in range(I):
        b = int(inst0[i]["req_begin"])
        nr, nq = int(inst0[i]["n_run"]), int(inst0[i]["n_queue"])
        nr2 = min(nr, cap)
        nq2 = min(nq, cap - nr2)
        req[i * cap:i * cap + nr2] = req0[b:b + nr2]
        dead[i * cap:i * cap + nr2] = dead0[b:b + nr2]
        req[i * cap + nr2:i * cap + nr2 + nq2] = req0[b + nr:b + nr + nq2]
        dead[i * cap + nr2:i * cap + nr2 + nq2] = dead0[b + nr:b + nr + nq2]
        inst[i]["req_begin"] = i * cap
        inst[i]["n_run"], inst[i]["n_queue"] = nr2, nq2
    t0 = float(inst["t_cur"].max())
    for i in range(I):                       # one common clock; deadlines keep their slack
        dead[i * cap:(i + 1) * cap] += t0 - float(inst[i]["t_cur"])
    inst["t_cur"] = t0
    rng = np.random.default_rng([rc.seed, 99])
    n = rc.n_requests
    nb = len(RPS_PROFILE)
    bins = rng.choice(nb, size=n, p=RPS_PROFILE / RPS_PROFILE.sum())
    t = t0 + (bins + rng.random(n)) * (rc.span_s / nb)
    t.sort()
    owner = np.arange(n) % I                 # round-robin dealing
    order = np.lexsort((t, owner))           # by instance, then time
    t, owner = t[order], owner[order]
    H = cfg.H
    r = _lognormal_int(rng, 250.0, 0.5, 10, min(700, H), n)
    q = _lognormal_int(rng, 600.0, 0.9, 1, 4000, n)
    arr_req = np.zeros(n, REQ_DTYPE)
    arr_req["q"], arr_req["r"] = q, r
    slo = np.vectorize(E2E_SLO.get)(inst["tp"][owner]).astype(np.float64)
    arr_off = np.concatenate([[0], np.cumsum(np.bincount(owner, minlength=I))]).astype(np.int64)
    return dict(inst=inst, req=req, t_dead=dead, arr_t=t, arr_req=arr_req, arr_dead=t + slo, arr_off=arr_off,
                freq=freq_levels(cfg.F, cfg.f_lo, cfg.f_hi), tbt_slo=np.float32(cfg.tbt_slo), H=H, slot_cap=cap,
                t0=t0)
