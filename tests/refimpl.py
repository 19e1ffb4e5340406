"""Independent, test-only re-derivations used to PIN the oracle (never the CUDA path).

None of this calls oracle/ code; each helper restates a definition from PAPER.md in
a different form than oracle.c uses, so a slip in either shows up as a mismatch:

* ``token_alloc_curve``  -- a token-by-token paged-KV allocator
  instead of Eq. 1's closed form;
* ``BoxModel``           -- evaluates an ensemble by leaf-box membership
  (each leaf owns the half-open box its root path carves) instead of a walk;
* ``brute_decide``       -- the whole decision with exact ``Fraction`` times,
  the token allocator and BoxModel, for tiny inputs;
* ``replay_completion``  -- iteration-by-iteration engine replay at a fixed
  frequency (SPEC's zero-drift property).
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np

LOST = 1
ST_EMPTY, ST_BYPASS_LOST, ST_INFEASIBLE, ST_KV_OVER = 1, 2, 4, 8
ST_QUEUE_BLOCKED, ST_IPS_CLAMPED, ST_BAD_INPUT = 16, 32, 64


def token_alloc_curve(a: int, q: int, r: int, N: int, H: int) -> list[int]:
    """Blocks held by one request at iterations k..k+H-1 (m = 1..H).

    The request was scheduled at s = k - a with its |q| prompt tokens cached;
    every iteration after s appends one generated token; blocks of N tokens are
    allocated on demand (a new block when all held blocks are full); the entry is
    struck after r iterations."""
    out = []
    tokens = blocks = 0

    def push():
        nonlocal tokens, blocks
        if tokens == blocks * N:
            blocks += 1
        tokens += 1

    for _ in range(q):
        push()
    step = 0                      # iterations since s
    while step < a + H:
        if step >= a:
            out.append(blocks if step < r else 0)
        push()
        step += 1
    return out


class BoxModel:
    """Ensemble evaluated by box membership, fp32 accumulation in tree order."""

    def __init__(self, ens):
        self.base = np.float32(ens.base)
        self.trees = []
        for nodes in ens.trees:
            leaves = []

            def rec(i, box):
                nd = nodes[i]
                if nd.feature == -1:
                    leaves.append((box, np.float32(nd.leaf)))
                    return
                lo, hi = box[nd.feature]
                lb = list(box); lb[nd.feature] = (lo, min(hi, nd.threshold))
                rb = list(box); rb[nd.feature] = (max(lo, nd.threshold), hi)
                rec(nd.left, lb)     # x < thr
                rec(nd.right, rb)    # x >= thr
            rec(0, [(-np.inf, np.inf)] * 4)
            self.trees.append(leaves)

    def leaf_values(self, X: np.ndarray, t: int) -> np.ndarray:
        X = np.asarray(X, dtype=np.float32)
        out = np.full(len(X), np.nan, dtype=np.float32)
        hits = np.zeros(len(X), dtype=np.int64)
        for box, v in self.trees[t]:
            inside = np.ones(len(X), dtype=bool)
            for f, (lo, hi) in enumerate(box):
                inside &= (X[:, f] >= np.float32(lo) if lo != -np.inf else True)
                inside &= (X[:, f] < np.float32(hi) if hi != np.inf else True)
            out[inside] = v
            hits += inside
        assert (hits == 1).all(), "boxes must partition feature space"
        return out

    def raw(self, X) -> np.ndarray:
        X = np.atleast_2d(np.asarray(X, dtype=np.float32))
        acc = np.full(len(X), self.base, dtype=np.float32)
        for t in range(len(self.trees)):
            acc = (acc + self.leaf_values(X, t)).astype(np.float32)
        return acc

    def ips(self, X):
        raw = self.raw(X)
        c = np.where(np.isnan(raw), np.float32(2.0 ** -4), np.clip(raw, np.float32(2.0 ** -4), np.float32(2.0 ** 17)))
        return c.astype(np.float32), (np.isnan(raw) | (c != raw))


def valid_inputs(inst, reqs, H, n_req) -> bool:
    """The validity rules of include/tp.h / DESIGN.md §3 (BAD_INPUT otherwise)."""
    LIM = 1 << 24
    if inst["N"] < 1 or inst["tp"] < 1 or inst["tp"] >= LIM or inst["n_run"] < 0 or inst["n_queue"] < 0:
        return False
    if inst["kv_cap"] < 0 or inst["max_batch"] < 0 or inst["req_begin"] < 0:
        return False
    if int(inst["req_begin"]) + int(inst["n_run"]) + int(inst["n_queue"]) > n_req:
        return False
    foot = 0
    for e, rq in enumerate(reqs):
        a, q, r = int(rq["a"]), int(rq["q"]), int(rq["r"])
        l = r - a
        if a < 0 or q < 1 or r < 1 or a >= LIM or q >= LIM or not (1 <= l <= H):
            return False
        if e >= inst["n_run"] and a != 0:
            return False
        foot += -(-(a + l - 1 + q) // int(inst["N"]))
    return foot < LIM


def _times(box, tpf, B, KV, n, f):
    """Exact T_R (Fractions) at frequency f over m = 1..n, and whether a value was clamped."""
    X = np.array([[tpf, B[m], KV[m], f] for m in range(n)], dtype=np.float32)
    ips, clamped = box.ips(X)
    TR, s = [], Fraction(0)
    for v in ips:
        s += Fraction(float(np.float32(1.0) / np.float32(v)))
        TR.append(s)
    return TR, bool(clamped.any())


def brute_decide(box: BoxModel, inst, reqs, deads, H, freq, tbt, admission=0, search="exhaustive"):
    """Full decision for ONE instance with exact rationals; returns dict like the oracle's.
    admission=1: the paper's admission control (checks 1-3 at f_max, lost marking)."""
    F = len(freq)
    res = dict(B=[0] * H, KV=[0] * H, n=0, n_adm=0, status=0, level=0, adm_lost=0)
    if not valid_inputs(inst, reqs, H, 10 ** 12):
        res.update(status=ST_BAD_INPUT, level=F - 1)
        return res
    N, C, mb = int(inst["N"]), int(inst["kv_cap"]), int(inst["max_batch"])
    nr, nq = int(inst["n_run"]), int(inst["n_queue"])
    B = [0] * H
    KV = [0] * H
    for rq in reqs[:nr]:
        cur = token_alloc_curve(int(rq["a"]), int(rq["q"]), int(rq["r"]), N, H)
        for m in range(H):
            KV[m] += cur[m]
            B[m] += cur[m] > 0
    st = ST_KV_OVER if max(KV) > C else 0
    adm = 0
    marked = set()
    tpf = float(inst["tp"])
    for c, rq in enumerate(reqs[nr:nr + nq]):
        if admission and c >= 32:
            st |= ST_QUEUE_BLOCKED
            break
        cur = token_alloc_curve(0, int(rq["q"]), int(rq["r"]), N, H)
        if not (B[0] + 1 <= mb and max(KV[m] + cur[m] for m in range(H)) <= C):
            st |= ST_QUEUE_BLOCKED
            break
        lost_c = False
        if admission:
            B2 = [B[m] + (cur[m] > 0) for m in range(H)]
            KV2 = [KV[m] + cur[m] for m in range(H)]
            members = list(range(nr + c + 1))
            nv = max(int(reqs[e]["r"]) - int(reqs[e]["a"]) for e in members)
            TR, _ = _times(box, tpf, B2, KV2, nv, freq[F - 1])
            ok2 = TR[-1] / nv <= Fraction(float(np.float32(tbt)))
            others = self_ = False
            for e in members:
                if int(reqs[e]["flags"]) & LOST or (e >= nr and (e - nr) in marked and e != nr + c):
                    continue
                l = int(reqs[e]["r"]) - int(reqs[e]["a"])
                slack = Fraction(float(np.float64(deads[e]) - np.float64(inst["t_cur"])))
                if not TR[l - 1] < slack:
                    if e == nr + c:
                        self_ = True
                    else:
                        others = True
            if not ok2 or others:
                st |= ST_QUEUE_BLOCKED
                break
            lost_c = self_
        for m in range(H):
            KV[m] += cur[m]
            B[m] += cur[m] > 0
        if lost_c:
            marked.add(c)
            res["adm_lost"] |= 1 << c
        adm += 1
    sched = list(range(nr + adm))
    n = max([int(reqs[e]["r"]) - int(reqs[e]["a"]) for e in sched], default=0)
    res.update(B=B, KV=KV, n=n, n_adm=adm)
    if n == 0:
        res.update(status=st | ST_EMPTY, level=0)
        return res
    if any(int(reqs[e]["flags"]) & LOST for e in sched) or marked:
        res.update(status=st | ST_BYPASS_LOST, level=F - 1)
        return res
    flags = [st]

    def passes(u):
        TR, clamped = _times(box, tpf, B, KV, n, freq[u])
        if clamped:
            flags[0] |= ST_IPS_CLAMPED
        ok = TR[-1] / n <= Fraction(float(np.float32(tbt)))
        for e in sched:
            l = int(reqs[e]["r"]) - int(reqs[e]["a"])
            slack = Fraction(float(np.float64(deads[e]) - np.float64(inst["t_cur"])))
            ok = ok and TR[l - 1] < slack
        return ok

    if search == "exhaustive":
        ok = [passes(u) for u in range(F)]
        level = ok.index(True) if any(ok) else None
    else:
        # binary search over the frequency range; the top level must pass
        level = None
        if passes(F - 1):
            lo, hi = 0, F - 1
            while lo < hi:
                mid = (lo + hi) // 2
                if passes(mid):
                    hi = mid
                else:
                    lo = mid + 1
            level = lo
    st = flags[0]
    if level is None:
        level = F - 1
        st |= ST_INFEASIBLE
    res.update(status=st, level=level)
    return res


def replay_completion(box: BoxModel, inst, reqs, n_sched: int, freq_u: float, N: int):
    """Engine replay at a fixed frequency: iterate m = 1, 2, ... with the live batch
    (requests not yet finished) and live KV (token allocator), advance time by the
    fp32 reciprocal of the model's IPS, exactly.  Returns each scheduled request's
    completion time (Fraction, seconds after t_cur)."""
    state = []
    for e in range(n_sched):
        rq = reqs[e]
        a, q, r = int(rq["a"]), int(rq["q"]), int(rq["r"])
        toks = q + a
        state.append(dict(left=r - a, tokens=toks, blocks=-(-toks // N)))
    now = Fraction(0)
    done = [None] * n_sched
    while any(d is None for d in done):
        live = [i for i in range(n_sched) if done[i] is None]
        kv = sum(state[i]["blocks"] for i in live)
        ips, _ = box.ips(np.array([[float(inst["tp"]), len(live), kv, freq_u]], dtype=np.float32))
        now += Fraction(float(np.float32(1.0) / ips[0]))
        for i in live:          # every live request emits one token this iteration
            s = state[i]
            s["left"] -= 1
            if s["left"] == 0:
                done[i] = now
            else:
                if s["tokens"] == s["blocks"] * N:
                    s["blocks"] += 1
                s["tokens"] += 1
    return done


def replay_advance(inst, req, t_dead, arr_next, data, dec, oracle_model, freq, cap, adm_lost=None):
    """One engine iteration per instance (the semantics include/tp.h states for tp_replay_advance),
    written independently of replay.cu.  dec: oracle decision dict for the same state."""
    inst = inst.copy()
    req_out = np.zeros_like(req)
    dead_out = np.zeros_like(t_dead)
    arr_next = arr_next.copy()
    stats = np.zeros(5, np.int64)
    for i in range(len(inst)):
        b = i * cap
        nr, nq = int(inst[i]["n_run"]), int(inst[i]["n_queue"])
        if dec["status"][i] & ST_BAD_INPUT:
            req_out[b:b + nr + nq] = req[b:b + nr + nq]
            dead_out[b:b + nr + nq] = t_dead[b:b + nr + nq]
            continue
        n, nadm, u = int(dec["n"][i]), int(dec["n_adm"][i]), int(dec["level"][i])
        t_cur = float(inst[i]["t_cur"])
        j0, j1 = int(arr_next[i]), int(data["arr_off"][i + 1])
        if n > 0:
            raw = oracle_model.predict_raw(inst[i]["tp"], dec["B"][i, 0], dec["KV"][i, 0], freq[u])
            ips = np.float32(2.0 ** -4) if np.isnan(raw) else np.clip(raw, np.float32(2.0 ** -4), np.float32(2.0 ** 17))
            t_new = t_cur + float(np.float32(1.0) / np.float32(ips))
            it = 1
        else:
            t_new = t_cur
            if j0 < j1 and data["arr_t"][j0] > t_new:
                t_new = float(data["arr_t"][j0])
            it = 0
        out = []
        for e in range(nr + nadm if it else 0):
            r = req[b + e].copy()
            if adm_lost is not None and e >= nr and e - nr < 32 and (int(adm_lost[i]) >> (e - nr)) & 1:
                r["flags"] |= LOST
            r["a"] += 1
            if r["r"] - r["a"] == 0:
                stats[0] += 1
                stats[1] += t_new < t_dead[b + e]
            else:
                out.append((r, t_dead[b + e]))
        nrun = len(out)
        q0 = nr + nadm if it else nr
        for e in range(q0, nr + nq):
            out.append((req[b + e], t_dead[b + e]))
        arrived = 0
        while j0 + arrived < j1 and data["arr_t"][j0 + arrived] <= t_new:
            arrived += 1
        take = min(arrived, max(cap - len(out), 0))
        for k in range(take):
            r = data["arr_req"][j0 + k].copy()
            r["a"] = 0
            out.append((r, data["arr_dead"][j0 + k]))
        for k, (r, d) in enumerate(out):
            req_out[b + k] = r
            dead_out[b + k] = d
        stats[2] += arrived - take
        stats[3] += it
        stats[4] += nadm if it else 0
        inst[i]["n_run"], inst[i]["n_queue"] = nrun, len(out) - nrun
        inst[i]["k"] += it
        inst[i]["t_cur"] = t_new
        arr_next[i] = j0 + arrived
    return inst, req_out, dead_out, arr_next, stats
