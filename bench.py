#!/usr/bin/env python
"""Benchmark of the throttLL'eM frequency-selection hot path (BASELINE.json metric: frequency
decisions/s and GBDT grid evals/s at 1/2/4/8 B200, vs roofline).

One step = one decision round over the workload: K1c projection (+ pieces, cell claims, Eq. 4
minima) -> K2 GBDT on the distinct cells -> K3c SLO scan + frequency choice (+ one NCCL all-gather
of the decisions when N > 1).  Inputs are synthetic and seeded (paper_2408_05235_b200/workload.py),
already resident in HBM when the timed region starts.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C5] [--impl ours|reference]

Default workload C5 = BASELINE.json configs[4], the configuration the metric is quoted on: 262,144
instances sharded over the N GPUs (strong scaling: rank r decides 262,144/N of them, grouped by
engine size, shard.shard_by_engine).  N > 1
runs under torchrun, one process per GPU, NCCL.  --workload C2/C3 time the other configs (C2: weak
scaling, 1,024 instances per GPU); --workload C4 is the trace replay.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2408_05235_b200 import workload as W  # noqa: E402

DESCR = {
    "C1": "BASELINE configs[0]: 1 instance, 8 running + 4 queued, 16 KV blocks/req cap, 8 freq levels, 64-iter horizon, 50-tree depth-6 GBDT",
    "C2": "BASELINE configs[1]: 1,024 instances, batch<=64, 16 freq levels, 512-iter horizon, 200-tree depth-8 GBDT",
    "C3": "BASELINE configs[2]: 65,536 instances, synthetic Azure-like trace, batch<=256, 32 freq levels, 1,024-iter horizon (200-tree depth-8 assumed)",
    "C4": "BASELINE configs[3]: trace replay, 1M requests across 4,096 TP instance states re-decided every iteration, 500-tree depth-8 GBDT",
    "C5": "BASELINE configs[4]: scaling sweep, 262,144 instances sharded over N B200 with NCCL gather of decisions (C3 generator, 200-tree depth-8)",
}
SKIP = 64 | 1 | 2
METRIC = "frequency decisions/sec"


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def parse_emulate(s):
    """'R/N' -> (R, N); None -> (0, 1)."""
    if not s:
        return 0, 1
    r, n = (int(x) for x in s.split("/"))
    if not (0 <= r < n):
        raise SystemExit(f"--emulate-shard {s}: need 0 <= R < N")
    return r, n


def shard_of(cfg, rank, world):
    """Instance range [i0, i1) of this rank and the global instance count (shard.py)."""
    from paper_2408_05235_b200 import shard
    if cfg.name == "C2":            # weak scaling: 1,024 new instances per GPU
        return (*shard.weak_range(cfg.n_inst, rank), cfg.n_inst * world)
    return (*shard.shard_range(cfg.n_inst, rank, world), cfg.n_inst)   # strong: fixed total


class Clocks:
    """nvidia-smi sampling during the timed region (clock line of B200_PROFILING.md)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev_index):
        self.dev = dev_index
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "100", "-i", str(self.dev)], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.25)
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return platform.processor() or "unknown"


def stratified(n_total, k, offset=0):
    """k instances spread evenly over [0, n_total) (the oracle's bounded sample of a workload)."""
    k = max(1, min(k, n_total))
    return np.unique((np.arange(k, dtype=np.int64) * n_total) // k + offset % max(1, n_total // k))


def sample_inputs(inputs, idx):
    """A self-contained round of the instances idx (request rows copied, req_begin rebased)."""
    inst = inputs["inst"][idx].copy()
    b = inputs["inst"]["req_begin"][idx].astype(np.int64)
    c = (inputs["inst"]["n_run"][idx] + inputs["inst"]["n_queue"][idx]).astype(np.int64)
    rows = np.concatenate([np.arange(x, x + y) for x, y in zip(b, c)]) if len(idx) else np.zeros(0, np.int64)
    inst["req_begin"] = np.concatenate([[0], np.cumsum(c)[:-1]]).astype(np.int32)
    return dict(inputs, inst=inst, req=inputs["req"][rows], t_dead=inputs["t_dead"][rows])


def oracle_time(blob, sub, threads, search):
    from oracle import oracle
    m = oracle.Model(blob)
    t = time.perf_counter()
    oracle.decide(m, sub["inst"], sub["req"], sub["t_dead"], sub["H"], sub["freq"], sub["tbt_slo"],
                  want_grid=False, want_curves=False, threads=threads, search=search)
    return time.perf_counter() - t


def cpu_baseline(cfg, blob, inputs, search="exhaustive", budget_s=15.0):
    """The oracle, as it stands, on this host's cores, on a bounded stratified sample of the same
    workload (all threads, plus a 1-thread figure on a smaller sample)."""
    threads = os.cpu_count() or 1
    I = len(inputs["inst"])
    k = min(I, max(threads * 4, 32))
    dt = oracle_time(blob, sample_inputs(inputs, stratified(I, k)), threads, search)
    if k < I and dt < budget_s:
        k = min(I, max(k, int(k * budget_s / max(dt, 1e-3))))
        dt = oracle_time(blob, sample_inputs(inputs, stratified(I, k)), threads, search)
    k1 = max(1, min(I, int(k * 2.0 / max(dt * threads, 1e-3))))        # ~2 s single-threaded
    dt1 = oracle_time(blob, sample_inputs(inputs, stratified(I, k1, 1)), 1, search)
    return {"value": k / dt, "unit": "decisions/s", "cores": threads, "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": f"{k} of {len(inputs['inst'])} instances of {cfg.name} (stratified, every "
                      f"{max(1, I // k)}th) on {threads} threads, {dt:.1f} s; "
                      + ("all F levels evaluated" if search == "exhaustive" else "the paper's binary search"),
            "one_thread": {"value": k1 / dt1, "unit": "decisions/s", "cores": 1,
                           "sample": f"{k1} instances (stratified), {dt1:.1f} s"}}


def bench_reference(args, cfg):
    """--impl reference: the CPU oracle is this tier's reference arm (rank 0 only), on the same
    workload as our arm: each step decides a bounded stratified sample of it."""
    if env_int("RANK", 0) != 0:
        return
    blob = W.write_blob(W.config_ensemble(cfg))
    world = max(args.gpus, env_int("WORLD_SIZE", 1))
    _, _, I_glob = shard_of(cfg, 0, world)
    inputs = W.config_inputs(dataclasses_replace(cfg, I_glob))
    per_step = args.ref_per_step or {"C1": 1, "C2": 256, "C3": 256, "C4": 128, "C5": 256}[cfg.name]
    threads = os.cpu_count() or 1
    subs = [sample_inputs(inputs, stratified(I_glob, per_step, s)) for s in range(args.warmup + args.steps)]
    for s in range(args.warmup):
        oracle_time(blob, subs[s], threads, args.search)
    dt = sum(oracle_time(blob, subs[args.warmup + s], threads, args.search) for s in range(args.steps))
    v = per_step * args.steps / dt
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "decisions/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak" if cfg.name == "C2" else "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": DESCR[cfg.name], "name": cfg.name, "global_instances": I_glob,
                       "instances_per_step": per_step, "search": args.search,
                       "sample": "each step decides a different stratified sample of the same workload"},
            "cpu_baseline": {"value": v, "unit": "decisions/s", "cores": threads, "kind": "oracle",
                             "cpu_model": cpu_model(),
                             "sample": f"{per_step} of {I_glob} instances of {cfg.name} per step (stratified)"},
            "e2e": {"value": v, "unit": "decisions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def slice_replay(data, i0, i1):
    """Instances [i0, i1) of a replay (fixed request slots, per-instance arrival streams)."""
    cap = int(data["slot_cap"])
    inst = data["inst"][i0:i1].copy()
    inst["req_begin"] -= i0 * cap
    a0, a1 = int(data["arr_off"][i0]), int(data["arr_off"][i1])
    return dict(data, inst=inst, req=data["req"][i0 * cap:i1 * cap], t_dead=data["t_dead"][i0 * cap:i1 * cap],
                arr_t=data["arr_t"][a0:a1], arr_req=data["arr_req"][a0:a1], arr_dead=data["arr_dead"][a0:a1],
                arr_off=data["arr_off"][i0:i1 + 1] - a0)


def bench_replay(args, cfg, rank, world, local, dist, dist_test):
    """BASELINE configs[3]: 1M requests over 4,096 instance states, all re-decided every iteration.
    A round = decide every instance (tp_decide: K1c -> K2 -> K3c) + advance every instance one
    engine iteration (tp_replay_advance), all on the GPU; instances are split over ranks.  The
    WHOLE replay is timed (every round until every arrival is consumed and every request has
    finished, or --replay-cap rounds): sustained decisions/s = instances x rounds / sum of round
    times, per-round p50 / p90.  e2e: the same replay through the public API with the trace
    uploaded from pinned host memory inside the timed region and every round's (level, status)
    read back."""
    import torch
    from paper_2408_05235_b200 import replay, runner, shard, tp
    dev = torch.device("cuda", local)
    rc = W.ReplayConfig()
    data = W.gen_replay(rc)
    i0, i1 = shard.shard_range(rc.n_inst, rank, world)
    data = slice_replay(data, i0, i1)
    I = i1 - i0
    blob = W.write_blob(W.config_ensemble(cfg))
    model = tp.Gbdt(blob, local)
    info = model.info()
    rp = replay.Replay(data, model, dev, admission=args.admission, search=args.search)
    stream = torch.cuda.current_stream(dev)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    for _ in range(max(args.warmup, 3)):              # warm-up rounds (then back to the initial state)
        rp.round(stream)
    rp.reset(stream)
    torch.cuda.synchronize(dev)
    cap = args.replay_cap

    phase = [None]

    def whole(ev_pairs, readback=None):
        """Rounds until drained, or until every arrival has been consumed and no instance has a
        running request left (what remains is queued and blocked for good: FIFO head-of-line
        requests whose KV footprint exceeds their instance's capacity), or cap; checked every 100
        rounds."""
        r = 0
        phase[0] = None
        while r < cap:
            n = min(100, cap - r)
            for k in range(n):
                a, b = ev_pairs[r + k]
                a.record(stream)
                rp.round(stream)
                if readback is not None:
                    readback.copy_(torch.stack([rp.level, rp.status]), non_blocking=True)
                b.record(stream)
            r += n
            torch.cuda.synchronize(dev)
            if rp.finished():
                break
            if rp.arrivals_consumed():
                if phase[0] is None:
                    phase[0] = r         # (within 100 rounds) every arrival has joined a queue
                if rp.running() == 0:
                    break                # what is left is queued and blocked for good
        return r

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(cap)]
    clocks = Clocks(local)
    if world > 1:
        dist.barrier()
    clocks.start()
    time.sleep(0.3)
    rounds = whole(ev)
    clk = clocks.stop()
    round_ms = np.array([a.elapsed_time(b) for a, b in ev[:rounds]])
    arrivals_rounds = phase[0] or rounds
    stats = rp.stats_dict()
    drained = rp.finished()
    blocked = rp.in_flight()
    # e2e: the trace uploaded from pinned host memory inside the timed region, every round's
    # decisions read back to pinned host memory
    out_h = torch.empty((2, max(I, 1)), dtype=torch.int32).pin_memory()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    e0.record(stream)
    rp.reset(stream)
    ev2 = [(torch.cuda.Event(enable_timing=False), torch.cuda.Event(enable_timing=False)) for _ in range(cap)]
    rounds2 = whole(ev2, readback=out_h[:, :I])
    e1.record(stream)
    torch.cuda.synchronize(dev)
    e2e_ms = e0.elapsed_time(e1) - 0.0
    # per-kernel breakdown and rooflines on snapshots of the replay state (initial and mid-replay):
    # the compact path's kernels on exactly those inputs, with events between the kernels
    snaps = []
    rp.reset(stream)
    for target in (0, rounds // 2):
        while rp.rounds < target:
            rp.round(stream)
        inst_h, req_h, td_h, _ = rp.state()
        snaps.append(dict(inst=inst_h, req=req_h, t_dead=td_h, H=data["H"], freq=data["freq"],
                          tbt_slo=data["tbt_slo"]))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    kern_rows = []
    for sn in snaps:
        rnd = runner.Round(sn, dev, k2_mode="compact", model=model, search=args.search)
        rnd.bkv = False
        for _ in range(2):
            rnd.run(model, stream)
        evk = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(10)]
        for e in evk:
            flush.zero_()
            e[0].record(stream)
            rnd.project(stream)
            e[1].record(stream)
            rnd.predict(model, stream)
            e[2].record(stream)
            rnd.select(stream)
            e[3].record(stream)
        torch.cuda.synchronize(dev)
        k_ms = np.array([[e[j].elapsed_time(e[j + 1]) for j in range(3)] for e in evk]).mean(axis=0)
        cs = tp.compact_stats(model, rnd.work, rnd.I, rnd.H, rnd.F)
        nadm = rnd.n_adm[:rnd.I].cpu().numpy().astype(np.int64)
        kern_rows.append((sn, k_ms, cs, int(sn["inst"]["n_run"].astype(np.int64).sum() + nadm.sum())))
        del rnd
    tot = torch.tensor([float(round_ms.sum()), e2e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        c = tot.cpu() if dist_test else tot
        dist.all_reduce(c, op=dist.ReduceOp.MAX)
        tot = c.to(dev)
    if rank != 0:
        return
    peaks = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", 6553.6))
    smax = float(peaks.get("sm_max_mhz", 1965.0))
    lds_peak = sms * 128 * smax * 1e6 / 1e9
    per_row = info.n_trees * (info.depth + 1) * 4
    snaps_out = []
    for (sn, k_ms, cs, n_sched), tag in zip(kern_rows, ("initial state", f"state after {rounds // 2} rounds")):
        n_req = int((sn["inst"]["n_run"].astype(np.int64) + sn["inst"]["n_queue"]).sum())
        Is = len(sn["inst"])
        k1b = 48 * Is + 16 * n_req + 8 * n_sched + 12 * Is + 16 * cs["pieces"]
        k3b = 12 * Is + 16 * cs["pieces"]
        kern = {"k1": roof("hbm", "K1c", k1b, k_ms[0], hbm, None, basis="as the C5 line"),
                "k2": roof("smem", "k2_cells_phase", cs["cells"] * len(sn["freq"]) * per_row, k_ms[1], lds_peak,
                           None, basis=f"{per_row} B per evaluated row"),
                "k3": roof("hbm", "K3c", k3b, k_ms[2], hbm, None, basis="as the C5 line")}
        snaps_out.append({"state": tag, "per_kernel": kern, "counts": dict(cs, instances=Is, requests=n_req)})
    dom = max(snaps_out[0]["per_kernel"], key=lambda k: snaps_out[0]["per_kernel"][k]["ms"])
    roofline = dict(snaps_out[0]["per_kernel"][dom], dominant=dom, snapshots=snaps_out)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, blob, snaps[0], search=args.search)
        cpu["sample"] += " (instances of the replay's initial state)"
    t_ms = float(tot[0])
    line = {
        "metric": METRIC, "value": I * world * rounds / (t_ms / 1e3), "unit": "decisions/s",
        "n_gpus": world, "steps": rounds, "warmup": max(args.warmup, 3),
        "ms_per_step": t_ms / rounds, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": DESCR["C4"], "name": "C4", "instances": rc.n_inst, "requests": rc.n_requests,
                   "span_s": rc.span_s, "trees": cfg.n_trees, "depth": cfg.depth, "F": cfg.F, "H": cfg.H,
                   "step": "one round: decide all instances + advance all instances one engine iteration "
                           "(GPU-resident replay)",
                   "timed": f"the whole replay: {rounds} rounds"
                            + (" until drained" if drained else
                               f" until every arrival was consumed and no request was running "
                               f"({blocked} queued requests blocked for good by their instance's KV capacity)"
                               if rounds < cap else f" (cap {cap}, not drained)"),
                   "admission": (f"full admission control (checks 1-3 at f_max, lost marking), q_max={args.admission}"
                                 if args.admission else "check 1 + batch cap gate"),
                   "search": args.search,
                   "l2": "not flushed: the replay state (~60 MB) is re-used every round by design"},
        "drained": drained,
        "arrival_phase": {"rounds": arrivals_rounds,
                          "decisions_per_sec": I * world * arrivals_rounds / (float(round_ms[:arrivals_rounds].sum()) / 1e3),
                          "note": "rounds until every arrival had joined a queue (checked every 100 rounds); "
                                  "the rest of the replay drains the queues"},
        "blocked_requests_at_end": blocked,
        "round_ms_pctl": {"p10": float(np.percentile(round_ms, 10)), "p50": float(np.percentile(round_ms, 50)),
                          "p90": float(np.percentile(round_ms, 90)), "max": float(round_ms.max())},
        "replay_stats": stats,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": {"value": I * world * rounds2 / (float(tot[1]) / 1e3), "unit": "decisions/s",
                "h2d_bytes_per_step": rp.host_bytes() / max(rounds2, 1), "d2h_bytes_per_step": 8 * I,
                "api": "Replay.reset (trace + state uploaded from pinned host memory, timed) + every round "
                       "tp_decide + tp_replay_advance + (level, status) read back to pinned host memory",
                "rounds": rounds2},
        # per round: K1c (+ its hand-over kernel at large batches), the cell-list collector, the K2
        # phases, K3c, the advance
        "gpu_launches": (None if args.admission else
                         (4 + k2_phases(info) + int(I * 2 > sms * 32)) * rounds),
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="C5", choices=sorted(DESCR))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--ref-per-step", type=int, default=None,
                    help="reference arm: instances the oracle decides per step (default per workload)")
    ap.add_argument("--instances", type=int, default=None,
                    help="override the workload's global instance count (tests; the line says so)")
    ap.add_argument("--emulate-shard", default=None,
                    help="R/N: one process decides rank R's shard of an N-way C5 sweep (no gather; a "
                         "per-rank step time for DESIGN.md's scaling projection, not a multi-GPU number)")
    ap.add_argument("--dump-decisions", default=None,
                    help="rank 0 writes the gathered [2, I] (level, status) rows of the last step (.npy)")
    ap.add_argument("--replay-cap", type=int, default=60000,
                    help="C4: at most this many rounds (the replay normally drains before)")
    ap.add_argument("--admission", type=int, default=0,
                    help="C4 replay: run the paper's full admission control on up to N queued requests per instance")
    ap.add_argument("--search", default="exhaustive", choices=["exhaustive", "binary"],
                    help="K3 order: lowest passing level over all levels (reading A-13, default) or the "
                         "paper's binary search (P:555, reading A-24)")
    ap.add_argument("--graph", dest="graph", action="store_true", default=True,
                    help="time the step as a replayed CUDA graph of its kernels (default; SURVEY §8d)")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="launch the kernels one by one in the timed steps")
    args = ap.parse_args()
    cfg = W.CONFIGS[args.workload]
    if args.instances:
        cfg = dataclasses_replace(cfg, args.instances)
    if args.impl == "reference":
        return bench_reference(args, cfg)

    import torch
    import torch.distributed as dist
    from paper_2408_05235_b200 import runner, shard, tp

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE", file=sys.stderr)
    # TP_BENCH_DIST_TEST=1 (test aid only): several ranks on ONE GPU over gloo, to exercise the
    # multi-rank code path on a 1-GPU box; real runs use one GPU per rank and NCCL.
    dist_test = os.environ.get("TP_BENCH_DIST_TEST") == "1"
    if dist_test:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if dist_test:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def all_reduce(t, op):
        if not dist_test:
            dist.all_reduce(t, op=op)
            return
        c = t.cpu()
        dist.all_reduce(c, op=op)
        t.copy_(c)

    if cfg.name == "C4":
        bench_replay(args, cfg, rank, world, local, dist, dist_test)
        if world > 1:
            dist.destroy_process_group()
        return
    i0, i1, I_glob = shard_of(cfg, rank, world)
    blob = W.write_blob(W.config_ensemble(cfg))
    em_r, em_n = parse_emulate(args.emulate_shard)
    shard_ix, perm = None, None
    if cfg.name != "C2" and (world > 1 or em_n > 1):
        # strong scaling grouped by engine size (shard.shard_by_engine): every rank generates the
        # global round (untimed) and keeps its instances
        cfg_g = dataclasses_replace(cfg, I_glob)
        tpv = W.tp_of(cfg_g)
        r_, n_ = (rank, world) if world > 1 else (em_r, em_n)
        shard_ix = shard.shard_by_engine(tpv, r_, n_)
        perm = np.concatenate([shard.shard_by_engine(tpv, r, n_) for r in range(n_)])
        inputs = W.select_instances(W.config_inputs(cfg_g), shard_ix)
    else:
        inputs = W.config_inputs(dataclasses_replace(cfg, I_glob), i0, i1)
    I, R = len(inputs["inst"]), len(inputs["req"])
    model = tp.Gbdt(blob, local)
    info = model.info()
    counts = [shard_of(cfg, r, world)[1] - shard_of(cfg, r, world)[0] for r in range(world)]
    gather = shard.DecisionGather(counts, dev, host_staging=dist_test) if world > 1 else None
    rows = gather.rows() if gather else torch.empty((2, max(I, 1)), dtype=torch.int32, device=dev)
    # the exact step (runner.BenchStep): K1c -> K2 cell phases -> K3c, B/KV on chip, PDL, one graph;
    # level / status written straight into the gather's send rows
    step = runner.BenchStep(inputs, dev, model, search=args.search, graph=args.graph, level=rows[0],
                            status=rows[1])
    rnd = step.rnd
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)     # > 126 MB L2

    def one_step(evs=None):
        if evs:
            evs[0].record(stream)
        if evs and len(evs) == 5:     # instrumented: kernel by kernel, events between kernels
            rnd.project(stream)
            evs[1].record(stream)
            rnd.predict(model, stream)
            evs[2].record(stream)
            rnd.select(stream)
            evs[3].record(stream)
        else:
            step.run(stream)
        if gather is not None:
            gather.gather()
        if evs:
            evs[-1].record(stream)

    for _ in range(max(args.warmup, 3)):
        one_step()
    torch.cuda.synchronize(dev)

    # algorithmic sizes of this rank's step (from K1c's outputs; read once, untimed)
    n_h = rnd.n[:I].cpu().numpy().astype(np.int64)
    st_h = rnd.status[:I].cpu().numpy().view(np.uint32)
    nadm_h = rnd.n_adm[:I].cpu().numpy().astype(np.int64)
    live = (st_h & SKIP) == 0
    grid = int((n_h * live).sum()) * rnd.F
    cs = tp.compact_stats(model, rnd.work, I, rnd.H, rnd.F)
    evaluated = cs["cells"] * rnd.F          # K2's model evaluations (LUT rows x levels)
    n_req_all = int((inputs["inst"]["n_run"].astype(np.int64) + inputs["inst"]["n_queue"]).sum())
    n_sched = int(inputs["inst"]["n_run"].astype(np.int64).sum() + nadm_h.sum())

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    clocks = Clocks(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks.start()
    time.sleep(0.3)
    for k in range(args.steps):
        flush.zero_()                      # untimed L2 flush between timed steps
        one_step(evs[k])
    torch.cuda.synchronize(dev)
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    step_ms = np.array([a.elapsed_time(b) for a, b in evs])            # ms, the K timed steps
    t_total = float(step_ms.sum())
    if args.dump_decisions:
        res = (gather.result() if gather is not None else rows[:, :I]).cpu().numpy()
        if gather is not None and perm is not None:      # engine-grouped shards -> global order
            glob = np.zeros_like(res)
            glob[:, perm] = res
            res = glob
        if rank == 0:
            np.save(args.dump_decisions, res)
    # per-kernel breakdown (the kernel times of the rooflines): a second pass of K steps kernel by
    # kernel with events between the kernels, same inputs, same L2 flushes
    evk = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    for k in range(args.steps):
        flush.zero_()
        one_step(evk[k])
    torch.cuda.synchronize(dev)
    per = np.array([[e[j].elapsed_time(e[j + 1]) for j in range(4)] for e in evk])   # ms
    k_ms = per.mean(axis=0)
    # the north_star's direct K2 (one descent per grid point) on the same inputs, where its ips
    # grid fits (I x F x H fp32)
    d_ms = None
    if I * rnd.F * rnd.H * 4 <= (16 << 30):
        rd = runner.Round(inputs, dev, k2_mode="direct")
        rd.project(stream)
        rd.predict(model, stream)
        de = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(5 if grid < 10**9 else 2)]
        for a, b in de:
            flush.zero_()
            a.record(stream)
            rd.predict(model, stream)
            b.record(stream)
        torch.cuda.synchronize(dev)
        d_ms = float(np.median([a.elapsed_time(b) for a, b in de]))
        del rd
    tot = torch.tensor([t_total, grid, I, evaluated], dtype=torch.float64, device=dev)
    if world > 1:
        mx = tot[:1].clone()
        sm = tot[1:].clone()
        all_reduce(mx, dist.ReduceOp.MAX)
        all_reduce(sm, dist.ReduceOp.SUM)
        tot = torch.cat([mx, sm])
    t_max_ms, grid_all, inst_all, eval_all = (float(x) for x in tot)
    sec = t_max_ms / 1e3
    decisions_per_s = inst_all * args.steps / sec

    # end to end through the C ABI with host buffers (pinned), copies inside the timed region
    ctx = tp.Ctx(local, I, R, rnd.H, rnd.F, model)
    ctx.set_search(args.search)
    bi, br, bd = inputs["inst"].nbytes, inputs["req"].nbytes, inputs["t_dead"].nbytes
    h_in = torch.empty(bi + br + bd, dtype=torch.uint8).pin_memory()     # [inst | req | t_dead]: one copy
    h_in[:bi].copy_(torch.from_numpy(inputs["inst"].view(np.uint8)))
    h_in[bi:bi + br].copy_(torch.from_numpy(inputs["req"].view(np.uint8)))
    h_in[bi + br:].copy_(torch.from_numpy(np.ascontiguousarray(inputs["t_dead"]).view(np.uint8)))
    h_inst, h_req, h_td = h_in[:bi], h_in[bi:bi + br], h_in[bi + br:].view(torch.float64)
    h_out = torch.empty((2, max(I, 1)), dtype=torch.int32).pin_memory()   # [level | status]: one copy
    ke = args.e2e_steps or min(args.steps, 10)
    for _ in range(3):
        ctx.decide_host(model, h_inst, I, h_req, R, h_td, rnd.freq, rnd.tbt, h_out[0], h_out[1], stream)
    torch.cuda.synchronize(dev)
    ee = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(ke)]
    for k in range(ke):
        flush.zero_()
        ee[k][0].record(stream)
        ctx.decide_host(model, h_inst, I, h_req, R, h_td, rnd.freq, rnd.tbt, h_out[0], h_out[1], stream)
        ee[k][1].record(stream)
    torch.cuda.synchronize(dev)
    te = torch.tensor([sum(a.elapsed_time(b) for a, b in ee)], dtype=torch.float64, device=dev)
    if world > 1:
        all_reduce(te, dist.ReduceOp.MAX)
    ok = np.array_equal(h_out[0, :I].numpy(), rows[0, :I].cpu().numpy())
    e2e = {"value": inst_all * ke / (float(te[0]) / 1e3), "unit": "decisions/s",
           "h2d_bytes_per_step": int(bi + br + bd), "d2h_bytes_per_step": int(I * 8),
           "api": "tp_decide_host (pinned host buffers, one H2D + one D2H copy per step)",
           "matches_device_path": bool(ok)}
    ctx.free()

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peaks = measured_peaks()
    smax = float(peaks.get("sm_max_mhz", 1965.0))
    hbm = float(peaks.get("hbm_gbs", 6553.6))
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    traffic = load_traffic(cfg.name)
    # K1c (HBM): header 48 B + 16 B per request record + 8 B t_dead per scheduled request read;
    # n / n_adm / status 12 B + 16 B per piece record (start, cell id, Dmin) written
    k1_bytes = 48 * I + 16 * n_req_all + 8 * n_sched + 12 * I + 16 * cs["pieces"]
    # K2 (shared-memory loads): T * (D + 1) 4-byte node / leaf words per evaluated row
    per_row = info.n_trees * (info.depth + 1) * 4
    # K3c (HBM): n + status 8 B in, 16 B per piece record in, level 4 B out; the T' LUT reads
    # (F * 8 B per piece) stay on chip / in L2
    k3_bytes = 12 * I + 16 * cs["pieces"]
    lds_peak = sms * 128 * smax * 1e6 / 1e9
    kern = {
        "k1": roof("hbm", "k1_packed / k1_compact (K1c: projection, gate, pieces, cell claims, Eq. 4 minima)",
                   k1_bytes, k_ms[0], hbm, traffic.get("k1"),
                   basis="48 + 16 (R+Q) + 8 (R+Q_adm) + 12 + 16 pieces bytes per instance"),
        "k2": roof("smem", f"k2_cells_phase<{info.depth},2> x {k2_phases(info)} tree-resident phases",
                   evaluated * per_row, k_ms[1], lds_peak, traffic.get("k2"),
                   basis=f"{per_row} B of node/leaf words per evaluated row (cells x levels); peak {sms} SMs x "
                         f"128 B/clk x {smax:.0f} MHz"),
        "k3": roof("hbm", "k3_compact<W> (K3c: exact T_R per piece, Eq. 4, TBT, ballot argmin)",
                   k3_bytes, k_ms[2], hbm, traffic.get("k3"),
                   basis="12 + 16 pieces bytes per instance (LUT reads are L2 traffic)",
                   extra={"lut_bytes_l2": (4 if info.tick_shift == 8 else 8) * rnd.F * cs["pieces"],
                          "tick_updates_per_s": rnd.F * cs["pieces"] / (k_ms[2] / 1e3)}),
    }
    for k, v in load_traffic(cfg.name, "ncu_limiters").items():
        if k in kern:
            kern[k]["ncu_limiters"] = v
    dom = max(kern, key=lambda k: kern[k]["ms"])
    roofline = dict(kern[dom], dominant=dom, per_kernel=kern)
    if d_ms is not None:
        da = grid * per_row / (d_ms / 1e3) / 1e9
        roofline["direct_k2"] = {"ms": d_ms, "achieved": da, "frac": da / lds_peak,
                                 "note": "tp_predict_ips (one descent per grid point) on the same inputs"}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, blob, inputs, search=args.search)
    dist_info = None
    if world > 1:
        dist_info = {"backend": dist.get_backend(), "world_size": world,
                     "nccl": ".".join(map(str, torch.cuda.nccl.version())) if not dist_test else None}
    line = {
        "metric": METRIC, "value": decisions_per_s, "unit": "decisions/s",
        "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": t_max_ms / args.steps,
        "higher_is_better": True, "scaling": "weak" if cfg.name == "C2" else "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": DESCR[cfg.name], "name": cfg.name, "instances_per_gpu": I,
                   "global_instances": int(inst_all), "H": cfg.H, "F": cfg.F, "trees": info.n_trees,
                   "depth": info.depth,
                   "parallelism": f"instance-sharded x{world}"
                                  + (", grouped by engine size" if shard_ix is not None and world > 1 else "")
                                  + (" + NCCL all-gather" if world > 1 else ""),
                   "emulated_shard": args.emulate_shard,
                   "l2": "flushed between timed steps (256 MiB device write, untimed)",
                   "path": "compact: K1c -> K2 cell phases -> K3c (B/KV on chip), PDL, "
                           + ("one CUDA graph per step" if args.graph else "kernel by kernel"),
                   "search": args.search,
                   "instances_override": bool(args.instances)},
        "grid_evals_per_sec": grid_all * args.steps / sec,
        "grid_evals_note": "(instance, level, m <= n) grid points whose IPS each step determines (sum F*n_i); "
                           "the model is evaluated once per distinct cell and level (model_evals_per_sec)",
        "model_evals_per_sec": eval_all * args.steps / sec,
        "model_evals_per_sec_k2_only": evaluated / (k_ms[1] / 1e3),
        "counts_per_step_rank0": {"instances": I, "requests": n_req_all, "scheduled": n_sched,
                                  "pieces": cs["pieces"], "end_positions": cs["ends"], "cells": cs["cells"],
                                  "grid_points": grid},
        "step_ms_pctl": {"p10": float(np.percentile(step_ms, 10)), "p50": float(np.percentile(step_ms, 50)),
                         "p90": float(np.percentile(step_ms, 90)), "rank": "0"},
        "per_kernel_ms": {"k1_project": k_ms[0], "k2_gbdt": k_ms[1], "k3_select": k_ms[2], "gather": k_ms[3],
                          "note": "second pass of the same steps, kernel by kernel with events between the kernels "
                                  "(the timed steps replay one graph with events only at their ends)"},
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        # our kernels per step: K1c (k1_packed + the hand-over k1_compact<1,1> at one warp per
        # instance, i.e. when the batch exceeds 16 warps per SM), the cell-list collector, the K2
        # phases, K3c
        "gpu_launches": (3 + k2_phases(info) + int(I * 2 > sms * 32)) * args.steps,
        "clocks": clk,
        "dist": dist_info,
        "paper_context": "paper controller on host CPU (A100 box): projection <2 ms, model ~3 ms per call, "
                         "scheduler+throttle 35 ms per decision (P:466, P:495, P:557)",
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def roof(bound, kernel, algo_bytes, ms, peak_gbs, traffic, basis, extra=None):
    achieved = algo_bytes / (ms / 1e3) / 1e9
    r = {"bound": bound, "kernel": kernel, "achieved": achieved, "peak": peak_gbs, "unit": "GB/s",
         "frac": achieved / peak_gbs, "traffic": traffic, "ms": ms, "algorithmic_bytes": int(algo_bytes),
         "basis": basis}
    if extra:
        r.update(extra)
    return r


def load_traffic(name, key="dram_bytes_per_launch"):
    """ncu dram__bytes (read + write) per launch of each kernel (or, key="ncu_limiters", its issue /
    L1 data-pipe / DRAM / warp utilisation), from the committed capture of this workload
    (profiles/traffic_<name>.json), or {}."""
    try:
        with open(os.path.join(ROOT, "profiles", f"traffic_{name}.json")) as f:
            return json.load(f).get(key, {})
    except (OSError, ValueError):
        return {}


def k2_phases(info):
    """Launches of k2_cells_phase per step (k2_gbdt.cu launch_phases: <= 200 KB of trees each)."""
    tw = max(4, 2 << info.depth) * 4
    per = max(1, min((200 * 1024) // tw, 512))
    return max(1, -(-info.n_trees // per))


def dataclasses_replace(cfg, n_inst):
    import dataclasses
    return dataclasses.replace(cfg, n_inst=n_inst)


if __name__ == "__main__":
    main()
