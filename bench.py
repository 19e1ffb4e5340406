#!/usr/bin/env python
"""Benchmark of the throttLL'eM frequency-selection hot path (BASELINE.json metric: frequency
decisions/s and GBDT grid evals/s vs roofline).

One step = one decision round over the workload: K1 projection -> K2 GBDT grid -> K3 SLO scan
(+ one NCCL all-gather of the decisions when N > 1).  Inputs are synthetic and seeded
(paper_2408_05235_b200/workload.py), already resident in HBM when the timed region starts.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C2] [--impl ours|reference]

N > 1 runs under torchrun (one process per GPU, NCCL).  Default workload C2 = BASELINE.json
configs[1]; per-GPU work is fixed (weak scaling: rank r decides instances [r*I, (r+1)*I) of the
same generator).  --workload C5 is the strong-scaling sweep (262,144 instances split over N).
"""
from __future__ import annotations

import argparse
import json
import os
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
    "C5": "BASELINE configs[4]: 262,144 instances sharded over N GPUs (strong scaling), 200-tree depth-8",
}
SKIP = 64 | 1 | 2


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def shard_of(cfg, rank, world):
    """Instance range of this rank and the global instance count (paper_2408_05235_b200/shard.py)."""
    from paper_2408_05235_b200 import shard
    if cfg.name == "C5":            # strong scaling: fixed total
        return (*shard.shard_range(cfg.n_inst, rank, world), cfg.n_inst)
    return (*shard.weak_range(cfg.n_inst, rank), cfg.n_inst * world)   # weak: fixed per GPU


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


def cpu_baseline(cfg, blob, inputs, budget_s=15.0, search="exhaustive"):
    """The oracle, as it stands, on this host's cores, on a bounded prefix of the workload."""
    from oracle import oracle
    m = oracle.Model(blob)
    threads = os.cpu_count() or 1
    inst = inputs["inst"]

    def run(k):
        sub = inst[:k]
        last = int(sub[-1]["req_begin"] + sub[-1]["n_run"] + sub[-1]["n_queue"])
        t = time.perf_counter()
        oracle.decide(m, sub, inputs["req"][:last], inputs["t_dead"][:last], inputs["H"], inputs["freq"],
                      inputs["tbt_slo"], want_grid=False, want_curves=False, threads=threads, search=search)
        return time.perf_counter() - t

    k = min(len(inst), max(threads, 8))
    dt = run(k)
    while k < len(inst) and dt < 1.0:
        k = min(len(inst), k * 4)
        dt = run(k)
    if k < len(inst) and dt < budget_s:
        k = min(len(inst), max(k, int(k * budget_s / max(dt, 1e-3))))
        dt = run(k)
    return {"value": k / dt, "unit": "decisions/s", "cores": threads, "kind": "oracle",
            "sample": f"first {k} of {len(inst)} instances of {cfg.name} ("
                      + ("all F levels evaluated" if search == "exhaustive" else "the paper's binary search")
                      + f", {threads} threads), {dt:.1f} s"}


def bench_reference(args, cfg):
    """--impl reference: the CPU oracle is this tier's reference arm (rank 0 only)."""
    rank = env_int("RANK", 0)
    if rank != 0:
        return
    blob = W.write_blob(W.config_ensemble(cfg))
    per_step = {"C1": 1, "C2": 64, "C3": 16, "C4": 8, "C5": 16}[cfg.name]
    inputs = W.config_inputs(cfg, 0, max(per_step, 1))
    from oracle import oracle
    m = oracle.Model(blob)
    threads = os.cpu_count() or 1

    def step():
        oracle.decide(m, inputs["inst"], inputs["req"], inputs["t_dead"], inputs["H"], inputs["freq"],
                      inputs["tbt_slo"], want_grid=False, want_curves=False, threads=threads, search=args.search)
    for _ in range(args.warmup):
        step()
    t = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t
    v = per_step * args.steps / dt
    line = {"impl": "reference", "metric": "frequency decisions/sec", "value": v, "unit": "decisions/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak" if cfg.name != "C5" else "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": DESCR[cfg.name], "name": cfg.name, "instances_per_step": per_step,
                       "search": args.search},
            "cpu_baseline": {"value": v, "unit": "decisions/s", "cores": threads, "kind": "oracle",
                             "sample": f"first {per_step} instances of {cfg.name} per step"},
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
    A step = one round: decide every instance (tp_decide) + advance every instance one engine
    iteration (tp_replay_advance), all on the GPU.  Instances are split over ranks."""
    import torch
    from paper_2408_05235_b200 import replay, shard, tp
    dev = torch.device("cuda", local)
    rc = W.ReplayConfig()
    data = W.gen_replay(rc)
    i0, i1 = shard.shard_range(rc.n_inst, rank, world)
    data = slice_replay(data, i0, i1)
    model = tp.Gbdt(W.write_blob(W.config_ensemble(cfg)), local)
    rp = replay.Replay(data, model, dev, admission=args.admission, search=args.search)
    stream = torch.cuda.current_stream(dev)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    for _ in range(max(args.warmup, 3)):
        rp.round(stream)
    torch.cuda.synchronize(dev)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    clocks = Clocks(local)
    if world > 1:
        dist.barrier()
    clocks.start()
    time.sleep(0.3)
    for k in range(args.steps):
        ev[k][0].record(stream)
        rp.decide(stream)
        ev[k][1].record(stream)
        rp.advance(stream)
        ev[k][2].record(stream)
    torch.cuda.synchronize(dev)
    clk = clocks.stop()
    dec_ms = float(sum(e[0].elapsed_time(e[1]) for e in ev))
    adv_ms = float(sum(e[1].elapsed_time(e[2]) for e in ev))
    tot = torch.tensor([dec_ms + adv_ms, dec_ms], dtype=torch.float64, device=dev)
    if world > 1:
        c = tot.cpu() if dist_test else tot
        dist.all_reduce(c, op=dist.ReduceOp.MAX)
        tot = c.to(dev)
    if rank != 0:
        return
    I = rc.n_inst
    st = rp.stats_dict()
    line = {
        "metric": "frequency decisions/sec", "value": I * args.steps / (float(tot[0]) / 1e3), "unit": "decisions/s",
        "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3),
        "ms_per_step": float(tot[0]) / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": DESCR["C4"], "name": "C4", "instances": I, "requests": rc.n_requests,
                   "span_s": rc.span_s, "trees": cfg.n_trees, "depth": cfg.depth, "F": cfg.F, "H": cfg.H,
                   "step": "decide all instances + advance all instances one iteration (GPU-resident replay)",
                   "admission": (f"full admission control (checks 1-3 at f_max, lost marking), q_max={args.admission}"
                                 if args.admission else "check 1 + batch cap gate"),
                   "search": args.search,
                   "l2": "not flushed: the replay state (~20 MB) is re-used every round by design"},
        "decisions_per_sec_decide_only": I * args.steps / (float(tot[1]) / 1e3),
        "per_round_ms": {"decide": dec_ms / args.steps, "advance": adv_ms / args.steps},
        "replay_stats_after_warmup_and_steps": st,
        # per round without admission: K1c (+ hand-over kernel at one warp per instance), the K2
        # phases, K3c, the replay advance; with admission control the prefix pass adds its own
        "gpu_launches": (None if args.admission else
                         (3 + k2_phases(model.info()) + int((i1 - i0) * 2 > sms * 32)) * args.steps),
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="C2", choices=sorted(DESCR))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--admission", type=int, default=0,
                    help="C4 replay: run the paper's full admission control on up to N queued requests per instance")
    ap.add_argument("--search", default="exhaustive", choices=["exhaustive", "binary"],
                    help="K3 order: lowest passing level over all levels (reading A-13, default) or the "
                         "paper's binary search (P:555, reading A-24; needs --k2 fused)")
    ap.add_argument("--graph", dest="graph", action="store_true", default=True,
                    help="time the step as a replayed CUDA graph of its kernels (default; SURVEY §8d)")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="launch the kernels one by one in the timed steps")
    ap.add_argument("--k2", default="compact", choices=["compact", "fused", "cells", "runs", "direct"],
                    help="path: compact (K1c runs + deadline list -> K2 on the cells -> K3c, default), "
                         "cell-memoised fused with K3, cell-memoised with the ips grid, run-compressed, or "
                         "one evaluation per grid point")
    args = ap.parse_args()
    cfg = W.CONFIGS[args.workload]
    if args.impl == "reference":
        return bench_reference(args, cfg)

    import torch
    import torch.distributed as dist
    from paper_2408_05235_b200 import runner, tp

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

    def _coll(t, fn):
        if not dist_test:
            return fn(t)
        c = t.cpu()
        fn(c)
        t.copy_(c)

    def all_reduce(t, op):
        _coll(t, lambda x: dist.all_reduce(x, op=op))

    if cfg.name == "C4":
        bench_replay(args, cfg, rank, world, local, dist, dist_test)
        if world > 1:
            dist.destroy_process_group()
        return
    i0, i1, I_glob = shard_of(cfg, rank, world)
    blob = W.write_blob(W.config_ensemble(cfg))
    inputs = W.config_inputs(dataclasses_replace(cfg, I_glob), i0, i1)
    I, R = len(inputs["inst"]), len(inputs["req"])
    model = tp.Gbdt(blob, local)
    info = model.info()
    rnd = runner.Round(inputs, dev, k2_mode=args.k2, model=model, search=args.search)
    rnd.bkv = False          # compact path: the B/KV curves stay on chip
    dec = torch.empty((2, max(I, 1)), dtype=torch.int32, device=dev)   # level, status rows
    rnd.level, rnd.status = dec[0], dec[1]
    # equal shards (C2 weak, C5 = 262144 / {1,2,4,8}): one preallocated all-gather of [2, I] rows
    gathered = torch.empty((world * 2, max(I, 1)), dtype=torch.int32, device=dev) if world > 1 else None
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)     # > 126 MB L2

    def kernels(strm):
        rnd.project(strm)
        rnd.predict(model, strm)
        rnd.select(strm)

    graph = None
    if args.graph:           # the K1 -> K2 -> K3 sequence captured once, replayed every step
        gs = torch.cuda.Stream(dev)
        with torch.cuda.stream(gs):
            kernels(gs)      # warm-up on the capture stream (attributes, lazy module loading)
        torch.cuda.synchronize(dev)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=gs):
            kernels(gs)
        torch.cuda.synchronize(dev)

    def step(evs=None, split=True):
        # split=False: events only around the whole step (an event between two kernels stops the
        # second from launching early -- programmatic dependent launch -- and costs ~4 us each)
        if evs:
            evs[0].record(stream)
        if graph is not None and not split:
            graph.replay()
        else:
            rnd.project(stream)
            if evs and split:
                evs[1].record(stream)
            rnd.predict(model, stream)
            if evs and split:
                evs[2].record(stream)
            rnd.select(stream)
            if evs and split:
                evs[3].record(stream)
        if world > 1:
            if dist_test:
                g = torch.empty(gathered.shape, dtype=gathered.dtype)
                dist.all_gather_into_tensor(g, dec.cpu())
                gathered.copy_(g)
            else:
                dist.all_gather_into_tensor(gathered, dec)
        if evs:
            evs[4].record(stream)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize(dev)

    # algorithmic grid size of this rank (from K1's outputs; not timed)
    n_h = rnd.n[:I].cpu().numpy().astype(np.int64)
    st_h = rnd.status[:I].cpu().numpy().view(np.uint32)
    grid = int((n_h * ((st_h & SKIP) == 0)).sum()) * rnd.F
    padded = int((((n_h + 31) // 32) * 32 * ((st_h & SKIP) == 0)).sum()) * rnd.F
    evaluated = {"runs": lambda: tp.runs_total(rnd.work, I, rnd.H) * rnd.F,
                 "cells": lambda: tp.cells_total(rnd.work, model, I, rnd.H, rnd.F) * rnd.F,
                 "fused": lambda: tp.cells_total(rnd.work, model, I, rnd.H, rnd.F) * rnd.F,
                 "compact": lambda: tp.cells_total(rnd.work, model, I, rnd.H, rnd.F) * rnd.F,
                 "direct": lambda: grid}[args.k2]()

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    clocks = Clocks(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks.start()
    time.sleep(0.3)
    for k in range(args.steps):
        flush.zero_()                      # untimed L2 flush between timed steps
        step(evs[k], split=False)
    torch.cuda.synchronize(dev)
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    step_ms = np.array([e[0].elapsed_time(e[4]) for e in evs])            # ms, the K timed steps
    t_total = float(step_ms.sum())
    # per-kernel breakdown (and the K2 time of the roofline): a second pass of K steps with events
    # between the kernels, same inputs, same L2 flushes
    evk = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    for k in range(args.steps):
        flush.zero_()
        step(evk[k])
    torch.cuda.synchronize(dev)
    per = np.array([[e[j].elapsed_time(e[j + 1]) for j in range(4)] for e in evk])   # ms
    k_ms = per.mean(axis=0)
    # the north_star's direct K2 (one descent per grid point), timed on the same inputs for reference
    d_ms = None
    if args.k2 != "direct":
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
    tot = torch.tensor([t_total, grid, I], dtype=torch.float64, device=dev)
    if world > 1:
        mx = tot[:1].clone()
        sm = tot[1:].clone()
        all_reduce(mx, dist.ReduceOp.MAX)
        all_reduce(sm, dist.ReduceOp.SUM)
        tot = torch.cat([mx, sm])
    t_max_ms, grid_all, inst_all = float(tot[0]), float(tot[1]), float(tot[2])
    sec = t_max_ms / 1e3
    decisions_per_s = inst_all * args.steps / sec
    grid_per_s = grid_all * args.steps / sec

    # end to end through the C ABI with host buffers (pinned), copies inside the timed region
    e2e = None
    if True:
        ctx = tp.Ctx(local, I, R, rnd.H, rnd.F, model if args.k2 in ("cells", "fused", "compact") else None)
        ctx.set_k2_mode({"direct": tp.K2_DIRECT, "compact": tp.K2_COMPACT}.get(args.k2, tp.K2_RUNS))
        ctx.set_search(args.search)
        # one pinned host buffer [inst | req | t_dead] (tp_decide_host then copies it in one go) and
        # one [level | status] buffer for the results
        bi, br, bd = inputs["inst"].nbytes, inputs["req"].nbytes, inputs["t_dead"].nbytes
        h_in = torch.empty(bi + br + bd, dtype=torch.uint8).pin_memory()
        h_in[:bi].copy_(torch.from_numpy(inputs["inst"].view(np.uint8)))
        h_in[bi:bi + br].copy_(torch.from_numpy(inputs["req"].view(np.uint8)))
        h_in[bi + br:].copy_(torch.from_numpy(np.ascontiguousarray(inputs["t_dead"]).view(np.uint8)))
        h_inst, h_req, h_td = h_in[:bi], h_in[bi:bi + br], h_in[bi + br:].view(torch.float64)
        h_out = torch.empty((2, max(I, 1)), dtype=torch.int32).pin_memory()
        h_level, h_status = h_out[0], h_out[1]
        ke = args.e2e_steps or args.steps
        for _ in range(3):
            ctx.decide_host(model, h_inst, I, h_req, R, h_td, rnd.freq, rnd.tbt, h_level, h_status, stream)
        torch.cuda.synchronize(dev)
        ee = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(ke)]
        for k in range(ke):
            flush.zero_()
            ee[k][0].record(stream)
            ctx.decide_host(model, h_inst, I, h_req, R, h_td, rnd.freq, rnd.tbt, h_level, h_status, stream)
            ee[k][1].record(stream)
        torch.cuda.synchronize(dev)
        te = torch.tensor([sum(a.elapsed_time(b) for a, b in ee)], dtype=torch.float64, device=dev)
        if world > 1:
            all_reduce(te, dist.ReduceOp.MAX)
        ok = np.array_equal(h_level[:I].numpy(), dec[0, :I].cpu().numpy())
        e2e = {"value": inst_all * ke / (float(te[0]) / 1e3), "unit": "decisions/s",
               "h2d_bytes_per_step": int(I * 48 + R * 16 + R * 8), "d2h_bytes_per_step": int(I * 8),
               "matches_device_path": bool(ok)}
        ctx.free()

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peaks = measured_peaks()
    smax = float(peaks.get("sm_max_mhz", 1965.0))
    # K2 roofline: shared-memory load bandwidth, 128 B/clk/SM (B200_PROFILING / B300_MICROARCH
    # LDS crossbar) x 148 SMs x max SM clock.  Algorithmic bytes per grid point: T*(D+1) 4-byte
    # node/leaf words.
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    per_pt = info.n_trees * (info.depth + 1) * 4
    k2_s = k_ms[1] / 1e3
    achieved = evaluated * per_pt / k2_s / 1e9     # this rank's K2 (incl. the run pre-pass), GB/s
    peak = sms * 128 * smax * 1e6 / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "k2_traffic.json")) as f:
            tj = json.load(f)
        if tj.get("workload") == cfg.name:
            traffic = tj.get("dram_bytes_per_launch")
    except (OSError, ValueError):
        pass
    roof = {"bound": "smem", "kernel": {"direct": "k2_gbdt", "runs": "k2_gbdt<runs> (+ k2_runs pre-pass)",
                                        "cells": "k2_gbdt<cells> (+ k2_runs pre-pass, k2_expand)",
                                        "fused": "k2_gbdt<cells> (+ k2_runs pre-pass)",
                                        "compact": f"k2_cells_phase<{info.depth},2> x {k2_phases(info)} "
                                                   "tree-resident phases (runs built by K1c)"}[args.k2],
            "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic,
            "peak_basis": f"{sms} SMs x 128 B/clk (LDS) x sm_max_mhz {smax:.0f} (MEASURED_PEAKS.json clock)",
            "frac_at_observed_clock": (achieved / (sms * 128 * clk["sm_mhz"] * 1e6 / 1e9)) if clk["sm_mhz"] else None,
            "bytes_per_evaluated_row": per_pt, "evaluated_rows_per_launch": evaluated,
            "grid_points_per_launch": grid, "padded_grid_points": padded}
    if d_ms is not None:
        da = grid * per_pt / (d_ms / 1e3) / 1e9
        roof["direct_k2"] = {"ms": d_ms, "achieved": da, "frac": da / peak,
                             "note": "tp_predict_ips (one descent per grid point) on the same inputs"}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, blob, inputs, search=args.search)
    line = {
        "metric": "frequency decisions/sec", "value": decisions_per_s, "unit": "decisions/s",
        "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": t_max_ms / args.steps,
        "higher_is_better": True, "scaling": "strong" if cfg.name == "C5" else "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": DESCR[cfg.name], "name": cfg.name, "instances_per_gpu": I,
                   "global_instances": int(inst_all), "H": cfg.H, "F": cfg.F, "trees": info.n_trees,
                   "depth": info.depth, "parallelism": f"instance-sharded x{world}" + (" + NCCL all-gather" if world > 1 else ""),
                   "l2": "flushed between timed steps (256 MiB device write, untimed)", "k2": args.k2,
                   "cuda_graph": bool(args.graph),
                   "search": args.search},
        "grid_evals_per_sec": grid_per_s,
        "step_ms_pctl": {"p10": float(np.percentile(step_ms, 10)), "p50": float(np.percentile(step_ms, 50)),
                         "p90": float(np.percentile(step_ms, 90)), "rank": "0"},
        "per_kernel_ms": {"k1_project": k_ms[0], "k2_gbdt": k_ms[1], "k3_select": k_ms[2],
                          "gather": k_ms[3],
                          "note": "from a second pass of the same steps with events between the kernels "
                                  "(those events stop programmatic dependent launch; the timed steps carry "
                                  "events only at their ends)"},
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": e2e,
        # our kernels per step: k1_project / k1_compact, [k2_runs], k2_gbdt, [k2_expand], k3_select* / k3_compact
        # compact: K1c (+ the hand-over kernel after k1_packed at one warp per instance, i.e. when
        # the batch exceeds 16 warps per SM), the K2 phases, K3c
        "gpu_launches": {"direct": 3, "runs": 4, "cells": 5, "fused": 4,
                         "compact": 2 + k2_phases(info) + int(I * 2 > sms * 32)}[args.k2] * args.steps,
        "clocks": clk,
        "paper_context": "paper controller on host CPU (A100 box): projection <2 ms, model ~3 ms per call, "
                         "scheduler+throttle 35 ms per decision (P:466, P:495, P:557)",
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


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
