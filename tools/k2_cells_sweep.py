"""Cell-mode K2 timing sweep over rows per lane / CTA size / chunk (each setting in its own process).
Usage (GPU box): python tools/k2_cells_sweep.py C2 [reps]"""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

def one(wl, reps):
    import torch
    from paper_2408_05235_b200 import runner, tp, workload as W
    cfg = W.CONFIGS[wl]
    model = tp.Gbdt(W.write_blob(W.config_ensemble(cfg)), 0)
    r = runner.Round(W.config_inputs(cfg), "cuda:0", k2_mode="fused", model=model)
    r.project(); r.predict(model); torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
    for k in range(reps):
        ev[2 * k].record(); r.predict(model); ev[2 * k + 1].record()
    torch.cuda.synchronize()
    ts = sorted(ev[2 * k].elapsed_time(ev[2 * k + 1]) for k in range(reps))
    return ts[len(ts) // 2]

if __name__ == "__main__":
    if os.environ.get("K2_SWEEP_CHILD"):
        print(json.dumps({"ms": one(sys.argv[1], int(sys.argv[2]))}))
        sys.exit(0)
    wl = sys.argv[1] if len(sys.argv) > 1 else "C2"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    grid = [(ru, th, ck) for ru in [1, 2] for th in [128, 256] for ck in [16, 24, 32]]
    if len(sys.argv) > 3:
        grid = [tuple(int(v) for v in g.split(",")) for g in sys.argv[3:]]
    for ru, th, ck in grid:
        if True:
            if True:
                env = dict(os.environ, K2_SWEEP_CHILD="1", TP_K2_RU_CELLS=str(ru), TP_K2_THREADS=str(th),
                           TP_K2_CHUNK_KB=str(ck))
                out = subprocess.run([sys.executable, __file__, wl, str(reps)], env=env, capture_output=True, text=True)
                line = [l for l in out.stdout.splitlines() if l.startswith("{")]
                print(wl, "ru", ru, "threads", th, "chunk_kb", ck, line[-1] if line else out.stderr[-300:], flush=True)
