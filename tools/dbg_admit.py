import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import cases
from paper_2408_05235_b200 import workload as W, runner, tp
from oracle import oracle
rng = np.random.default_rng(21)
for trial in range(80):
    ens, inst, req, td, H, freq, tbt = cases.random_tiny_case(rng)
    blob = W.write_blob(ens)
    inputs = dict(inst=inst, req=req, t_dead=td, H=H, freq=freq, tbt_slo=tbt)
    model = tp.Gbdt(blob, 0)
    I, R = len(inst), len(req)
    ctx = tp.Ctx(0, I, max(R, 1), H, len(freq), model); ctx.enable_admission(32)
    r = runner.Round(inputs, "cuda:0", k2_mode="direct")
    n_adm = torch.full((I,), -7, dtype=torch.int32, device="cuda:0"); lost = torch.full((I,), -7, dtype=torch.int32, device="cuda:0")
    ctx.decide_admit(model, r.inst, I, r.req, R, r.t_dead, freq, tbt, r.level, r.status, n_adm, lost)
    torch.cuda.synchronize()
    ref = oracle.decide(oracle.Model(blob), inst, req, td, H, freq, tbt, want_grid=False, admission=1)
    g = dict(level=r.level.cpu().numpy(), status=r.status.cpu().numpy().view(np.uint32), n_adm=n_adm.cpu().numpy(), lost=lost.cpu().numpy().view(np.uint32))
    bad = [i for i in range(I) if (g['level'][i], g['status'][i], g['n_adm'][i], g['lost'][i]) != (ref['level'][i], ref['status'][i], ref['n_adm'][i], ref['adm_lost'][i])]
    if bad:
        print('trial', trial, 'H', H, 'F', len(freq), 'bad', bad)
        for i in bad:
            print(' inst', inst[i], '\n  reqs', req[int(inst[i]['req_begin']):int(inst[i]['req_begin']+inst[i]['n_run']+inst[i]['n_queue'])])
            print('  gpu', {k: int(v[i]) for k, v in g.items()}, 'ref', {k: int(ref[k][i]) for k in ['level','status','n_adm','adm_lost']})
        break
print('done')
