import os, sys, time, json, numpy as np, torch
sys.path.insert(0, '/root/repo')
import datagen, paper_2601_02826_b200 as fs
name = sys.argv[1]; flags = int(sys.argv[2]) if len(sys.argv) > 2 else 0
prob = datagen.make(name)
Xd = torch.from_numpy(prob.X).cuda(); yd = torch.from_numpy(prob.y).cuda()
taus = [prob.taus[0]] if name == 'm' else list(prob.taus)
res = {}
states = {}
for mode in ['bulk', 'tcp']:
    os.environ['FSQR_K1'] = mode
    S = fs.Solver(Xd, prob.storage, prob.n, prob.p, prob.ld, yd, taus, [1.0]*len(taus), G=prob.G, flags=flags)
    lm = S.lambda_max(); S.set_lambda([prob.lam_frac * v for v in lm])
    S.iterate(200)
    torch.cuda.synchronize()
    st, tot = fs.fsqr_profile_iterate(S.ctx, 200)
    states[mode] = S.state()
    res[mode] = dict(k2=st[0]/200, k1=st[1]/200, fin=st[2]/200, nnz=int(S.trace(1)[-1,0,4]))
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record(); S.iterate(600); e1.record(); torch.cuda.synchronize()
    res[mode]['graph_ms'] = e0.elapsed_time(e1)/600
    del S
same = all(np.array_equal(a, b) for a, b in zip(states['bulk'], states['tcp']))
print(json.dumps(dict(name=name, flags=flags, same=same, **res)))
