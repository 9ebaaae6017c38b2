"""K1 timing on a fixed state: `save` runs the correct library 200 iterations and stores the
state; `time` (any library, e.g. a measurement variant via FSQR_LIB) restores it and profiles
single iterations from it, so every variant sees the same support."""
import os, sys, json, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen, paper_2601_02826_b200 as fs
what, name, flags = sys.argv[1], sys.argv[2], int(sys.argv[3])
path = f"/tmp/k1state_{name}.npz"
prob = datagen.make(name)
Xd = torch.from_numpy(prob.X).cuda(); yd = torch.from_numpy(prob.y).cuda()
taus = [prob.taus[0]] if name == 'm' else list(prob.taus)
out = {}
for mode in (sys.argv[4].split(',') if len(sys.argv) > 4 else ['bulk', 'tcp']):
    os.environ['FSQR_K1'] = mode
    S = fs.Solver(Xd, prob.storage, prob.n, prob.p, prob.ld, yd, taus, [1.0]*len(taus), G=prob.G, flags=flags,
                  eta=[1.0] * prob.G if what == 'time' else None)
    if what == 'save':
        lm = S.lambda_max(); S.set_lambda([prob.lam_frac * v for v in lm])
        S.iterate(200)
        b, z, t = S.state()
        np.savez(path, b=b, z=z, t=t, lam=[prob.lam_frac * v for v in lm], eta=S.eta())
        print("saved", int(S.trace(1)[-1, 0, 4]))
        break
    d = np.load(path)
    del S
    S = fs.Solver(Xd, prob.storage, prob.n, prob.p, prob.ld, yd, taus, list(d['lam']), G=prob.G, flags=flags,
                  eta=list(d['eta']))
    ks = []
    for rep in range(20):
        S.set_state(d['b'], d['z'], d['t'])
        st, tot = fs.fsqr_profile_iterate(S.ctx, 1)
        ks.append(st[1])
    out[mode] = float(np.median(ks[2:]))
    del S
print(json.dumps(dict(name=name, **out)))
