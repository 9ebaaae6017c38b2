import os, sys, json, numpy as np, torch
sys.path.insert(0, '/root/repo')
import datagen, paper_2601_02826_b200 as fs
prob = datagen.make('c5')
X = torch.from_numpy(prob.X).cuda(); y = torch.from_numpy(prob.y).cuda()
S = fs.Solver(X, 1, prob.n, prob.p, prob.ld, y, list(prob.taus), [0.05]*9, G=48, flags=1, eta=[30.0]*48)
S.iterate(20)
st, tot = fs.fsqr_profile_iterate(S.ctx, 20)
print(os.environ.get('FSQR_LIB'), 'k2 ms', st[0]/20)
