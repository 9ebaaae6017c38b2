"""K2 time of the 2-bit kernel at C5 size for R RHS (argv[1], default 9), for A/B builds via FSQR_LIB."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import datagen, paper_2601_02826_b200 as fs
R = int(sys.argv[1]) if len(sys.argv) > 1 else 9
prob = datagen.make('c5')
X = torch.from_numpy(prob.X).cuda(); y = torch.from_numpy(prob.y).cuda()
taus = list(prob.taus)[:R] if R <= 9 else [0.05 + 0.9 * k / (R - 1) for k in range(R)]
S = fs.Solver(X, 1, prob.n, prob.p, prob.ld, y, taus, [0.05] * R, G=48, flags=1, eta=[30.0] * 48)
S.iterate(20)
st, tot = fs.fsqr_profile_iterate(S.ctx, 20)
print(os.environ.get('FSQR_LIB', 'default'), 'R', R, 'k2 ms', round(st[0] / 20, 4))
