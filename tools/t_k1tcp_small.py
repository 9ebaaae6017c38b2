import os, sys
sys.path.insert(0, '/root/repo')
import datagen, paper_2601_02826_b200 as fs, torch
def to_device(p):
    return torch.from_numpy(p.X).cuda(), torch.from_numpy(p.y).cuda()
os.environ['FSQR_K1'] = 'tcp'
b = datagen.make("c5", n=1500, p=2600, storage=2)
X, y = to_device(b)
try:
    S = fs.Solver(X, 2, b.n, b.p, b.ld, y, [0.5], [0.02], G=5, eta=[40.0]*5)
    S.iterate(3); print(os.environ.get('FSQR_LIB'), 'ok', S.objective())
except Exception as e:
    print(os.environ.get('FSQR_LIB'), 'ERR', str(e)[:150])
