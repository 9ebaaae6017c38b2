"""Per-CTA timeline of one fused forward-product + finalize launch (k1_tcp) at M, from a measurement
build with -DK1P_TIMING=<iteration> (tools/build_variant.sh k1t k1_tcp.cu -DK1P_TIMING=230).
Prints phase times relative to the earliest CTA start (us)."""
import os
import statistics

import numpy as np
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ['FSQR_LIB'] = os.path.join(ROOT, 'build_var', os.environ.get('K1T', 'k1t'), 'libfsqr.so')
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2601_02826_b200 as fs  # noqa: E402

prob = datagen.make(os.environ.get('K1T_CONFIG', 'm'))
X = torch.from_numpy(prob.X).cuda()
y = torch.from_numpy(prob.y).cuda()
S = fs.Solver(X, prob.storage, prob.n, prob.p, prob.ld, y, [prob.taus[0]], [1.0], G=prob.G, mu=2 / prob.n,
              flags=fs.DESIGN_PACK2)
lm = S.lambda_max()[0]
S.set_lambda([prob.lam_frac * lm])
S.iterate(240)
torch.cuda.synchronize()
st = fs.fsqr_debug_stamps(S.ctx).astype('int64')
cta = st[:8 * 148].reshape(148, 8)
t0 = cta[:, 0].min()
prod = cta[(cta[:, 6] >> 32) == 0]
names = ["start", "itemsdone", "barrier", "recdone", "published"]
for k, nm in enumerate(names):
    v = (prod[:, k] - t0) / 1000.0
    print(f"{nm:10s} min {v.min():7.2f} med {statistics.median(v):7.2f} max {v.max():7.2f} us")
print("reducer: records complete %.2f us, iteration done %.2f us" % ((st[8 * 148 + 70] - t0) / 1e3,
                                                                     (st[8 * 148 + 40] - t0) / 1e3))
