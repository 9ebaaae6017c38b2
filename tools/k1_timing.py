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
names = ["start", "itemsdone", "barrier", "recwork", "fence", "ticket"]
for k, nm in enumerate(names):
    v = (cta[:, k] - t0) / 1000.0
    print(f"{nm:10s} min {v.min():7.2f} med {statistics.median(v):7.2f} max {v.max():7.2f} us")
print("reduce (before requant) %.2f us, requant %d" % ((st[8 * 148 + 50] - t0) / 1e3, st[8 * 148 + 51]))
print("reduce_rhs0 done %.2f us, tail end %.2f us" % ((st[8 * 148] - t0) / 1e3, (st[8 * 148 + 40] - t0) / 1e3))
slow = sorted(range(148), key=lambda c: -cta[c, 4])[:10]
print("slowest fences (cta, sm, us):", [(c, int(cta[c, 6] & 0xffffffff), round((cta[c, 4] - t0) / 1e3, 2)) for c in slow])

rec = st[1300:1300 + 4 * 40].reshape(40, 4)
for nm, k in (("rec start", 0), ("loads done", 1), ("rows+warp red", 2), ("group bar", 3)):
    v = (rec[:, k] - t0) / 1e3
    print(f"{nm:14s} min {v.min():7.2f} med {statistics.median(v):7.2f} max {v.max():7.2f} us")

lc = st[8 * 148:8 * 148 + 80]
print("last CTA: after fence %.2f, reduced %.2f us (requant mask %d)" % (
    (lc[70] - t0) / 1e3, (st[1234] - t0) / 1e3, st[1235]))
print("warp reduce of RHS 0: loads done %.2f, butterfly done %.2f, scalars done %.2f us" % tuple((st[1234 + q] - t0) / 1e3 for q in (20, 21, 22)))
cyc = st[8 * 148 + 200: 8 * 148 + 200 + 148]
print("record phase cycles per CTA (records CTAs): min %d med %d max %d" % (cyc[cyc > 0].min(), np.median(cyc[cyc > 0]), cyc.max()))
print("last CTA fin_reduce_all cycles: %d" % st[8 * 148 + 74])
