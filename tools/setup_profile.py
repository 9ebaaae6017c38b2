"""Setup (create) cost breakdown at a config: wall time of fsqr_create with eta computed (Lanczos,
power) and with eta given, and the per-kernel launch list when run under ncu (launch-list pass)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2601_02826_b200 as fs  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "m"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
prob = datagen.make(cfg)
X = torch.from_numpy(prob.X).cuda()
y = torch.from_numpy(prob.y).cuda()
flags = fs.DESIGN_PACK2 if prob.storage == 1 else 0
out = {"config": cfg, "n": prob.n, "p": prob.p}


def create(**kw):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    S = fs.Solver(X, prob.storage, prob.n, prob.p, prob.ld, y, [prob.taus[0]], [1.0], G=prob.G, mu=2 / prob.n,
                  flags=flags, **kw)
    torch.cuda.synchronize()
    return S, time.perf_counter() - t0


for name, kw in (("lanczos", {}), ("power", {"eta_method": fs.ETA_POWER})):
    ts = []
    for _ in range(reps):
        S, dt = create(**kw)
        ts.append(dt)
        eta = S.eta() if hasattr(S, "eta") else None
        del S
    out[name + "_s"] = ts
S, _ = create()
eta = fs.fsqr_get_eta(S.ctx, prob.G) if hasattr(fs, "fsqr_get_eta") else None
del S
if eta is not None:
    ts = []
    for _ in range(reps):
        S, dt = create(eta=eta)
        ts.append(dt)
        del S
    out["eta_given_s"] = ts
print(json.dumps(out))
