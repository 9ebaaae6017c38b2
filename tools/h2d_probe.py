"""Probe: pinned host->device copy rate for the M design size, and fsqr_fit_host phase times."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import datagen, paper_2601_02826_b200 as fs
prob = datagen.make("m")
Xp = torch.empty(prob.X.shape, dtype=torch.uint8, pin_memory=True); Xp.numpy()[:] = prob.X
yp = torch.empty(prob.n, dtype=torch.float64, pin_memory=True); yp.numpy()[:] = prob.y
d = torch.empty(prob.X.shape, dtype=torch.uint8, device="cuda")
for i in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(Xp, non_blocking=True); torch.cuda.synchronize()
    dt = time.perf_counter() - t0; print(f"H2D {prob.X.nbytes/1e9:.1f} GB: {dt:.3f} s = {prob.X.nbytes/dt/1e9:.1f} GB/s")
del d; torch.cuda.empty_cache()
eta = [1.0] * prob.G
for k in (0, 600, 600):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    fs.fsqr_fit_host(Xp.numpy(), 1, prob.n, prob.p, prob.ld, yp.numpy(), [0.5], [0.002], k,
                     opt=fs.default_options(G=prob.G), eta=eta, flags=fs.DESIGN_PACK2)
    torch.cuda.synchronize(); print(f"fit_host pack2 iters={k}: {time.perf_counter()-t0:.3f} s")
