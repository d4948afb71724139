"""Race proxy (compute-sanitizer is not available on the pool): repeated applies,
residuals and diagonals of the element-kernel families must be bitwise equal
run to run at sizes where every SM holds several CTAs."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2408_12479_b200 import emfgpu as G  # noqa: E402
from paper_2408_12479_b200 import inputs as I  # noqa: E402

prm = G.MaterialParams(mu=1.0, lam=10.0, kappa_b=50.0)
cases = [(17, 3, m, s, prec, 0.05) for m in ("cnh", "inh", "fiber") for s in ("none", "scalar", "tensor", "cachedF")
         for prec in (64, 32)]
cases += [(13, 4, m, s, prec, 0.05) for m in ("inh", "fiber") for s in ("none", "tensor", "cachedF") for prec in (64, 32)]
cases += [(17, 3, "cnh", s, prec, 0.0) for s in ("none", "tensor") for prec in (64, 32)]
cases += [(21, 2, "inh", "tensor", 32, 0.0), (21, 2, "cnh", "none", 32, 0.0)]
bad = 0
for n, p, model, strat, prec, mp in cases:
    lev = G.FeLevel(n, p=p, map_param=(mp,))
    op = G.ElasticOperator(lev, model, prm, strat, prec)
    u0 = I.make_u0(n, n, n, p, amp=0.02, noise=1e-4)
    op.update_linearization(u0)
    dt = torch.float64 if prec == 64 else torch.float32
    x = torch.tensor(I.make_v(lev.n_dofs), dtype=dt, device="cuda")
    du = torch.tensor(u0, dtype=dt, device="cuda")
    y0 = torch.empty_like(x)
    r0 = torch.empty_like(x)
    op.apply_tangent_device(x, y0)
    op.evaluate_residual_device(du, r0)
    ok = bool(torch.isfinite(y0).all()) and bool(torch.isfinite(r0).all())
    y = torch.empty_like(x)
    r = torch.empty_like(x)
    for _ in range(30):
        op.apply_tangent_device(x, y)
        op.evaluate_residual_device(du, r)
        ok = ok and torch.equal(y, y0) and torch.equal(r, r0)
    print(n, p, model, strat, prec, mp, "OK" if ok else "MISMATCH", flush=True)
    bad += 0 if ok else 1
print("bad", bad)
sys.exit(1 if bad else 0)
