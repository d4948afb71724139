"""Small driver for ncu captures: cfg1 (32^3 Q3 cNH) tangent applies of one
variant.  Usage: python tools/profile_apply.py [precision] [strategy] [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2408_12479_b200 import emfgpu as G  # noqa: E402
from paper_2408_12479_b200 import inputs as I  # noqa: E402

prec = int(sys.argv[1]) if len(sys.argv) > 1 else 64
strat = sys.argv[2] if len(sys.argv) > 2 else "none"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
model = sys.argv[4] if len(sys.argv) > 4 else "cnh"
n, p = (32, 3) if len(sys.argv) <= 5 else (int(sys.argv[5]), int(sys.argv[6]))
lev = G.FeLevel(n, p=p)
print("affine", lev.affine, "cartesian", lev.cartesian)
op = G.ElasticOperator(lev, model, G.MaterialParams(mu=1.0, lam=10.0, kappa_b=1000.0), strat, prec)
op.update_linearization(I.make_u0(n, n, n, p))
dt = torch.float64 if prec == 64 else torch.float32
x = torch.tensor(I.make_v(lev.n_dofs), dtype=dt, device="cuda")
y = torch.empty_like(x)
for _ in range(reps):
    op.apply_tangent_device(x, y)
torch.cuda.synchronize()
print("ok", float(torch.linalg.norm(y.double())))
