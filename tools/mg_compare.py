"""cfg4-style hp-MG parity at intermediate sizes: the reference's
MgHierarchy<float> + fp64 PCG (oracle/_ref, here in the build container:
`python tools/mg_compare.py ref N`) against the device hierarchy (on the GPU
box: `python tools/mg_compare.py gpu N`), same seeded r / b, kappa/mu = 50,
u0 = 0, Q4, dense coarse solve; prints V-cycle rel. difference and PCG
iterations."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2408_12479_b200 import inputs as I  # noqa: E402

mode, n = sys.argv[1], int(sys.argv[2])
lim = int(sys.argv[3]) if len(sys.argv) > 3 else 2000
p = int(sys.argv[4]) if len(sys.argv) > 4 else 4
out = os.path.join(ROOT, "tools", f"mgcmp_{n}_{lim}_{p}.npz")
if mode == "ref":
    from oracle import refbind as R
    n0, lv = {6: (6, 0), 12: (6, 1), 24: (6, 2), 48: (6, 3), 8: (1, 3), 16: (1, 4), 4: (1, 2), 3: (3, 0), 2: (2, 0)}[n]
    L = R.RefLevel(n0, lv, p, 0.0, 1)
    prm = R.material_params(mu=1.0, lam=10.0, kappa=50.0)
    mg = R.RefMg(L, "inh", prm, degree=5, coarse_direct_limit=lim)
    mg.update_linearization(np.zeros(L.ndofs))
    r = I.make_v(L.ndofs, 11)
    z = mg.precondition(r)
    op = R.RefOperator(L, "inh", prm, "none", 64)
    op.update_linearization(np.zeros(L.ndofs))
    b = I.make_v(L.ndofs, 2)
    b[I.dirichlet_mask(n, n, n, p, 1)] = 0.0
    x, its, hist = R.pcg_solve(op, mg, b, 1e-8, 300)
    np.savez(out, r=r, z=z, b=b, its=its, hist=hist, levels=mg.n_levels)
    print("ref", n, "levels", mg.n_levels, "its", its)
else:
    import torch
    from paper_2408_12479_b200 import emfgpu as G
    g = np.load(out)
    lev = G.FeLevel(n, p=p)
    prm = G.MaterialParams(mu=1.0, lam=10.0, kappa_b=50.0)
    coarse = {6: 6, 12: 6, 24: 6, 48: 6, 3: 3, 2: 2}.get(n, 1)
    mg = G.MgHierarchy(lev, "inh", prm, degree=5, coarse_n=coarse, precision=32, coarse_direct_limit=lim)
    mg.update_linearization(torch.zeros(lev.n_dofs, dtype=torch.float64, device="cuda"))
    r = torch.tensor(g["r"], device="cuda")
    z = torch.empty_like(r)
    mg.precondition(r, z)
    torch.cuda.synchronize()
    zz = z.cpu().numpy()
    print("gpu", n, "levels", mg.n_levels, mg.levels(), "V-cycle rel diff %.3e" % (np.linalg.norm(zz - g["z"]) / np.linalg.norm(g["z"])))
    op = G.ElasticOperator(lev, "inh", prm, "none", 64)
    op.update_linearization(np.zeros(lev.n_dofs))
    b = torch.tensor(g["b"], device="cuda")
    x = torch.empty_like(b)
    its, hist = G.pcg_solve(op, mg, b, x, 1e-8, 300)
    print("its gpu", its, "ref", int(g["its"]))
    h = g["hist"]
    for k in range(0, min(len(hist), len(h)), 5):
        print(k, "%.3e %.3e" % (hist[k], h[k]))
