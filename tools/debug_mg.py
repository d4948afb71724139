import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2408_12479_b200 import emfgpu as G
prm = G.MaterialParams(mu=1.0, lam=10.0, kappa_b=50.0)
for (n, p) in [(1, 1), (2, 1), (4, 1), (4, 2)]:
    lev = G.FeLevel(n, p=p)
    op = G.ElasticOperator(lev, "inh", prm, "none", 32)
    op.update_linearization(np.zeros(lev.n_dofs))
    d, nb = op.compute_diagonal()
    print(n, p, "ndofs", lev.n_dofs, "diag min/max", d.min(), d.max(), "nbad", nb, "nan", np.isnan(d).any())
    # dense K via applies
    N = lev.n_dofs
    K = np.zeros((N, N))
    for j in range(N):
        e = np.zeros(N, np.float32); e[j] = 1
        K[:, j] = op.apply_tangent(e)
    print("   sym", np.abs(K - K.T).max(), "eig min", np.linalg.eigvalsh(0.5 * (K + K.T)).min(), "diag match", np.abs(np.diag(K) - d).max())
lev = G.FeLevel(4, p=2)
mg = G.MgHierarchy(lev, "inh", prm, degree=5, coarse_n=1, precision=32, coarse_maxit=5000)
print(mg.levels())
u0 = torch.zeros(lev.n_dofs, dtype=torch.float64, device="cuda")
mg.update_linearization(u0)
r = torch.randn(lev.n_dofs, dtype=torch.float64, device="cuda")
z = torch.empty_like(r)
try:
    mg.precondition(r, z); torch.cuda.synchronize()
    print("z norm", z.norm().item())
except Exception as ex:
    print("precondition failed:", ex)
