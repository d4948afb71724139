import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2408_12479_b200 import emfgpu as G
from paper_2408_12479_b200 import workloads as W
w = W.cfg4(wellposed=True); lev = w.level()
op = G.ElasticOperator(lev, w.model, w.material(), "none", 64); op.update_linearization(np.zeros(lev.n_dofs))
mg = G.MgHierarchy(lev, w.model, w.material(), degree=5, coarse_n=6, precision=32)
mg.update_linearization(torch.zeros(lev.n_dofs, dtype=torch.float64, device="cuda"))
b = torch.tensor(W.rhs(w), device="cuda"); x = torch.empty_like(b)
for warm in (True, False, False):
    if warm:
        try: G.pcg_solve(op, mg, b, x, 1e-8, 2)
        except G.EmfGpuError as e: print("warm-up:", e)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    its, hist = G.pcg_solve(op, mg, b, x, 1e-8, 300); torch.cuda.synchronize()
    print("its", its, "solve_s %.4f" % (time.perf_counter() - t0), flush=True)
