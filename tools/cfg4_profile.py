"""cfg4 (well-posed variant) PCG + fp32 hp-MG solve, for an ncu launch list
(python tools/cfg4_profile.py [iterations [reps [level strategy]]]); prints the solve time."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2408_12479_b200 import emfgpu as G  # noqa: E402
from paper_2408_12479_b200 import workloads as W  # noqa: E402

its_max = int(sys.argv[1]) if len(sys.argv) > 1 else 300
w = W.cfg4(wellposed=True)
lev = w.level()
op_strategy = sys.argv[4] if len(sys.argv) > 4 else "none"  # strategy of the outer fp64 operator
op = G.ElasticOperator(lev, w.model, w.material(), op_strategy, 64)
op.update_linearization(np.zeros(lev.n_dofs))
mg_strategy = sys.argv[3] if len(sys.argv) > 3 else "none"  # storage strategy of the V-cycle's level operators
t0 = time.perf_counter()
mg = G.MgHierarchy(lev, w.model, w.material(), strategy=mg_strategy, degree=5, coarse_n=6, precision=32)
mg.update_linearization(torch.zeros(lev.n_dofs, dtype=torch.float64, device="cuda"))
torch.cuda.synchronize()
print("hierarchy (%s levels) create + linearize %.3f s" % (mg_strategy, time.perf_counter() - t0))
b = torch.tensor(W.rhs(w), device="cuda")
x = torch.empty_like(b)
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
for _ in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    try:
        its, hist = G.pcg_solve(op, mg, b, x, 1e-8, its_max)
    except G.EmfGpuError as e:  # a capped iteration count (launch lists) stops unconverged
        its = its_max
        print(e)
    torch.cuda.synchronize()
    print("its", its, "solve_s %.4f" % (time.perf_counter() - t0), "levels", mg.levels(), flush=True)
