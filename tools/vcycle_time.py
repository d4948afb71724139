import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2408_12479_b200 import emfgpu as G, workloads as W
w = W.cfg4(wellposed=True)
lev = w.level()
op = G.ElasticOperator(lev, w.model, w.material(), "none", 64)
op.update_linearization(np.zeros(lev.n_dofs))
mg = G.MgHierarchy(lev, w.model, w.material(), degree=5, coarse_n=6, precision=32)
mg.update_linearization(torch.zeros(lev.n_dofs, dtype=torch.float64, device="cuda"))
b = torch.tensor(W.rhs(w), device="cuda"); z = torch.empty_like(b); y = torch.empty_like(b)
ts = []; ta = []
for i in range(40):
    e0, e1, e2 = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    t0 = time.perf_counter()
    e0.record(); mg.precondition(b, z); e1.record(); op.apply_tangent_device(b, y); e2.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1)); ta.append(e1.elapsed_time(e2))
print("vcycle ms:", " ".join("%.1f" % t for t in ts))
print("apply ms:", " ".join("%.2f" % t for t in ta))
