"""Break down the cfg4 (48^3 Q4 iNH) solver setup time: hierarchy creation and
update_linearization (cold and warm)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2408_12479_b200 import emfgpu as G  # noqa: E402
from paper_2408_12479_b200 import workloads as W  # noqa: E402

w = W.cfg4(wellposed=True)
t = time.perf_counter()
lev = w.level()
torch.cuda.synchronize()
print("fine level create %.3f s" % (time.perf_counter() - t))
t = time.perf_counter()
mg = G.MgHierarchy(lev, w.model, w.material(), degree=5, coarse_n=6, precision=32)
torch.cuda.synchronize()
print("hierarchy create %.3f s (%d levels)" % (time.perf_counter() - t, mg.n_levels))
u = torch.zeros(lev.n_dofs, dtype=torch.float64, device="cuda")
for k in range(3):
    t = time.perf_counter()
    mg.update_linearization(u)
    torch.cuda.synchronize()
    print("update_linearization #%d %.3f s" % (k, time.perf_counter() - t))
op = G.ElasticOperator(lev, w.model, w.material(), "none", 64)
t = time.perf_counter()
op.update_linearization_device(u)
torch.cuda.synchronize()
print("fine op linearize (device u) %.4f s" % (time.perf_counter() - t))
d = torch.empty_like(u)
t = time.perf_counter()
op.compute_diagonal_device(d)
torch.cuda.synchronize()
print("fine diagonal %.4f s" % (time.perf_counter() - t))
