"""Where the cfg4 setup time goes (host wall clock, synchronised after each step)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2408_12479_b200 import emfgpu as G  # noqa: E402
from paper_2408_12479_b200 import workloads as W  # noqa: E402

torch.zeros(1, device="cuda")
w = W.cfg4(wellposed=True)


def step(name, fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    print("%-44s %.3f s" % (name, time.perf_counter() - t), flush=True)
    return r


for rep in range(2):
    print("rep", rep)
    lev = step("FeLevel (mesh, geometry)", lambda: w.level())
    op = step("ElasticOperator(none, fp64)", lambda: G.ElasticOperator(lev, w.model, w.material(), "none", 64))
    u0 = np.zeros(lev.n_dofs)
    step("op.update_linearization(host u0)", lambda: op.update_linearization(u0))
    strat = sys.argv[1] if len(sys.argv) > 1 else "none"
    mg = step("MgHierarchy(%s, fp32) create" % strat,
              lambda: G.MgHierarchy(lev, w.model, w.material(), strategy=strat, degree=5, coarse_n=6, precision=32))
    du = torch.zeros(lev.n_dofs, dtype=torch.float64, device="cuda")
    step("mg.update_linearization(device u)", lambda: mg.update_linearization(du))
    step("mg.update_linearization again", lambda: mg.update_linearization(du))
    del mg, op, lev
