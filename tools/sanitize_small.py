"""Small applies of every element-kernel family for compute-sanitizer runs:
python tools/sanitize_small.py  (run under compute-sanitizer --tool memcheck|racecheck)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2408_12479_b200 import emfgpu as G  # noqa: E402
from paper_2408_12479_b200 import inputs as I  # noqa: E402

prm = G.MaterialParams(mu=1.0, lam=10.0, kappa_b=50.0)
cases = [(4, 3, "cnh", s, prec, d) for s in ("none", "scalar", "tensor", "cachedF") for prec in (64, 32)
         for d in ("material",)] + [(4, 3, "inh", s, prec, "spatial") for s in ("none", "tensor") for prec in (64, 32)]
cases += [(4, 2, "fiber", "none", 32, "material"), (2, 4, "inh", "none", 64, "material"),
          (4, 1, "cnh", "none", 64, "material")]
# the collocated Q3 / Q4 kernels, the push-forward tensor cache (iNH, fibre), odd element counts
cases += [(3, 3, "inh", s, prec, "material") for s in ("none", "tensor") for prec in (64, 32)]
cases += [(3, 3, "fiber", "tensor", prec, "material") for prec in (64, 32)]
cases += [(2, 4, m, s, prec, "material") for m in ("inh", "fiber") for s in ("tensor", "cachedF") for prec in (64, 32)]
cases += [(2, 4, "inh", "none", 32, "material"), (3, 2, "cnh", "tensor", 64, "material")]
for n, p, model, strat, prec, dom in cases:
    for mp in (0.0, 0.05):
        lev = G.FeLevel(n, p=p, map_param=(mp,))
        op = G.ElasticOperator(lev, model, prm, strat, prec, domain=dom)
        op.update_linearization(I.make_u0(n, n, n, p, amp=0.05))
        y = op.apply_tangent(I.make_v(lev.n_dofs))
        d, nb = op.compute_diagonal()
        r = op.evaluate_residual(I.make_u0(n, n, n, p, amp=0.05))
        assert np.isfinite(y).all() and np.isfinite(d).all() and np.isfinite(r).all()
print("ok")
