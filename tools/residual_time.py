"""evaluate_residual device time (L2 flushed) on cfg2 (64^3 Q4 curved iNH) and
cfg1 (32^3 Q3 cNH), fp64 and fp32, both domains:
EMFGPU_LIB=... python tools/residual_time.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2408_12479_b200 import emfgpu as G  # noqa: E402
from paper_2408_12479_b200 import inputs as I  # noqa: E402
from paper_2408_12479_b200 import workloads as W  # noqa: E402

flush = torch.empty(256 * 2 ** 20 // 4, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream()
lib = os.path.basename(os.environ.get("EMFGPU_LIB", "libemfgpu.so"))


def run(name, lev, model, mat, u0, prec, dom):
    op = G.ElasticOperator(lev, model, mat, "none", prec, domain=dom)
    op.update_linearization(u0)
    dt = torch.float64 if prec == 64 else torch.float32
    du = torch.tensor(u0, dtype=dt, device="cuda")
    r = torch.empty_like(du)
    for _ in range(3):
        op.evaluate_residual_device(du, r)
    ts = []
    for _ in range(10):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        op.evaluate_residual_device(du, r)
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    t = ts[len(ts) // 2]
    print("%s %s fp%d %s: residual %.4f ms (%.3e DoF/s) ||r|| %.12e" % (
        lib, name, prec, dom, t, lev.n_dofs / (t * 1e-3), float(torch.linalg.vector_norm(r.double()))), flush=True)


w = W.cfg2()
lev2 = w.level()
u2 = w.u0()
for prec in (64, 32):
    for dom in ("material", "spatial"):
        run("cfg2", lev2, "inh", w.material(), u2, prec, dom)
del lev2
lev1 = G.FeLevel(32, p=3)
u1 = I.make_u0(32, 32, 32, 3, noise=1e-3 * 8 / 32)
for prec in (64, 32):
    run("cfg1", lev1, "cnh", G.MaterialParams(mu=1.0, lam=10.0, kappa_b=1000.0), u1, prec, "material")
