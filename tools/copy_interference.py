"""Element/node kernel time of cfg1 fp64 none alone and with a concurrent
large H2D, D2H or both (separate streams): does PCIe DMA slow the kernels?"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2408_12479_b200 import emfgpu as G  # noqa: E402
from paper_2408_12479_b200 import inputs as I  # noqa: E402

lev = G.FeLevel(32, p=3)
op = G.ElasticOperator(lev, "cnh", G.MaterialParams(mu=1.0, lam=10.0), "none", 64)
op.update_linearization(I.make_u0(32, 32, 32, 3))
dx = torch.tensor(I.make_v(lev.n_dofs), device="cuda")
dy = torch.empty_like(dx)
hb = torch.empty(64 * 2 ** 20, dtype=torch.float64).pin_memory()
db = torch.empty_like(hb, device="cuda")
hb2 = torch.empty_like(hb).pin_memory()
db2 = torch.empty_like(db)
sc, s1, s2 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def timed(kind):
    torch.cuda.synchronize()
    if kind in ("h2d", "both"):
        with torch.cuda.stream(s1):
            db.copy_(hb, non_blocking=True)
    if kind in ("d2h", "both"):
        with torch.cuda.stream(s2):
            hb2.copy_(db2, non_blocking=True)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record(sc)
    for _ in range(10):
        op.apply_elements(dx, 0, 32, stream=sc)
    e[1].record(sc)
    for _ in range(10):
        op.apply_nodes(dx, dy, 0, 96, stream=sc)
    e[2].record(sc)
    torch.cuda.synchronize()
    return e[0].elapsed_time(e[1]) / 10, e[1].elapsed_time(e[2]) / 10


for k in ("none", "h2d", "d2h", "both", "none"):
    el, nd = timed(k)
    print("%-5s elements %.4f ms  nodes %.4f ms" % (k, el, nd))
