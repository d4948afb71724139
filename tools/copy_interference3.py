"""Element kernel time (full cfg1 and a 4-layer chunk) while a pinned H2D copy
of 19 MB or 512 MB, or a D2D copy, runs on another stream."""
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
small_h = torch.empty(int(19e6 / 8), dtype=torch.float64).pin_memory()
small_d = torch.empty_like(small_h, device="cuda")
big_h = torch.empty(64 * 2 ** 20, dtype=torch.float64).pin_memory()
big_d = torch.empty_like(big_h, device="cuda")
big_d2 = torch.empty_like(big_d)
sc, s1 = torch.cuda.Stream(), torch.cuda.Stream()


def t(kind, layers):
    torch.cuda.synchronize()
    with torch.cuda.stream(s1):
        if kind == "h2d19MB":
            small_d.copy_(small_h, non_blocking=True)
        elif kind == "h2d512MB":
            big_d.copy_(big_h, non_blocking=True)
        elif kind == "d2d512MB":
            big_d2.copy_(big_d, non_blocking=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(sc)
    op.apply_elements(dx, 0, layers, stream=sc)
    e1.record(sc)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


for layers in (4, 32):
    for kind in ("none", "h2d19MB", "h2d512MB", "d2d512MB", "none"):
        v = sorted(t(kind, layers) for _ in range(5))
        print("layers %2d %-9s %.4f ms (min) %.4f (max)" % (layers, kind, v[0], v[-1]))
