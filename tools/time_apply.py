"""Device-resident apply timing (L2 flushed) of one configuration:
python tools/time_apply.py n p model strategy precision [curved_amp] [domain]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2408_12479_b200 import emfgpu as G  # noqa: E402
from paper_2408_12479_b200 import inputs as I  # noqa: E402

n, p, model, strat, prec = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4], int(sys.argv[5])
amp = float(sys.argv[6]) if len(sys.argv) > 6 else 0.0
dom = sys.argv[7] if len(sys.argv) > 7 else "material"
lev = G.FeLevel(n, p=p, map_param=(amp,))
op = G.ElasticOperator(lev, model, G.MaterialParams(mu=1.0, lam=10.0, kappa_b=1000.0), strat, prec, domain=dom)
op.update_linearization(I.make_u0(n, n, n, p, noise=1e-3 * 8 / n))
dt = torch.float64 if prec == 64 else torch.float32
x = torch.tensor(I.make_v(lev.n_dofs), dtype=dt, device="cuda")
y = torch.empty_like(x)
flush = torch.empty(256 * 2 ** 20 // 4, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream()
for _ in range(3):
    op.apply_tangent_device(x, y)
ts = []
for _ in range(15):
    flush.fill_(1.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    op.apply_elements(x, 0, n)
    e1.record(s)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
print("%s n=%d p=%d %s %s fp%d: element phase %.4f ms, %.3e DoF/s (elements only)" % (
    dom, n, p, model, strat, prec, ts[len(ts) // 2], lev.n_dofs / (ts[len(ts) // 2] * 1e-3)))
