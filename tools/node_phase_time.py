"""Node-phase (element-result assembly) time of cfg1 right after the element
phase (L2-warm loc, as in a real apply).  Usage: python tools/node_phase_time.py [prec]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2408_12479_b200 import emfgpu as G  # noqa: E402
from paper_2408_12479_b200 import inputs as I  # noqa: E402

prec = int(sys.argv[1]) if len(sys.argv) > 1 else 64
lev = G.FeLevel(32, p=3)
op = G.ElasticOperator(lev, "cnh", G.MaterialParams(mu=1.0, lam=10.0), "none", prec)
op.update_linearization(I.make_u0(32, 32, 32, 3))
dt = torch.float64 if prec == 64 else torch.float32
x = torch.tensor(I.make_v(lev.n_dofs), dtype=dt, device="cuda")
y = torch.empty_like(x)
s = torch.cuda.current_stream()
ts = []
for it in range(25):
    op.apply_elements(x, 0, 32)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    op.apply_nodes(x, y, 0, 96)
    e1.record(s)
    torch.cuda.synchronize()
    if it >= 5:
        ts.append(e0.elapsed_time(e1))
ts.sort()
import hashlib  # noqa: E402
print("EMFGPU_NODE_FLAT=%s y sha1 %s node phase median %.4f ms min %.4f ms" % (
    os.environ.get("EMFGPU_NODE_FLAT", "1"), hashlib.sha1(y.cpu().numpy().tobytes()).hexdigest()[:12],
    ts[len(ts) // 2], ts[0]))
