"""cfg3 (fibre tube 16x128x256 Q3, per-qp frames, strategy tensor) element-phase
and whole-apply time, L2 flushed: EMFGPU_LIB=... python tools/cfg3_time.py [64 32]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2408_12479_b200 import emfgpu as G  # noqa: E402
from paper_2408_12479_b200 import workloads as W  # noqa: E402

precs = [int(a) for a in sys.argv[1:]] or [64, 32]
w = W.cfg3()
lev = w.level()
u0 = W.tube_u0(w, lev.node_coords())
v = w.v()
flush = torch.empty(256 * 2 ** 20 // 4, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream()
lib = os.path.basename(os.environ.get("EMFGPU_LIB", "libemfgpu.so"))
for prec in precs:
    op = G.ElasticOperator(lev, "fiber", w.material(), "tensor", prec)
    op.set_fibre_frame("cylindrical")
    op.update_linearization(u0)
    dt = torch.float64 if prec == 64 else torch.float32
    x = torch.tensor(v, dtype=dt, device="cuda")
    y = torch.empty_like(x)
    for _ in range(3):
        op.apply_tangent_device(x, y)
    res = {}
    for name, fn in (("apply", lambda: op.apply_tangent_device(x, y)), ("elements", lambda: op.apply_elements(x, 0, lev.nz))):
        ts = []
        for _ in range(10):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            fn()
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        res[name] = ts[len(ts) // 2]
    print("%s cfg3 fp%d tensor: apply %.4f ms (%.3e DoF/s), elements %.4f ms, ||y|| %.12e" % (
        lib, prec, res["apply"], lev.n_dofs / (res["apply"] * 1e-3), res["elements"],
        float(torch.linalg.vector_norm(y.double()))), flush=True)
    del op, x, y
