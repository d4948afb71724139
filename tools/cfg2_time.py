"""cfg2 (64^3 Q4 curved iNH) element-phase and whole-apply timing, L2 flushed,
with the full-size known answers checked (tests/golden/cfg2_full.json):
EMFGPU_LIB=... python tools/cfg2_time.py [prec:strategy ...]   (default 64:none)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2408_12479_b200 import emfgpu as G  # noqa: E402
from paper_2408_12479_b200 import workloads as W  # noqa: E402

cases = sys.argv[1:] or ["64:none"]
ref = json.load(open(os.path.join(ROOT, "tests", "golden", "cfg2_full.json")))
w = W.cfg2()
lev = w.level()
u0, v = w.u0(), w.v()
flush = torch.empty(256 * 2 ** 20 // 4, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream()
lib = os.path.basename(os.environ.get("EMFGPU_LIB", "libemfgpu.so"))
for c in cases:
    prec, strat = c.split(":")
    prec = int(prec)
    op = G.ElasticOperator(lev, "inh", w.material(), strat, prec)
    op.update_linearization(u0)
    dt = torch.float64 if prec == 64 else torch.float32
    x = torch.tensor(v, dtype=dt, device="cuda")
    y = torch.empty_like(x)
    op.apply_tangent_device(x, y)
    torch.cuda.synchronize()
    yn = float(torch.linalg.vector_norm(y.double()))
    err = abs(yn - ref["norm_y64"]) / ref["norm_y64"]
    for _ in range(3):
        op.apply_tangent_device(x, y)
    res = {}
    for name, fn in (("apply", lambda: op.apply_tangent_device(x, y)), ("elements", lambda: op.apply_elements(x, 0, 64))):
        ts = []
        for _ in range(12):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            fn()
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        res[name] = ts[len(ts) // 2]
    print("%s fp%d %s: apply %.4f ms (%.3e DoF/s), elements %.4f ms, | ||y|| rel err %.1e" % (
        lib, prec, strat, res["apply"], lev.n_dofs / (res["apply"] * 1e-3), res["elements"], err), flush=True)
    del op, x, y
