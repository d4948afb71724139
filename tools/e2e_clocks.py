"""SM clocks (nvidia-smi, 100 ms samples) while the pipelined host apply runs
back to back for ~3 s, and the same for device-resident applies."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2408_12479_b200 import emfgpu as G  # noqa: E402
from paper_2408_12479_b200 import inputs as I  # noqa: E402

lev = G.FeLevel(32, p=3)
op = G.ElasticOperator(lev, "cnh", G.MaterialParams(mu=1.0, lam=10.0), "none", 64)
op.update_linearization(I.make_u0(32, 32, 32, 3))
hx = torch.tensor(I.make_v(lev.n_dofs)).pin_memory()
hy = torch.empty_like(hx).pin_memory()
dx = hx.cuda()
dy = torch.empty_like(dx)
for label, fn in (("e2e", lambda: G.lib().emfgpu_op_apply_host(op.h, hx.data_ptr(), hy.data_ptr())),
                  ("device", lambda: op.apply_tangent_device(dx, dy))):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    with bench.ClockSampler(0) as cs:
        t0 = time.time()
        k = 0
        while time.time() - t0 < 3.0:
            fn()
            k += 1
        torch.cuda.synchronize()
    print(label, "calls", k, "ms/call %.3f" % (3000.0 / k), cs.summary())
