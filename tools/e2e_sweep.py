"""e2e (pinned host vectors) apply time of cfg1 fp64 none vs the z-chunk count
of the pipelined host apply (EMFGPU_E2E_CHUNKS).  Usage: python tools/e2e_sweep.py"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, ROOT)
    import time

    import torch

    from paper_2408_12479_b200 import emfgpu as G
    from paper_2408_12479_b200 import inputs as I
    lev = G.FeLevel(32, p=3)
    op = G.ElasticOperator(lev, "cnh", G.MaterialParams(mu=1.0, lam=10.0), "none", 64)
    op.update_linearization(I.make_u0(32, 32, 32, 3))
    hx = torch.tensor(I.make_v(lev.n_dofs)).pin_memory()
    hy = torch.empty_like(hx).pin_memory()
    for _ in range(5):
        G.lib().emfgpu_op_apply_host(op.h, hx.data_ptr(), hy.data_ptr())
    ts = []
    for _ in range(30):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        G.lib().emfgpu_op_apply_host(op.h, hx.data_ptr(), hy.data_ptr())
        ts.append(time.perf_counter() - t0)
    ts.sort()
    print(os.environ.get("EMFGPU_E2E_CHUNKS"), "median %.4f ms  min %.4f ms" % (1e3 * ts[len(ts) // 2], 1e3 * ts[0]))
else:
    for n in (1, 2, 4, 8, 12, 16, 32):
        env = dict(os.environ, EMFGPU_E2E_CHUNKS=str(n))
        subprocess.run([sys.executable, __file__, "child"], env=env, check=True)
