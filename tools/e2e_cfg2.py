"""e2e (pinned host vectors, emfgpu_op_apply_host) time of cfg2 fp64 none vs
the z-chunk schedule of the pipelined host apply (EMFGPU_E2E_CHUNKS,
EMFGPU_E2E_TAIL), and the plain copy floors: python tools/e2e_cfg2.py [chunks:tail ...]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, ROOT)
    import time

    import torch

    from paper_2408_12479_b200 import emfgpu as G
    from paper_2408_12479_b200 import workloads as W
    w = W.cfg2()
    lev = w.level()
    op = G.ElasticOperator(lev, "inh", w.material(), "none", 64)
    op.update_linearization(w.u0())
    hx = torch.tensor(w.v()).pin_memory()
    hy = torch.empty_like(hx).pin_memory()
    for _ in range(3):
        G.lib().emfgpu_op_apply_host(op.h, hx.data_ptr(), hy.data_ptr())
    ts = []
    for _ in range(8):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        G.lib().emfgpu_op_apply_host(op.h, hx.data_ptr(), hy.data_ptr())
        ts.append(time.perf_counter() - t0)
    ts.sort()
    dx = torch.empty(hx.numel(), dtype=torch.float64, device="cuda")
    dy = torch.empty_like(dx)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    cp = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(s1):
            dx.copy_(hx, non_blocking=True)
        with torch.cuda.stream(s2):
            hy.copy_(dy, non_blocking=True)
        torch.cuda.synchronize()
        cp.append(time.perf_counter() - t0)
    h2d = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dx.copy_(hx, non_blocking=True)
        torch.cuda.synchronize()
        h2d.append(time.perf_counter() - t0)
    print("chunks %s tail %s: e2e %.3f ms (min %.3f); duplex copy floor %.3f ms; H2D alone %.3f ms (%.1f GB/s)" % (
        os.environ.get("EMFGPU_E2E_CHUNKS", "default"), os.environ.get("EMFGPU_E2E_TAIL", "default"), 1e3 * ts[len(ts) // 2], 1e3 * ts[0], 1e3 * min(cp),
        1e3 * min(h2d), hx.numel() * 8 / min(h2d) / 1e9), flush=True)
else:
    for c in (sys.argv[1:] or ["16:0", "16:4"]):  # chunks:tail
        ch, tl = c.split(":")
        subprocess.run([sys.executable, __file__, "child"], env=dict(os.environ, EMFGPU_E2E_CHUNKS=ch, EMFGPU_E2E_TAIL=tl))
