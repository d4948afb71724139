"""PCIe probe: H2D / D2H / concurrent bandwidth of 21.9 MB pinned buffers and the
pipelined host-vector apply at several chunk counts (cfg1, fp64 none)."""
import os, sys, time, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
n = 2738019
h = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=20):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
mb = n * 8 / 1e6
for name, fn in [("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h2.copy_(d2, non_blocking=True)), ("both", both)]:
    dt = t(fn); print(f"{name:5s} {dt*1e3:.3f} ms  {mb/dt/1e3:.1f} GB/s per direction")
for ch in [4, 8, 16, 32]:
    out = subprocess.run([sys.executable, "-c", f"""
import os, sys, time; sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})
os.environ['EMFGPU_E2E_CHUNKS']='{ch}'
import torch, numpy as np
from paper_2408_12479_b200 import emfgpu as G, inputs as I
lev = G.FeLevel(32, p=3); op = G.ElasticOperator(lev, 'cnh', G.MaterialParams(mu=1.0, lam=10.0), 'none', 64)
op.update_linearization(I.make_u0(32,32,32,3))
hx = torch.tensor(I.make_v(lev.n_dofs)).pin_memory(); hy = torch.empty_like(hx).pin_memory()
for _ in range(3): G.lib().emfgpu_op_apply_host(op.h, hx.data_ptr(), hy.data_ptr())
ts=[]
for _ in range(20):
    t0=time.perf_counter(); G.lib().emfgpu_op_apply_host(op.h, hx.data_ptr(), hy.data_ptr()); ts.append(time.perf_counter()-t0)
print('%.3f' % (1e3*sum(ts)/len(ts)))
"""], capture_output=True, text=True)
    print("chunks", ch, "apply_host ms", out.stdout.strip(), out.stderr[-200:])
