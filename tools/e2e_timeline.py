"""Timeline of the chunked host-vector apply on cfg2 (fp64 none), replayed
through the public split API with timing events on the three streams, plus
copy-only variants of the same schedule:
python tools/e2e_timeline.py [schedule ...]   schedule = N (uniform chunks) or
comma-separated layer counts, e.g. 2,12,18,18,12,2; --timeline prints events"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2408_12479_b200 import emfgpu as G  # noqa: E402
from paper_2408_12479_b200 import workloads as W  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")] or ["16"]
show = "--timeline" in sys.argv
w = W.cfg2()
lev = w.level()
op = G.ElasticOperator(lev, "inh", w.material(), "none", 64)
op.update_linearization(w.u0())
hx = torch.tensor(w.v()).pin_memory()
hy = torch.empty_like(hx).pin_memory()
dx = torch.empty(hx.numel(), dtype=torch.float64, device="cuda")
dy = torch.empty_like(dx)
nz, p = lev.nz, lev.p
mx, my = lev.nx * p + 1, lev.ny * p + 1
mz = nz * p + 1
plane = 3 * mx * my
sh, sc, sd = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def bounds_of(spec):
    if "," in spec:
        ks = [int(v) for v in spec.split(",")]
    else:
        c = int(spec)
        per = (nz + c - 1) // c
        ks = [min(per, nz - i * per) for i in range(c) if i * per < nz]
    assert sum(ks) == nz, spec
    b = np.cumsum([0] + ks)
    return [(int(b[i]), int(b[i + 1])) for i in range(len(ks))]


def run(mode, timeline=False):
    """mode: full | copies | nocompute-dep"""
    ev = lambda: torch.cuda.Event(enable_timing=timeline)  # noqa: E731
    t0 = ev()
    t0.record(torch.cuda.current_stream())
    for s in (sh, sc, sd):
        s.wait_event(t0)
    eh, ec, ed = [], [], []
    done = -1
    for i in range(nch):
        k1 = bnd[i][1]
        hi = k1 * p
        with torch.cuda.stream(sh):
            if hi > done:
                dx[(done + 1) * plane:(hi + 1) * plane].copy_(hx[(done + 1) * plane:(hi + 1) * plane], non_blocking=True)
                done = hi
            e = ev()
            e.record(sh)
            eh.append(e)
    for i in range(nch):
        k0, k1 = bnd[i]
        c0, c1 = k0 * p, (mz - 1 if k1 == nz else k1 * p - 1)
        with torch.cuda.stream(sc):
            sc.wait_event(eh[i])
            if mode == "full":
                op.apply_elements(dx, k0, k1, stream=sc.cuda_stream)
                op.apply_nodes(dx, dy, c0, c1, stream=sc.cuda_stream)
            e = ev()
            e.record(sc)
            ec.append(e)
        with torch.cuda.stream(sd):
            sd.wait_event(ec[i])
            hy[c0 * plane:(c1 + 1) * plane].copy_(dy[c0 * plane:(c1 + 1) * plane], non_blocking=True)
            e = ev()
            e.record(sd)
            ed.append(e)
    torch.cuda.synchronize()
    if timeline:
        f = lambda e: t0.elapsed_time(e)  # noqa: E731
        for i in range(nch):
            print(f"  chunk {i:2d}: h2d done {f(eh[i]):7.3f}  compute done {f(ec[i]):7.3f}  d2h done {f(ed[i]):7.3f}")


for spec in args:
    bnd = bounds_of(spec)
    nch = len(bnd)
    res = []
    for mode in ("full", "copies"):
        for _ in range(2):
            run(mode)
        ts = []
        for _ in range(6):
            torch.cuda.synchronize()
            a = time.perf_counter()
            run(mode)
            ts.append(time.perf_counter() - a)
        res.append(1e3 * np.median(ts))
    print(f"schedule {spec:28s}: full {res[0]:.3f} ms  copies only {res[1]:.3f} ms", flush=True)
    if show:
        print("timeline (full, timing events):")
        run("full", timeline=True)
op_ts = []
for _ in range(3):
    G.lib().emfgpu_op_apply_host(op.h, hx.data_ptr(), hy.data_ptr())
for _ in range(6):
    torch.cuda.synchronize()
    a = time.perf_counter()
    G.lib().emfgpu_op_apply_host(op.h, hx.data_ptr(), hy.data_ptr())
    op_ts.append(time.perf_counter() - a)
print(f"emfgpu_op_apply_host: median {1e3 * np.median(op_ts):.3f} ms")
