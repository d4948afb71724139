"""PCIe copy behaviour behind the e2e apply (cfg2 sized, 407 MB each way,
pinned host memory): whole vs chunked copies, one direction or both at
once.  python tools/pcie_chunks.py"""
import time

import numpy as np
import torch

n = 3 * 257 ** 3
hx = torch.empty(n, dtype=torch.float64).pin_memory()
hy = torch.empty(n, dtype=torch.float64).pin_memory()
hx.uniform_()
dx = torch.empty(n, dtype=torch.float64, device="cuda")
dy = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        a = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - a)
    return 1e3 * np.median(ts)


def h2d(ch):
    def f():
        with torch.cuda.stream(s1):
            for c in range(ch):
                a, b = c * n // ch, (c + 1) * n // ch
                dx[a:b].copy_(hx[a:b], non_blocking=True)
    return f


def d2h(ch):
    def f():
        with torch.cuda.stream(s2):
            for c in range(ch):
                a, b = c * n // ch, (c + 1) * n // ch
                hy[a:b].copy_(dy[a:b], non_blocking=True)
    return f


def both(ch):
    f1, f2 = h2d(ch), d2h(ch)
    return lambda: (f1(), f2())


def pipelined(ch):
    """D2H of chunk c waits for H2D of chunk c (the e2e schedule, no compute)"""
    def f():
        evs = []
        with torch.cuda.stream(s1):
            for c in range(ch):
                a, b = c * n // ch, (c + 1) * n // ch
                dx[a:b].copy_(hx[a:b], non_blocking=True)
                e = torch.cuda.Event()
                e.record(s1)
                evs.append(e)
        with torch.cuda.stream(s2):
            for c in range(ch):
                a, b = c * n // ch, (c + 1) * n // ch
                s2.wait_event(evs[c])
                hy[a:b].copy_(dy[a:b], non_blocking=True)
    return f


gb = n * 8 / 1e9
for ch in (1, 4, 16, 64):
    t1, t2, t3 = timeit(h2d(ch)), timeit(d2h(ch)), timeit(both(ch))
    t4 = timeit(pipelined(ch)) if ch > 1 else float("nan")
    print(f"chunks {ch:3d}: H2D {t1:.3f} ms ({gb / t1 * 1e3:.1f} GB/s)  D2H {t2:.3f} ms ({gb / t2 * 1e3:.1f} GB/s)  "
          f"both {t3:.3f} ms  pipelined {t4:.3f} ms", flush=True)
