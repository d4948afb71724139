"""Device apply (emfgpu_op_apply) vs the split-phase entry points
(apply_elements + apply_nodes): bitwise equality and device time per apply
(L2 flushed), for a list of configurations.  With EMFGPU_LIB pointing at a
variant build (tools/build_variant.sh) it is the launch-bound A/B harness.
python tools/apply_ab.py [n p model strategy precision [amp]]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2408_12479_b200 import emfgpu as G  # noqa: E402
from paper_2408_12479_b200 import inputs as I  # noqa: E402

CASES = [
    (32, 3, "cnh", "none", 64, 0.0),
    (32, 3, "cnh", "scalar", 64, 0.0),
    (32, 3, "cnh", "none", 64, 0.05),
    (24, 4, "inh", "none", 64, 0.1),
    (32, 2, "cnh", "none", 64, 0.0),
    (32, 1, "cnh", "none", 64, 0.0),
]


def timed(fn, flush, reps=15):
    s = torch.cuda.current_stream()
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn()
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    cases = CASES
    if len(sys.argv) > 1:
        a = sys.argv[1:]
        cases = [(int(a[0]), int(a[1]), a[2], a[3], int(a[4]), float(a[5]) if len(a) > 5 else 0.0,
                  a[6] if len(a) > 6 else "material")]
    flush = torch.empty(256 * 2 ** 20 // 4, dtype=torch.float32, device="cuda")
    for case in cases:
        n, p, model, strat, prec, amp = case[:6]
        dom = case[6] if len(case) > 6 else "material"
        lev = G.FeLevel(n, p=p, map_param=(amp,), dirichlet_faces=1)
        op = G.ElasticOperator(lev, model, G.MaterialParams(mu=1.0, lam=10.0, kappa_b=1000.0), strat, prec,
                               domain=dom)
        op.update_linearization(I.make_u0(n, n, n, p, noise=1e-3 * 8 / n))
        dt = torch.float64 if prec == 64 else torch.float32
        x = torch.tensor(I.make_v(lev.n_dofs), dtype=dt, device="cuda")
        y1 = torch.empty_like(x)
        y2 = torch.empty_like(x)
        mz = n * p + 1

        def whole():
            op.apply_tangent_device(x, y1)

        def split():
            op.apply_elements(x, 0, n)
            op.apply_nodes(x, y2, 0, mz - 1)

        whole()
        split()
        torch.cuda.synchronize()
        same = torch.equal(y1, y2)
        for _ in range(3):  # repeated launches must rewind the ticket counters
            whole()
        torch.cuda.synchronize()
        same = same and torch.equal(y1, y2)
        tf, ts = timed(whole, flush), timed(split, flush)
        print("n=%d p=%d %s %s %s fp%d amp=%g: bitwise %s  apply %.4f ms  split %.4f ms  (%.1f%%)  %.3e DoF/s" % (
            n, p, model, dom[:3], strat, prec, amp, same, tf, ts, 100 * (ts - tf) / ts, lev.n_dofs / (tf * 1e-3)), flush=True)


if __name__ == "__main__":
    main()
