"""Exact version of tools/pencil_map.py: a MILP (scipy.optimize.milp) finds a
thread -> pencil assignment of the Q4 fp64 sweeps whose half-warps are free of
shared-memory bank conflicts for every access class, or proves none exists,
for a layout (SY, SZ, SIZE); with --search it scans small paddings and also
checks the per-point accesses (thread = point, lanes in point order)."""
import sys

import numpy as np
from scipy.optimize import Bounds, LinearConstraint, milp

sys.path.insert(0, __import__("os").path.dirname(__file__))
from pencil_map import GROUPS, KS, N, base, decode  # noqa: E402


def solve(o, SY, SZ, SIZE, ks=None):
    ks = ks or KS[o]
    P, G = 3 * N * N, len(GROUPS)
    nv = P * G
    A, lo, hi = [], [], []
    for p in range(P):  # each pencil in exactly one group
        row = np.zeros(nv)
        row[p * G:(p + 1) * G] = 1
        A.append(row); lo.append(1); hi.append(1)
    for g, (g0, g1) in enumerate(GROUPS):  # group sizes
        row = np.zeros(nv)
        row[g::G] = 1
        A.append(row); lo.append(g1 - g0); hi.append(g1 - g0)
    for k, _ in ks:
        res = []
        for p in range(P):
            c, u, v = decode(o, p)
            res.append((k * c * SIZE + base(o, SY, SZ, u, v)) % 16)
        for g in range(G):
            for r in range(16):
                row = np.zeros(nv)
                for p in range(P):
                    if res[p] == r:
                        row[p * G + g] = 1
                if row.sum() > 1:
                    A.append(row); lo.append(0); hi.append(1)
    r = milp(c=np.zeros(nv), constraints=LinearConstraint(np.array(A), lo, hi), integrality=np.ones(nv),
             bounds=Bounds(0, 1), options={"time_limit": 20})
    if r.x is None or r.status != 0:
        return None
    x = r.x.reshape(P, G).round().astype(int)
    lanes = []
    for g, (g0, g1) in enumerate(GROUPS):
        lanes += [p for p in range(P) if x[p, g]]
    return lanes


def point_ok(SY, SZ, SIZE):
    for h0 in range(0, 128, 16):
        seen = {}
        for q in range(h0, min(h0 + 16, N ** 3)):
            w = q % N + SY * ((q // N) % N) + SZ * (q // (N * N))
            if w % 16 in seen:
                return False
            seen[w % 16] = 1
    return True


if __name__ == "__main__":
    if "--search" in sys.argv:
        for SY in range(5, 8):
            for SZ in range(4 * SY + 5, 4 * SY + 5 + 8):
                if not point_ok(SY, SZ, 0):
                    continue
                for SIZE in range(4 + 4 * SY + 4 * SZ + 1, 4 + 4 * SY + 4 * SZ + 1 + 16):
                    ok = all(solve(o, SY, SZ, SIZE) is not None for o in 'xyz')
                    print(SY, SZ, SIZE, ok, flush=True)
                    if ok:
                        sys.exit(0)
    else:
        SY, SZ, SIZE = (int(x) for x in sys.argv[1:4])
        for o in 'xyz':
            print(o, solve(o, SY, SZ, SIZE))


def solve_min(o, SY, SZ, SIZE, k=1):
    """Minimum-wavefront assignment (one access class k): minimise the sum over
    half-warps of the largest bank-pair multiplicity."""
    P, G = 3 * N * N, len(GROUPS)
    nv = P * G + G  # x[p,g] and m[g]
    A, lo, hi = [], [], []
    for p in range(P):
        row = np.zeros(nv)
        row[p * G:(p + 1) * G] = 1
        A.append(row); lo.append(1); hi.append(1)
    for g, (g0, g1) in enumerate(GROUPS):
        row = np.zeros(nv)
        row[g:P * G:G] = 1
        A.append(row); lo.append(g1 - g0); hi.append(g1 - g0)
    res = []
    for p in range(P):
        c, u, v = decode(o, p)
        res.append((k * c * SIZE + base(o, SY, SZ, u, v)) % 16)
    for g in range(G):
        for r in range(16):
            row = np.zeros(nv)
            for p in range(P):
                if res[p] == r:
                    row[p * G + g] = 1
            row[P * G + g] = -1
            A.append(row); lo.append(-np.inf); hi.append(0)
    cost = np.zeros(nv)
    cost[P * G:] = 1
    integ = np.ones(nv)
    r = milp(c=cost, constraints=LinearConstraint(np.array(A), lo, hi), integrality=integ,
             bounds=Bounds(0, [1] * (P * G) + [16] * G), options={"time_limit": 60})
    x = r.x[:P * G].reshape(P, G).round().astype(int)
    lanes = []
    for g in range(G):
        lanes += [p for p in range(P) if x[p, g]]
    return int(round(r.fun)), lanes


def solve_groups(res, groups, banks, time_limit=60):
    """Assign pencils (residue list `res`, index = pencil id) to lane groups
    (list of sizes) minimising the sum over groups of the largest residue
    multiplicity; returns (cost, [pencil ids in lane order])."""
    P, G = len(res), len(groups)
    assert sum(groups) == P
    nv = P * G + G
    A, lo, hi = [], [], []
    for p in range(P):
        row = np.zeros(nv)
        row[p * G:(p + 1) * G] = 1
        A.append(row); lo.append(1); hi.append(1)
    for g, sz in enumerate(groups):
        row = np.zeros(nv)
        row[g:P * G:G] = 1
        A.append(row); lo.append(sz); hi.append(sz)
    for g in range(G):
        for r in range(banks):
            row = np.zeros(nv)
            for p in range(P):
                if res[p] == r:
                    row[p * G + g] = 1
            if not row.any():
                continue
            row[P * G + g] = -1
            A.append(row); lo.append(-np.inf); hi.append(0)
    cost = np.zeros(nv)
    cost[P * G:] = 1
    r = milp(c=cost, constraints=LinearConstraint(np.array(A), lo, hi), integrality=np.ones(nv),
             bounds=Bounds(0, [1] * (P * G) + [32] * G), options={"time_limit": time_limit})
    x = r.x[:P * G].reshape(P, G).round().astype(int)
    lanes = []
    for g in range(G):
        lanes += [p for p in range(P) if x[p, g]]
    return int(round(r.fun)), lanes


def f32_q4_maps(SY=5, SZ=25, SIZE=125):
    """fp32 Q4 (4-byte words, 32 banks): the fused x/u_k forward sweeps
    (fwc_*: 150 pencils, two rounds over 125 threads: lane groups 32, 32, 32,
    29 then 25) and the transposed sweeps (75 pencils: 32, 32, 11), arrays
    direction-major (every access c + const)."""
    lat = lambda a, b, c: a + SY * b + SZ * c
    out = {}
    # fused: pencil wk: vc = wk / 25, r = wk % 25; x: j = r % 5, k = r / 5; y: i = r % 5, k = r / 5; z: i, j
    for o in 'xyz':
        res = []
        for wk in range(150):
            vc, r = wk // 25, wk % 25
            u, v = r % 5, r // 5
            base = {'x': lat(0, u, v), 'y': lat(u, 0, v), 'z': lat(u, v, 0)}[o]
            res.append((vc * SIZE + base) % 32)
        out['fwc_' + o] = solve_groups(res, [32, 32, 32, 29, 25], 32)
    # transposed: z / y: c = wk / 25, (i, j) / (i, k); x (fp32 order): c = wk / 25, j = r % 5, k = r / 5
    for o in 'xyz':
        res = []
        for wk in range(75):
            c, r = wk // 25, wk % 25
            u, v = r % 5, r // 5
            base = {'x': lat(0, u, v), 'y': lat(u, 0, v), 'z': lat(u, v, 0)}[o]
            res.append((c * SIZE + base) % 32)
        out['tr_' + o] = solve_groups(res, [32, 32, 11], 32)
    return out



# A sub-pencil variant of the fp64 Q4 y / z sweeps (225 single-line items over
# two thread rounds, warp-uniform tables, MILP-mapped like the maps above) was
# built and measured in round 2: 2.21 -> 3.53 ms per element phase with the
# items processed one after the other (short-scoreboard stalls on the 5-value
# line loads) and 600-800 B of spills when both items' loads were issued
# first, so it was dropped.


def f64_q4_fused_maps(SY=5, SZ=25, SIZE=125):
    """fp64 Q4 with the x / u_k forward sweeps fused (fwc_*: 150 pencils,
    vc = wk / 25 over the 6 staged arrays; round 1 over threads 0-124, round 2
    over threads 0-24): half-warp groups, 8-byte words (16 bank pairs)."""
    lat = lambda a, b, c: a + SY * b + SZ * c
    groups = [16] * 7 + [13] + [16, 9]
    out = {}
    for o in 'xyz':
        res = []
        for wk in range(150):
            vc, r = wk // 25, wk % 25
            u, v = r % 5, r // 5
            base = {'x': lat(0, u, v), 'y': lat(u, 0, v), 'z': lat(u, v, 0)}[o]
            res.append((vc * SIZE + base) % 16)
        out['fwc_' + o] = solve_groups(res, groups, 16)
    return out
