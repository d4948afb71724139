"""Shared-memory wavefront model of the Q4 (n = 5) fp64 element kernel's
accesses (apply_v2.cuh, one element per CTA, 125 threads) for a given padded
layout (SY, SZ, SIZE) and pencil orders; used to pick the Q4 layout.
Model: an 8-byte warp access is served per half-warp; a half-warp takes as
many wavefronts as the largest number of distinct 8-byte words that share a
bank pair (word mod 16)."""
import itertools
import sys

N = 5


def wavefronts(words, active):
    """words: list of 32 word offsets (None for inactive lanes)."""
    total = 0
    for h in (0, 1):
        lanes = [w for l, w in enumerate(words[16 * h:16 * h + 16]) if w is not None]
        if not lanes:
            continue
        banks = {}
        for w in set(lanes):
            banks.setdefault(w % 16, set()).add(w)
        total += max(len(s) for s in banks.values())
    return total


def run_sites(sites, nthreads):
    """sites: list of functions lane_index -> word offset (or None); returns wavefronts per element."""
    tot = 0
    for f in sites:
        for w0 in range(0, nthreads, 32):
            words = [f(t) if t < nthreads else None for t in range(w0, w0 + 32)]
            tot += wavefronts(words, None)
    return tot


def model(SY, SZ, SIZE, orders, verbose=False):
    lat = lambda a, b, c: a + SY * b + SZ * c
    res = {}
    P = 3 * N * N  # pencils

    def pen(order, wk):
        # order: permutation of ('c', 'u', 'v') major..minor  (u, v: the two in-plane line indices)
        dims = {'c': 3, 'u': N, 'v': N}
        idx = {}
        r = wk
        for d in reversed(order):
            idx[d] = r % dims[d]
            r //= dims[d]
        return idx['c'], idx['u'], idx['v']

    def sweep(name, order, loads, stores):
        sites = []
        for arr, posf in loads + stores:
            for t in range(N):
                def f(wk, arr=arr, posf=posf, t=t):
                    if wk >= P:
                        return None
                    c, u, v = pen(order, wk)
                    return arr(c) * SIZE + posf(u, v, t)
                sites.append(f)
        res[name] = run_sites(sites, 128)

    X = lambda u, v, t: lat(t, u, v)   # x-pencil: line (j=u, k=v), running a
    Y = lambda u, v, t: lat(u, t, v)   # y-pencil: (i=u, k=v)
    Z = lambda u, v, t: lat(u, v, t)   # z-pencil: (i=u, j=v)
    o = orders
    # forward (per vector): fw_x 3 in-arrays c, out tb (c), td (3+c)
    sweep('fw_x', o['x'], [(lambda c: c, X)], [(lambda c: c, X), (lambda c: 3 + c, X)])
    sweep('fw_y', o['y'], [(lambda c: c, Y), (lambda c: 3 + c, Y)],
          [(lambda c: c, Y), (lambda c: 3 + c, Y), (lambda c: 6 + c, Y)])
    sweep('fw_z', o['z'], [(lambda c: c, Z), (lambda c: 3 + c, Z), (lambda c: 6 + c, Z)],
          [(lambda c: 3 * c, Z), (lambda c: 3 * c + 1, Z), (lambda c: 3 * c + 2, Z)])
    sweep('tr_z', o['z'], [(lambda c: 3 * c + t, Z) for t in range(3)], [(lambda c: 3 * c + t, Z) for t in range(3)])
    sweep('tr_y', o['y'], [(lambda c: 3 * c + t, Y) for t in range(3)], [(lambda c: c, Y), (lambda c: 3 + c, Y)])
    sweep('tr_x', o['x'], [(lambda c: c, X), (lambda c: 3 + c, X)], [])
    # per point: thread q -> (i, j, k), 9 reads (x grad) + 9 reads (u_k grad) + 9 writes + 6 staged writes
    pt = lambda m: (lambda q: m * SIZE + lat(q % N, (q // N) % N, q // (N * N)) if q < N ** 3 else None)
    res['point'] = run_sites([pt(m) for m in range(9)], 128) * 3 + run_sites([pt(m) for m in range(6)], 128)
    total = 2 * (res['fw_x'] + res['fw_y'] + res['fw_z']) + res['tr_z'] + res['tr_y'] + res['tr_x'] + res['point']
    res['total'] = total
    return res


def ideal():
    return model(5, 25, 125, {'x': ('v', 'c', 'u'), 'y': 'cvu', 'z': 'cvu'})


if __name__ == "__main__":
    cur = {'x': ('v', 'c', 'u'), 'y': ('c', 'v', 'u'), 'z': ('c', 'v', 'u')}
    print("current", model(5, 25, 125, cur))
    best = []
    orders = list(itertools.permutations('cuv'))
    for SY in range(5, 9):
        for SZ in range(4 * SY + 5, 4 * SY + 5 + 12):
            for SIZE in range(4 + 4 * SY + 4 * SZ + 1, 4 + 4 * SY + 4 * SZ + 1 + 12):
                r = {}
                tot = 0
                for sw in ('x', 'y', 'z'):
                    bestsw = None
                    for od in orders:
                        oo = dict(cur)
                        oo[sw] = od
                        m = model(SY, SZ, SIZE, oo)
                        key = {'x': m['fw_x'] * 2 + m['tr_x'], 'y': m['fw_y'] * 2 + m['tr_y'],
                               'z': m['fw_z'] * 2 + m['tr_z']}[sw]
                        if bestsw is None or key < bestsw[0]:
                            bestsw = (key, od)
                    r[sw] = bestsw[1]
                m = model(SY, SZ, SIZE, r)
                best.append((m['total'], SY, SZ, SIZE, r, m))
    best.sort(key=lambda x: x[0])
    for b in best[:10]:
        print(b[0], b[1:4], b[4], {k: v for k, v in b[5].items() if k != 'total'})
