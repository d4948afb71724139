"""Search for a conflict-free thread -> pencil assignment of the Q4 (n = 5)
fp64 sweeps (apply_v2.cuh, one element per 125-thread CTA): 75 pencils per
orientation are placed on the lanes of 3 warps so that, in every half-warp,
the pencils' shared-memory words fall on distinct bank pairs (8-byte word
mod 16) for every access of the sweep.  The layout is a + SY b + SZ c with
array stride SIZE; the array of an access is k*c + const (k = 1 or 3, c the
pencil's component).  Output: per orientation the pencil index (in the
sweep's own decoding) of each thread, for the kernel's constant table."""
import random
import sys

N = 5
GROUPS = [(0, 16), (16, 32), (32, 48), (48, 64), (64, 75)]  # lanes of the 75 active threads


def decode(o, wk):
    """Pencil (c, u, v) of worker wk in the sweep's own order (apply_v2.cuh)."""
    if o == 'x':  # fp64 fw_x / tr_x: j fastest, then c, then k
        return (wk // N) % 3, wk % N, wk // (3 * N)  # c, j, k
    c, r = wk // (N * N), wk % (N * N)
    return c, r % N, r // N  # y: (i, k), z: (i, j)


def base(o, SY, SZ, u, v):
    return {'x': SY * u + SZ * v, 'y': u + SZ * v, 'z': u + SY * v}[o]


def cost(assign, o, SY, SZ, SIZE, ks):
    tot = 0
    for g0, g1 in GROUPS:
        for k, w in ks:
            seen = {}
            for wk in assign[g0:g1]:
                c, u, v = decode(o, wk)
                r = (k * c * SIZE + base(o, SY, SZ, u, v)) % 16
                seen[r] = seen.get(r, 0) + 1
            tot += w * max(seen.values())
    return tot


def ideal(ks):
    return sum(w for _, w in ks) * len(GROUPS)


def anneal(o, SY, SZ, SIZE, ks, iters=40000, seed=0):
    rnd = random.Random(seed)
    a = list(range(3 * N * N))
    rnd.shuffle(a)
    cur = cost(a, o, SY, SZ, SIZE, ks)
    best = (cur, a[:])
    T = 2.0
    for it in range(iters):
        i, j = rnd.randrange(75), rnd.randrange(75)
        if i // 16 == j // 16:
            continue
        a[i], a[j] = a[j], a[i]
        c = cost(a, o, SY, SZ, SIZE, ks)
        if c <= cur or rnd.random() < pow(2.718, (cur - c) / T):
            cur = c
            if c < best[0]:
                best = (c, a[:])
                if c == ideal(ks):
                    break
        else:
            a[i], a[j] = a[j], a[i]
        T = max(0.05, T * 0.9997)
    return best


# access classes per orientation: (k, number of accesses of that class per pencil)
KS = {'x': [(1, 15 * 2 + 10)],                 # fw_x (x2 vectors): 5 ld + 10 st; tr_x 10 ld
      'y': [(1, 25 * 2 + 10), (3, 15)],        # fw_y 10 ld + 15 st; tr_y ld 3c+t (15), st c / 3+c (10)
      'z': [(1, 15 * 2), (3, 15 * 2 + 30)]}    # fw_z ld c.. (15), st 3c+t (15); tr_z 15 ld + 15 st (3c+t)

if __name__ == "__main__":
    SY, SZ, SIZE = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (5, 25, 125)
    for o in 'xyz':
        natural = cost(list(range(75)), o, SY, SZ, SIZE, KS[o])
        c, a = anneal(o, SY, SZ, SIZE, KS[o])
        print(o, "natural", natural, "best", c, "ideal", ideal(KS[o]))
        print("  ", a)
