"""Dev prototype (not product, not oracle): the GPU algorithm for one bisection,
written sequentially in numpy so its *structure* — rounds to a fixpoint,
clamp-monoid sizes scan with speculated ties, tie verification, sequential
walk repair — can be validated against the C oracle and instrumented
(rounds per chunk, walk lengths) before the CUDA version exists.
"""
import sys
from math import ceil

import numpy as np

sys.path.insert(0, ".")
from oracle import oracle  # noqa: E402

INF = 1 << 40
JACOBI = int(__import__('os').environ.get('JACOBI', '0'))


def seed_reference(nodes, adj_lists, cap, passes=2):
    # sequential seed (seed.py) for the prototype only
    n = len(nodes)
    target = (n + 1) // 2
    deg = np.array([len(a) for a in adj_lists])
    order = np.lexsort((np.arange(n), -deg))
    picked = np.zeros(n, bool)
    from collections import deque
    q = deque(); count = 0; rp = 0
    while count < target:
        if not q:
            while picked[order[rp]]:
                rp += 1
            b = order[rp]; q.append(b); picked[b] = True; count += 1
            if count >= target:
                break
        v = q.popleft()
        for w in adj_lists[v]:
            if not picked[w]:
                picked[w] = True; count += 1; q.append(w)
                if count >= target:
                    break
    lab = np.where(picked, 0, 1).astype(np.int8)
    sizes = [target, n - target]
    for _ in range(passes):
        moved = False
        for i in range(n):
            side = lab[i]
            same = sum(1 for w in adj_lists[i] if lab[w] == side)
            other = len(adj_lists[i]) - same
            if other == 0:
                continue
            if other > same and sizes[1 - side] < cap:
                lab[i] = 1 - side; sizes[side] -= 1; sizes[1 - side] += 1; moved = True
        if not moved:
            break
    return lab


def chunk_struct(e):
    nodes, inv = np.unique(e.reshape(-1), return_inverse=True)
    loc = inv.reshape(-1, 2)
    mask = loc[:, 0] != loc[:, 1]
    return nodes, loc[mask]


def counts_round(loc, T, old, nn):
    # lower local index sees T (tentative), higher sees old
    u, v = loc[:, 0], loc[:, 1]
    lo = np.minimum(u, v); hi = np.maximum(u, v)
    # lo's count from hi: old[hi]; hi's count from lo: T[lo]
    c0 = np.bincount(lo[old[hi] == 0], minlength=nn) + np.bincount(hi[T[lo] == 0], minlength=nn)
    c1 = np.bincount(lo[old[hi] == 1], minlength=nn) + np.bincount(hi[T[lo] == 1], minlength=nn)
    return c0.astype(np.float64), c1.astype(np.float64)


def process_chunk_rounds(parts, nbr0, nbr1, sizes, cap, e, refine, stats, spec_mode="prev"):
    nodes, loc = chunk_struct(e)
    nn = len(nodes)
    old = parts[nodes].astype(np.int64)
    active = (old == -1) | bool(refine)
    isnew = old == -1
    o = ((old == 0) & active).astype(np.int64)
    lift = ((old != -1) & active).astype(np.int64)
    s0 = sizes[0] + sizes[1]
    x0 = sizes[0]
    s_before = s0 + np.concatenate([[0], np.cumsum(active & isnew)[:-1]])
    s_l = s_before - lift
    T = old.copy()
    xprev = None
    rounds = 0
    while True:
        rounds += 1
        c0, c1 = counts_round(loc, T, old, nn)
        a0 = np.where(isnew, c0, (nbr0[nodes] + c0) * 0.5)
        a1 = np.where(isnew, c1, (nbr1[nodes] + c1) * 0.5)
        pref = np.where(a0 < a1, 1, np.where(a1 < a0, 0, 2))
        pref = np.where(active, pref, 3)
        thr = np.where(pref == 0, cap - 1, np.where(pref == 1, s_l - cap, s_l // 2))
        # speculation for ties
        if xprev is None:
            if __import__('os').environ.get('HALF', '1') == '1':
                # half-step predictor: ties count +1/2 (clamp scan in doubled coords)
                X = np.empty(nn, np.int64); cur = 2 * x0
                for i in range(nn):
                    X[i] = cur; p = pref[i]
                    if p == 3: continue
                    if p == 0: cur = min(cur + 2 - 2 * o[i], 2 * cap)
                    elif p == 1: cur = max(cur - 2 * o[i], 2 * (s_l[i] - cap + 1))
                    else: cur = cur + 1 - 2 * o[i]
                spec = np.where(X - 2 * o <= 2 * (s_l // 2), 0, 1)
            else:
                spec = np.where(x0 - o <= s_l // 2, 0, 1)
        else:
            spec = np.where(xprev - o <= s_l // 2, 0, 1)
        for jac in range(JACOBI + 1):
            # clamp scan (sequential eval here; associative on the GPU)
            x = np.empty(nn + 1, dtype=np.int64)
            cur = x0
            for i in range(nn):
                x[i] = cur
                p = pref[i]
                if p == 3:
                    continue
                if p == 0:
                    cur = min(cur - o[i] + 1, cap)
                elif p == 1:
                    cur = max(cur - o[i], s_l[i] - cap + 1)
                else:
                    cur = cur - o[i] + (1 if spec[i] == 0 else 0)
            x[nn] = cur
            # verify ties
            bad = np.flatnonzero((pref == 2) & (((x[:nn] - o) <= thr).astype(int) != (1 - spec)))
            if not bad.size or jac == JACOBI:
                break
            stats["jacobi"] += 1
            # segment relaxation: exact local simulation from the scanned x at
            # each segment start -> locally consistent tie guesses
            SEG = int(__import__('os').environ.get('SEG', '256'))
            spec = spec.copy()
            for st in range(0, nn, SEG):
                xe = x[st]
                for i in range(st, min(st + SEG, nn)):
                    p = pref[i]
                    if p == 3:
                        continue
                    b0 = (xe - o[i]) <= thr[i]
                    if p == 2:
                        spec[i] = 0 if b0 else 1
                    xe = xe - o[i] + (1 if b0 else 0)
        walk = 0
        if bad.size and __import__('os').environ.get('BUNDLE') == '1':
            import tools.proto_bundle as pb
            # candidate centers: this round's speculative scan, and the previous
            # round's exact x (round 1: the half-step predictor)
            if xprev is not None:
                c2 = xprev
            else:
                Xh = np.empty(nn, np.int64); cur = 2 * x0
                for i in range(nn):
                    Xh[i] = cur; p = pref[i]
                    if p == 3: continue
                    if p == 0: cur = min(cur + 2 - 2 * o[i], 2 * cap)
                    elif p == 1: cur = max(cur - 2 * o[i], 2 * (s_l[i] - cap + 1))
                    else: cur = min(max(cur + 1 - 2 * o[i], 2 * (s_l[i] + 1 - cap)), 2 * cap)
                c2 = Xh // 2
            L = max(64, -(-nn // 4096))
            x = pb.bundle_exact(x0, pref, o, thr, s_l, cap, x[:nn], c2, L)
            bad = bad[:0]
        if bad.size:
            cursor = -1
            for k in bad:
                if k < cursor:
                    continue
                xe = x[k]
                i = k
                while True:
                    p = pref[i]
                    x[i] = xe
                    if p != 3:
                        b0 = (xe - o[i]) <= thr[i]
                        xe = xe - o[i] + (1 if b0 else 0)
                    i += 1
                    walk += 1
                    if i == nn or xe == x[i]:
                        break
                if i == nn:
                    x[nn] = xe
                cursor = i
        stats["walk"] += walk
        stats["flagged"] += int(bad.size)
        b = np.where(((x[:nn] - o) <= thr), 0, 1)
        Tn = np.where(active, b, old)
        xprev = x[:nn].copy()
        if np.array_equal(Tn, T):
            break
        T = Tn
    stats["rounds"] += rounds
    stats["max_rounds"] = max(stats["max_rounds"], rounds)
    stats["visits"] += nn
    parts[nodes[active]] = T[active]
    nbr0[nodes[active]] = a0[active]
    nbr1[nodes[active]] = a1[active]
    sizes[0] = int(x[nn])
    sizes[1] = int(s0 + int((active & isnew).sum()) - x[nn])


def bisect_proto(edges, n, chunk, cap, refine=True, passes=1, stats=None):
    parts = np.full(n, -1, dtype=np.int64)
    nbr0 = np.zeros(n); nbr1 = np.zeros(n)
    sizes = [0, 0]
    m = len(edges)
    nch = ceil(m / chunk) if m else 0
    for ps in range(passes):
        for ci in range(nch):
            e = edges[ci * chunk:(ci + 1) * chunk]
            if ps == 0 and ci == 0:
                nodes, loc = chunk_struct(e)
                adj = [[] for _ in range(len(nodes))]
                for a, b in loc.tolist():
                    adj[a].append(b); adj[b].append(a)
                adj = [sorted(x) for x in adj]
                lab = seed_reference(nodes, adj, cap)
                parts[nodes] = lab
                sizes = [int((parts == 0).sum()), int((parts == 1).sum())]
                for i, g in enumerate(nodes):
                    nbr0[g] = sum(1 for w in adj[i] if lab[w] == 0)
                    nbr1[g] = sum(1 for w in adj[i] if lab[w] == 1)
            else:
                process_chunk_rounds(parts, nbr0, nbr1, sizes, cap, e, refine, stats)
    # fill (closed form)
    un = np.flatnonzero(parts == -1)
    d = sizes[1] - sizes[0]
    j = np.arange(un.size)
    lab = np.where(j < abs(d), 0 if d > 0 else 1, (j - abs(d)) % 2)
    parts[un] = lab
    return parts


if __name__ == "__main__":
    import time
    sys.path.insert(0, "paper_2502_17846_b200")
    from paper_2502_17846_b200 import synth
    n, m, beta = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 11
    frac = float(sys.argv[4]) if len(sys.argv) > 4 else 0.1
    slack = float(sys.argv[5]) if len(sys.argv) > 5 else 0.0
    edges = synth.powerlaw_edges(n, m, beta=beta, seed=0)
    chunk = max(1, ceil(frac * m))
    cap = ceil((1.0 + slack) * n / 2)
    stats = dict(rounds=0, max_rounds=0, visits=0, walk=0, flagged=0, jacobi=0)
    t = time.time()
    mine = bisect_proto(edges, n, chunk, cap, stats=stats)
    t1 = time.time()
    ref = oracle.bisect(edges, n, chunk, cap)
    print("equal", np.array_equal(mine, ref), stats, "proto %.1fs" % (t1 - t))
