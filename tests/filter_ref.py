"""Reference of the filtering phase's SET semantics (test infrastructure only).

An independent, slow, plain-Python restatement of what the candidate sets are
after each stage, used to pin the CUDA filter kernels exactly (not only their
soundness).  It shares no code with the CUDA path or the oracle.

  stage 0  kernel_check (Def. 3; reading R12): label (or wildcard),
           bound id (concept node), #distinct out-(in-)neighbours of u in
           the query <= #distinct (target, label) out-(in-)arcs of v.
  stage 1  initialisation (Alg. 2): for u in the visit order O,
           prune C(u) to the vertices with, for every T-edge at u, a fitting arc
           to the current C(v) (lines 14-18), then shrink every T-neighbour's C(v)
           to the fitting neighbours of the surviving C(u) (lines 19-22, reading R15).
  stage 2  refinement (reading R17): rounds over the reversed
           discovery order of the vertices kept by the low-connectivity rule,
           pruning against every kept neighbour.

The plan (O, the spanning tree T, the discovery order) is re-derived here from
P:677-688 with the tie-breaks of readings R13/R14: ranking f(u) = deg(u)/freq(u)
as exact fractions, seed edge with maximal f(a)+f(b) (first in (a, b) order),
started from its endpoint with the larger f (ties: a); then repeatedly the
T-vertex with unvisited neighbours and maximal f (ties: lowest id); T grows by
u's edges to vertices not yet in T, in increasing id.
"""
from fractions import Fraction

import numpy as np


def _arcs(g):
    src = g.src.astype(np.int64)
    dst = g.dst.astype(np.int64)
    lab = g.elab.astype(np.int64) if g.elab is not None else np.zeros_like(src)
    if g.undirected:
        src, dst, lab = np.concatenate([src, dst]), np.concatenate([dst, src]), np.concatenate([lab, lab])
    out = [set() for _ in range(g.n)]
    inn = [set() for _ in range(g.n)]
    for a, b, l in zip(src.tolist(), dst.tolist(), lab.tolist()):
        out[a].add((b, l))
        inn[b].add((a, l))
    return out, inn


def plan(g, q):
    """(O, parent, discovery) of P:677-688 with readings R13/R14."""
    k = q.k
    adj = [set() for _ in range(k)]
    for a, b, _ in q.edges:
        adj[a].add(b)
        adj[b].add(a)
    vlab = g.vlab.astype(np.int64) if g.vlab is not None else np.zeros(g.n, np.int64)
    hist = np.bincount(vlab, minlength=1)

    def freq(u):
        if q.bound[u] >= 0:
            return 1
        if q.vlabels[u] < 0:
            return g.n
        return int(hist[q.vlabels[u]]) if q.vlabels[u] < hist.shape[0] else 0

    f = [Fraction(len(adj[u]), freq(u)) for u in range(k)]
    if k == 1:
        return [0], [-1], [0]
    best = None
    for a in range(k):
        for b in range(a + 1, k):
            if b in adj[a] and (best is None or f[a] + f[b] > f[best[0]] + f[best[1]]):
                best = (a, b)
    u = best[0] if f[best[0]] >= f[best[1]] else best[1]
    order, discovery, parent, inT = [u], [u], [-1] * k, {u}

    def grow(x):
        for v in range(k):
            if v in adj[x] and v not in inT:
                inT.add(v)
                parent[v] = x
                discovery.append(v)

    grow(u)
    while len(inT) < k:
        pick = None
        for x in range(k):
            if x in inT and adj[x] - inT and (pick is None or f[x] > f[pick]):
                pick = x
        order.append(pick)
        grow(pick)
    return order, parent, discovery


def candidates(g, q, stage, refine_rounds=1, reverse_refine=True, lowconn_threshold=1):
    """(k, n) bool array of the candidate sets after `stage` (0, 1 or 2)."""
    out, inn = _arcs(g)
    k, n = q.k, g.n
    vlab = g.vlab.astype(np.int64) if g.vlab is not None else np.zeros(n, np.int64)
    qout = [set() for _ in range(k)]
    qin = [set() for _ in range(k)]
    for a, b, _ in q.edges:
        qout[a].add(b)
        qin[b].add(a)
    if g.undirected:   # reading R12: undirected data compares distinct neighbours with the degree
        both = [qout[u] | qin[u] for u in range(k)]
        qout, qin = both, both
    C = []
    for u in range(k):
        s = set()
        for v in range(n):
            if q.vlabels[u] >= 0 and vlab[v] != q.vlabels[u]:
                continue
            if q.bound[u] >= 0 and v != q.bound[u]:
                continue
            if len(out[v]) >= len(qout[u]) and len(inn[v]) >= len(qin[u]):
                s.add(v)
        C.append(s)
    if stage >= 1:
        order, parent, discovery = plan(g, q)

        def constraints(u, nbrs):
            cs = []
            for a, b, lab in q.edges:
                if a == u and b in nbrs:
                    cs.append((b, 0, lab))
                elif b == u and a in nbrs:
                    cs.append((a, 1, lab))
            return cs

        def fitting(x, d, lab):   # neighbours of data vertex x through arcs of direction d with label lab
            return {y for (y, l) in (out[x] if d == 0 else inn[x]) if (lab < 0 or l == lab) and y != x}

        def prune(u, cs):
            C[u] = {x for x in C[u] if all(fitting(x, d, lab) & C[v] for v, d, lab in cs)}

        for u in order:
            tn = {v for v in range(k) if parent[v] == u or parent[u] == v}
            cs = constraints(u, tn)
            if not cs:
                continue
            prune(u, cs)
            new = {}
            for v, d, lab in cs:
                reach = set()
                for x in C[u]:
                    reach |= fitting(x, d, lab)
                new[v] = (new[v] if v in new else C[v]) & reach
            for v, s in new.items():
                C[v] = s
    if stage >= 2:
        adj = [set() for _ in range(k)]
        for a, b, _ in q.edges:
            adj[a].add(b)
            adj[b].add(a)
        kept = {u for u in range(k) if q.bound[u] >= 0 or len(adj[u]) > lowconn_threshold}
        for _ in range(refine_rounds):
            seq = list(reversed(discovery)) if reverse_refine else list(discovery)
            for u in seq:
                if u not in kept:
                    continue
                cs = constraints(u, kept & adj[u])
                if cs:
                    prune(u, cs)
    res = np.zeros((k, n), bool)
    for u in range(k):
        res[u, sorted(C[u])] = True
    return res
