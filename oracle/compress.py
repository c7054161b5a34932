"""f3 multi-level graph compression -- TEST INFRASTRUCTURE ONLY (the CPU oracle).

Only tests/ may import this module; it never imports the CUDA package and the
CUDA package never imports it.  Plain Python over the raw arc list, following
PAPER.md §"Multi-level Graph Compression" step by step, with the
readings DESIGN.md lists as R33-R36 where the text is garbled or silent:

  level i: nodes of G_{i-1} that are SIMILAR are combined pairwise into weighted
  nodes ("at each level i, similar nodes are combined to form a weighted
  node"; "u in V_i is a combination of p, q in V_{i-1}"); M(u) is the
  mapping list (the original vertices combined into u).

  R33 similarity (garbled: max(|adj(u)|/|common|, |adj(v)|/|common|) >= delta
      always holds for 0 < delta <= 1): u, v are similar iff they carry the same
      vertex label and |common(u, v)| >= delta * max(|A(u)|, |A(v)|), where A(u) is
      the set of labelled edge ends (direction, edge label, neighbour node) of u in
      G_{i-1} and common(u, v) = A(u) & A(v) ("common edge e(l_u, v)").
  R34 pairing: nodes in increasing id order; an unpaired p combines with the
      smallest-id unpaired similar q > p.  Level-i ids follow the smallest member.
  R35 weights: w_out(u) = max over x in M(u) of the number of arcs
      x -> M(u) ("the maximum degree among nodes in the graph constructed by
      M(p) u M(q)"), w_in likewise; edge weights start at the number of arcs x -> y
      ("the initial weight of all edges in the original graph is 1", one per
      labelled arc) and follow P:850's recursion generalised to singletons:
      w_i(U, V) = sum over parts V' of V of max over parts U' of U of w_{i-1}(U', V').
  R36 candidate test (P:905 definition): X is a candidate of query vertex u iff
      the labels agree (or u is *), the bound id (if any) is in M(X), and
      qout(u) <= w_out(X) + sum_{Z != X} w_out(X, Z), qin(u) likewise with in-weights
      (qout / qin = distinct query out-/in-neighbours, R12).
"""
from __future__ import annotations

from collections import defaultdict

import numpy as np


def _arcs(g):
    """Set of (src, dst, label) arcs from the raw edge list (undirected: both directions)."""
    el = np.zeros(len(g.src), np.int64) if g.elab is None else np.asarray(g.elab, np.int64)
    arcs = set()
    for s, d, l in zip(np.asarray(g.src, np.int64).tolist(), np.asarray(g.dst, np.int64).tolist(), el.tolist()):
        arcs.add((s, d, l))
        if g.undirected:
            arcs.add((d, s, l))
    return arcs


class Level:
    """One compression level: group[x] = node of original vertex x; members[U] = M(U)."""

    def __init__(self, group, members, label, w_out, w_in, e_out, e_in):
        self.group = group          # list, len n
        self.members = members      # list of sorted lists
        self.label = label          # list, label of each node
        self.w_out = w_out          # list, node weights
        self.w_in = w_in
        self.e_out = e_out          # dict (U, V) -> weight, U != V or U == V
        self.e_in = e_in

    @property
    def n_nodes(self) -> int:
        return len(self.members)


def _node_weights(arcs, group, nn):
    cnt_out = defaultdict(int)
    cnt_in = defaultdict(int)
    for (s, d, _) in arcs:
        if group[s] == group[d]:
            cnt_out[s] += 1
            cnt_in[d] += 1
    w_out = [0] * nn
    w_in = [0] * nn
    for x, c in cnt_out.items():
        w_out[group[x]] = max(w_out[group[x]], c)
    for x, c in cnt_in.items():
        w_in[group[x]] = max(w_in[group[x]], c)
    return w_out, w_in


def compress(g, deltas):
    """Levels G_1..G_L of the compression with thresholds deltas[0..L) (each in (0, 1]).
    Returns the list of Level objects (level 0 = the original graph is not included)."""
    n = int(g.n)
    arcs = _arcs(g)
    vl = [0] * n if g.vlab is None else [int(x) for x in g.vlab]
    # level 0
    group = list(range(n))
    label = list(vl)
    e_out = defaultdict(int)
    e_in = defaultdict(int)
    for (s, d, _) in arcs:
        e_out[(s, d)] += 1      # base weight: one per labelled arc x -> y
        e_in[(d, s)] += 1       # in-weight of d towards s
    levels = []
    nn = n
    for delta in deltas:
        if not (0.0 < delta <= 1.0):
            raise ValueError("delta must be in (0, 1]")
        # A(U): labelled edge ends of the current nodes
        A = [set() for _ in range(nn)]
        for (s, d, l) in arcs:
            A[group[s]].add(("o", l, group[d]))
            A[group[d]].add(("i", l, group[s]))
        partner = [-1] * nn
        for p in range(nn):
            if partner[p] >= 0:
                continue
            for q in range(p + 1, nn):
                if partner[q] >= 0 or label[q] != label[p]:
                    continue
                common = len(A[p] & A[q])
                if common >= delta * max(len(A[p]), len(A[q])):
                    partner[p], partner[q] = q, p
                    break
        # new ids in increasing order of the first part
        new_id = [-1] * nn
        parts = []
        for p in range(nn):
            if partner[p] >= 0 and partner[p] < p:
                continue
            new_id[p] = len(parts)
            parts.append([p] if partner[p] < 0 else [p, partner[p]])
        for p in range(nn):
            if new_id[p] < 0:
                new_id[p] = new_id[partner[p]]
        nn2 = len(parts)
        # edge-weight recursion (R35) over the previous level's weighted edges
        def recur(e_prev):
            best = {}   # (U, V, V') -> max over U' of w(U', V')
            for (u1, v1), w in e_prev.items():
                key = (new_id[u1], new_id[v1], v1)
                if w > best.get(key, 0):
                    best[key] = w
            out = defaultdict(int)
            for (U, V, _), w in best.items():
                out[(U, V)] += w
            return out
        e_out = recur(e_out)
        e_in = recur(e_in)
        group = [new_id[group[x]] for x in range(n)]
        label = [label[pt[0]] for pt in parts]
        members = [[] for _ in range(nn2)]
        for x in range(n):
            members[group[x]].append(x)
        w_out, w_in = _node_weights(arcs, group, nn2)
        levels.append(Level(list(group), members, label, w_out, w_in, dict(e_out), dict(e_in)))
        nn = nn2
    return levels


def _qdeg(q):
    outs = [set() for _ in range(q.k)]
    ins = [set() for _ in range(q.k)]
    for (a, b, _) in q.edges:
        outs[a].add(b)
        ins[b].add(a)
    return [len(s) for s in outs], [len(s) for s in ins]


def weighted_candidates(level: Level, q):
    """Per query vertex, the sorted weighted nodes passing R36's test."""
    qo, qi = _qdeg(q)
    tot_out = list(level.w_out)
    tot_in = list(level.w_in)
    for (U, V), w in level.e_out.items():
        if U != V:
            tot_out[U] += w
    for (U, V), w in level.e_in.items():
        if U != V:
            tot_in[U] += w
    res = []
    for u in range(q.k):
        c = []
        for X in range(level.n_nodes):
            if q.vlabels[u] != -1 and q.vlabels[u] != level.label[X]:
                continue
            if q.bound[u] != -1 and q.bound[u] not in level.members[X]:
                continue
            if qo[u] <= tot_out[X] and qi[u] <= tot_in[X]:
                c.append(X)
        res.append(c)
    return res


def expanded_candidates(level: Level, q):
    """Per query vertex, the sorted original vertices of its weighted candidates' mapping lists."""
    return [sorted(x for X in cs for x in level.members[X]) for cs in weighted_candidates(level, q)]
