"""Seeded query generators and the reconstructed worked example (no method arithmetic).

A Query has k vertices 0..k-1, per-vertex label (-1 = wildcard '*'), per-vertex
bound data id (-1 = free variable; a bound vertex is a "concept node"),
and directed labelled arcs (a, b, label) with label -1 = wildcard (a "variable
edge").  For undirected data graphs (DataGraph.undirected) an arc is an
unordered edge.
"""
from __future__ import annotations

import dataclasses
from typing import List, Tuple

import numpy as np

from .graphs import DataGraph

ANY = -1


@dataclasses.dataclass
class Query:
    k: int
    vlabels: List[int]
    bound: List[int]
    edges: List[Tuple[int, int, int]]

    def to_json(self) -> dict:
        return {"k": self.k, "vlabels": list(map(int, self.vlabels)),
                "bound": list(map(int, self.bound)),
                "edges": [list(map(int, e)) for e in self.edges]}

    @staticmethod
    def from_json(d: dict) -> "Query":
        return Query(int(d["k"]), list(d["vlabels"]), list(d["bound"]),
                     [tuple(e) for e in d["edges"]])


def triangle_tail(labels=None) -> Query:
    """Triangle (q0,q1,q2) plus tail q3 on q2 (BASELINE.json configs[0])."""
    lab = list(labels) if labels is not None else [ANY] * 4
    return Query(4, lab, [ANY] * 4, [(0, 1, ANY), (1, 2, ANY), (2, 0, ANY), (2, 3, ANY)])


def complete_query(k: int) -> Query:
    return Query(k, [ANY] * k, [ANY] * k, [(i, j, ANY) for i in range(k) for j in range(i + 1, k)])


def fixture_fig3_example():
    """Appendix A reconstruction of `fig3:example`.

    Labels A..E -> 0..4; u_i -> query id i-1, v_i -> data id i-1.
    Returns (DataGraph, Query).  Undirected, vertex-labelled.
    Text constraints it satisfies: unique embedding {(u1,v1),(u2,v2),(u3,v3),
    (u4,v6),(u5,v7),(u6,v8)}; u3 label B, degree 3, C(u3)={v3,v4}
    (P:624); adj(u3)={u2,u4,u5}; C(u1)={v1,v3,v4};
    visit order u5, u2.
    """
    A, B, C, D, E = range(5)
    q = Query(6, [B, A, B, C, D, E], [ANY] * 6,
              [(0, 1, ANY), (1, 2, ANY), (2, 3, ANY), (2, 4, ANY), (3, 4, ANY), (4, 5, ANY), (1, 4, ANY)])
    de = [(0, 1), (1, 2), (2, 5), (2, 6), (5, 6), (6, 7), (1, 6), (3, 4), (3, 5), (3, 7)]
    g = DataGraph(n=8, src=np.array([a for a, _ in de], np.uint32),
                  dst=np.array([b for _, b in de], np.uint32), elab=None,
                  vlab=np.array([B, A, B, B, A, C, D, E], np.uint16), undirected=True)
    return g, q


def random_connected_query(rng: np.random.Generator, k: int, extra: int, n_elabels: int,
                           n_vlabels: int, p_wild_v: float = 0.5, p_wild_e: float = 0.5,
                           bound_choices=None, p_bound: float = 0.0) -> Query:
    """Random connected query: random spanning tree + `extra` random arcs."""
    edges = []
    for i in range(1, k):
        p = int(rng.integers(0, i))
        a, b = (p, i) if rng.random() < 0.5 else (i, p)
        edges.append((a, b))
    for _ in range(extra):
        a, b = rng.choice(k, 2, replace=False)
        edges.append((int(a), int(b)))
    arcs = []
    for a, b in edges:
        lab = ANY if (n_elabels <= 1 or rng.random() < p_wild_e) else int(rng.integers(0, n_elabels))
        arcs.append((a, b, lab))
    vl = [ANY if (n_vlabels <= 1 or rng.random() < p_wild_v) else int(rng.integers(0, n_vlabels))
          for _ in range(k)]
    bound = [ANY] * k
    if bound_choices is not None:
        for u in range(k):
            if rng.random() < p_bound:
                bound[u] = int(rng.choice(bound_choices))
    return Query(k, vl, bound, arcs)


class _Skeleton:
    """Undirected view of a DataGraph's arcs, for BFS extraction only."""

    def __init__(self, g: DataGraph):
        s = g.src.astype(np.int64)
        d = g.dst.astype(np.int64)
        lab = g.elab.astype(np.int64) if g.elab is not None else np.zeros_like(s)
        # entry: neighbour, arc index, forward flag
        nb = np.concatenate([d, s])
        own = np.concatenate([s, d])
        aid = np.concatenate([np.arange(s.shape[0]), np.arange(s.shape[0])])
        fwd = np.concatenate([np.ones_like(s), np.zeros_like(s)])
        order = np.argsort(own, kind="stable")
        self.nb, self.aid, self.fwd = nb[order], aid[order], fwd[order]
        cnt = np.bincount(own, minlength=g.n)
        self.off = np.zeros(g.n + 1, np.int64)
        np.cumsum(cnt, out=self.off[1:])
        self.deg = cnt
        self.s, self.d, self.lab = s, d, lab


_SKEL_CACHE: dict = {}


def _skeleton(g: DataGraph) -> _Skeleton:
    key = id(g)
    sk = _SKEL_CACHE.get(key)
    if sk is None or sk[0] is not g:
        sk = (g, _Skeleton(g))
        _SKEL_CACHE.clear()
        _SKEL_CACHE[key] = sk
    return sk[1]


def bfs_query(g: DataGraph, k: int, seed: int, induced: bool = False,
              keep_vlabels: bool = True, keep_elabels: bool = True,
              p_wild_v: float = 0.0, bind_seed: bool = False,
              top_fraction: float = 0.1, max_children: int = 0, prefer_hubs: bool = False,
              max_extra: int = -1, max_vertex_degree: int = 0) -> Query:
    """BFS-extracted query ("picking a node ... following breadth-first
    search ... nodes in the dense area").

    Seed: uniform among the top `top_fraction` vertices by total degree.
    BFS over the undirected skeleton with a seeded shuffle of each neighbour
    list; the discovering arc (its direction and label) becomes a tree edge.
    induced=True adds every data arc among the chosen vertices (cyclic queries).
    Vertex labels kept from the data (each replaced by '*' with prob p_wild_v);
    edge labels kept unless keep_elabels=False.  max_children > 0 caps how many
    new vertices one BFS expansion may add (deeper, less star-like trees around
    hubs).  prefer_hubs expands the highest-degree neighbours first (dense core ->
    induced queries with cycles).  bind_seed binds query vertex 0
    to the seed (concept node).  The identity image is always an
    embedding, so the result set is never empty.
    """
    rng = np.random.default_rng(seed)
    sk = _skeleton(g)
    order = np.argsort(-sk.deg, kind="stable")
    if max_vertex_degree > 0:
        order = order[sk.deg[order] <= max_vertex_degree]
    top = order[: max(1, int(g.n * top_fraction))]
    for _attempt in range(64):
        root = int(rng.choice(top))
        chosen = [root]
        pos = {root: 0}
        tree = []
        head = 0
        while head < len(chosen) and len(chosen) < k:
            x = chosen[head]
            head += 1
            lo, hi = sk.off[x], sk.off[x + 1]
            idx = np.arange(lo, hi)
            rng.shuffle(idx)
            if prefer_hubs:
                idx = idx[np.argsort(-sk.deg[sk.nb[idx]], kind="stable")]
            added = 0
            for e in idx:
                if max_children and added >= max_children:
                    break
                y = int(sk.nb[e])
                if y == x or y in pos:
                    continue
                if max_vertex_degree > 0 and sk.deg[y] > max_vertex_degree:
                    continue
                pos[y] = len(chosen)
                chosen.append(y)
                a = int(sk.aid[e])
                tree.append(a)
                added += 1
                if len(chosen) == k:
                    break
        if len(chosen) == k:
            break
    else:
        raise RuntimeError("could not extract a connected query of size %d" % k)
    if induced:
        sel = np.zeros(g.n, bool)
        sel[chosen] = True
        arcs = np.nonzero(sel[sk.s] & sel[sk.d] & (sk.s != sk.d))[0].tolist()
        if max_extra >= 0:
            tset = set(int(a) for a in tree)
            tpairs = {(min(int(sk.s[a]), int(sk.d[a])), max(int(sk.s[a]), int(sk.d[a]))) for a in tree}
            extra = [a for a in arcs if a not in tset and
                     (min(int(sk.s[a]), int(sk.d[a])), max(int(sk.s[a]), int(sk.d[a]))) not in tpairs]
            extra = [extra[i] for i in rng.permutation(len(extra))]
            chosen_extra, epairs = [], set()
            for a in extra:
                pk = (min(int(sk.s[a]), int(sk.d[a])), max(int(sk.s[a]), int(sk.d[a])))
                if pk in epairs:
                    continue
                epairs.add(pk)
                chosen_extra.append(a)
                if len(chosen_extra) >= max_extra:
                    break
            arcs = [int(a) for a in tree] + chosen_extra
    else:
        arcs = tree
    edges = []
    seen = set()
    pairs = set()
    for a in arcs:
        qa, qb = pos[int(sk.s[a])], pos[int(sk.d[a])]
        lab = int(sk.lab[a]) if (keep_elabels and g.elab is not None) else ANY
        key = (qa, qb, lab)
        if key in seen:
            continue
        if induced:   # at most one arc per unordered vertex pair (the first found), <= 64 arcs
            pk = (min(qa, qb), max(qa, qb))
            if pk in pairs or len(edges) >= 64:
                continue
            pairs.add(pk)
        seen.add(key)
        edges.append(key)
    if g.vlab is not None and keep_vlabels:
        vl = [int(g.vlab[v]) for v in chosen]
    else:
        vl = [ANY] * k
    if p_wild_v > 0:
        vl = [ANY if rng.random() < p_wild_v else x for x in vl]
    bound = [ANY] * k
    if bind_seed:
        bound[0] = root
    return Query(k, vl, bound, edges)
