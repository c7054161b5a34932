"""Pins of the f3 compression oracle (oracle/compress.py) against what PAPER.md fixes:
Theorem 1 (every Def. 3 candidate lies in the mapping list of a weighted candidate),
the mapping lists partition V with one label per node (Theorem 1's proof), delta = 1
combines exactly nodes with identical labelled adjacency (R33 at delta = 1), the weight
bounds the recursion must satisfy, the level-1 closed form of the recursion,
and a hand-worked example."""
import itertools

import numpy as np
import pytest

from oracle import compress, oracle
from synth import DataGraph, Query, random_connected_query, random_multigraph


def _arcs(g):
    return compress._arcs(g)


def _def3(g, q):
    """Def. 3 candidates by brute force (label, bound, out/in arc counts >= distinct query degree, R12)."""
    arcs = _arcs(g)
    od = [0] * g.n
    idg = [0] * g.n
    for (s, d, _) in arcs:
        od[s] += 1
        idg[d] += 1
    qo = [len({b for (a, b, _) in q.edges if a == u}) for u in range(q.k)]
    qi = [len({a for (a, b, _) in q.edges if b == u}) for u in range(q.k)]
    vl = [0] * g.n if g.vlab is None else g.vlab.tolist()
    res = []
    for u in range(q.k):
        res.append([v for v in range(g.n)
                    if (q.vlabels[u] == -1 or q.vlabels[u] == vl[v]) and (q.bound[u] == -1 or q.bound[u] == v)
                    and od[v] >= qo[u] and idg[v] >= qi[u]])
    return res


def _graph(seed, n=None):
    rng = np.random.default_rng(9000 + seed)
    n = n or int(rng.integers(6, 14))
    # few labels and a "hub" pattern so that identical adjacencies exist
    g = random_multigraph(n, int(rng.integers(n, 3 * n)), n_elabels=2, n_vlabels=2, seed=seed,
                          undirected=seed % 3 == 0, dup_prob=0.3)
    return g, rng


@pytest.mark.parametrize("seed", range(25))
def test_theorem1_and_partition(seed):
    g, rng = _graph(seed)
    deltas = [1.0, 1.0] if seed % 2 else [0.6, 0.8]
    levels = compress.compress(g, deltas)
    vl = [0] * g.n if g.vlab is None else g.vlab.tolist()
    for lev in levels:
        allm = sorted(x for m in lev.members for x in m)
        assert allm == list(range(g.n))                       # mapping lists partition V
        for U, m in enumerate(lev.members):
            assert len({vl[x] for x in m}) == 1 and lev.label[U] == vl[m[0]]
            assert all(lev.group[x] == U for x in m)
    k = int(rng.integers(2, 5))
    q = random_connected_query(rng, k, extra=1, n_elabels=2, n_vlabels=2, p_wild_v=0.6, p_wild_e=0.7,
                               bound_choices=list(range(g.n)), p_bound=0.1)
    d3 = _def3(g, q)
    emb = oracle.match(oracle.OracleGraph(g), q)
    for lev in levels:
        ex = compress.expanded_candidates(lev, q)
        for u in range(q.k):
            assert set(d3[u]) <= set(ex[u]), (u, d3[u], ex[u])      # Theorem 1
            assert set(emb[:, u].tolist()) <= set(ex[u])            # Theorem 2's consequence


@pytest.mark.parametrize("seed", range(25))
def test_delta1_merges_identical_adjacency(seed):
    g, _ = _graph(seed)
    lev = compress.compress(g, [1.0])[0]
    arcs = _arcs(g)
    A = [set() for _ in range(g.n)]
    for (s, d, l) in arcs:
        A[s].add(("o", l, d))
        A[d].add(("i", l, s))
    vl = [0] * g.n if g.vlab is None else g.vlab.tolist()
    for m in lev.members:
        assert len(m) <= 2
        if len(m) == 2:
            assert A[m[0]] == A[m[1]] and vl[m[0]] == vl[m[1]]
    single = [m[0] for m in lev.members if len(m) == 1]
    for a, b in itertools.combinations(single, 2):           # greedy pairing leaves no similar pair
        assert not (A[a] == A[b] and vl[a] == vl[b])


@pytest.mark.parametrize("seed", range(25))
def test_weights_bound_degrees_and_level1_closed_form(seed):
    g, _ = _graph(seed)
    levels = compress.compress(g, [1.0, 0.7, 1.0])
    arcs = _arcs(g)
    cnt = {}
    for (s, d, _) in arcs:
        cnt[(s, d)] = cnt.get((s, d), 0) + 1
    od = [0] * g.n
    idg = [0] * g.n
    for (s, d, _) in arcs:
        od[s] += 1
        idg[d] += 1
    for lev in levels:
        for X, m in enumerate(lev.members):
            so = lev.w_out[X] + sum(w for (U, V), w in lev.e_out.items() if U == X and V != X)
            si = lev.w_in[X] + sum(w for (U, V), w in lev.e_in.items() if U == X and V != X)
            for x in m:
                assert od[x] <= so and idg[x] <= si               # P:925 degree(v) <= weight(x)
                # w(X) is the max internal degree, here recomputed from its definition
            assert lev.w_out[X] == max(sum(1 for (s, d, _) in arcs if s == x and d in m) for x in m)
    lev1 = levels[0]
    for (U, V), w in lev1.e_out.items():                       # level 1: parts of V are vertices
        assert w == sum(max(cnt.get((x, y), 0) for x in lev1.members[U]) for y in lev1.members[V])


def test_hand_worked_example():
    """P:838-856 in miniature: v0 and v1 both have arcs -r0-> v2 and -r1-> v3 (identical
    labelled adjacency), so delta = 1 combines them into u0' = {v0, v1}; v2, v3 stay single.
    Weights by hand: w(u0') = 0 (no arc inside {v0, v1}); w_out(u0', v2) = max(1, 1) = 1,
    w_out(u0', v3) = 1; w_in(v2, u0') = 1 + 1 = 2 (v2's in-weight sums the parts
    v0, v1 of u0').  The query a -> b, a -> c with a of label 0 and b, c of label 1 has
    weighted candidates {u0'} for a (out-degree 2 <= 0 + 1 + 1) and {v2', v3'} for b and c."""
    src = np.array([0, 0, 1, 1], np.uint32)
    dst = np.array([2, 3, 2, 3], np.uint32)
    el = np.array([0, 1, 0, 1], np.uint16)
    vl = np.array([0, 0, 1, 1], np.uint16)
    g = DataGraph(4, src, dst, el, vl, False)
    lev = compress.compress(g, [1.0])[0]
    assert lev.members == [[0, 1], [2], [3]]
    assert lev.w_out == [0, 0, 0] and lev.w_in == [0, 0, 0]
    assert lev.e_out == {(0, 1): 1, (0, 2): 1}
    assert lev.e_in == {(1, 0): 2, (2, 0): 2}
    q = Query(3, [0, 1, 1], [-1, -1, -1], [(0, 1, -1), (0, 2, -1)])
    assert compress.weighted_candidates(lev, q) == [[0], [1, 2], [1, 2]]
    assert compress.expanded_candidates(lev, q) == [[0, 1], [2, 3], [2, 3]]
