"""Pins for the CPU oracle (oracle/oracle.c) against things other than itself.

Each pin is chosen so a plausible oracle bug (a dropped label test, a reversed
arc direction, a missing injectivity check, duplicate rows from parallel arcs,
a bound vertex ignored) fails at least one of them:

  * brute force over ALL injective maps on tiny directed, edge-labelled
    multigraphs with wildcards and bound vertices (Def. 2);
  * networkx MultiDiGraphMatcher.subgraph_monomorphisms_iter (independent library);
  * closed forms on the config-1 graph: tr(A^3), 4-cycles,
    wedges, the labelled triangle-plus-tail formula, and the label-partition
    identity over all 8^4 labelled variants;
  * the worked example of P:612-618 (SURVEY Appendix A fixture, tests/golden);
  * special cases with textbook counts: K_n / K_k -> n!/(n-k)!, K4 triangle -> 24
    (S:454), star S_m edge query -> 2m, unsatisfiable label -> 0.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import closed_forms  # noqa: F401  (tests/ on sys.path via conftest)
from oracle import oracle
from synth import (DataGraph, Query, complete_graph, complete_query, config_graph,
                   fixture_fig3_example, random_connected_query, random_multigraph,
                   star_graph, triangle_tail)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def brute_force(g: DataGraph, q: Query) -> np.ndarray:
    """Enumerate every injective map V_q -> V_g and keep those satisfying Def. 2
    (generalised: directed labelled arcs, '*' labels, bound vertices)."""
    arcs = set()
    pairs = set()
    lab = g.elab if g.elab is not None else np.zeros(g.m, np.uint16)
    for s, d, l in zip(g.src.tolist(), g.dst.tolist(), lab.tolist()):
        arcs.add((s, d, l)); pairs.add((s, d))
        if g.undirected:
            arcs.add((d, s, l)); pairs.add((d, s))
    vl = g.vlab.tolist() if g.vlab is not None else [0] * g.n
    rows = []
    for f in itertools.permutations(range(g.n), q.k):
        if any(q.vlabels[u] != -1 and q.vlabels[u] != vl[f[u]] for u in range(q.k)):
            continue
        if any(q.bound[u] != -1 and q.bound[u] != f[u] for u in range(q.k)):
            continue
        ok = True
        for a, b, l in q.edges:
            if l == -1:
                ok = (f[a], f[b]) in pairs
            else:
                ok = (f[a], f[b], l) in arcs
            if not ok:
                break
        if ok:
            rows.append(f)
    return oracle.sort_rows(np.array(rows, np.uint32).reshape(-1, q.k))


def _eq(a, b):
    return a.shape == b.shape and np.array_equal(a, b)


@pytest.mark.parametrize("seed", range(60))
def test_oracle_equals_brute_force(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(4, 8))
    undirected = seed % 3 == 0
    g = random_multigraph(n, int(rng.integers(n, 3 * n)), n_elabels=3, n_vlabels=2,
                          seed=seed, undirected=undirected, self_loops=True, dup_prob=0.3)
    k = int(rng.integers(1, min(5, n) + 1))
    q = random_connected_query(rng, k, extra=int(rng.integers(0, 3)) if k > 2 else 0,
                               n_elabels=3, n_vlabels=2, p_wild_v=0.5, p_wild_e=0.5,
                               bound_choices=list(range(n)), p_bound=0.15)
    og = oracle.OracleGraph(g)
    got = oracle.match(og, q)
    want = brute_force(g, q)
    assert _eq(got, want), (seed, got.shape, want.shape)
    assert oracle.count(og, q) == want.shape[0]


def _nx_rows(g: DataGraph, q: Query):
    nx = pytest.importorskip("networkx")
    from networkx.algorithms import isomorphism as iso
    G = nx.MultiDiGraph()
    vl = g.vlab.tolist() if g.vlab is not None else [0] * g.n
    for v in range(g.n):
        G.add_node(v, lab=vl[v], vid=v)
    lab = g.elab.tolist() if g.elab is not None else [0] * g.m
    seen = set()
    for s, d, l in zip(g.src.tolist(), g.dst.tolist(), lab):
        for (x, y) in ([(s, d), (d, s)] if g.undirected else [(s, d)]):
            if (x, y, l) not in seen:
                seen.add((x, y, l))
                G.add_edge(x, y, lab=l)
    Q = nx.MultiDiGraph()
    for u in range(q.k):
        Q.add_node(u, lab=q.vlabels[u], bound=q.bound[u])
    for a, b, l in q.edges:
        Q.add_edge(a, b, lab=l)

    def node_match(dn, qn):
        return (qn["lab"] == -1 or qn["lab"] == dn["lab"]) and (qn["bound"] == -1 or qn["bound"] == dn["vid"])

    def edge_match(de, qe):
        want = [e["lab"] for e in qe.values()]
        have = {e["lab"] for e in de.values()}
        return all(w == -1 or w in have for w in want)

    M = iso.MultiDiGraphMatcher(G, Q, node_match=node_match, edge_match=edge_match)
    rows = []
    for mp in M.subgraph_monomorphisms_iter():
        inv = {u: v for v, u in mp.items()}
        rows.append([inv[u] for u in range(q.k)])
    return oracle.sort_rows(np.array(rows, np.uint32).reshape(-1, q.k))


@pytest.mark.parametrize("seed", range(12))
def test_oracle_equals_networkx(seed):
    rng = np.random.default_rng(2000 + seed)
    n = int(rng.integers(20, 60))
    g = random_multigraph(n, 4 * n, n_elabels=3, n_vlabels=3, seed=500 + seed,
                          undirected=seed % 4 == 0, self_loops=True, dup_prob=0.2)
    k = int(rng.integers(2, 6))
    q = random_connected_query(rng, k, extra=int(rng.integers(0, 3)) if k > 2 else 0,
                               n_elabels=3, n_vlabels=3, p_wild_v=0.6, p_wild_e=0.6,
                               bound_choices=list(range(n)), p_bound=0.1)
    # networkx's multigraph matcher counts parallel query arcs; keep one arc per ordered pair
    uniq = {}
    for a, b, l in q.edges:
        uniq.setdefault((a, b), (a, b, l))
    q = Query(q.k, q.vlabels, q.bound, list(uniq.values()))
    og = oracle.OracleGraph(g)
    assert _eq(oracle.match(og, q), _nx_rows(g, q))


@pytest.fixture(scope="module")
def cfg1():
    g = config_graph(1)
    # float64 so numpy uses BLAS; every entry stays an integer far below 2^53
    A = np.zeros((g.n, g.n), np.float64)
    A[g.src, g.dst] = 1
    A[g.dst, g.src] = 1
    return g, A, oracle.OracleGraph(g)


def test_cfg1_generator_shape(cfg1):
    g, A, og = cfg1
    assert g.n == 1000 and g.m == 5000 and g.undirected
    assert np.all(np.diag(A) == 0) and A.sum() == 2 * 5000   # simple graph
    assert og.arcs == 10000


def test_closed_form_triangles(cfg1):
    g, A, og = cfg1
    tri = Query(3, [-1] * 3, [-1] * 3, [(0, 1, -1), (1, 2, -1), (2, 0, -1)])
    assert oracle.count(og, tri) == int(round(np.trace(A @ A @ A)))


def test_closed_form_four_cycles(cfg1):
    g, A, og = cfg1
    d = A.sum(1)
    c4 = Query(4, [-1] * 4, [-1] * 4, [(0, 1, -1), (1, 2, -1), (2, 3, -1), (3, 0, -1)])
    A2 = A @ A
    want = int(round(np.trace(A2 @ A2) - 2 * (d * d).sum() + 2 * g.m))
    assert oracle.count(og, c4) == want


def test_closed_form_wedges(cfg1):
    g, A, og = cfg1
    d = A.sum(1)
    wedge = Query(3, [-1] * 3, [-1] * 3, [(0, 1, -1), (1, 2, -1)])
    assert oracle.count(og, wedge) == int(round((d * (d - 1)).sum()))


def _tt_exact(A, vlab, la, lb, lc, ld):
    """Labelled triangle (q0,q1,q2) + tail q3 on q2:
    sum_c T_c * (N_c - [f(q0) fits q3] - [f(q1) fits q3]) with T_c counted per
    label class of q0/q1 so the subtraction is exact even with wildcards."""
    ones = np.ones(A.shape[0], np.float64)

    def D(l):
        return ones if l == -1 else (vlab == l).astype(np.float64)
    Da, Db, Dc, Dd = D(la), D(lb), D(lc), D(ld)
    N = A @ Dd
    # T_c: ordered (a, b) with a~b, b~c, c~a, labels fitting
    T = np.diag((Dc[:, None] * A) @ (Da[:, None] * A) @ (Db[:, None] * A)) * Dc
    # T_c^{a fits d}: same but a additionally fits q3's label
    Tad = np.diag((Dc[:, None] * A) @ ((Da * Dd)[:, None] * A) @ (Db[:, None] * A)) * Dc
    Tbd = np.diag((Dc[:, None] * A) @ (Da[:, None] * A) @ ((Db * Dd)[:, None] * A)) * Dc
    return int(round((T * N).sum() - Tad.sum() - Tbd.sum()))


def test_closed_form_triangle_tail_labelled(cfg1):
    g, A, og = cfg1
    vlab = g.vlab.astype(np.int64)
    rng = np.random.default_rng(7)
    cases = [(-1, -1, -1, -1), (0, 1, 2, 3), (1, 1, 1, 1), (2, 2, 5, 2), (-1, 3, -1, 3)]
    cases += [tuple(int(x) for x in rng.integers(0, 8, 4)) for _ in range(6)]
    for lab in cases:
        q = triangle_tail(lab)
        assert oracle.count(og, q) == _tt_exact(A, vlab, *lab), lab


def test_label_partition_identity(cfg1):
    """sum over all 8^4 labelled variants of count = count of the all-'*' query."""
    g, A, og = cfg1
    total = 0
    for lab in itertools.product(range(8), repeat=4):
        total += oracle.count(og, triangle_tail(lab))
    assert total == oracle.count(og, triangle_tail())


def test_cfg1_triangle_tail_networkx(cfg1):
    g, A, og = cfg1
    q = triangle_tail((1, -1, 2, -1))
    assert _eq(oracle.match(og, q), _nx_rows(g, q))


def test_worked_example_fig3():
    """the unique match {(u1,v1),(u2,v2),(u3,v3),(u4,v6),(u5,v7),(u6,v8)}."""
    with open(os.path.join(GOLDEN, "fig3_example.json")) as fh:
        gold = json.load(fh)
    g, q = fixture_fig3_example()
    rows = oracle.match(oracle.OracleGraph(g), q)
    assert rows.tolist() == gold["embeddings"]
    assert rows.tolist() == [[0, 1, 2, 5, 6, 7]]


@pytest.mark.parametrize("n,k", [(4, 3), (6, 3), (6, 4), (7, 5)])
def test_complete_graph_counts(n, k):
    og = oracle.OracleGraph(complete_graph(n))
    assert oracle.count(og, complete_query(k)) == math.perm(n, k)


def test_k4_triangle_24():
    """triangle query in K4 (unlabelled) -> 24 injective maps."""
    og = oracle.OracleGraph(complete_graph(4))
    assert oracle.count(og, complete_query(3)) == 24


@pytest.mark.parametrize("m", [1, 3, 10])
def test_star_edge_query(m):
    og = oracle.OracleGraph(star_graph(m))
    assert oracle.count(og, Query(2, [-1, -1], [-1, -1], [(0, 1, -1)])) == 2 * m


def test_bound_and_unsatisfiable():
    og = oracle.OracleGraph(star_graph(5))
    # centre bound: 5 leaves
    assert oracle.count(og, Query(2, [-1, -1], [0, -1], [(0, 1, -1)])) == 5
    # leaf bound on both sides of a 2-path through the centre: the other leaf varies
    assert oracle.count(og, Query(3, [-1] * 3, [1, -1, -1], [(0, 1, -1), (1, 2, -1)])) == 4
    # a label nobody carries
    assert oracle.count(og, Query(2, [3, -1], [-1, -1], [(0, 1, -1)])) == 0
    # an edge label nobody carries (graph has only label 0)
    assert oracle.count(og, Query(2, [-1, -1], [-1, -1], [(0, 1, 4)])) == 0


def test_directed_semantics():
    # 0 -> 1 -> 2 (directed path): directed 2-path query has exactly one match
    g = DataGraph(3, np.array([0, 1], np.uint32), np.array([1, 2], np.uint32), None, None, False)
    og = oracle.OracleGraph(g)
    assert oracle.match(og, Query(3, [-1] * 3, [-1] * 3, [(0, 1, -1), (1, 2, -1)])).tolist() == [[0, 1, 2]]
    # reversed arc direction in the query: still one match, mapped in reverse
    assert oracle.match(og, Query(3, [-1] * 3, [-1] * 3, [(1, 0, -1), (2, 1, -1)])).tolist() == [[2, 1, 0]]


def test_parallel_arcs_no_duplicate_rows():
    # two parallel arcs 0->1 (labels 0 and 1) and exact duplicates: one wildcard match only
    g = DataGraph(2, np.array([0, 0, 0], np.uint32), np.array([1, 1, 1], np.uint32),
                  np.array([0, 1, 1], np.uint16), None, False)
    og = oracle.OracleGraph(g)
    assert oracle.match(og, Query(2, [-1, -1], [-1, -1], [(0, 1, -1)])).tolist() == [[0, 1]]
    assert oracle.count(og, Query(2, [-1, -1], [-1, -1], [(0, 1, 1)])) == 1
    assert oracle.count(og, Query(2, [-1, -1], [-1, -1], [(0, 1, 2)])) == 0
    # both labels demanded at once: satisfied by the two parallel arcs
    assert oracle.count(og, Query(2, [-1, -1], [-1, -1], [(0, 1, 0), (0, 1, 1)])) == 1


def test_errors():
    og = oracle.OracleGraph(complete_graph(4))
    with pytest.raises(ValueError):   # disconnected
        oracle.count(og, Query(3, [-1] * 3, [-1] * 3, [(0, 1, -1)]))
    with pytest.raises(ValueError):   # self loop
        oracle.count(og, Query(2, [-1] * 2, [-1] * 2, [(0, 0, -1), (0, 1, -1)]))
    with pytest.raises(ValueError):   # bound id out of range
        oracle.count(og, Query(2, [-1] * 2, [9, -1], [(0, 1, -1)]))


# ------------------------------------------------------------------ closed forms of config 4
@pytest.mark.parametrize("seed", range(6))
def test_closed_forms_large_families_vs_oracle(seed):
    """tests/closed_forms.py (used to pin config 4 at 10^8 scale) against the oracle on small graphs."""
    import closed_forms as cf
    from synth.large import in_star, out_star, path2
    g = random_multigraph(60, 700, n_elabels=3, n_vlabels=3, seed=900 + seed, undirected=False,
                          self_loops=False, dup_prob=0.3)
    og = oracle.OracleGraph(g)
    keys = cf.pair_keys(g)
    rng = np.random.default_rng(seed)
    for _ in range(4):
        la, lb, lc = (int(x) for x in rng.integers(-1, 3, 3))
        k = int(rng.integers(1, 4))
        assert oracle.count(og, out_star(k, la, lb)) == cf.out_star(g, keys, k, la, lb)
        assert oracle.count(og, in_star(k, la, lb)) == cf.in_star(g, keys, k, la, lb)
        assert oracle.count(og, path2(la, lb, lc)) == cf.path2(g, keys, la, lb, lc)


# ---------------------------------------------------------------- f2 named variable edges
def brute_force_named(g: DataGraph, q: Query, edge_var, project):
    """Every injective map V_q -> V_g and every assignment of present labels to the named
    variables, kept when Def. 2 holds with each named edge carrying its variable's label."""
    arcs, pairs = set(), set()
    lab = g.elab if g.elab is not None else np.zeros(g.m, np.uint16)
    for s, d, l in zip(g.src.tolist(), g.dst.tolist(), lab.tolist()):
        arcs.add((s, d, l)); pairs.add((s, d))
        if g.undirected:
            arcs.add((d, s, l)); pairs.add((d, s))
    present = sorted(set(lab.tolist())) or [0]
    names = sorted({v for v in edge_var if v >= 0})
    vl = g.vlab.tolist() if g.vlab is not None else [0] * g.n
    out = set()
    for f in itertools.permutations(range(g.n), q.k):
        if any(q.vlabels[u] != -1 and q.vlabels[u] != vl[f[u]] for u in range(q.k)):
            continue
        if any(q.bound[u] != -1 and q.bound[u] != f[u] for u in range(q.k)):
            continue
        for beta in itertools.product(present, repeat=len(names)):
            ok = True
            for (a, b, l), v in zip(q.edges, edge_var):
                if v >= 0:
                    ok = (f[a], f[b], beta[names.index(v)]) in arcs
                elif l == -1:
                    ok = (f[a], f[b]) in pairs
                else:
                    ok = (f[a], f[b], l) in arcs
                if not ok:
                    break
            if ok:
                out.add(tuple(f[p] for p in project) + tuple(beta))
    w = len(project) + len(names)
    return np.array(sorted(out), np.uint32).reshape(-1, w)


@pytest.mark.parametrize("seed", range(30))
def test_oracle_named_edges_equal_brute_force(seed):
    rng = np.random.default_rng(5000 + seed)
    n = int(rng.integers(4, 7))
    g = random_multigraph(n, int(rng.integers(2 * n, 4 * n)), n_elabels=3, n_vlabels=2,
                          seed=seed, undirected=seed % 4 == 0, dup_prob=0.4)
    k = int(rng.integers(2, min(4, n) + 1))
    q = random_connected_query(rng, k, extra=int(rng.integers(0, 2)), n_elabels=3, n_vlabels=2,
                               p_wild_v=0.6, p_wild_e=0.8)
    # name some of the variable edges, from a pool of 2 names (so names repeat)
    ev = [int(rng.integers(0, 2)) if (l == -1 and rng.random() < 0.7) else -1 for (_, _, l) in q.edges]
    proj = sorted(rng.choice(k, size=int(rng.integers(1, k + 1)), replace=False).tolist())
    got = oracle.match_named(g, oracle.OracleGraph(g), q, ev, proj)
    want = brute_force_named(g, q, ev, proj)
    assert _eq(got, want), (seed, got.shape, want.shape)


def test_oracle_named_edges_worked_example():
    """Hand-worked (P:592-594 reading): data arcs person -eats(1)-> bread, person -eats(1)-> soup,
    person -likes(2)-> soup, cook -makes(3)-> soup, cook -makes(3)-> bread.  Query ?p -?x-> ?f <-?y- ?c
    with ?x, ?y distinct names: ?p = person (0), ?c = cook (3):  f = soup: x in {eats, likes},
    y = makes; f = bread: x = eats, y = makes.  With ?x = ?y (one name) nothing matches (no label
    both eats/likes and makes).  Projection onto ?f only: (bread, 1, 3), (soup, 1, 3), (soup, 2, 3)."""
    person, bread, soup, cook = 0, 1, 2, 3
    src = np.array([person, person, person, cook, cook], np.uint32)
    dst = np.array([bread, soup, soup, soup, bread], np.uint32)
    el = np.array([1, 1, 2, 3, 3], np.uint16)
    g = DataGraph(4, src, dst, el, None, False)
    q = Query(3, [-1, -1, -1], [person, -1, cook], [(0, 1, -1), (2, 1, -1)])
    og = oracle.OracleGraph(g)
    rows = oracle.match_named(g, og, q, [0, 1])
    assert rows.tolist() == [[person, bread, cook, 1, 3], [person, soup, cook, 1, 3], [person, soup, cook, 2, 3]]
    assert oracle.match_named(g, og, q, [0, 0]).shape == (0, 4)
    assert oracle.match_named(g, og, q, [0, 1], [1]).tolist() == [[bread, 1, 3], [soup, 1, 3], [soup, 2, 3]]
    # one named edge, one plain variable edge: the plain one binds nothing
    assert oracle.match_named(g, og, q, [-1, 7], [1]).tolist() == [[bread, 3], [soup, 3]]
