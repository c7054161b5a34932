"""f2 -- commonsense query semantics.

* Projection ("we only need to find the matches of nodes in a subset of
  variable nodes, termed projection"): gps_match_project returns the SET of projected
  tuples, i.e. np.unique(oracle rows[:, project], axis=0) -- the plain definition of the
  projection of Emb(Q, G) -- in lexicographic order; gps_count_project its size.
* The commonsense visit order (the concept node of maximum degree first, then the
  neighbour with the most nodes not yet in the order, until the order's edges cover the
  query) is pinned on hand-built queries, and never changes a result.
* gps_load_triples ("direct transformation" of a KB into a labelled graph): the
  graph built from (subject, relation, object) triples gives the oracle's matches, the
  oracle building its own adjacency from the same triples.
"""
import json
import os

import numpy as np
import pytest

import corpus
from oracle import oracle
from synth import DataGraph, Query, config_graph, triangle_tail

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def gps():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1807_08804_b200 import gpsense
    return gpsense


@pytest.fixture(scope="module")
def ctx(gps):
    c = gps.Context(0)
    yield c
    c.close()


def _proj(rows, cols):
    if rows.shape[0] == 0:
        return np.zeros((0, len(cols)), np.uint32)
    return np.unique(rows[:, cols], axis=0).astype(np.uint32)


@pytest.mark.parametrize("seed", range(0, 200, 4))
def test_projection_corpus(gps, ctx, seed):
    g, q = corpus.instance(seed)
    og = oracle.OracleGraph(g)
    try:
        if oracle.count(og, q, limit=300_000) == oracle.ELIMIT:
            pytest.skip("too many embeddings")
    except ValueError:
        pytest.skip("oracle rejects the instance")
    rows = oracle.match(og, q)
    G = ctx.load_graph(g)
    rng = np.random.default_rng(seed)
    for kp in (1, 2, min(3, q.k), q.k):
        cols = [int(x) for x in rng.permutation(q.k)[:kp]]
        want = _proj(rows, cols)
        got = ctx.match_project(G, q, cols)
        assert np.array_equal(got, want), (kp, cols)
        assert ctx.count_project(G, q, cols) == want.shape[0]


def test_projection_qa_batch(gps, ctx):
    """Config-5 QA queries (a bound concept node): the answers are the distinct images of the
    variable nodes, as in P:592-594's example."""
    g = config_graph(2)
    G = ctx.load_graph(g)
    og = oracle.OracleGraph(g)
    d = json.load(open(os.path.join(ROOT, "synth", "data", "cfg5_queries.json")))["queries"]
    for x in d[:40]:
        q = Query.from_json(x["query"])
        var = [u for u in range(q.k) if q.bound[u] < 0]
        rows = oracle.match(og, q)
        for cols in ([var[0]], var[:2], var):
            want = _proj(rows, cols)
            assert np.array_equal(ctx.match_project(G, q, cols), want)
        o = gps.default_opts(plan_mode=gps.GPS_PLAN_COMMONSENSE)
        assert ctx.count(G, q, o) == x["oracle_count"]


def test_projection_errors(gps, ctx):
    g = config_graph(1)
    G = ctx.load_graph(g)
    for bad in ([], [4], [-1]):
        with pytest.raises(gps.GpsError) as e:
            ctx.match_project(G, triangle_tail(), bad)
        assert e.value.status == gps.GPS_EINVAL


def test_commonsense_order(gps, ctx):
    """P:937-939 on hand-built queries."""
    g = config_graph(1)
    G = ctx.load_graph(g)
    o = gps.default_opts(plan_mode=gps.GPS_PLAN_COMMONSENSE)
    # star with a bound centre 2 and a path 0-1-3-4 hanging off leaf 1: the concept node first,
    # then its neighbour 1 (two unordered neighbours: 3 and... ) -- order covers every edge
    q = Query(6, [-1] * 6, [-1, -1, 7, -1, -1, -1], [(2, 0, -1), (2, 1, -1), (2, 5, -1), (1, 3, -1), (3, 4, -1)])
    order, _ = ctx.plan(G, q, o)
    assert order[0] == 2                      # the (only) concept node
    assert order[1] == 1                      # neighbour with the most nodes outside the order (3)
    assert order == [2, 1, 3]                 # {2, 1, 3} covers all five edges
    # two concept nodes: the one of larger degree first
    q2 = Query(5, [-1] * 5, [5, -1, 9, -1, -1], [(0, 1, -1), (2, 1, -1), (2, 3, -1), (2, 4, -1), (3, 4, -1)])
    order2, _ = ctx.plan(G, q2, o)
    assert order2[0] == 2
    # no concept node: the vertex of maximum degree
    q3 = triangle_tail()
    assert ctx.plan(G, q3, o)[0][0] == 2


@pytest.mark.parametrize("seed", range(0, 200, 8))
def test_commonsense_order_same_result(gps, ctx, seed):
    g, q = corpus.instance(seed)
    og = oracle.OracleGraph(g)
    try:
        if oracle.count(og, q, limit=300_000) == oracle.ELIMIT:
            pytest.skip("too many embeddings")
    except ValueError:
        pytest.skip("oracle rejects the instance")
    G = ctx.load_graph(g)
    o = gps.default_opts(plan_mode=gps.GPS_PLAN_COMMONSENSE)
    want = oracle.match(og, q)
    got = oracle.sort_rows(ctx.match(G, q, o).cpu().numpy().astype(np.uint32))
    assert np.array_equal(got, want)


def test_load_triples(gps, ctx):
    rng = np.random.default_rng(11)
    n, m = 400, 3000
    s = rng.integers(0, n, m).astype(np.uint32)
    o_ = rng.integers(0, n, m).astype(np.uint32)
    r = rng.integers(0, 5, m).astype(np.uint16)
    G = ctx.load_triples(n, s, r, o_)
    g = DataGraph(n=n, src=s, dst=o_, elab=r, vlab=None, undirected=False)
    og = oracle.OracleGraph(g)
    assert G.arcs == og.arcs
    for q in (Query(3, [-1] * 3, [-1] * 3, [(0, 1, 2), (1, 2, -1)]),
              Query(3, [-1] * 3, [int(s[0]), -1, -1], [(0, 1, -1), (1, 2, 3), (2, 0, -1)])):
        want = oracle.match(og, q)
        got = oracle.sort_rows(ctx.match(G, q).cpu().numpy().astype(np.uint32))
        assert np.array_equal(got, want)
    with pytest.raises(gps.GpsError):
        ctx.load_triples(10, [1, 2], [0, 0], [3, 10])


# ------------------------------------------------------------ named variable edges
def _named_instance(seed):
    """A corpus instance with some variable edges named from a pool of 2 names (names repeat)."""
    g, q = corpus.instance(seed)
    rng = np.random.default_rng(77 + seed)
    ev = [int(rng.integers(0, 2)) if (l == -1 and rng.random() < 0.6) else -1 for (_, _, l) in q.edges]
    return g, q, ev


@pytest.mark.parametrize("seed", range(0, 200, 4))
def test_named_edges_corpus(gps, ctx, seed):
    """gps_match_named / gps_count_named equal the oracle's plain definition (oracle.match_named:
    embeddings x label assignments with each named edge carrying its name's label) as sorted
    sets, for all vertices and for a projection."""
    g, q, ev = _named_instance(seed)
    og = oracle.OracleGraph(g)
    try:
        if oracle.count(og, q, limit=100_000) == oracle.ELIMIT:
            pytest.skip("too many embeddings")
    except ValueError:
        pytest.skip("oracle rejects the instance")
    G = ctx.load_graph(g)
    rng = np.random.default_rng(seed)
    for proj in (None, sorted(rng.permutation(q.k)[:max(1, q.k // 2)].tolist())):
        want = oracle.match_named(g, og, q, ev, proj)
        got = ctx.match_named(G, q, ev, proj)
        assert np.array_equal(got, want), (proj, got.shape, want.shape)
        assert ctx.count_named(G, q, ev, proj) == want.shape[0]


def test_named_edges_worked_example(gps, ctx):
    """The hand-worked example of tests/test_oracle_pins.py (values written out by hand)."""
    person, bread, soup, cook = 0, 1, 2, 3
    g = DataGraph(4, np.array([0, 0, 0, 3, 3], np.uint32), np.array([1, 2, 2, 2, 1], np.uint32),
                  np.array([1, 1, 2, 3, 3], np.uint16), None, False)
    q = Query(3, [-1, -1, -1], [person, -1, cook], [(0, 1, -1), (2, 1, -1)])
    G = ctx.load_graph(g)
    assert ctx.match_named(G, q, [0, 1]).tolist() == [[person, bread, cook, 1, 3], [person, soup, cook, 1, 3],
                                                      [person, soup, cook, 2, 3]]
    assert ctx.match_named(G, q, [0, 0]).shape == (0, 4)
    assert ctx.match_named(G, q, [5, 9], [1]).tolist() == [[bread, 1, 3], [soup, 1, 3], [soup, 2, 3]]
    assert ctx.match_named(G, q, [-1, 7], [1]).tolist() == [[bread, 3], [soup, 3]]
    assert ctx.count_named(G, q, [-1, -1]) == 2   # no names: the distinct embeddings


def test_named_edges_errors(gps, ctx):
    g = DataGraph(3, np.array([0, 1], np.uint32), np.array([1, 2], np.uint32), np.array([0, 1], np.uint16), None, False)
    G = ctx.load_graph(g)
    q = Query(3, [-1] * 3, [-1] * 3, [(0, 1, 0), (1, 2, -1)])
    with pytest.raises(gps.GpsError):   # a named edge must be a variable edge
        ctx.match_named(G, q, [0, 1])
    with pytest.raises(gps.GpsError):
        ctx.match_named(G, q, [-1, 0], [3])


def test_named_edges_cfg5_queries(gps, ctx):
    """ConceptNet-shaped graph (34 edge labels): QA queries whose variable edges share one name
    (the commonsense "same relation" question), against the oracle."""
    path = os.path.join(ROOT, "synth", "data", "cfg5_queries.json")
    if not os.path.exists(path):
        pytest.skip("cfg5 queries not generated")
    with open(path) as fh:
        data = json.load(fh)
    g = config_graph(5)
    og = oracle.OracleGraph(g)
    G = ctx.load_graph(g)
    done = 0
    for item in data["queries"][:400]:
        q0 = Query.from_json(item["query"])
        # the query with its relations replaced by variable edges: names 0, 1, 0, 1, ...
        q = Query(q0.k, q0.vlabels, q0.bound, [(a, b, -1) for (a, b, _) in q0.edges])
        ev = [i % 2 for i in range(len(q.edges))]
        if oracle.count(og, q, limit=20_000) == oracle.ELIMIT:
            continue
        want = oracle.match_named(g, og, q, ev)
        assert np.array_equal(ctx.match_named(G, q, ev), want), item["seed"]
        done += 1
        if done == 6:
            break
    assert done > 0
