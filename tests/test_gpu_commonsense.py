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
