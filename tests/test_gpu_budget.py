"""Depth-first chunking of oversized join tables (reading R27 / SURVEY A27, PAPER P:941
"intermediate results ... a key challenge") and the per-query limits of a batch.

The result set never depends on the row budget: with a budget so small that nearly every
join step is split into pair ranges (and each range carried through the remaining steps
before the next starts), gps_match returns the oracle's sorted set and gps_count its
count.  A batch whose candidate-edge tables exceed the 32-bit value positions defers the
queries that do not fit to a later chunk; a query that alone exceeds them fails with
GPS_EOVERFLOW and the others are unaffected (GPS_EC_PAIR_LIMIT lowers the limit).
"""
import json
import os

import numpy as np
import pytest

import corpus
from oracle import oracle
from synth import Query, config_graph, triangle_tail

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


def _rows(t):
    a = t.cpu().numpy() if hasattr(t, "cpu") else np.asarray(t)
    return oracle.sort_rows(a.astype(np.uint32))


@pytest.mark.parametrize("fast", [True, False])
@pytest.mark.parametrize("seed", range(0, 200, 4))
def test_corpus_tiny_budget(gps, ctx, seed, fast, monkeypatch):
    if not fast:
        monkeypatch.setenv("GPS_NO_FAST_JOIN", "1")
    g, q = corpus.instance(seed)
    og = oracle.OracleGraph(g)
    try:
        c = oracle.count(og, q, limit=300_000)
    except ValueError:
        pytest.skip("oracle rejects the instance")
    if c == oracle.ELIMIT:
        pytest.skip("too many embeddings for this test")
    G = ctx.load_graph(g)
    o = gps.default_opts(row_budget_bytes=2048)
    ctx.reset_stats()
    assert ctx.count(G, q, o) == c
    want = oracle.match(og, q)
    assert np.array_equal(_rows(ctx.match(G, q, o)), want)
    if c > 2048:   # some step was split: no table the budget does not allow
        assert ctx.stats()["join_rows_max"] * 8 <= 2048


def test_cfg2_batch_small_budget(gps, ctx):
    """A whole batch falls to the depth-first path (every query of an oversized step)."""
    g = config_graph(2)
    G = ctx.load_graph(g)
    d = json.load(open(os.path.join(ROOT, "synth", "data", "cfg2_queries.json")))
    qs = [Query.from_json(x["query"]) for x in d["queries"][:30]]
    want = [x["oracle_count"] for x in d["queries"][:30]]
    o = gps.default_opts(row_budget_bytes=1 << 20)
    assert ctx.count_batch(G, qs, o).tolist() == want
    outs = ctx.match_batch(G, qs, o)
    assert [t.shape[0] for t in outs] == want
    og = oracle.OracleGraph(g)
    for i in sorted(range(30), key=lambda i: want[i])[:3]:
        assert np.array_equal(_rows(outs[i]), oracle.match(og, qs[i]))


def test_ec_deferral_and_per_query_overflow(gps, ctx, monkeypatch):
    g = config_graph(1)
    G = ctx.load_graph(g)
    og = oracle.OracleGraph(g)
    qs = [triangle_tail(lab) for lab in [(-1, -1, -1, -1), (0, 1, 2, 3), (1, -1, 2, -1), (-1, 2, -1, 5)]] * 4
    want = [oracle.count(og, q) for q in qs]
    ctx.set_workers(1)
    # room for about one query's candidate-edge pairs per chunk: most queries are deferred
    monkeypatch.setenv("GPS_EC_PAIR_LIMIT", "90000")
    counts, st = ctx.count_batch(G, qs, statuses=True)
    assert st.tolist() == [0] * len(qs)
    assert counts.tolist() == want
    outs = ctx.match_batch(G, qs)
    assert [t.shape[0] for t in outs] == want
    # a limit below the all-wildcard query's own need: it alone fails, the others complete
    monkeypatch.setenv("GPS_EC_PAIR_LIMIT", "30000")
    counts, st = ctx.count_batch(G, qs, statuses=True)
    for i, q in enumerate(qs):
        if st[i] == 0:
            assert counts[i] == want[i]
        else:
            assert st[i] == gps.GPS_EOVERFLOW
    assert (st == gps.GPS_EOVERFLOW).any() and (st == 0).any()
    monkeypatch.delenv("GPS_EC_PAIR_LIMIT")
    ctx.set_workers(0)


def test_batch_results_outlive_workers(gps, ctx):
    """Device rows of a batch stay valid after the worker pool is rebuilt (they belong to the
    caller's ctx) and are released in order after the torch stream that reads them."""
    import torch
    g = config_graph(1)
    G = ctx.load_graph(g)
    og = oracle.OracleGraph(g)
    qs = [triangle_tail(), triangle_tail((0, -1, -1, -1))]
    ctx.set_workers(2)
    outs = ctx.match_batch(G, qs)
    ctx.set_workers(3)            # destroys the workers that produced the rows
    torch.cuda.synchronize()
    for t, q in zip(outs, qs):
        s = t.to(torch.int64).sum()   # a torch kernel reads the rows
        assert np.array_equal(_rows(t), oracle.match(og, q))
        assert int(s) == int(oracle.match(og, q).astype(np.int64).sum())
    del outs
    torch.cuda.synchronize()
    ctx.set_workers(0)
