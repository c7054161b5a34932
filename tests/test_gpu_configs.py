"""Parity on BASELINE configs[2] (cyclic 8/10/12-vertex queries) and configs[4]
(QA batch of 10,000 small queries with a bound concept vertex), full size.

Expected counts are the CPU oracle's (stored by scripts/gen_queries.py, which
calls only synth/ and oracle/); sorted embedding sets are recomputed by the
oracle live for a sample.
"""
import json
import os

import numpy as np
import pytest

from oracle import oracle
from synth import Query, config_graph

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1807_08804_b200 import gpsense
    ctx = gpsense.Context(0)
    g = config_graph(2)
    G = ctx.load_graph(g)
    yield gpsense, ctx, g, G
    ctx.close()


def _load(name):
    d = json.load(open(os.path.join(ROOT, "synth", "data", f"{name}_queries.json")))
    return [Query.from_json(x["query"]) for x in d["queries"]], [x["oracle_count"] for x in d["queries"]]


def _rows(t):
    return oracle.sort_rows(t.cpu().numpy().astype(np.uint32))


def _load_full(name):
    return json.load(open(os.path.join(ROOT, "synth", "data", f"{name}_queries.json")))["queries"]


def test_cfg3_cyclic_counts(env):
    """All 30 cyclic queries: gps_count_batch and single gps_count equal the oracle's counts."""
    gps, ctx, g, G = env
    qs, counts = _load("cfg3")
    assert ctx.count_batch(G, qs).tolist() == counts
    for q, c in zip(qs[:6], counts[:6]):
        assert ctx.count(G, q) == c


@pytest.mark.parametrize("i", range(30))
def test_cfg3_cyclic_sets(env, i):
    """Every cyclic query's full result set (up to ~10^8 rows, tables >= 10^7 rows on the
    oracle's BFS prefixes): count and multiset hash equal the oracle's, every row is a valid
    embedding and no row repeats (tests/rowcheck.py) -- together the oracle's set.  The
    smallest results are also compared as sorted sets, and one first-column partition of
    each query row by row (SURVEY §8(d) streaming comparison)."""
    import torch
    import rowcheck
    gps, ctx, g, G = env
    d = _load_full("cfg3")[i]
    q = Query.from_json(d["query"])
    ctx.reset_stats()
    t = ctx.match(G, q)
    assert t.shape == (d["oracle_count"], q.k)
    assert rowcheck.multiset_hash(t.view(torch.int32)) == int(d["oracle_hash"])
    assert rowcheck.all_distinct(t.view(torch.int32))
    ga = getattr(test_cfg3_cyclic_sets, "_ga", None)
    if ga is None:
        ga = test_cfg3_cyclic_sets._ga = rowcheck.GraphArrays(g, t.device)
    assert rowcheck.all_valid(t.view(torch.int32), ga, q)
    og = getattr(test_cfg3_cyclic_sets, "_og", None)
    if og is None:
        og = test_cfg3_cyclic_sets._og = oracle.OracleGraph(g)
    if d["oracle_count"] <= 300_000:
        assert np.array_equal(_rows(t), oracle.match(og, q))
    # one first-column partition, row by row: [lo, hi) chosen around the median image of vertex 0
    x = t.view(torch.int32)
    col0 = x[:, 0].to(torch.int64) & 0xFFFFFFFF
    if col0.numel():
        mid = int(col0.median().item())
        lo, hi = max(0, mid - 200), mid + 200
        sel = x[(col0 >= lo) & (col0 < hi)]
        r = oracle.run(og, q, col0_range=(lo, hi), rows=True, cap=max(1, sel.shape[0]) + 1, threads=os.cpu_count())
        assert r["count"] == sel.shape[0]
        assert np.array_equal(_rows(sel), r["rows"])
    del t, x


def test_cfg5_qa_batch_counts(env):
    gps, ctx, g, G = env
    qs, counts = _load("cfg5")
    got = ctx.count_batch(G, qs)
    assert got.tolist() == counts


def test_cfg5_qa_batch_sets(env):
    gps, ctx, g, G = env
    qs, counts = _load("cfg5")
    rng = np.random.default_rng(55)
    idx = rng.choice(len(qs), 60, replace=False)
    sub = [qs[i] for i in idx]
    outs = ctx.match_batch(G, sub)
    og = oracle.OracleGraph(g)
    for t, i in zip(outs, idx):
        assert t.shape[0] == counts[i]
        assert np.array_equal(_rows(t), oracle.match(og, qs[i]))
