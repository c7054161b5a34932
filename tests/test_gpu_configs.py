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


def test_cfg3_cyclic_counts(env):
    gps, ctx, g, G = env
    qs, counts = _load("cfg3")
    assert ctx.count_batch(G, qs).tolist() == counts
    for q, c in zip(qs[:6], counts[:6]):
        assert ctx.count(G, q) == c


def test_cfg3_cyclic_sets(env):
    gps, ctx, g, G = env
    qs, counts = _load("cfg3")
    og = oracle.OracleGraph(g)
    outs = ctx.match_batch(G, qs)
    for i in sorted(range(len(qs)), key=lambda i: counts[i])[:6]:
        assert np.array_equal(_rows(outs[i]), oracle.match(og, qs[i]))
    ctx.reset_stats()
    ctx.count_batch(G, qs)
    st = ctx.stats()
    assert st["join_rows_max"] > 0


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
