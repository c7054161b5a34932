"""Pins of tests/filter_ref.py (the filter-set reference) against the paper and the oracle.

CPU only.  The worked example fixes O's prefix and the check results (P:618-624,
P:688, tests/golden/fig3_example.json); on the random corpus every
embedding the oracle finds must survive every stage (soundness: filtering never
removes a true image, Alg. 1), stages only shrink the sets, and the filter is not
vacuous (it removes something on a good share of instances).
"""
import json
import os

import numpy as np
import pytest

import corpus
import filter_ref
from oracle import oracle
from synth import fixture_fig3_example

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_fig3_plan_and_check():
    gold = json.load(open(os.path.join(GOLDEN, "fig3_example.json")))
    g, q = fixture_fig3_example()
    order, parent, discovery = filter_ref.plan(g, q)
    assert order[:2] == gold["visit_order_prefix"]          # u5, u2
    c0 = filter_ref.candidates(g, q, 0)
    assert np.nonzero(c0[2])[0].tolist() == gold["candidates_u3_after_check"]
    assert np.nonzero(c0[0])[0].tolist() == gold["candidates_u1_after_check"]
    rows = np.array(gold["embeddings"])
    for stage in (1, 2):
        c = filter_ref.candidates(g, q, stage)
        for u in range(q.k):
            assert c[u][rows[:, u]].all()


def test_plan_is_a_spanning_tree():
    for seed in range(0, 200, 3):
        g, q = corpus.instance(seed)
        order, parent, discovery = filter_ref.plan(g, q)
        assert sorted(discovery) == list(range(q.k)) and len(set(order)) == len(order)
        assert sum(p < 0 for p in parent) == 1
        edges = {(a, b) for a, b, _ in q.edges} | {(b, a) for a, b, _ in q.edges}
        assert all(p < 0 or (p, v) in edges for v, p in enumerate(parent))


@pytest.mark.parametrize("seed", range(0, 200, 4))
def test_reference_filter_sound_and_monotone(seed):
    g, q = corpus.instance(seed)
    og = oracle.OracleGraph(g)
    try:
        if oracle.count(og, q, limit=200_000) == oracle.ELIMIT:
            pytest.skip("too many embeddings")
    except ValueError:
        pytest.skip("oracle rejects the instance")
    rows = oracle.match(og, q)
    prev = None
    for stage in (0, 1, 2):
        c = filter_ref.candidates(g, q, stage)
        for u in range(q.k):
            assert c[u][rows[:, u]].all(), (stage, u)
        if prev is not None:
            assert not (c & ~prev).any()
        prev = c


def test_reference_filter_not_vacuous():
    shrunk = 0
    for seed in range(0, 200, 10):
        g, q = corpus.instance(seed)
        shrunk += int(filter_ref.candidates(g, q, 2).sum() < filter_ref.candidates(g, q, 0).sum())
    assert shrunk >= 5
