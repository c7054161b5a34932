"""Pins of the oracle's bookkeeping (oracle.c oracle_run): the OpenMP timing variant,
the multiset row hash, the per-depth partial-map counts and the first-column
partitions (SURVEY §8(c) step 4, §8(d) "Comparison of results").

Each is pinned against something other than the oracle's own search:
  * the rows of the parallel variant and of every partition equal brute force over
    all injective maps (Def. 2), so neither can drop or duplicate rows;
  * the hash equals a pure-Python restatement of splitmix64 over the brute-force
    rows (a wrong constant, shift or column order fails);
  * levels[i] equals the brute-force count of embeddings of the sub-query INDUCED
    on the first i+1 BFS vertices (the quantity the config-3/4 acceptance uses).
"""
import numpy as np
import pytest

from oracle import oracle
from synth import Query, config_graph, random_connected_query, random_multigraph, triangle_tail
from test_oracle_pins import brute_force


def _instance(seed):
    rng = np.random.default_rng(5000 + seed)
    n = int(rng.integers(5, 8))
    g = random_multigraph(n, int(rng.integers(2 * n, 4 * n)), n_elabels=2, n_vlabels=2, seed=seed,
                          undirected=seed % 4 == 0, self_loops=True, dup_prob=0.2)
    k = int(rng.integers(2, min(5, n) + 1))
    q = random_connected_query(rng, k, extra=int(rng.integers(0, 3)) if k > 2 else 0, n_elabels=2,
                               n_vlabels=2, p_wild_v=0.6, p_wild_e=0.6,
                               bound_choices=list(range(n)), p_bound=0.1)
    return g, q


def _sub_query(q: Query, verts):
    """The sub-query induced on `verts` (relabelled 0..len-1 in that order)."""
    idx = {u: i for i, u in enumerate(verts)}
    edges = [(idx[a], idx[b], l) for a, b, l in q.edges if a in idx and b in idx]
    return Query(len(verts), [q.vlabels[u] for u in verts], [q.bound[u] for u in verts], edges)


@pytest.mark.parametrize("seed", range(40))
def test_run_matches_brute_force(seed):
    g, q = _instance(seed)
    og = oracle.OracleGraph(g)
    want = brute_force(g, q)
    for threads in (1, 3):
        r = oracle.run(og, q, threads=threads, rows=True, cap=max(1, want.shape[0]))
        assert r["count"] == want.shape[0]
        assert np.array_equal(r["rows"], want)
        assert r["hash"] == oracle.multiset_hash_py(want.tolist())
        # levels: #embeddings of the sub-query induced on each BFS prefix
        order = r["order"]
        assert sorted(order) == list(range(q.k)) and order[0] == 0
        for i in range(q.k):
            sub = _sub_query(q, order[: i + 1])
            assert r["levels"][i] == brute_force(g, sub).shape[0], (threads, i)
        assert r["levels"][q.k - 1] == r["count"]


@pytest.mark.parametrize("seed", range(12))
def test_partitions_cover_the_set(seed):
    g, q = _instance(seed)
    og = oracle.OracleGraph(g)
    want = brute_force(g, q)
    cuts = [0, 2, 3, g.n]
    parts, hs, n = [], 0, 0
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        r = oracle.run(og, q, col0_range=(lo, hi), rows=True, cap=max(1, want.shape[0]))
        sel = want[(want[:, 0] >= lo) & (want[:, 0] < hi)] if want.shape[0] else want
        assert np.array_equal(r["rows"], sel)
        parts.append(r["rows"])
        hs = (hs + r["hash"]) % (1 << 64)
        n += r["count"]
    assert n == want.shape[0]
    assert hs == oracle.multiset_hash_py(want.tolist())


def test_parallel_variant_on_config1():
    """cfg1 triangle+tail (9,720 rows): the parallel variant equals the serial one, row for row."""
    g = config_graph(1)
    og = oracle.OracleGraph(g)
    q = triangle_tail()
    a = oracle.run(og, q, threads=1, rows=True, cap=20000)
    b = oracle.run(og, q, threads=4, rows=True, cap=20000)
    assert a["count"] == b["count"] == oracle.count(og, q)
    assert a["hash"] == b["hash"] and a["levels"] == b["levels"]
    assert np.array_equal(a["rows"], b["rows"])


def test_hash_of_known_rows():
    """The row hash is order-sensitive within a row and order-free across rows."""
    h1 = oracle.row_hash_py([1, 2, 3])
    h2 = oracle.row_hash_py([3, 2, 1])
    assert h1 != h2
    assert oracle.multiset_hash_py([[1, 2], [3, 4]]) == oracle.multiset_hash_py([[3, 4], [1, 2]])
    assert oracle.multiset_hash_py([[1, 2], [3, 4]]) != oracle.multiset_hash_py([[1, 4], [3, 2]])
    # splitmix64 reference value (Vigna's splitmix64 with state 0 -> first output)
    assert oracle._splitmix64(0) == 0xE220A8397B1DCDAF
