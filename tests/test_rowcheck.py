"""Pins of tests/rowcheck.py (the device-side large-set checks) on CPU torch tensors.

multiset_hash equals the pure-Python splitmix64 restatement (oracle.row_hash_py, itself
pinned in test_oracle_run.py) and the oracle's own hash; all_distinct / all_valid agree
with brute force on small instances (a duplicated row, a wrong label, a missing arc,
a repeated vertex each fail)."""
import numpy as np
import torch

import rowcheck
from oracle import oracle
from synth import config_graph, random_connected_query, random_multigraph, triangle_tail


def test_hash_matches_python_and_oracle():
    rng = np.random.default_rng(3)
    rows = rng.integers(0, 2**32, size=(257, 5), dtype=np.uint64).astype(np.uint32)
    t = torch.as_tensor(rows.view(np.int32))
    assert rowcheck.multiset_hash(t, chunk=64) == oracle.multiset_hash_py(rows.tolist())
    g = config_graph(1)
    og = oracle.OracleGraph(g)
    r = oracle.run(og, triangle_tail(), rows=True, cap=20000)
    assert rowcheck.multiset_hash(torch.as_tensor(r["rows"].view(np.int32))) == r["hash"]


def test_distinct_and_valid():
    g = config_graph(1)
    og = oracle.OracleGraph(g)
    q = triangle_tail((0, -1, -1, 2))
    rows = oracle.match(og, q)
    t = torch.as_tensor(rows.astype(np.int64))
    ga = rowcheck.GraphArrays(g, "cpu")
    assert rowcheck.all_distinct(t) and rowcheck.all_valid(t, ga, q)
    dup = torch.cat([t, t[:1]])
    assert not rowcheck.all_distinct(dup)
    bad = t.clone()
    bad[0, 1] = bad[0, 2]          # repeated vertex
    assert not rowcheck.all_valid(bad, ga, q)
    bad = t.clone()
    bad[0, 3] = int(np.nonzero(g.vlab != 2)[0][0])   # wrong label
    assert not rowcheck.all_valid(bad, ga, q)
    # random directed labelled multigraphs: valid rows are exactly the oracle's (brute force size)
    for seed in range(10):
        rng = np.random.default_rng(seed)
        gg = random_multigraph(7, 25, n_elabels=2, n_vlabels=2, seed=seed, undirected=seed % 2 == 0)
        qq = random_connected_query(rng, 3, extra=1, n_elabels=2, n_vlabels=2, p_wild_v=0.5, p_wild_e=0.5)
        ga = rowcheck.GraphArrays(gg, "cpu")
        allmaps = torch.tensor([[a, b, c] for a in range(7) for b in range(7) for c in range(7)])
        valid = [bool(rowcheck.all_valid(allmaps[i:i + 1], ga, qq)) for i in range(allmaps.shape[0])]
        want = {tuple(r) for r in oracle.match(oracle.OracleGraph(gg), qq).tolist()}
        got = {tuple(allmaps[i].tolist()) for i in range(allmaps.shape[0]) if valid[i]}
        assert got == want, seed
