"""f3 multi-level graph compression on the device against
the CPU oracle (oracle/compress.py): every level's mapping (group of each vertex), labels,
node weights and weighted edges equal the oracle's; the expanded weighted candidates equal
the oracle's; with the compression attached the filter starts from them and every match
set still equals the oracle's (Theorem 1)."""
import json
import os

import numpy as np
import pytest

import corpus
from oracle import compress as ocomp
from oracle import oracle
from synth import DataGraph, Query, config_graph, random_connected_query, random_multigraph

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


def _same_level(dev, ref):
    assert dev["nodes"] == ref.n_nodes
    assert dev["group"].tolist() == ref.group
    assert dev["label"].tolist() == ref.label
    assert dev["w_out"].tolist() == ref.w_out and dev["w_in"].tolist() == ref.w_in
    assert dev["edges_out"] == ref.e_out and dev["edges_in"] == ref.e_in


def _star_forest(seed):
    """Hubs with many leaves carrying identical arcs: merges at several levels."""
    rng = np.random.default_rng(seed)
    hubs, leaves = 3, 40
    src, dst, el = [], [], []
    n = hubs + hubs * leaves
    for h in range(hubs):
        for i in range(leaves):
            leaf = hubs + h * leaves + i
            src.append(leaf); dst.append(h); el.append(int(rng.integers(0, 2)) if i % 5 == 0 else 0)
    vl = np.zeros(n, np.uint16)
    return DataGraph(n, np.array(src, np.uint32), np.array(dst, np.uint32), np.array(el, np.uint16), vl, False)


def _leafy(seed):
    """A random core plus pendant leaves hanging off a few hubs (labels from 2, arc labels
    from 2): many leaves share their labelled adjacency, so levels keep merging."""
    rng = np.random.default_rng(300 + seed)
    core = 30
    g0 = random_multigraph(core, 90, n_elabels=2, n_vlabels=2, seed=seed, undirected=False, dup_prob=0.2)
    src, dst = list(g0.src.tolist()), list(g0.dst.tolist())
    el, vl = list(g0.elab.tolist()), list(g0.vlab.tolist())
    n = core
    for _ in range(150):
        h = int(rng.integers(0, 4))
        if rng.random() < 0.5:
            src.append(n); dst.append(h)
        else:
            src.append(h); dst.append(n)
        el.append(int(rng.integers(0, 2)))
        vl.append(int(rng.integers(0, 2)))
        n += 1
    return DataGraph(n, np.array(src, np.uint32), np.array(dst, np.uint32), np.array(el, np.uint16),
                     np.array(vl, np.uint16), seed % 2 == 1)


def _graphs():
    out = []
    for seed in range(12):
        rng = np.random.default_rng(9000 + seed)
        n = int(rng.integers(6, 40))
        out.append(random_multigraph(n, int(rng.integers(n, 3 * n)), n_elabels=2, n_vlabels=2, seed=seed,
                                     undirected=seed % 3 == 0, dup_prob=0.3))
    out += [_star_forest(s) for s in range(3)]
    out += [_leafy(s) for s in range(4)]
    out.append(config_graph(2, scale=0.01))
    return out


@pytest.mark.parametrize("gi", range(20))
def test_levels_equal_oracle(gps, ctx, gi):
    g = _graphs()[gi]
    G = ctx.load_graph(g)
    cg = ctx.compress(G, [1.0, 1.0, 1.0])
    ref = ocomp.compress(g, [1.0, 1.0, 1.0])
    for lv in range(1, 4):
        _same_level(cg.level(lv), ref[lv - 1])
    cg.free()


@pytest.mark.parametrize("seed", range(0, 200, 5))
def test_corpus_candidates_and_matches(gps, ctx, seed):
    g, q = corpus.instance(seed)
    og = oracle.OracleGraph(g)
    try:
        if oracle.count(og, q, limit=500_000) == oracle.ELIMIT:
            pytest.skip("too many embeddings")
    except ValueError:
        pytest.skip("oracle rejects the instance")
    G = ctx.load_graph(g)
    cg = ctx.compress(G, [1.0, 1.0])
    ref = ocomp.compress(g, [1.0, 1.0])
    for lv in (1, 2):
        _same_level(cg.level(lv), ref[lv - 1])
        want = ocomp.expanded_candidates(ref[lv - 1], q)
        got = cg.candidates(lv, q)
        for u in range(q.k):
            assert np.nonzero(got[u])[0].tolist() == want[u], (lv, u)
    want_rows = oracle.match(og, q)
    cg.attach(2)
    rows = oracle.sort_rows(ctx.match(G, q).cpu().numpy())
    assert np.array_equal(rows, want_rows)
    assert ctx.count(G, q) == want_rows.shape[0]
    cg.free()


def test_cfg1_graph_levels(gps, ctx):
    g = config_graph(1)
    G = ctx.load_graph(g)
    cg = ctx.compress(G, [1.0, 1.0])
    ref = ocomp.compress(g, [1.0, 1.0])
    for lv in (1, 2):
        _same_level(cg.level(lv), ref[lv - 1])


def test_cfg2_theorem1_and_counts(gps, ctx):
    """Config-2 graph: the expanded weighted candidates contain Def. 3's (stage-0 bitmaps), and
    with the compression attached gps_count equals the stored oracle counts."""
    path = os.path.join(ROOT, "synth", "data", "cfg2_queries.json")
    data = json.load(open(path))
    g = config_graph(2)
    G = ctx.load_graph(g)
    cg = ctx.compress(G, [1.0, 1.0])
    n1, n2 = cg.level(1)["nodes"], cg.level(2)["nodes"]
    assert n2 <= n1 < g.n
    for item in data["queries"][:10]:
        q = Query.from_json(item["query"])
        c0 = ctx.candidates(G, q, 0)
        ex = cg.candidates(2, q)
        assert not (c0 & ~ex).any()
    cg.attach(2)
    for item in data["queries"][:20]:
        assert ctx.count(G, Query.from_json(item["query"])) == item["oracle_count"], item["seed"]
    cg.free()


def test_errors(gps, ctx):
    g = _graphs()[0]
    G = ctx.load_graph(g)
    with pytest.raises(gps.GpsError):
        ctx.compress(G, [0.8])          # delta < 1: not built on the device
    with pytest.raises(gps.GpsError):
        ctx.compress(G, [1.5])
    cg = ctx.compress(G, [1.0])
    G2 = ctx.load_graph(g)
    with pytest.raises(gps.GpsError):
        lib = gps.lib
        gps._check(lib.gps_graph_attach_compressed(G2.handle, cg.handle, 1))
    with pytest.raises(gps.GpsError):
        cg.attach(2)                    # only one level
    cg.free()


def test_free_while_attached_detaches(gps, ctx):
    """gps_free_compressed on an attached compression detaches it: later matches run without it."""
    g, q = corpus.instance(10)
    og = oracle.OracleGraph(g)
    G = ctx.load_graph(g)
    cg = ctx.compress(G, [1.0])
    cg.attach(1)
    gps._check(gps.lib.gps_free_compressed(cg.handle))   # the C call alone, no Python-side detach
    cg._h = None
    rows = oracle.sort_rows(ctx.match(G, q).cpu().numpy())
    assert np.array_equal(rows, oracle.match(og, q))
