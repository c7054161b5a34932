"""Parity of the CUDA path (through the C-ABI) with the CPU oracle.

Bar: the path is integer-only, so every comparison is
bit-exact -- the sorted embedding set of gps_match equals the oracle's sorted
set, and gps_count equals the oracle's count.  Inputs are seeded synth/
generators; expected values come only from oracle/ (or tests/golden, cited).
"""
import json
import os

import numpy as np
import pytest

import corpus
import filter_ref
from oracle import oracle
from synth import (DataGraph, Query, bfs_query, config_graph, fixture_fig3_example,
                   random_connected_query, random_multigraph, triangle_tail)

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


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


def _check(ctx, G, og, q, opts=None):
    want = oracle.match(og, q)
    got = _rows(ctx.match(G, q, opts))
    assert got.shape == want.shape, (got.shape, want.shape)
    assert np.array_equal(got, want)
    assert ctx.count(G, q, opts) == want.shape[0]
    return want


# ---------------------------------------------------------------- worked example
def test_fig3_example(ctx):
    gold = json.load(open(os.path.join(GOLDEN, "fig3_example.json")))
    g, q = fixture_fig3_example()
    G = ctx.load_graph(g)
    rows = _rows(ctx.match(G, q))
    assert rows.tolist() == gold["embeddings"]
    assert ctx.count(G, q) == 1
    order, rank = ctx.plan(G, q)
    assert order[:2] == gold["visit_order_prefix"]        # u5, u2
    for (d, f), (gd, gf) in zip(rank, gold["rank_f"]):     # f(u) = deg/freq
        assert d * gf == gd * f
    c0 = ctx.candidates(G, q, 0)
    assert np.nonzero(c0[2])[0].tolist() == gold["candidates_u3_after_check"]
    assert np.nonzero(c0[0])[0].tolist() == gold["candidates_u1_after_check"]
    assert c0[0][:6].tolist() == gold["c_set_u1_flags_v1_to_v6"]


# ------------------------------------------------------------- random corpus
def _instance(seed):
    return corpus.instance(seed)


@pytest.mark.parametrize("seed", range(200))
def test_random_corpus(ctx, seed):
    """S:499 acceptance corpus: data <= 300 nodes, avg degree <= 8, <= 20 labels, BFS queries of 4-8 nodes."""
    g, q = _instance(seed)
    og = oracle.OracleGraph(g)
    try:
        oracle.count(og, q, limit=2_000_000)
    except ValueError:
        pytest.skip("oracle rejects the instance")
    if oracle.count(og, q, limit=2_000_000) == oracle.ELIMIT:
        pytest.skip("too many embeddings for the oracle")
    _check(ctx, ctx.load_graph(g), og, q)


@pytest.mark.parametrize("env", ["GPS_SINGLE_PASS_BYTES=0", "GPS_NO_FAST_JOIN=1", "GPS_SINGLE_PASS_BYTES=256",
                                 "GPS_NO_CLOSE_DIR=1"])
@pytest.mark.parametrize("seed", range(0, 200, 5))
def test_random_corpus_other_join_paths(ctx, seed, env, monkeypatch):
    """Same corpus with the closing-free fast path off (GPS_NO_FAST_JOIN: look-back tiles) and
    additionally: the single pass off (GPS_SINGLE_PASS_BYTES=0: count -> exact allocation ->
    write); a 256-byte single-pass buffer (nearly every step overflows it and reruns its tail);
    closing arcs only in the direction built first (GPS_NO_CLOSE_DIR: per-pair rank lookups)."""
    monkeypatch.setenv("GPS_NO_FAST_JOIN", "1")
    k, v = env.split("=")
    monkeypatch.setenv(k, v)
    g, q = _instance(seed)
    og = oracle.OracleGraph(g)
    try:
        if oracle.count(og, q, limit=2_000_000) == oracle.ELIMIT:
            pytest.skip("too many embeddings for the oracle")
    except ValueError:
        pytest.skip("oracle rejects the instance")
    ctx.reset_stats()
    _check(ctx, ctx.load_graph(g), og, q)


@pytest.mark.parametrize("env", ["GPS_JOIN_NO_BULK=1", "GPS_JOIN_WIDE_STAGED=1"])
@pytest.mark.parametrize("seed", range(0, 200, 5))
def test_random_corpus_kernel_variants(ctx, seed, env, monkeypatch):
    """Same corpus through the kernel variants the default path replaced: the closing-free
    write loading its row inputs as it goes (k_join_fast instead of the bulk-staged
    k_join_bulk), and wide output rows staged + bulk-stored instead of stored word-parallel."""
    k, v = env.split("=")
    monkeypatch.setenv(k, v)
    g, q = _instance(seed)
    og = oracle.OracleGraph(g)
    try:
        if oracle.count(og, q, limit=2_000_000) == oracle.ELIMIT:
            pytest.skip("too many embeddings for the oracle")
    except ValueError:
        pytest.skip("oracle rejects the instance")
    _check(ctx, ctx.load_graph(g), og, q)


@pytest.mark.parametrize("seed", range(0, 200, 7))
def test_filter_soundness_and_monotone(ctx, seed):
    """No oracle-embedding image is ever pruned; stages only shrink the sets."""
    g, q = _instance(seed)
    og = oracle.OracleGraph(g)
    if oracle.count(og, q, limit=200_000) == oracle.ELIMIT:
        pytest.skip("too many embeddings")
    rows = oracle.match(og, q)
    G = ctx.load_graph(g)
    prev = None
    for stage in (0, 1, 2):
        c = ctx.candidates(G, q, stage)
        for u in range(q.k):
            assert c[u][rows[:, u]].all(), (stage, u)
        if prev is not None:
            assert not (c & ~prev).any()
        prev = c


@pytest.mark.parametrize("seed", range(0, 200, 3))
def test_filter_sets_equal_reference(gps, ctx, seed):
    """Candidate bitmaps after check / initialisation / refinement == tests/filter_ref.py exactly,
    and the visit order O == the reference planner's."""
    g, q = _instance(seed)
    G = ctx.load_graph(g)
    try:
        order, _ = ctx.plan(G, q)
    except Exception:
        pytest.skip("planner rejects the instance")
    assert order == filter_ref.plan(g, q)[0]
    for stage in (0, 1, 2):
        assert np.array_equal(ctx.candidates(G, q, stage), filter_ref.candidates(g, q, stage)), stage
    for rounds, rev, low in [(0, 1, 1), (2, 0, 2), (1, 1, 0)]:
        o = gps.default_opts(refine_rounds=rounds, reverse_refine=rev, lowconn_threshold=low)
        want = filter_ref.candidates(g, q, 2, refine_rounds=rounds, reverse_refine=bool(rev), lowconn_threshold=low)
        assert np.array_equal(ctx.candidates(G, q, 2, o), want), (rounds, rev, low)
    # the fixpoint version ("until convergence"): equal to the reference refined for so
    # many rounds that it no longer changes
    for rev in (1, 0):
        o = gps.default_opts(refine_rounds=UNTIL_STABLE, reverse_refine=rev)
        want = filter_ref.candidates(g, q, 2, refine_rounds=48, reverse_refine=bool(rev))
        assert np.array_equal(want, filter_ref.candidates(g, q, 2, refine_rounds=49, reverse_refine=bool(rev)))
        assert np.array_equal(ctx.candidates(G, q, 2, o), want), ("fixpoint", rev)


UNTIL_STABLE = 0xFFFFFFFF   # GPS_REFINE_UNTIL_STABLE


@pytest.mark.parametrize("rounds,rev,low", [(0, 1, 1), (1, 0, 1), (3, 1, 1), (1, 1, 0), (2, 0, 2),
                                            (UNTIL_STABLE, 1, 1), (UNTIL_STABLE, 0, 1)])
def test_refinement_variants_same_result(gps, ctx, rounds, rev, low):
    """P:997-1008 refinement variants change work, never the result."""
    for seed in (3, 11, 22, 40):
        g, q = _instance(seed)
        og = oracle.OracleGraph(g)
        if oracle.count(og, q, limit=500_000) == oracle.ELIMIT:
            continue
        o = gps.default_opts(refine_rounds=rounds, reverse_refine=rev, lowconn_threshold=low)
        _check(ctx, ctx.load_graph(g), og, q, o)


# ------------------------------------------------------------------ config 1
@pytest.fixture(scope="module")
def cfg1(ctx):
    g = config_graph(1)
    return g, ctx.load_graph(g), oracle.OracleGraph(g)


def test_cfg1_graph_layout(cfg1):
    g, G, og = cfg1
    assert G.n == 1000 and G.arcs == 10000 == og.arcs


@pytest.mark.parametrize("labels", [(-1, -1, -1, -1), (0, 1, 2, 3), (1, 1, 1, 1), (2, -1, 5, 2), (-1, 3, -1, 3),
                                    (7, 7, 0, -1)])
def test_cfg1_triangle_tail(ctx, cfg1, labels):
    g, G, og = cfg1
    _check(ctx, G, og, triangle_tail(labels))


def test_cfg1_label_partition(ctx, cfg1):
    """sum over the 8^4 labelled variants = all-'*' count (checked on the CUDA path, 512 variants sampled)."""
    g, G, og = cfg1
    rng = np.random.default_rng(5)
    for _ in range(64):
        lab = tuple(int(x) for x in rng.integers(0, 8, 4))
        assert ctx.count(G, triangle_tail(lab)) == oracle.count(og, triangle_tail(lab))


# ------------------------------------------------------------------ config 2
@pytest.fixture(scope="module")
def cfg2(ctx):
    path = os.path.join(ROOT, "synth", "data", "cfg2_queries.json")
    data = json.load(open(path))
    g = config_graph(2)
    return g, ctx.load_graph(g), data


def test_cfg2_graph_layout(cfg2):
    g, G, data = cfg2
    assert G.n == 300_000 and G.arcs == 1_500_000 and G.elabel_bits == 6


def test_cfg2_counts_all_queries(ctx, cfg2):
    """Full-size config 2 (the bench workload): gps_count == stored oracle count for all 100 queries."""
    g, G, data = cfg2
    for item in data["queries"]:
        q = Query.from_json(item["query"])
        assert ctx.count(G, q) == item["oracle_count"], item["seed"]


@pytest.mark.parametrize("env", ["GPS_SINGLE_PASS_BYTES=0", "GPS_NO_FAST_JOIN=1"])
def test_cfg2_other_join_paths(ctx, cfg2, env, monkeypatch):
    """Full-size config 2 through the look-back-tile join and the count -> write join."""
    monkeypatch.setenv("GPS_NO_FAST_JOIN", "1")
    k, v = env.split("=")
    monkeypatch.setenv(k, v)
    g, G, data = cfg2
    for item in data["queries"][:20]:
        assert ctx.count(G, Query.from_json(item["query"])) == item["oracle_count"], item["seed"]
    item = min(data["queries"], key=lambda d: d["oracle_count"])
    assert ctx.match(G, Query.from_json(item["query"])).shape[0] == item["oracle_count"]


def test_cfg2_match_sets(ctx, cfg2):
    """Full-size config 2: complete sorted-set equality for the queries the oracle enumerates quickly."""
    g, G, data = cfg2
    og = oracle.OracleGraph(g)
    small = sorted(data["queries"], key=lambda d: d["oracle_count"])[:12]
    big = max(data["queries"], key=lambda d: d["oracle_count"])
    for item in small + [big]:
        q = Query.from_json(item["query"])
        got = _rows(ctx.match(G, q))
        assert got.shape[0] == item["oracle_count"]
        assert np.array_equal(got, oracle.match(og, q))


# ---------------------------------------------------------------- edge cases
def test_single_vertex_query(ctx, cfg1):
    g, G, og = cfg1
    for lab in (-1, 3):
        _check(ctx, G, og, Query(1, [lab], [-1], []))
    _check(ctx, G, og, Query(1, [-1], [17], []))


def test_bound_vertices(ctx, cfg1):
    g, G, og = cfg1
    hub = int(np.bincount(np.concatenate([g.src, g.dst])).argmax())
    _check(ctx, G, og, Query(3, [-1, -1, -1], [hub, -1, -1], [(0, 1, -1), (1, 2, -1)]))
    _check(ctx, G, og, Query(3, [-1, -1, -1], [-1, hub, -1], [(0, 1, -1), (1, 2, -1), (2, 0, -1)]))


def test_empty_results(ctx, cfg1):
    g, G, og = cfg1
    assert ctx.count(G, triangle_tail((9, -1, -1, -1))) == 0          # label nobody has
    assert ctx.match(G, Query(2, [-1, -1], [-1, -1], [(0, 1, 3)])).shape == (0, 2)   # edge label absent
    assert ctx.count(G, Query(5, [-1] * 5, [-1] * 5,
                              [(i, j, -1) for i in range(5) for j in range(i + 1, 5)])) == \
        oracle.count(og, Query(5, [-1] * 5, [-1] * 5, [(i, j, -1) for i in range(5) for j in range(i + 1, 5)]))


def test_errors(gps, ctx, cfg1):
    g, G, og = cfg1
    with pytest.raises(gps.GpsError) as e:
        ctx.count(G, Query(3, [-1] * 3, [-1] * 3, [(0, 1, -1)]))
    assert e.value.status == gps.GPS_EDISCONNECTED
    with pytest.raises(gps.GpsError) as e:
        ctx.count(G, Query(2, [-1] * 2, [-1] * 2, [(0, 0, -1), (0, 1, -1)]))
    assert e.value.status == gps.GPS_EINVAL
    with pytest.raises(gps.GpsError) as e:
        ctx.count(G, Query(2, [-1] * 2, [5000, -1], [(0, 1, -1)]))
    assert e.value.status == gps.GPS_EINVAL
    with pytest.raises(gps.GpsError) as e:
        ctx.load_graph_csr(3, np.array([0, 1, 1, 5], np.uint64), np.array([1], np.uint32))
    assert e.value.status == gps.GPS_EINVAL
    with pytest.raises(gps.GpsError) as e:
        ctx.load_graph_csr(3, np.array([0, 1, 1, 1], np.uint64), np.array([7], np.uint32))
    assert e.value.status == gps.GPS_EINVAL


def test_parallel_arcs_and_duplicates(ctx):
    g = DataGraph(4, np.array([0, 0, 0, 1, 2, 2], np.uint32), np.array([1, 1, 1, 2, 0, 3], np.uint32),
                  np.array([0, 1, 1, 2, 0, 5], np.uint16), None, False)
    G = ctx.load_graph(g)
    og = oracle.OracleGraph(g)
    assert G.arcs == 5
    for q in [Query(2, [-1, -1], [-1, -1], [(0, 1, -1)]), Query(2, [-1, -1], [-1, -1], [(0, 1, 1)]),
              Query(2, [-1, -1], [-1, -1], [(0, 1, 0), (0, 1, 1)]),
              Query(3, [-1] * 3, [-1] * 3, [(0, 1, -1), (1, 2, -1), (2, 0, -1)]),
              Query(3, [-1] * 3, [-1] * 3, [(0, 1, -1), (1, 2, -1)])]:
        _check(ctx, G, og, q)


def test_graph_without_arcs(ctx):
    g = DataGraph(5, np.zeros(0, np.uint32), np.zeros(0, np.uint32), None, None, False)
    G = ctx.load_graph(g)
    assert G.arcs == 0
    assert ctx.count(G, Query(1, [-1], [-1], [])) == 5
    assert ctx.count(G, Query(2, [-1, -1], [-1, -1], [(0, 1, -1)])) == 0


def test_match_host_and_overflow(gps, ctx, cfg1):
    g, G, og = cfg1
    q = triangle_tail((1, -1, 2, -1))
    want = oracle.match(og, q)
    out = np.zeros((want.shape[0] + 5, 4), np.uint32)
    got = ctx.match_host(G, q, out)
    assert np.array_equal(oracle.sort_rows(np.array(got)), want)
    small = np.zeros((max(want.shape[0] - 1, 0), 4), np.uint32)
    with pytest.raises(gps.GpsError) as e:
        ctx.match_host(G, q, small)
    assert e.value.status == gps.GPS_EOVERFLOW
    host = ctx.match(G, q, device=False)
    assert np.array_equal(oracle.sort_rows(host), want)


def test_determinism(ctx, cfg1):
    g, G, og = cfg1
    q = triangle_tail()
    a = ctx.match(G, q).cpu().numpy()
    b = ctx.match(G, q).cpu().numpy()
    assert np.array_equal(a, b)   # row order is deterministic too (reading R25)


def test_stats_count_launches(ctx, cfg1):
    g, G, og = cfg1
    ctx.reset_stats()
    ctx.count(G, triangle_tail())
    st = ctx.stats()
    assert st["queries"] == 1 and st["launches"] > 5
    assert st["kernels"]["join_write"]["launches"] >= 1   # single-pass join steps count and write


# ------------------------------------------------------------ batched execution
def test_cfg2_match_batch(ctx, cfg2):
    """gps_match_batch (worker pool, concurrent streams) == stored oracle counts; sets for a sample."""
    g, G, data = cfg2
    qs = [Query.from_json(d["query"]) for d in data["queries"]]
    outs = ctx.match_batch(G, qs)
    assert len(outs) == len(qs)
    for t, d in zip(outs, data["queries"]):
        assert t.shape == (d["oracle_count"], 6)
    og = oracle.OracleGraph(g)
    small = sorted(range(len(qs)), key=lambda i: data["queries"][i]["oracle_count"])[:5]
    for i in small:
        assert np.array_equal(_rows(outs[i]), oracle.match(og, qs[i]))
    counts = ctx.count_batch(G, qs)
    assert counts.tolist() == [d["oracle_count"] for d in data["queries"]]


def test_batch_workers_and_errors(gps, ctx, cfg1):
    g, G, og = cfg1
    qs = [triangle_tail(lab) for lab in [(-1, -1, -1, -1), (0, 1, 2, 3), (1, -1, 2, -1)]] * 5
    for w in (1, 3, 8):
        ctx.set_workers(w)
        assert ctx.count_batch(G, qs).tolist() == [oracle.count(og, q) for q in qs]
    bad = qs[:2] + [Query(3, [-1] * 3, [-1] * 3, [(0, 1, -1)])]
    with pytest.raises(gps.GpsError) as e:
        ctx.count_batch(G, bad)
    assert e.value.status == gps.GPS_EDISCONNECTED
    ctx.set_workers(0)


def test_cfg2_match_batch_host(ctx, cfg2):
    """gps_match_batch_host: every result copied into one caller-owned host buffer."""
    g, G, data = cfg2
    qs = [Query.from_json(d["query"]) for d in data["queries"][:40]]
    want_rows = [d["oracle_count"] for d in data["queries"][:40]]
    buf = np.zeros(sum(r * 6 for r in want_rows) + 10, np.uint32)
    offs, rows = ctx.match_batch_host(G, qs, buf)
    assert rows.tolist() == want_rows
    og = oracle.OracleGraph(g)
    for i in sorted(range(40), key=lambda i: want_rows[i])[:4]:
        got = buf[int(offs[i]): int(offs[i]) + int(rows[i]) * 6].reshape(-1, 6)
        assert np.array_equal(oracle.sort_rows(got), oracle.match(og, qs[i]))
    br = ctx.match_batch_raw(G, qs[:5])
    assert br.rows().tolist() == want_rows[:5]
    t = br.tensor(0)
    assert t.shape == (want_rows[0], 6)
    br.free()


def test_recovers_after_allocation_failures(gps, ctx, cfg1, monkeypatch):
    """Every device-allocation failure path (GPS_FAULT_ALLOC=N fails the N-th allocation) reports
    GPS_ENOMEM and leaves the context usable: the next calls still give the oracle's answers
    (A27: GPS_ENOMEM is a reported resource error, never a corrupted context)."""
    g, G, og = cfg1
    q = triangle_tail()
    q2 = Query(4, [-1] * 4, [-1] * 4, [(0, 1, -1), (1, 2, -1), (2, 3, -1), (3, 0, -1)])   # closing edge
    want, want2 = oracle.match(og, q), oracle.count(og, q2)
    failed = 0
    for n in range(1, 80):
        monkeypatch.setenv("GPS_FAULT_ALLOC", str(n))
        try:
            ctx.match(G, q)
            ctx.count(G, q2)
            ctx.match_batch(G, [q, q2, q])
        except gps.GpsError as e:
            assert "ENOMEM" in str(e), e
            failed += 1
        monkeypatch.delenv("GPS_FAULT_ALLOC")
        assert np.array_equal(_rows(ctx.match(G, q)), want), n
        assert ctx.count(G, q2) == want2, n
    assert failed > 10   # the hook reached many allocation sites


def test_torch_caching_allocator(gps, cfg2):
    """gps_ctx_opts.dev_alloc / dev_free: with torch's caching allocator the
    library's device memory (scratch, tables, results) is torch memory -- results equal the
    oracle's, batch workers use it too, and a held result shows in torch.cuda.memory_allocated."""
    import torch
    c = gps.Context(0, torch_allocator=True)
    try:
        for seed in range(0, 200, 25):
            g, q = _instance(seed)
            og = oracle.OracleGraph(g)
            try:
                if oracle.count(og, q, limit=200_000) == oracle.ELIMIT:
                    continue
            except ValueError:
                continue
            _check(c, c.load_graph(g), og, q)
        g, G, data = cfg2[0], c.load_graph(cfg2[0]), cfg2[2]
        qs = [Query.from_json(d["query"]) for d in data["queries"][:12]]
        c.set_workers(2)
        c.set_slice(3)
        counts = c.count_batch(G, qs)
        assert counts.tolist() == [d["oracle_count"] for d in data["queries"][:12]]
        torch.cuda.synchronize()
        before = torch.cuda.memory_allocated(0)
        big = max(data["queries"], key=lambda d: d["oracle_count"])
        t = c.match(G, Query.from_json(big["query"]))
        torch.cuda.synchronize()
        assert t.shape[0] == big["oracle_count"]
        assert torch.cuda.memory_allocated(0) >= before + t.shape[0] * t.shape[1] * 4
        del t
    finally:
        c.close()


@pytest.mark.parametrize("k", [13, 16, 20, 24, 28, 32])
@pytest.mark.parametrize("induced", [False, True])
def test_large_queries_k13_to_32(gps, ctx, k, induced, monkeypatch):
    """Queries of 13-32 vertices (BFS trees and induced cyclic queries on the config-1 graph):
    rows of 13-32 columns exercise the wide-row join paths -- the k_join<2> single pass, the
    count -> exact allocation -> write path (GPS_SINGLE_PASS_BYTES=0) and the depth-first path
    under a 4 KB row budget -- each with full sorted-set equality with the oracle and the count."""
    g = config_graph(1)
    og = oracle.OracleGraph(g)
    q = bfs_query(g, k, seed=(200 if induced else 100), induced=induced, max_children=3)
    if oracle.count(og, q, limit=300_000) == oracle.ELIMIT:
        pytest.skip("too many embeddings for the oracle")
    G = ctx.load_graph(g)
    _check(ctx, G, og, q)
    _check(ctx, G, og, q, gps.default_opts(row_budget_bytes=4096))
    monkeypatch.setenv("GPS_SINGLE_PASS_BYTES", "0")
    _check(ctx, G, og, q)
