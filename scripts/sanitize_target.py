"""Small workload for compute-sanitizer runs (memcheck / racecheck / synccheck / initcheck):
the worked example, cfg1 queries, corpus instances through every join path, a batch, the
row budget's depth-first path and 2 in-process ranks of the row-sharded join."""
import os, sys, threading
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import corpus
from oracle import oracle
from synth import config_graph, fixture_fig3_example, triangle_tail, Query
from paper_1807_08804_b200 import gpsense as gps

ctx = gps.Context(0)
nchk = 0


def check(G, og, q, o=None):
    global nchk
    want = oracle.match(og, q)
    got = oracle.sort_rows(ctx.match(G, q, o).cpu().numpy().astype(np.uint32))
    assert np.array_equal(got, want), (got.shape, want.shape)
    assert ctx.count(G, q, o) == want.shape[0]
    nchk += 1


g, q = fixture_fig3_example()
check(ctx.load_graph(g), oracle.OracleGraph(g), q)
g1 = config_graph(1)
G1, og1 = ctx.load_graph(g1), oracle.OracleGraph(g1)
for lab in [(-1, -1, -1, -1), (0, 1, 2, 3), (1, -1, 2, -1)]:
    check(G1, og1, triangle_tail(lab))
check(G1, og1, Query(4, [-1] * 4, [-1] * 4, [(0, 1, -1), (1, 2, -1), (2, 3, -1), (3, 0, -1)]))
seeds = [int(x) for x in os.environ.get("SEEDS", "0,3,4,9,12,17,22").split(",")]
for env in ({}, {"GPS_NO_FAST_JOIN": "1"}, {"GPS_SINGLE_PASS_BYTES": "256"}, {"GPS_SINGLE_PASS_BYTES": "0"}):
    os.environ.update(env)
    for s in seeds:
        g, q = corpus.instance(s)
        og = oracle.OracleGraph(g)
        if oracle.count(og, q, limit=50_000) == oracle.ELIMIT:
            continue
        G = ctx.load_graph(g)
        check(G, og, q)
        check(G, og, q, gps.default_opts(row_budget_bytes=2048))
        check(G, og, q, gps.default_opts(refine_rounds=0xFFFFFFFF))
    for k in env:
        del os.environ[k]
ctx.set_workers(2)
qs = [triangle_tail(lab) for lab in [(-1, -1, -1, -1), (0, 1, 2, 3), (1, -1, 2, -1)]] * 3
assert ctx.count_batch(G1, qs).tolist() == [oracle.count(og1, q) for q in qs]
outs = ctx.match_batch(G1, qs)
assert [t.shape[0] for t in outs] == [oracle.count(og1, q) for q in qs]
ctx.set_workers(0)
# 2 in-process ranks of the row-sharded join
comm = gps.LocalComm(2)
ctxs = [gps.Context(0, local_comm=comm, rank=r, world=2) for r in range(2)]
Gs = [c.load_graph(g1) for c in ctxs]
res = [None, None]
q = triangle_tail()


def body(r):
    res[r] = ctxs[r].match_shard(Gs[r], q, gps.default_opts(rebalance_threshold=0.0))


th = [threading.Thread(target=body, args=(r,)) for r in range(2)]
[t.start() for t in th]
[t.join() for t in th]
union = oracle.sort_rows(np.concatenate([res[0][0], res[1][0]]))
assert np.array_equal(union, oracle.match(og1, q))
# f2 named edges, f3 compression (attached), f4 relations
from oracle import compress as ocomp, relate  # noqa: E402
for s_ in seeds[:3]:
    g, q = corpus.instance(s_)
    og = oracle.OracleGraph(g)
    if oracle.count(og, q, limit=20_000) == oracle.ELIMIT:
        continue
    G = ctx.load_graph(g)
    ev = [i % 2 if l == -1 else -1 for i, (_, _, l) in enumerate(q.edges)]
    assert np.array_equal(ctx.match_named(G, q, ev), oracle.match_named(g, og, q, ev))
    cg = ctx.compress(G, [1.0, 1.0])
    cg.attach(2)
    check(G, og, q)
    cg.free()
rng = np.random.default_rng(1)
a, b = rng.integers(0, 30, 80).astype(np.uint32), rng.integers(0, 30, 80).astype(np.uint32)
assert np.array_equal(ctx.rel_join(a, b, b, a), relate.join(a, b, b, a))
assert np.array_equal(ctx.rel_closure(a, b)[0], relate.closure(a, b)[0])
os.environ["GPS_JOIN_NO_BULK"] = "1"
check(G1, og1, triangle_tail((-1, -1, -1, -1)))
del os.environ["GPS_JOIN_NO_BULK"]
print(f"sanitize target ok: {nchk} checked match+count pairs")
