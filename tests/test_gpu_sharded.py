"""Row-sharded join with several in-process ranks on one GPU.

Every rank (a thread with its own gps_ctx on a LocalComm) runs the same query;
the filter and edge candidates are replicated, the join's pair space is split,
per-step counts are all-gathered and rows are exchanged when unbalanced.  Checks:
gps_count is the GLOBAL count on every rank; the shards are disjoint and their
union (rank order) equals the oracle's embedding set -- for rebalancing forced
on every step (threshold 0), the default (1.10) and never (1e30).
"""
import json
import os
import threading

import numpy as np
import pytest

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


def _run_ranks(gps, world, g, fn):
    comm = gps.LocalComm(world)
    ctxs = [gps.Context(0, local_comm=comm, rank=r, world=world) for r in range(world)]
    graphs = [c.load_graph(g) for c in ctxs]
    out = [None] * world
    err = []

    def body(r):
        try:
            out[r] = fn(ctxs[r], graphs[r])
        except Exception as e:  # noqa: BLE001
            err.append(e)

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not err, err
    for c in ctxs:
        c.close()
    return out


def _queries():
    """cfg2 trees (smallest and largest results) and the smallest cyclic cfg3 queries."""
    d2 = json.load(open(os.path.join(ROOT, "synth", "data", "cfg2_queries.json")))["queries"]
    d3 = json.load(open(os.path.join(ROOT, "synth", "data", "cfg3_queries.json")))["queries"]
    picks = sorted(d2, key=lambda x: x["oracle_count"])
    cyc = [x for x in sorted(d3, key=lambda x: x["oracle_count"]) if x["oracle_count"] <= 300_000][:2]
    return [Query.from_json(x["query"]) for x in picks[:2] + picks[-2:] + cyc]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("thr", [0.0, 1.10, 1e30])
def test_sharded_cfg2_cfg3(gps, world, thr):
    g = config_graph(2)
    og = oracle.OracleGraph(g)
    qs = _queries()
    want = [oracle.match(og, q) for q in qs]
    o = gps.default_opts(rebalance_threshold=thr)

    def fn(ctx, G):
        res = []
        for q in qs:
            c = ctx.count(G, q, o)
            rows, glob = ctx.match_shard(G, q, o)
            res.append((c, rows, glob))
        return res

    out = _run_ranks(gps, world, g, fn)
    for i, w in enumerate(want):
        counts = {out[r][i][0] for r in range(world)}
        globs = {out[r][i][2] for r in range(world)}
        assert counts == {w.shape[0]} and globs == {w.shape[0]}
        shards = [out[r][i][1] for r in range(world)]
        union = np.concatenate(shards, axis=0)
        assert union.shape == w.shape
        assert np.array_equal(oracle.sort_rows(union), w)   # disjoint + complete


def test_sharded_cfg1(gps):
    g = config_graph(1)
    og = oracle.OracleGraph(g)
    qs = [triangle_tail(), triangle_tail((1, -1, 2, -1)), Query(1, [3], [-1], [])]
    want = [oracle.match(og, q) for q in qs]

    def fn(ctx, G):
        return [ctx.match_shard(G, q, gps.default_opts(rebalance_threshold=0.0)) for q in qs]

    out = _run_ranks(gps, 4, g, fn)
    for i, w in enumerate(want):
        union = np.concatenate([out[r][i][0] for r in range(4)], axis=0)
        assert np.array_equal(oracle.sort_rows(union), w)
        assert {out[r][i][1] for r in range(4)} == {w.shape[0]}


@pytest.mark.parametrize("world", [1, 2, 4])
def test_sharded_corpus_cyclic(gps, world):
    """Random-corpus instances (closing arcs, wildcards, bound vertices, undirected graphs),
    every step rebalanced (threshold 0): shards in rank order are disjoint and complete."""
    import corpus
    for seed in range(0, 200, 10):
        g, q = corpus.instance(seed)
        og = oracle.OracleGraph(g)
        try:
            if oracle.count(og, q, limit=200_000) == oracle.ELIMIT:
                continue
        except ValueError:
            continue
        w = oracle.match(og, q)

        def fn(ctx, G):
            o = gps.default_opts(rebalance_threshold=0.0)
            return ctx.count(G, q, o), ctx.match_shard(G, q, o)

        out = _run_ranks(gps, world, g, fn)
        assert {out[r][0] for r in range(world)} == {w.shape[0]}, seed
        union = np.concatenate([out[r][1][0] for r in range(world)], axis=0)
        assert np.array_equal(oracle.sort_rows(union), w), seed


NCCL_WORKER = r"""
import os, sys, json
sys.path.insert(0, {root!r})
import numpy as np, torch, torch.distributed as dist
from paper_1807_08804_b200 import gpsense as gps
from synth import config_graph, triangle_tail, Query
from oracle import oracle
local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
r, w = dist.get_rank(), dist.get_world_size()
backend = dist.group.WORLD._get_backend(torch.device("cuda", local))
ptr = backend._comm_ptr()
ctx = gps.Context(local, nccl_comm=ptr, rank=r, world=w)
g = config_graph(1)
G = ctx.load_graph(g)
og = oracle.OracleGraph(g)
qs = [triangle_tail(), triangle_tail((1, -1, 2, -1)),
      Query(4, [-1] * 4, [-1] * 4, [(0, 1, -1), (1, 2, -1), (2, 3, -1), (3, 0, -1)])]
res = []
for q in qs:
    want = oracle.match(og, q)
    for thr in (0.0, 1.10):
        o = gps.default_opts(rebalance_threshold=thr)
        c = ctx.count(G, q, o)
        rows, glob = ctx.match_shard(G, q, o)
        assert c == want.shape[0] and glob == want.shape[0], (c, glob, want.shape)
        if w == 1:
            assert np.array_equal(oracle.sort_rows(rows), want)
        res.append(int(rows.shape[0]))
ctx.close()
dist.destroy_process_group()
open(os.path.join({tmp!r}, "nccl%d" % r), "w").write(json.dumps(res))
"""


def test_nccl_backend_world1(gps, tmp_path):
    """The NCCL backend of the row-sharded join (ncclAllGather / grouped send-recv on the
    communicator torch created, ProcessGroupNCCL._comm_ptr()) executes for real: one rank,
    every step's collectives run, results equal the oracle's."""
    import socket
    import subprocess
    import sys
    script = tmp_path / "n.py"
    script.write_text(NCCL_WORKER.format(root=ROOT, tmp=str(tmp_path)))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(script)]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert (tmp_path / "nccl0").exists()
