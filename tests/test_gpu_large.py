"""Config 4 at full size: 20M vertices, 100M labelled arcs (HBM-resident CSR, ~1 GB
per direction on the device) and joins of 10^7..10^9 embeddings.

Pins (independent of oracle and CUDA path): closed-form counts of labelled stars
and 2-paths (tests/closed_forms.py); every written row is checked against the data
arcs and labels, for injectivity and for distinctness (tests/rowcheck.py).  The cyclic
config-4 queries (synth/data/cfg4_queries.json) are checked against the oracle's stored
count and multiset hash.
"""
import json
import os

import numpy as np
import pytest

import closed_forms as cf
from synth import config_graph
from synth.large import CFG4

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1807_08804_b200 import gpsense
    ctx = gpsense.Context(0)
    g = config_graph(4)
    G = ctx.load_graph(g)
    keys = cf.pair_keys(g)
    yield ctx, g, G, keys
    ctx.close()


def _closed(g, keys, name):
    return {
        "out_star2_leaf0": lambda: cf.out_star(g, keys, 2, leaf_label=0),
        "in_star2_c0_leaf0": lambda: cf.in_star(g, keys, 2, leaf_label=0, centre_label=0),
        "path2_mid3": lambda: cf.path2(g, keys, -1, 3, -1),
        "out_star3_c0_leaf0": lambda: cf.out_star(g, keys, 3, leaf_label=0, centre_label=0),
    }[name]()


def test_cfg4_graph(env):
    ctx, g, G, keys = env
    assert G.n == 20_000_000 and G.arcs == 100_000_000


@pytest.mark.parametrize("i", range(len(CFG4)))
def test_cfg4_counts_closed_form(env, i):
    ctx, g, G, keys = env
    name, q, mode = CFG4[i]
    assert ctx.count(G, q) == _closed(g, keys, name)


@pytest.mark.parametrize("i", [0, 1, 2])
def test_cfg4_rows_all_valid_distinct(env, i):
    """Every written row of the closed-form joins (10^7..10^8 rows) is a valid embedding and
    no row repeats; with the closed-form count this is the full set."""
    import torch
    import rowcheck
    ctx, g, G, keys = env
    name, q, mode = CFG4[i]
    t = ctx.match(G, q)
    assert t.shape[0] == _closed(g, keys, name)
    x = t.view(torch.int32)
    assert rowcheck.all_distinct(x)
    assert rowcheck.all_valid(x, _ga(env, t.device), q)
    del t, x


def _ga(env, device):
    import rowcheck
    if not hasattr(_ga, "v"):
        _ga.v = rowcheck.GraphArrays(env[1], device)
    return _ga.v


def _cyclic():
    p = os.path.join(ROOT, "synth", "data", "cfg4_queries.json")
    return json.load(open(p))["queries"] if os.path.exists(p) else []


@pytest.mark.parametrize("i", range(len(_cyclic())))
def test_cfg4_cyclic_parity(env, i):
    """BASELINE configs[3] cyclic queries (oracle BFS-prefix tables >= 10^9 rows): gps_count
    equals the oracle's count (scripts/gen_queries_cfg4.py, OpenMP oracle on the GPU host);
    the gps_match rows have the oracle's multiset hash, are all valid embeddings and all
    distinct -- the oracle's set."""
    import torch
    import rowcheck
    from synth import Query
    ctx, g, G, keys = env
    d = _cyclic()[i]
    q = Query.from_json(d["query"])
    assert ctx.count(G, q) == d["oracle_count"]
    ctx.reset_stats()
    t = ctx.match(G, q)
    st = ctx.stats()
    assert t.shape == (d["oracle_count"], q.k)
    x = t.view(torch.int32)
    assert rowcheck.multiset_hash(x) == int(d["oracle_hash"])
    assert rowcheck.all_distinct(x)
    assert rowcheck.all_valid(x, _ga(env, t.device), q)
    print(f"cfg4 cyclic {i}: {d['oracle_count']} rows, join_rows_max {st['join_rows_max']}")
    del t, x
