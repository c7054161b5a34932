"""Config 4 at full size: 20M vertices, 100M labelled arcs (HBM-resident CSR, ~1 GB
per direction on the device) and joins of 10^7..10^9 embeddings.

Pins (independent of oracle and CUDA path): closed-form counts of labelled stars
and 2-paths (tests/closed_forms.py).  Written rows are checked on a random sample
against the data arcs and labels, and for pairwise-distinct vertices.
"""
import numpy as np
import pytest

import closed_forms as cf
from synth import config_graph
from synth.large import CFG4

pytestmark = pytest.mark.gpu


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


@pytest.mark.parametrize("i", [0, 2])
def test_cfg4_rows_valid_sample(env, i):
    import torch
    ctx, g, G, keys = env
    name, q, mode = CFG4[i]
    t = ctx.match(G, q)
    assert t.shape[0] == _closed(g, keys, name)
    rng = np.random.default_rng(i)
    idx = torch.as_tensor(rng.choice(t.shape[0], 4096, replace=False), device=t.device)
    rows = t.view(torch.int32)[idx].cpu().numpy().astype(np.int64)
    for u in range(q.k):
        if q.vlabels[u] >= 0:
            assert (g.vlab[rows[:, u]] == q.vlabels[u]).all()
        for v in range(u + 1, q.k):
            assert (rows[:, u] != rows[:, v]).all()
    for a, b, _ in q.edges:
        kk = rows[:, a] * g.n + rows[:, b]
        pos = np.minimum(np.searchsorted(keys, kk), keys.shape[0] - 1)
        assert (keys[pos] == kk).all()
    del t
