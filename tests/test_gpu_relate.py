"""f4 gSparql primitives on the device against the
relation oracle (oracle/relate.py): join, union, difference and the recursive-rule closure
(rows and round count) equal element by element, on random relations (duplicates, self
pairs, empty sides) and on a larger power-law relation taken from the config-2 graph."""
import numpy as np
import pytest

from oracle import relate
from synth import config_graph

pytestmark = pytest.mark.gpu


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


def _rel(rng, n, m):
    return rng.integers(0, n, m).astype(np.uint32), rng.integers(0, n, m).astype(np.uint32)


@pytest.mark.parametrize("seed", range(30))
def test_join_union_difference(gps, ctx, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 60))
    rs, rd = _rel(rng, n, int(rng.integers(0, 4 * n)))
    ss, sd = _rel(rng, n, int(rng.integers(0, 4 * n)))
    if seed % 7 == 0:   # large term ids (the high bits of the packed keys)
        rs, sd = rs + np.uint32(0xfffff000), sd + np.uint32(0xfffff000)
        rd = rd.copy()
    assert np.array_equal(ctx.rel_join(rs, rd, ss, sd), relate.join(rs, rd, ss, sd))
    assert np.array_equal(ctx.rel_union(rs, rd, ss, sd), relate.union(rs, rd, ss, sd))
    assert np.array_equal(ctx.rel_difference(rs, rd, ss, sd), relate.difference(rs, rd, ss, sd))


@pytest.mark.parametrize("seed", range(20))
def test_closure(gps, ctx, seed):
    rng = np.random.default_rng(500 + seed)
    n = int(rng.integers(1, 80))
    s, d = _rel(rng, n, int(rng.integers(0, 2 * n)))
    got, it = ctx.rel_closure(s, d)
    want, wit = relate.closure(s, d)
    assert np.array_equal(got, want)
    assert it == wit


def test_closure_path_and_bound(gps, ctx):
    s = np.arange(100, dtype=np.uint32)
    rows, it = ctx.rel_closure(s, s + 1)
    assert rows.shape[0] == 100 * 101 // 2 and it == 8       # ceil(log2 100) + 1
    with pytest.raises(gps.GpsError):
        ctx.rel_closure(s, s + 1, max_rounds=3)
    e = np.zeros(0, np.uint32)
    assert ctx.rel_join(e, e, s, s).shape == (0, 2)
    assert ctx.rel_closure(e, e)[0].shape == (0, 2)


def test_config2_relation(gps, ctx):
    """A power-law relation: the arcs among the 1,000 highest-degree vertices of the config-2
    graph (38K pairs; closure 155K pairs in 6 rounds) -- join with itself and closure."""
    g = config_graph(2)
    deg = np.bincount(g.src, minlength=g.n) + np.bincount(g.dst, minlength=g.n)
    top = np.zeros(g.n, bool)
    top[np.argsort(-deg, kind="stable")[:1000]] = True
    sel = top[g.src] & top[g.dst]
    s, d = g.src[sel], g.dst[sel]
    assert np.array_equal(ctx.rel_join(s, d, s, d), relate.join(s, d, s, d))
    got, it = ctx.rel_closure(s, d)
    want, wit = relate.closure(s, d)
    assert np.array_equal(got, want) and it == wit
