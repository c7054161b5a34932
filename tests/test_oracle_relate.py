"""Pins of the f4 relation oracle (oracle/relate.py): the join equals a dense
boolean matrix product, the recursive-rule loop's result equals BFS reachability, its number of
rounds on a path of L arcs is ceil(log2 L) + 1 (semi-naive doubling, worked out by hand), and
union / difference equal numpy set operations."""
import math

import numpy as np
import pytest

from oracle import relate


def _rel(rng, n, m):
    return rng.integers(0, n, m).astype(np.uint32), rng.integers(0, n, m).astype(np.uint32)


@pytest.mark.parametrize("seed", range(20))
def test_join_is_boolean_matrix_product(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 20))
    rs, rd = _rel(rng, n, int(rng.integers(0, 3 * n)))
    ss, sd = _rel(rng, n, int(rng.integers(0, 3 * n)))
    A = np.zeros((n, n), np.int64)
    B = np.zeros((n, n), np.int64)
    A[rs, rd] = 1
    B[ss, sd] = 1
    want = np.argwhere((A @ B) > 0).astype(np.uint32)
    assert np.array_equal(relate.join(rs, rd, ss, sd), want.reshape(-1, 2))


def _bfs_closure(n, src, dst):
    adj = [[] for _ in range(n)]
    for a, b in zip(src.tolist(), dst.tolist()):
        adj[a].append(b)
    out = []
    for x in range(n):
        seen, stack = set(), list(adj[x])
        while stack:
            v = stack.pop()
            if v in seen:
                continue
            seen.add(v)
            stack.extend(adj[v])
        out += [(x, z) for z in sorted(seen)]
    return np.array(out, np.uint32).reshape(-1, 2)


@pytest.mark.parametrize("seed", range(20))
def test_closure_is_reachability(seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(2, 25))
    s, d = _rel(rng, n, int(rng.integers(0, 2 * n)))
    rows, _ = relate.closure(s, d)
    assert np.array_equal(rows, _bfs_closure(n, s, d))


@pytest.mark.parametrize("L", [1, 2, 3, 4, 5, 8, 9, 10, 16, 17, 33])
def test_closure_rounds_on_a_path(L):
    s = np.arange(L, dtype=np.uint32)
    rows, it = relate.closure(s, s + 1)
    assert rows.shape[0] == L * (L + 1) // 2
    assert it == math.ceil(math.log2(L)) + 1


@pytest.mark.parametrize("seed", range(10))
def test_union_difference_are_set_operations(seed):
    rng = np.random.default_rng(200 + seed)
    a = np.stack(_rel(rng, 8, 20), 1)
    b = np.stack(_rel(rng, 8, 20), 1)
    ka = a[:, 0].astype(np.int64) * 8 + a[:, 1]
    kb = b[:, 0].astype(np.int64) * 8 + b[:, 1]
    u = np.union1d(ka, kb)
    d = np.setdiff1d(ka, kb)
    assert np.array_equal(relate.union(a[:, 0], a[:, 1], b[:, 0], b[:, 1]), np.stack([u // 8, u % 8], 1).astype(np.uint32))
    assert np.array_equal(relate.difference(a[:, 0], a[:, 1], b[:, 0], b[:, 1]),
                          np.stack([d // 8, d % 8], 1).astype(np.uint32).reshape(-1, 2))
