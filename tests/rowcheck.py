"""Device-side checks of large embedding sets (test infrastructure, plain torch ops).

Used where a full host-side sorted-set comparison is too large (configs 3 and 4, up to
10^8 rows): SURVEY §8(d) "an order-independent 64-bit multiset hash (sum of splitmix64
of the rows mod 2^64) as a fast pre-check", plus checks that hold at any size:
  * multiset_hash(rows) -- the same row hash as oracle.c row_hash (pinned against the
    pure-Python restatement in tests/test_rowcheck.py), summed mod 2^64;
  * all_distinct(rows)  -- exact: lexicographic sort by stable per-column sorts, then no
    two neighbours equal;
  * all_valid(rows, graph arrays, query) -- every row is an embedding by Def. 2
    (P:605-607): injective, vertex labels, bound vertices, every query arc present in
    the data with a fitting label.
With the oracle's count and hash, valid + distinct + equal count + equal hash establishes
the set (a wrong row fails validity; a missing row changes the count or the hash).
Shares no code with the CUDA library or the oracle.
"""
from __future__ import annotations

import numpy as np
import torch

_M64 = (1 << 64) - 1


def _s64(c: int) -> int:
    """Unsigned 64-bit constant as the int64 torch stores."""
    return c - (1 << 64) if c >= 1 << 63 else c


_C1, _C2, _C3 = _s64(0x9E3779B97F4A7C15), _s64(0xBF58476D1CE4E5B9), _s64(0x94D049BB133111EB)
_SEED = 0x243F6A8885A308D3


def _shr(x: torch.Tensor, s: int) -> torch.Tensor:
    """Logical right shift of int64 (torch's >> is arithmetic)."""
    return (x >> s) & ((1 << (64 - s)) - 1)


def _splitmix64(x: torch.Tensor) -> torch.Tensor:
    z = x + _C1
    z = (z ^ _shr(z, 30)) * _C2
    z = (z ^ _shr(z, 27)) * _C3
    return z ^ _shr(z, 31)


def multiset_hash(rows: torch.Tensor, chunk: int = 1 << 24) -> int:
    """Sum over rows of row_hash (oracle.c) mod 2^64.  rows: (R, k) uint32/int32 tensor."""
    R, k = rows.shape
    total = 0
    for a in range(0, R, chunk):
        blk = rows[a:a + chunk].to(torch.int64) & 0xFFFFFFFF
        h = torch.full((blk.shape[0],), _s64(_SEED ^ k), dtype=torch.int64, device=rows.device)
        for j in range(k):
            h = _splitmix64(h ^ blk[:, j])
        total = (total + int(h.sum().item())) & _M64
    return total


def all_distinct(rows: torch.Tensor) -> bool:
    R, k = rows.shape
    if R < 2:
        return True
    x = rows.to(torch.int64) & 0xFFFFFFFF
    perm = torch.arange(R, device=rows.device)
    for j in range(k - 1, -1, -1):   # LSD: stable sort by each column from the last
        _, o = torch.sort(x[perm, j], stable=True)
        perm = perm[o]
    s = x[perm]
    same = (s[1:] == s[:-1]).all(dim=1)
    return not bool(same.any().item())


class GraphArrays:
    """The data arcs as sorted device keys (built from the raw arc list, not from a CSR of
    the library): key = (src*n + dst) for wildcard arcs, key*L + label for labelled ones."""

    def __init__(self, g, device):
        n = int(g.n)
        s = torch.as_tensor(np.asarray(g.src, np.int64), device=device)
        d = torch.as_tensor(np.asarray(g.dst, np.int64), device=device)
        lab = (torch.as_tensor(np.asarray(g.elab, np.int64), device=device) if g.elab is not None
               else torch.zeros_like(s))
        if g.undirected:
            s, d, lab = torch.cat([s, d]), torch.cat([d, s]), torch.cat([lab, lab])
        self.n = n
        self.L = int(lab.max().item()) + 1 if lab.numel() else 1
        self.pairs = torch.unique(s * n + d)
        self.labelled = torch.unique((s * n + d) * self.L + lab)
        self.vlab = (torch.as_tensor(np.asarray(g.vlab, np.int64), device=device) if g.vlab is not None
                     else torch.zeros(n, dtype=torch.int64, device=device))


def _member(sorted_keys: torch.Tensor, x: torch.Tensor) -> torch.Tensor:
    i = torch.searchsorted(sorted_keys, x).clamp(max=sorted_keys.numel() - 1)
    return sorted_keys[i] == x


def all_valid(rows: torch.Tensor, ga: GraphArrays, q, chunk: int = 1 << 24) -> bool:
    R, k = rows.shape
    assert k == q.k
    for a0 in range(0, R, chunk):
        x = rows[a0:a0 + chunk].to(torch.int64) & 0xFFFFFFFF
        if (x >= ga.n).any():
            return False
        for u in range(k):
            if q.vlabels[u] >= 0 and not bool((ga.vlab[x[:, u]] == q.vlabels[u]).all()):
                return False
            if q.bound[u] >= 0 and not bool((x[:, u] == q.bound[u]).all()):
                return False
            for v in range(u + 1, k):
                if bool((x[:, u] == x[:, v]).any()):
                    return False
        for a, b, lab in q.edges:
            key = x[:, a] * ga.n + x[:, b]
            ok = _member(ga.pairs, key) if lab < 0 else _member(ga.labelled, key * ga.L + lab)
            if not bool(ok.all()):
                return False
    return True
