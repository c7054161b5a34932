"""Seeded data-graph generators (no method arithmetic; see package docstring).

A DataGraph is a labelled directed multigraph given as an arc list
(src[i] -> dst[i] with edge label elab[i]) plus optional vertex labels.
`undirected=True` means "each listed edge is unordered": consumers symmetrise it
themselves (the C-ABI via GPS_UNDIRECTED, the oracle in its own loader).

Recipes:
  cfg1  G(n=1000, m=5000) uniform simple undirected, 8 uniform vertex labels
        (seeds 1807 graph / 1808 labels), no edge labels.
  cfg2  ConceptNet-shaped directed Chung-Lu: n=300,000, m=1,500,000 distinct
        labelled arcs, out-weights (i+i0)^(-1/(g_out-1)), in-weights
        (i+i0)^(-1/(g_in-1)), g_out=2.5, g_in=2.1, independent seeded
        permutations, no self-loops, 34 edge labels ~ Zipf(1.3), 16 uniform
        vertex labels (seed 8804).
  cfg4  same weights at n=20,000,000, m=100,000,000 (seed 100), drawn with the
        closed-form inverse of the continuous weight CDF (chung_lu_directed_fast).
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np


@dataclasses.dataclass
class DataGraph:
    n: int
    src: np.ndarray            # uint32 [m]
    dst: np.ndarray            # uint32 [m]
    elab: Optional[np.ndarray]  # uint16 [m] or None (all label 0)
    vlab: Optional[np.ndarray]  # uint16 [n] or None (all label 0)
    undirected: bool = False

    @property
    def m(self) -> int:
        return int(self.src.shape[0])

    def to_csr(self):
        """CSR view of the arc list exactly as listed (row order = stable by src).

        Pure marshalling for the C-ABI input (offsets u64 [n+1], targets u32,
        edge labels u16).  Rows are NOT sorted or de-duplicated here: that is the
        library's load step (a0).
        """
        order = np.argsort(self.src, kind="stable")
        targets = np.ascontiguousarray(self.dst[order], dtype=np.uint32)
        elab = None
        if self.elab is not None:
            elab = np.ascontiguousarray(self.elab[order], dtype=np.uint16)
        counts = np.bincount(self.src.astype(np.int64), minlength=self.n)
        offsets = np.zeros(self.n + 1, dtype=np.uint64)
        np.cumsum(counts, out=offsets[1:])
        return offsets, targets, elab

    def stats(self) -> dict:
        outdeg = np.bincount(self.src.astype(np.int64), minlength=self.n)
        indeg = np.bincount(self.dst.astype(np.int64), minlength=self.n)
        d = {"n": self.n, "m": self.m, "max_out": int(outdeg.max(initial=0)),
             "max_in": int(indeg.max(initial=0)), "undirected": self.undirected}
        if self.elab is not None:
            d["n_elabels"] = int(self.elab.max(initial=0)) + 1
        if self.vlab is not None:
            d["n_vlabels"] = int(self.vlab.max(initial=0)) + 1
        return d


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def gnm_undirected(n: int, m: int, n_vlabels: int = 8, seed: int = 1807,
                   label_seed: int = 1808) -> DataGraph:
    """Uniform simple undirected G(n, m): m distinct unordered pairs, no loops."""
    rng = np.random.default_rng(seed)
    keys = np.empty(0, dtype=np.int64)
    while keys.shape[0] < m:
        need = (m - keys.shape[0]) * 2 + 16
        a = rng.integers(0, n, size=need, dtype=np.int64)
        b = rng.integers(0, n, size=need, dtype=np.int64)
        ok = a != b
        lo, hi = np.minimum(a, b)[ok], np.maximum(a, b)[ok]
        cand = np.concatenate([keys, lo * n + hi])
        _, first = np.unique(cand, return_index=True)
        keys = cand[np.sort(first)]
    keys = keys[:m]
    vlab = None
    if n_vlabels > 0:
        vlab = np.random.default_rng(label_seed).integers(
            0, n_vlabels, size=n, dtype=np.int64).astype(np.uint16)
    return DataGraph(n=n, src=_u32(keys // n), dst=_u32(keys % n), elab=None,
                     vlab=vlab, undirected=True)


def _zipf_labels(rng, size, n_labels, s):
    p = 1.0 / np.arange(1, n_labels + 1, dtype=np.float64) ** s
    p /= p.sum()
    return rng.choice(n_labels, size=size, p=p).astype(np.uint16)


def chung_lu_directed(n: int, m: int, gamma_out: float = 2.5, gamma_in: float = 2.1,
                      n_elabels: int = 34, zipf_s: float = 1.3, n_vlabels: int = 16,
                      i0: float = 4.0, seed: int = 8804) -> DataGraph:
    """Directed Chung-Lu power-law graph with m distinct (src, dst, label) arcs.

    src ~ w_out, dst ~ w_in with w_i = (i+i0)^(-1/(gamma-1)) applied through
    independent random permutations of the vertex ids; self-loops rejected;
    duplicate (src, dst, label) triples dropped (first draw wins), topped up
    until exactly m arcs remain.
    """
    rng = np.random.default_rng(seed)
    idx = np.arange(n, dtype=np.float64)
    w_out = (idx + i0) ** (-1.0 / (gamma_out - 1.0))
    w_in = (idx + i0) ** (-1.0 / (gamma_in - 1.0))
    c_out = np.cumsum(w_out); c_out /= c_out[-1]
    c_in = np.cumsum(w_in); c_in /= c_in[-1]
    perm_out = rng.permutation(n).astype(np.int64)
    perm_in = rng.permutation(n).astype(np.int64)
    zp = 1.0 / np.arange(1, n_elabels + 1, dtype=np.float64) ** zipf_s
    c_lab = np.cumsum(zp); c_lab /= c_lab[-1]
    L = np.int64(max(n_elabels, 1))
    keys = np.empty(0, dtype=np.int64)
    while keys.shape[0] < m:
        need = int((m - keys.shape[0]) * 1.15) + 1024
        s = perm_out[np.minimum(np.searchsorted(c_out, rng.random(need)), n - 1)]
        d = perm_in[np.minimum(np.searchsorted(c_in, rng.random(need)), n - 1)]
        lab = np.minimum(np.searchsorted(c_lab, rng.random(need)), n_elabels - 1).astype(np.int64)
        ok = s != d
        cand = np.concatenate([keys, (s[ok] * n + d[ok]) * L + lab[ok]])
        _, first = np.unique(cand, return_index=True)
        keys = cand[np.sort(first)]
    keys = keys[:m]
    lab = (keys % L).astype(np.uint16)
    sd = keys // L
    vlab = rng.integers(0, n_vlabels, size=n, dtype=np.int64).astype(np.uint16) if n_vlabels > 0 else None
    return DataGraph(n=n, src=_u32(sd // n), dst=_u32(sd % n),
                     elab=lab if n_elabels > 1 else None, vlab=vlab, undirected=False)


def chung_lu_directed_fast(n: int, m: int, gamma_out: float = 2.5, gamma_in: float = 2.1,
                           n_elabels: int = 34, zipf_s: float = 1.3, n_vlabels: int = 16,
                           i0: float = 4.0, seed: int = 100) -> DataGraph:
    """Large-scale variant of chung_lu_directed (config 4: 20M vertices, 100M arcs).

    Same weights w_i = (i+i0)^(-a), a = 1/(gamma-1), but ranks are drawn by
    inverting the CONTINUOUS approximation of the weight CDF (closed form, O(1)
    per draw) instead of a binary search in the exact discrete CDF, and the
    duplicate (src, dst, label) triples of a 1.04 m oversample are removed by one
    sort, the survivors subsampled to exactly m arcs.  Seeded; no self-loops.
    """
    rng = np.random.default_rng(seed)

    def draw(size, gamma):
        a = 1.0 / (gamma - 1.0)
        e = 1.0 - a                      # a != 1 for gamma != 2
        lo = i0 ** e
        hi = (n + i0) ** e
        u = rng.random(size)
        x = (lo + u * (hi - lo)) ** (1.0 / e) - i0
        return np.minimum(x.astype(np.int64), n - 1)

    perm_out = rng.permutation(n).astype(np.int64)
    perm_in = rng.permutation(n).astype(np.int64)
    zp = 1.0 / np.arange(1, n_elabels + 1, dtype=np.float64) ** zipf_s
    c_lab = np.cumsum(zp)
    c_lab /= c_lab[-1]
    L = np.int64(max(n_elabels, 1))
    keys = np.empty(0, dtype=np.int64)
    while keys.shape[0] < m:
        need = int((m - keys.shape[0]) * 1.04) + 1024
        sv = perm_out[draw(need, gamma_out)]
        dv = perm_in[draw(need, gamma_in)]
        lab = np.minimum(np.searchsorted(c_lab, rng.random(need)), n_elabels - 1).astype(np.int64)
        ok = sv != dv
        keys = np.concatenate([keys, (sv[ok] * n + dv[ok]) * L + lab[ok]])
        keys.sort()   # de-duplicate by one sort (np.unique's hashing path is slow at 10^8)
        keys = keys[np.concatenate([[True], keys[1:] != keys[:-1]])]
    if keys.shape[0] > m:
        keys = np.sort(rng.choice(keys, size=m, replace=False))
    lab = (keys % L).astype(np.uint16)
    sd = keys // L
    vlab = rng.integers(0, n_vlabels, size=n, dtype=np.int64).astype(np.uint16) if n_vlabels > 0 else None
    return DataGraph(n=n, src=_u32(sd // n), dst=_u32(sd % n),
                     elab=lab if n_elabels > 1 else None, vlab=vlab, undirected=False)


def random_multigraph(n: int, m: int, n_elabels: int, n_vlabels: int, seed: int,
                      undirected: bool = False, self_loops: bool = True,
                      dup_prob: float = 0.1) -> DataGraph:
    """Tiny/small random directed labelled multigraph for oracle pins and parity.

    Arcs drawn uniformly; with probability dup_prob an arc is repeated with
    another label (parallel arcs), and exact duplicates may occur (set semantics
    must absorb them).  Self-loops allowed when self_loops=True.
    """
    rng = np.random.default_rng(seed)
    s = rng.integers(0, n, size=m)
    d = rng.integers(0, n, size=m)
    if not self_loops:
        ok = s != d
        s, d = s[ok], d[ok]
    lab = rng.integers(0, max(n_elabels, 1), size=s.shape[0])
    extra = rng.random(s.shape[0]) < dup_prob
    s = np.concatenate([s, s[extra]])
    d = np.concatenate([d, d[extra]])
    lab = np.concatenate([lab, rng.integers(0, max(n_elabels, 1), size=int(extra.sum()))])
    vlab = rng.integers(0, n_vlabels, size=n).astype(np.uint16) if n_vlabels > 0 else None
    return DataGraph(n=n, src=_u32(s), dst=_u32(d),
                     elab=lab.astype(np.uint16) if n_elabels > 1 else None,
                     vlab=vlab, undirected=undirected)


def complete_graph(n: int) -> DataGraph:
    """Undirected K_n, unlabelled."""
    a, b = np.triu_indices(n, 1)
    return DataGraph(n=n, src=_u32(a), dst=_u32(b), elab=None, vlab=None, undirected=True)


def star_graph(m: int) -> DataGraph:
    """Undirected star S_m: centre 0 with leaves 1..m, unlabelled."""
    return DataGraph(n=m + 1, src=_u32(np.zeros(m)), dst=_u32(np.arange(1, m + 1)),
                     elab=None, vlab=None, undirected=True)


def config_graph(cfg: int, scale: float = 1.0) -> DataGraph:
    """The data graph of BASELINE.json config `cfg` (1-based).

    scale < 1 shrinks n and m proportionally (same recipe, same seed) for
    quick tests; the bench always uses scale=1.
    """
    if cfg == 1:
        return gnm_undirected(int(1000 * scale), int(5000 * scale), 8, 1807, 1808)
    if cfg in (2, 3, 5):
        return chung_lu_directed(int(300_000 * scale), int(1_500_000 * scale), seed=8804)
    if cfg == 4:
        return chung_lu_directed_fast(int(20_000_000 * scale), int(100_000_000 * scale), seed=100)
    raise ValueError(f"unknown config {cfg}")
