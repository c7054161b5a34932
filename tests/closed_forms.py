"""Closed-form embedding counts for query families used at full scale (config 4).

Independent of the oracle and of the CUDA path: plain numpy over the arc list.
A wildcard query edge matches a data vertex PAIR (reading R5: parallel arcs with
different labels count once), so neighbour sets are built from distinct
(src, dst) pairs (optionally restricted to one edge label).

  out-star  c -> x1..xk, leaves with label l (or *), centre label lc (or *):
            sum_c [lc fits c] * P(|N_out_l(c)|, k)          P(d, k) = d (d-1) ... (d-k+1)
  in-star   x1..xk -> c: same with in-neighbours
  2-path    a -> b -> c with vertex labels (la, lb, lc):
            sum_b [lb fits b] |N_in_la(b)| |N_out_lc(b)| - #{(a, b): a -> b, b -> a, a fits la and lc, b fits lb}
"""
import numpy as np


def pair_keys(g, label=None):
    """Sorted distinct src * n + dst keys (restricted to one edge label if given)."""
    s = g.src.astype(np.int64)
    d = g.dst.astype(np.int64)
    if label is not None:
        sel = g.elab == label
        s, d = s[sel], d[sel]
    k = s * g.n + d
    k.sort()
    return k[np.concatenate([[True], k[1:] != k[:-1]])] if k.shape[0] else k


def _fits(g, lab):
    return np.ones(g.n, bool) if lab < 0 else (g.vlab == lab)


def falling(d, k):
    out = np.ones_like(d, dtype=np.float64)
    for i in range(k):
        out *= np.maximum(d - i, 0)
    return out


def out_star(g, keys, k, leaf_label=-1, centre_label=-1):
    s, d = keys // g.n, keys % g.n
    ok = _fits(g, leaf_label)[d]
    deg = np.bincount(s[ok], minlength=g.n).astype(np.float64)
    return int(round(float((falling(deg, k) * _fits(g, centre_label)).sum())))


def in_star(g, keys, k, leaf_label=-1, centre_label=-1):
    s, d = keys // g.n, keys % g.n
    ok = _fits(g, leaf_label)[s]
    deg = np.bincount(d[ok], minlength=g.n).astype(np.float64)
    return int(round(float((falling(deg, k) * _fits(g, centre_label)).sum())))


def path2(g, keys, la=-1, lb=-1, lc=-1):
    s, d = keys // g.n, keys % g.n
    fa, fb, fc = _fits(g, la), _fits(g, lb), _fits(g, lc)
    nin = np.bincount(d[fa[s]], minlength=g.n).astype(np.float64)
    nout = np.bincount(s[fc[d]], minlength=g.n).astype(np.float64)
    total = float((nin * nout * fb).sum())
    # subtract a == c: arcs a->b whose reverse b->a exists, a fits la and lc, b fits lb
    cand = fa[s] & fc[s] & fb[d]          # label filter first: only these arcs can close a == c
    rev = np.sort(d[cand] * g.n + s[cand])  # sorted needles: cache-friendly membership test
    pos = np.minimum(np.searchsorted(keys, rev), keys.shape[0] - 1)
    return int(round(total - float((keys[pos] == rev).sum())))
