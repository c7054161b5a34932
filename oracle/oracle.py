"""ctypes wrapper around oracle.c -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module.  It never imports the CUDA package and
the CUDA package never imports it.  See oracle.c for what is computed and the
PAPER.md passages it follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

EINVAL, EDISCONNECTED, ELIMIT, ENOMEM = -1, -2, -3, -4


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        lib.oracle_graph_build.restype = P
        lib.oracle_graph_build.argtypes = [ctypes.c_uint32, ctypes.c_uint64, P, P, P, P, ctypes.c_int]
        lib.oracle_graph_free.argtypes = [P]
        lib.oracle_graph_arcs.restype = ctypes.c_uint64
        lib.oracle_graph_arcs.argtypes = [P]
        lib.oracle_match.restype = ctypes.c_int64
        lib.oracle_match.argtypes = [P, ctypes.c_uint32, P, P, ctypes.c_uint32, P, P, P, P,
                                     ctypes.c_uint64, ctypes.c_uint64]
        lib.oracle_set_work_limit.argtypes = [ctypes.c_uint64]
        lib.oracle_run.restype = None
        lib.oracle_run.argtypes = [P, ctypes.c_uint32, P, P, ctypes.c_uint32, P, P, P, ctypes.c_uint32,
                                   ctypes.c_uint32, ctypes.c_uint32, P, ctypes.c_uint64, ctypes.c_uint64, P]
        _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class OracleGraph:
    """The oracle's own adjacency, built from the raw edge list (never a CSR
    produced by the CUDA path)."""

    def __init__(self, g):
        lib = _load()
        self._keep = [np.ascontiguousarray(g.src, np.uint32), np.ascontiguousarray(g.dst, np.uint32),
                      None if g.elab is None else np.ascontiguousarray(g.elab, np.uint16),
                      None if g.vlab is None else np.ascontiguousarray(g.vlab, np.uint16)]
        s, d, el, vl = self._keep
        self.n = int(g.n)
        self._h = lib.oracle_graph_build(self.n, s.shape[0], _ptr(s), _ptr(d), _ptr(el), _ptr(vl),
                                         1 if g.undirected else 0)
        if not self._h:
            raise ValueError("oracle_graph_build rejected the input")
        self._keep = None

    @property
    def arcs(self) -> int:
        return int(_load().oracle_graph_arcs(self._h))

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.oracle_graph_free(self._h)
            self._h = None


def _qarrays(q):
    vl = np.array(q.vlabels, np.int32)
    bd = np.array(q.bound, np.int64)
    e = np.array(q.edges, np.int32).reshape(-1, 3)
    return vl, bd, np.ascontiguousarray(e[:, 0]), np.ascontiguousarray(e[:, 1]), np.ascontiguousarray(e[:, 2])


def set_work_limit(tries: int) -> None:
    """Abort searches after `tries` candidate tests (ELIMIT); 0 = unlimited.  Acceptance scripts only."""
    _load().oracle_set_work_limit(int(tries))


def count(og: OracleGraph, q, limit: int = 0) -> int:
    """#Emb(Q, G); raises on error, returns -3 (ELIMIT) when count > limit > 0."""
    vl, bd, a, b, lab = _qarrays(q)
    r = _load().oracle_match(og._h, q.k, _ptr(vl), _ptr(bd), a.shape[0], _ptr(a), _ptr(b), _ptr(lab),
                             None, 0, limit)
    if r < 0 and r != ELIMIT:
        raise ValueError(f"oracle error {r}")
    return int(r)


def match(og: OracleGraph, q, limit: int = 0) -> np.ndarray:
    """All embeddings as a lexicographically sorted (R, k) uint32 array."""
    c = count(og, q, limit)
    if c == ELIMIT:
        raise OverflowError("more than %d embeddings" % limit)
    rows = np.zeros((max(c, 1), q.k), np.uint32)
    vl, bd, a, b, lab = _qarrays(q)
    r = _load().oracle_match(og._h, q.k, _ptr(vl), _ptr(bd), a.shape[0], _ptr(a), _ptr(b), _ptr(lab),
                             _ptr(rows), c, 0)
    assert r == c
    rows = rows[:c]
    return sort_rows(rows)


def sort_rows(rows: np.ndarray) -> np.ndarray:
    """Lexicographic row sort (plain numpy; used to compare sets of rows)."""
    rows = np.ascontiguousarray(rows)
    if rows.shape[0] == 0:
        return rows
    order = np.lexsort(rows.T[::-1])
    return rows[order]


class _Result(ctypes.Structure):
    _fields_ = [("count", ctypes.c_int64), ("hash", ctypes.c_uint64), ("level", ctypes.c_uint64 * 32),
                ("pi", ctypes.c_uint32 * 32), ("threads", ctypes.c_uint32)]


def run(og: OracleGraph, q, threads: int = 1, col0_range=None, rows: bool = False, limit: int = 0,
        cap: int = 0) -> dict:
    """One oracle search with its bookkeeping (oracle.c oracle_run).

    threads > 1: the OpenMP timing variant (same result).  col0_range=(lo, hi): only
    embeddings whose image of query vertex 0 lies in [lo, hi).  rows=True also returns
    the sorted rows (cap rows at most: pass the count from a first run).  Returns
    dict(count, hash (multiset hash, see oracle.c row_hash), levels (#partial maps per
    BFS depth), order (the BFS order), threads, rows (if asked)).  count = ELIMIT when
    the search was cut by `limit` / the work limit."""
    lib = _load()
    vl, bd, a, b, lab = _qarrays(q)
    res = _Result()
    lo, hi = (0, 0) if col0_range is None else (int(col0_range[0]), int(col0_range[1]))
    if col0_range is not None and hi <= lo:
        out = dict(count=0, hash=0, levels=[0] * q.k, order=[], threads=threads)
        if rows:
            out["rows"] = np.zeros((0, q.k), np.uint32)
        return out
    buf = np.zeros((max(cap, 1), q.k), np.uint32) if rows else None
    lib.oracle_run(og._h, q.k, _ptr(vl), _ptr(bd), a.shape[0], _ptr(a), _ptr(b), _ptr(lab), int(threads),
                   lo, hi, _ptr(buf), cap if rows else 0, int(limit), ctypes.byref(res))
    c = int(res.count)
    if c < 0 and c != ELIMIT:
        raise ValueError(f"oracle error {c}")
    out = dict(count=c, hash=int(res.hash), levels=[int(res.level[i]) for i in range(q.k)],
               order=[int(res.pi[i]) for i in range(q.k)], threads=int(res.threads))
    if rows:
        if c > cap:
            raise OverflowError(f"{c} rows > cap {cap}")
        out["rows"] = sort_rows(buf[:max(c, 0)])
    return out


_M64 = (1 << 64) - 1


def _splitmix64(x: int) -> int:
    z = (x + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def row_hash_py(row) -> int:
    """Pure-Python restatement of oracle.c row_hash (for pinning it)."""
    h = 0x243F6A8885A308D3 ^ len(row)
    for v in row:
        h = _splitmix64(h ^ int(v))
    return h


def multiset_hash_py(rows) -> int:
    return sum(row_hash_py(r) for r in rows) & _M64


def match_named(g, og: OracleGraph, q, edge_var, project=None) -> np.ndarray:
    """Named variable edges (f2; "each variable-edge name as a binding reported in
    output, with equal names constrained equal"; DESIGN reading R32).  edge_var[e] >= 0 names
    query edge e (its label must be ANY), -1 leaves it unnamed.

    Plain definition: the set of tuples (f(project...), beta(v_0), beta(v_1), ...) -- the
    variables v_i in increasing id order -- over every embedding f (Def. 2, with the
    named edges as variable edges) and every assignment beta of labels to the variables
    such that each edge e = (a, b) named v has an arc f(a) -> f(b) labelled beta(v).  Rows are
    distinct and lexicographically sorted.  The arc labels come from the raw edge list g."""
    import itertools
    edges = [tuple(e) for e in q.edges]
    if len(edge_var) != len(edges):
        raise ValueError("edge_var needs one entry per query edge")
    names = sorted({int(v) for v in edge_var if v >= 0})
    for e, v in zip(edges, edge_var):
        if v >= 0 and e[2] != -1:
            raise ValueError("a named edge must be a variable (ANY) edge")
    proj = list(range(q.k)) if project is None else [int(x) for x in project]
    labels = {}   # (a, b) -> set of arc labels, from the raw edge list
    el = np.zeros(len(g.src), np.int64) if g.elab is None else np.asarray(g.elab, np.int64)
    for s, d, l in zip(np.asarray(g.src, np.int64), np.asarray(g.dst, np.int64), el):
        labels.setdefault((int(s), int(d)), set()).add(int(l))
        if g.undirected:
            labels.setdefault((int(d), int(s)), set()).add(int(l))
    out = set()
    for f in match(og, q):
        choices = []
        for v in names:
            s = None
            for (a, b, _), ev in zip(edges, edge_var):
                if ev == v:
                    ls = labels.get((int(f[a]), int(f[b])), set())
                    s = set(ls) if s is None else s & ls
            choices.append(sorted(s))
        head = tuple(int(f[c]) for c in proj)
        for beta in itertools.product(*choices):
            out.add(head + beta)
    width = len(proj) + len(names)
    if not out:
        return np.zeros((0, width), np.uint32)
    return np.array(sorted(out), np.uint32).reshape(-1, width)
