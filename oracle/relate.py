"""f4 gSparql primitives on binary relations -- TEST INFRASTRUCTURE ONLY (the CPU oracle).

Only tests/ may import this module; it never imports the CUDA package and the CUDA
package never imports it.  Plain Python sets, following PAPER.md Ch. 4:

  * a property table holds the (subject, object) pairs of one predicate;
  * a subject/object join rule joins two property tables on a shared term:
    join(R, S) = {(x, z) : (x, y) in R, (y, z) in S};
  * a pattern node merges (unions) its rule nodes' results;
  * a recursive rule is applied until no new triple is derived (Algorithm),
    read as (DESIGN R37; the text's "NewT := T minus InferT" is read as InferT minus T):
        NewT := T
        while NewT not empty:
            InferT := apply_rule(NewT, T)
            NewT := InferT minus T
            T := T union NewT
    with apply_rule for the transitive rule (x p y), (y p z) -> (x p z) being
    join(NewT, T) union join(T, NewT).
Results are sets of pairs, returned as lexicographically sorted (rows, 2) uint32 arrays.
"""
from __future__ import annotations

import numpy as np


def _pairs(src, dst):
    return {(int(a), int(b)) for a, b in zip(np.asarray(src).tolist(), np.asarray(dst).tolist())}


def _arr(s):
    if not s:
        return np.zeros((0, 2), np.uint32)
    return np.array(sorted(s), np.uint32).reshape(-1, 2)


def join_set(R, S):
    by_first = {}
    for (y, z) in S:
        by_first.setdefault(y, []).append(z)
    return {(x, z) for (x, y) in R for z in by_first.get(y, ())}


def join(r_src, r_dst, s_src, s_dst) -> np.ndarray:
    """Subject/object join rule: {(x, z) : (x, y) in R, (y, z) in S}."""
    return _arr(join_set(_pairs(r_src, r_dst), _pairs(s_src, s_dst)))


def union(a_src, a_dst, b_src, b_dst) -> np.ndarray:
    return _arr(_pairs(a_src, a_dst) | _pairs(b_src, b_dst))


def difference(a_src, a_dst, b_src, b_dst) -> np.ndarray:
    return _arr(_pairs(a_src, a_dst) - _pairs(b_src, b_dst))


def closure(src, dst):
    """Transitive closure by the recursive-rule loop; returns (rows, iterations)."""
    T = _pairs(src, dst)
    new = set(T)
    it = 0
    while new:
        infer = join_set(new, T) | join_set(T, new)
        new = infer - T
        T = T | new
        it += 1
    return _arr(T), it
