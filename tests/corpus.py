"""Seeded random instances of the S:499 acceptance corpus (shared by CPU and GPU tests).

Only draws inputs (synth generators); no matching arithmetic.
"""
import numpy as np

from synth import bfs_query, random_connected_query, random_multigraph


def instance(seed):
    rng = np.random.default_rng(10_000 + seed)
    n = int(rng.integers(20, 301))
    deg = float(rng.uniform(1.5, 8.0))
    undirected = seed % 4 == 0
    g = random_multigraph(n, int(n * deg / (2 if undirected else 1)), n_elabels=int(rng.integers(1, 5)),
                          n_vlabels=int(rng.integers(1, 21)), seed=seed, undirected=undirected,
                          self_loops=seed % 3 == 0, dup_prob=0.1)
    k = int(rng.integers(4, 9))
    if seed % 5 == 4:
        q = random_connected_query(rng, min(k, 6), extra=int(rng.integers(0, 4)),
                                   n_elabels=int(g.elab.max()) + 1 if g.elab is not None else 1,
                                   n_vlabels=int(g.vlab.max()) + 1, p_wild_v=0.6, p_wild_e=0.6,
                                   bound_choices=list(range(n)), p_bound=0.1)
    else:
        q = bfs_query(g, min(k, n), seed, induced=seed % 2 == 0, p_wild_v=float(rng.uniform(0, 1)),
                      keep_elabels=seed % 3 != 1, bind_seed=seed % 7 == 3, max_children=int(rng.integers(0, 3)))
    return g, q
