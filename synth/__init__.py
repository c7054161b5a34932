"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the CPU oracle.

This package holds NONE of the method's arithmetic (no candidate tests, no
filtering, no joining, no counting of embeddings).  It only draws graphs and
queries from seeded random generators and marshals them into the plain array
formats both sides accept (an edge list for the oracle, a CSR view for the C-ABI).
Recipes are documented in DESIGN.md §"Input recipe".
"""
from .graphs import (  # noqa: F401
    DataGraph,
    gnm_undirected,
    chung_lu_directed,
    chung_lu_directed_fast,
    random_multigraph,
    complete_graph,
    star_graph,
    config_graph,
)
from .queries import (  # noqa: F401
    Query,
    triangle_tail,
    bfs_query,
    fixture_fig3_example,
    random_connected_query,
    complete_query,
)
