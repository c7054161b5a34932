"""f1: refinement ablation on large synthetic cyclic queries (16 and 20 vertices).

The thesis reports that without refinement the joining phase needs "up to 150 times" more
intermediate memory on 20-vertex queries.  Here: N seeded BFS queries of 16 / 20
vertices from the dense core of the config-2 graph (induced arcs, wildcard edge labels, data
vertex labels kept), gps_count under each refinement variant; per query the intermediate rows
written by all join steps (join_rows_total) and the largest table (join_rows_max).  Counts must
agree across variants (refinement only prunes candidates that are in no embedding).
  python scripts/ablation_refine20.py [N]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from synth import bfs_query, config_graph  # noqa: E402
from paper_1807_08804_b200 import gpsense  # noqa: E402

# the four versions of P:1008 (until convergence; until convergence reversed; one round reversed --
# the default; none) plus one round forward
VARIANTS = [("none", dict(refine_rounds=0)), ("1 round reversed (default)", dict(refine_rounds=1, reverse_refine=1)),
            ("until stable", dict(refine_rounds=0xFFFFFFFF, reverse_refine=0)),
            ("until stable reversed", dict(refine_rounds=0xFFFFFFFF, reverse_refine=1)),
            ("1 round forward", dict(refine_rounds=1, reverse_refine=0))]


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    only = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else None
    g = config_graph(2)
    ctx = gpsense.Context(0)
    G = ctx.load_graph(g)
    rows = []
    for i in range(n):
        if only is not None and i not in only:
            continue
        k = (16, 20)[i % 2]
        q = bfs_query(g, k, 6000 + i, induced=True, max_children=2, prefer_hubs=True, top_fraction=0.01,
                      keep_elabels=False, p_wild_v=0.0)
        res = {}
        for name, o in VARIANTS:
            ctx.reset_stats()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            try:
                c = ctx.count(G, q, gpsense.default_opts(**o))
            except gpsense.GpsError as e:
                res[name] = (None, None, None, str(e)[:40])
                continue
            dt = time.perf_counter() - t0
            st = ctx.stats()
            res[name] = (c, st["join_rows_total"], st["join_rows_max"], dt * 1e3)
        counts = {v[0] for v in res.values() if v[0] is not None}
        assert len(counts) <= 1, (i, res)
        base = res["none"]
        ref = res["1 round reversed (default)"]
        ratio_t = base[1] / max(ref[1], 1) if base[1] is not None and ref[1] is not None else None
        ratio_m = base[2] / max(ref[2], 1) if base[2] is not None and ref[2] is not None else None
        rows.append((k, q.n_edges if hasattr(q, "n_edges") else len(q.edges), res, ratio_t, ratio_m))
        line = f"q{i:02d} k={k} e={len(q.edges):2d} count={next(iter(counts)) if counts else None}"
        for name, _ in VARIANTS:
            c, tot, mx, ms = res[name]
            line += f" | {name.split(' (')[0]}: rows {tot} max {mx} {ms if isinstance(ms, str) else f'{ms:.1f} ms'}"
        line += f" | none/default rows x{ratio_t:.1f} max x{ratio_m:.1f}" if ratio_t else ""
        print(line, flush=True)
    rt = [r[3] for r in rows if r[3]]
    rm = [r[4] for r in rows if r[4]]
    if rt:
        print(f"intermediate rows, no refinement / default: max x{max(rt):.1f}, median x{sorted(rt)[len(rt) // 2]:.1f}; "
              f"largest table: max x{max(rm):.1f}, median x{sorted(rm)[len(rm) // 2]:.1f}  ({len(rt)} queries)")


if __name__ == "__main__":
    main()
