import os, sys, time
sys.path.insert(0, "/root/repo")
import torch
from synth import bfs_query, config_graph
from paper_1807_08804_b200 import gpsense
i = int(sys.argv[1]); vars_ = [int(x) for x in sys.argv[2].split(",")]
g = config_graph(2)
ctx = gpsense.Context(0)
G = ctx.load_graph(g)
k = (16, 20)[i % 2]
q = bfs_query(g, k, 6000 + i, induced=True, max_children=2, prefer_hubs=True, top_fraction=0.01, keep_elabels=False, p_wild_v=0.0)
V = [dict(refine_rounds=0), dict(refine_rounds=1, reverse_refine=1), dict(refine_rounds=1, reverse_refine=0), dict(refine_rounds=4, reverse_refine=1)]
if os.environ.get("TRACE"):
    os.environ["GPS_TRACE"] = "1"
for var in vars_:
    try:
        ctx.reset_stats()
        c = ctx.count(G, q, gpsense.default_opts(**V[var]))
        torch.cuda.synchronize()
        print("variant", var, "count", c, ctx.stats()["join_rows_total"], ctx.stats()["join_rows_max"], flush=True)
    except Exception as e:
        print("variant", var, "ERR", e, flush=True)
