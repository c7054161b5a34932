"""Refinement ablation on config 2/3 (f1): time and intermediate rows per variant."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from synth import Query, config_graph
from paper_1807_08804_b200 import gpsense

ctx = gpsense.Context(0, workers=1)
ctx.set_slice(1000)
G = ctx.load_graph(config_graph(2))
for cfg in (2, 3):
    qs = [Query.from_json(d["query"]) for d in json.load(open(os.path.join(ROOT, "synth", "data", f"cfg{cfg}_queries.json")))["queries"]] * (4 if cfg == 2 else 8)
    for name, o in [("none", dict(refine_rounds=0)), ("1 round reversed", dict(refine_rounds=1, reverse_refine=1)),
                    ("1 round forward", dict(refine_rounds=1, reverse_refine=0)), ("3 rounds reversed", dict(refine_rounds=3)),
                    ("1 round, lowconn 0", dict(refine_rounds=1, lowconn_threshold=0))]:
        opts = gpsense.default_opts(**o)
        ctx.count_batch(G, qs[:50], opts)
        ctx.reset_stats()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        br = ctx.match_batch_raw(G, qs, opts)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        st = ctx.stats()
        br.free()
        print(f"cfg{cfg} {name:22s} {dt / len(qs) * 1e6:7.1f} us/query  join rows total {st['join_rows_total']:>12,}  max {st['join_rows_max']:>10,}", flush=True)
