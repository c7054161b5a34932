"""Config-4 step stability: the bench step (10 queries, one at a time) repeated, host wall time
per query, with GPS_TRACE phase deltas > 20 ms reported (stderr)."""
import json
import os
import sys
import time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from synth import Query, config_graph  # noqa: E402
from synth.large import CFG4  # noqa: E402
from paper_1807_08804_b200 import gpsense  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "batch"
ctx = gpsense.Context(0)
G = ctx.load_graph(config_graph(4))
qs = [(q, m) for _, q, m in CFG4]
qs += [(Query.from_json(d["query"]), "match") for d in
       json.load(open(os.path.join(ROOT, "synth", "data", "cfg4_queries.json")))["queries"]]


def run_one(q, m):
    if m == "count":
        return ctx.count(G, q)
    if mode == "batch":
        br = ctx.match_batch_raw(G, [q])
        n = int(br.rows().sum())
        br.free()
        return n
    t = ctx.match(G, q)
    n = t.shape[0]
    del t
    return n


for s in range(12):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    per = []
    for q, m in qs:
        a = time.perf_counter()
        run_one(q, m)
        torch.cuda.synchronize()
        per.append(1e3 * (time.perf_counter() - a))
    print(f"{mode} step {s}: {1e3 * (time.perf_counter() - t0):.1f} ms  per query " +
          " ".join(f"{x:.0f}" for x in per), flush=True)
