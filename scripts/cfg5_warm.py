"""Diagnostic: cfg5 batch step time over successive 3-step groups (warm-up convergence)."""
import json, os, sys, time
ROOT = sys.argv[1] if len(sys.argv) > 1 else os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from synth import Query, config_graph
from paper_1807_08804_b200 import gpsense
qs = [Query.from_json(d["query"]) for d in json.load(open(os.path.join(ROOT, "synth/data/cfg5_queries.json")))["queries"]]
ctx = gpsense.Context(0)
G = ctx.load_graph(config_graph(2))
qb = gpsense.QueryBatch(qs)
ctx.set_workers(3); ctx.set_slice(34)
out = []
for g in range(5):
    t0 = time.perf_counter()
    for _ in range(2): ctx.match_batch_raw(G, qb).free()
    torch.cuda.synchronize()
    out.append((time.perf_counter() - t0) / 2 * 1e3)
print(os.path.basename(ROOT.rstrip("/")), " ".join(f"{x:.0f}" for x in out), "ms/step", flush=True)
