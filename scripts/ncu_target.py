"""Small driver for ncu captures: one warm batch, then one profiled batch of the cfg2 queries."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from synth import Query, config_graph
from paper_1807_08804_b200 import gpsense
data = json.load(open(os.path.join(ROOT, "synth", "data", "cfg2_queries.json")))
qs = [Query.from_json(d["query"]) for d in data["queries"]]
ctx = gpsense.Context(0)
ctx.set_workers(1)
ctx.set_slice(int(os.environ.get("SLICE", "100")))
G = ctx.load_graph(config_graph(2))
if os.environ.get("MODE", "both") != "match":
    ctx.count_batch(G, qs)
outs = ctx.match_batch(G, qs)
torch.cuda.synchronize()
print("ok", sum(t.shape[0] for t in outs))
