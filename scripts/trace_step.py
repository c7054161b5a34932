"""One bench-shaped step (100 cfg2 queries, 4 workers x 25) with GPS_TRACE phase timestamps."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from synth import Query, config_graph
from paper_1807_08804_b200 import gpsense
qs = [Query.from_json(d["query"]) for d in json.load(open(os.path.join(ROOT, "synth", "data", "cfg2_queries.json")))["queries"]]
ctx = gpsense.Context(0)
ctx.set_workers(int(os.environ.get("W", "4")))
ctx.set_slice(int(os.environ.get("S", "25")))
G = ctx.load_graph(config_graph(2))
for _ in range(3):
    ctx.match_batch(G, qs)
torch.cuda.synchronize()
os.environ["GPS_TRACE"] = "1"
t0 = time.perf_counter()
outs = ctx.match_batch(G, qs)
torch.cuda.synchronize()
print(f"step wall {1e3 * (time.perf_counter() - t0):.3f} ms", file=sys.stderr)
