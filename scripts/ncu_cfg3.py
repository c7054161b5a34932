"""ncu target: config-3 cyclic queries (one warm batch, then one profiled batch, one worker)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from synth import Query, config_graph
from paper_1807_08804_b200 import gpsense
cfg = int(os.environ.get("CFG", "3"))
qs = [Query.from_json(d["query"]) for d in json.load(open(os.path.join(ROOT, "synth", "data", f"cfg{cfg}_queries.json")))["queries"]]
ctx = gpsense.Context(0)
ctx.set_workers(1)
ctx.set_slice(34)
G = ctx.load_graph(config_graph(4 if cfg == 4 else 2))
for _ in range(int(os.environ.get("PASSES", "2"))):
    if cfg == 4:
        for q in qs:
            ctx.match_batch_raw(G, [q]).free()
    else:
        ctx.match_batch_raw(G, qs).free()
    torch.cuda.synchronize()
print("ok")
