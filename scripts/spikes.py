"""Find host-side stalls in repeated config-3 batch steps (GPS_TRACE deltas > 20 ms)."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from synth import Query, config_graph
from paper_1807_08804_b200 import gpsense
qs = [Query.from_json(d["query"]) for d in json.load(open(os.path.join(ROOT, "synth", "data", "cfg3_queries.json")))["queries"]]
ctx = gpsense.Context(0)
ctx.set_workers(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
ctx.set_slice(34)
G = ctx.load_graph(config_graph(2))
qb = gpsense.QueryBatch(qs)
for _ in range(3):
    ctx.match_batch_raw(G, qb).free()
torch.cuda.synchronize()
os.environ["GPS_TRACE"] = "1"
for s in range(12):
    t0 = time.perf_counter()
    br = ctx.match_batch_raw(G, qb)
    t1 = time.perf_counter()
    br.free()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"STEP {s}: call {1e3 * (t1 - t0):.1f} ms, free+sync {1e3 * (t2 - t1):.1f} ms", file=sys.stderr, flush=True)
