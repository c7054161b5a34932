"""Phase timeline of one step of a config (GPS_TRACE host timestamps) + per-query timing.

  python scripts/trace_cfg.py CONFIG [workers] [slice]
"""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from synth import Query, config_graph
from paper_1807_08804_b200 import gpsense
cfg = int(sys.argv[1])
W = int(sys.argv[2]) if len(sys.argv) > 2 else 1
S = int(sys.argv[3]) if len(sys.argv) > 3 else 34
qs = [Query.from_json(d["query"]) for d in json.load(open(os.path.join(ROOT, "synth", "data", f"cfg{cfg}_queries.json")))["queries"]]
ctx = gpsense.Context(0)
ctx.set_workers(W)
ctx.set_slice(S)
G = ctx.load_graph(config_graph(4 if cfg == 4 else 2))
qb = gpsense.QueryBatch(qs)
for _ in range(2):
    ctx.match_batch_raw(G, qb).free()
torch.cuda.synchronize()
t0 = time.perf_counter()
ctx.match_batch_raw(G, qb).free()
torch.cuda.synchronize()
print(f"step wall {1e3 * (time.perf_counter() - t0):.3f} ms (workers {W}, slice {S})", flush=True)
os.environ["GPS_TRACE"] = "1"
t0 = time.perf_counter()
ctx.match_batch_raw(G, qb).free()
torch.cuda.synchronize()
print(f"traced step wall {1e3 * (time.perf_counter() - t0):.3f} ms", flush=True)
del os.environ["GPS_TRACE"]
ctx.set_workers(1)
ctx.set_slice(1)
for i, q in enumerate(qs[:12]):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    br = ctx.match_batch_raw(G, [q])
    n = int(br.rows().sum())
    br.free()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    ctx.reset_stats()
    ctx.count(G, q)
    st = ctx.stats()
    print(f"q{i} k={q.k} rows {n} {1e3 * dt:.2f} ms  (count: syncs {st['host_syncs']}, launches {st['launches']}, "
          f"join_rows_max {st['join_rows_max']})", flush=True)
