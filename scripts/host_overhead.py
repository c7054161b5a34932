"""Host-side cost breakdown of one bench step (marshalling, library call, result handling)."""
import ctypes, json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from synth import Query, config_graph
from paper_1807_08804_b200 import gpsense
from paper_1807_08804_b200.gpsense import lib
qs = [Query.from_json(d["query"]) for d in json.load(open(os.path.join(ROOT, "synth", "data", "cfg2_queries.json")))["queries"]]
ctx = gpsense.Context(0)
ctx.set_workers(4)
ctx.set_slice(25)
G = ctx.load_graph(config_graph(2))
for _ in range(3):
    ctx.match_batch_raw(G, qs).free()
torch.cuda.synchronize()
T = {"desc": 0, "call": 0, "rows": 0, "free": 0, "total": 0}
N = 20
for _ in range(N):
    t0 = time.perf_counter()
    qas, arr, qb = ctx._batch_desc(qs)
    t1 = time.perf_counter()
    n = len(qas)
    res = (ctypes.c_void_p * n)()
    st = np.zeros(n, np.int32)
    o = gpsense._with_device(gpsense.default_opts(), True)
    rc = lib.gps_match_batch(ctx._h, G.handle, arr, n, ctypes.byref(o), res, ctypes.c_void_p(st.ctypes.data))
    t2 = time.perf_counter()
    br = gpsense.BatchResult(ctx, res, n)
    t3 = time.perf_counter()
    br.free()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    for k, v in zip(("desc", "call", "rows", "free", "total"), (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t4 - t0)):
        T[k] += v
print({k: round(1e3 * v / N, 3) for k, v in T.items()}, "ms per step")
