"""Step time of the cfg2 batch for several (workers, slice) settings, interleaved repeats (diagnostic)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from synth import Query, config_graph  # noqa: E402
from paper_1807_08804_b200 import gpsense  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
data = json.load(open(os.path.join(ROOT, "synth", "data", f"cfg{cfg}_queries.json")))
qs = [Query.from_json(d["query"]) for d in data["queries"]]
ctx = gpsense.Context(0)
G = ctx.load_graph(config_graph(2))
qb = gpsense.QueryBatch(qs)
settings = [(4, 25), (3, 34), (2, 50), (5, 20), (3, 25), (4, 34)]
res = {s: [] for s in settings}
for rep in range(4):
    for w, s in settings:
        ctx.set_workers(w)
        ctx.set_slice(s)
        ctx.match_batch_raw(G, qb).free()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        per = []
        for _ in range(10):
            t1 = time.perf_counter()
            ctx.match_batch_raw(G, qb).free()
            torch.cuda.synchronize()
            per.append((time.perf_counter() - t1) * 1e3)
        res[(w, s)].append((time.perf_counter() - t0) / 10 * 1e3)
        if max(per) > 3 * min(per):
            print(f"  outlier workers={w} slice={s} rep={rep}: " + " ".join(f"{x:.2f}" for x in per), flush=True)
for k, v in res.items():
    print(f"workers={k[0]} slice={k[1]}: " + " ".join(f"{x:.3f}" for x in v) + " ms/step")
