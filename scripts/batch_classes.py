"""Per-kernel-class breakdown of the bench's batch workload (diagnostic).

One worker stream, SLICE-query batch-synchronous slices (bench default 25), every
kernel class event-timed: ms per step per class, launches, algorithmic GB/s.
Then the step time with W worker streams (bench default 4) and no profiling.
  python scripts/batch_classes.py [CONFIG=2] [SLICE=25]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from synth import Query, config_graph  # noqa: E402
from paper_1807_08804_b200 import gpsense  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    sl = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    data = json.load(open(os.path.join(ROOT, "synth", "data", f"cfg{cfg}_queries.json")))
    qs = [Query.from_json(d["query"]) for d in data["queries"]]
    ctx = gpsense.Context(0)
    G = ctx.load_graph(config_graph(2))
    qb = gpsense.QueryBatch(qs)
    ctx.set_workers(1)
    ctx.set_slice(sl)
    for _ in range(2):
        ctx.match_batch_raw(G, qb).free()
    ctx.set_profiling(gpsense.KERNEL_CLASSES)
    ctx.reset_stats()
    ctx.match_batch_raw(G, qb).free()
    torch.cuda.synchronize()
    st = ctx.stats()
    tot = 0.0
    print(f"== cfg{cfg} slice {sl}: launches/step {st['launches']}, syncs/step {st['host_syncs']}")
    for k, v in sorted(st["kernels"].items(), key=lambda kv: -kv[1]["ms"]):
        if v["launches"]:
            tot += v["ms"]
            print(f"   {k:12s} launches {v['launches']:5d}  ms {v['ms']:.4f}  avg us "
                  f"{1e3 * v['ms'] / max(v['timed'], 1):8.2f}  MB {v['bytes'] / 1e6:9.2f}  "
                  f"GB/s {v['bytes'] / max(v['ms'], 1e-9) / 1e6:8.1f}")
    print(f"   sum of kernel time {tot:.3f} ms/step")
    ctx.set_profiling([])
    for w, s in ((1, sl), (4, sl), (2, 50), (3, 34), (2, 25), (1, 100), (4, 13)):
        ctx.set_workers(w)
        ctx.set_slice(s)
        ctx.match_batch_raw(G, qb).free()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(10):
            ctx.match_batch_raw(G, qb).free()
        torch.cuda.synchronize()
        print(f"workers={w} slice={s}: {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms/step")


if __name__ == "__main__":
    main()
