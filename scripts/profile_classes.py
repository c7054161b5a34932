"""Per-kernel-class time breakdown of the config-2 bench workload (diagnostic).

Runs the 100 cfg2 queries one at a time (single stream) with every kernel class
event-timed, then prints ms/query per class, launches/query, syncs/query, and
the wall time per query -- the gap between the two is launch latency + host work.
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
    data = json.load(open(os.path.join(ROOT, "synth", "data", "cfg2_queries.json")))
    qs = [Query.from_json(d["query"]) for d in data["queries"]]
    ctx = gpsense.Context(0)
    G = ctx.load_graph(config_graph(2))
    for q in qs[:10]:
        ctx.count(G, q)
    for mode in ("match", "count"):
        ctx.set_profiling(gpsense.KERNEL_CLASSES)
        ctx.reset_stats()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for q in qs:
            if mode == "match":
                t = ctx.match(G, q)
                del t
            else:
                ctx.count(G, q)
        wall = (time.perf_counter() - t0) / len(qs) * 1e3
        st = ctx.stats()
        print(f"== {mode}: wall {wall:.3f} ms/query, launches/query {st['launches'] / len(qs):.1f}, "
              f"syncs/query {st['host_syncs'] / len(qs):.1f}")
        tot = 0.0
        for k, v in st["kernels"].items():
            if v["launches"]:
                ms = v["ms"] / len(qs)
                tot += ms
                print(f"   {k:12s} launches/q {v['launches'] / len(qs):5.1f}  gpu ms/q {ms:.4f}  "
                      f"avg us {1e3 * v['ms'] / max(v['timed'], 1):8.2f}  GB/s {v['bytes'] / max(v['ms'], 1e-9) / 1e6:8.1f}")
        print(f"   sum of kernel time {tot:.3f} ms/query")
    ctx.set_profiling([])
    for w in (4, 8, 16):
        ctx.set_workers(w)
        ctx.count_batch(G, qs)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            outs = ctx.match_batch(G, qs)
            del outs
        torch.cuda.synchronize()
        print(f"batch workers={w}: {(time.perf_counter() - t0) / 3 / len(qs) * 1e3:.3f} ms/query")


if __name__ == "__main__":
    main()
