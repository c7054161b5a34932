"""Batch-mode tuning / breakdown on the config-2 bench workload (diagnostic).

Sweeps (workers, slice) for gps_match_batch over the 100 cfg2 queries, then
prints a per-kernel-class breakdown (event-timed) for one configuration.
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
    reps = int(os.environ.get("REPS", "4"))
    qs = qs * reps
    ctx = gpsense.Context(0)
    G = ctx.load_graph(config_graph(2))
    combos = [(1, 400), (1, 100), (1, 50), (2, 50), (2, 25), (4, 25), (4, 13), (8, 13), (8, 7), (16, 7)]
    for w, s in combos:
        ctx.set_workers(w)
        ctx.set_slice(s)
        ctx.count_batch(G, qs[:100])
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(3):
            t0 = time.perf_counter()
            outs = ctx.match_batch(G, qs)
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
            del outs
        print(f"workers={w:2d} slice={s:3d}: {best / len(qs) * 1e6:8.1f} us/query  {len(qs) / best:9.0f} q/s",
              flush=True)
    w, s = [int(x) for x in os.environ.get("PROFILE", "1,100").split(",")]
    ctx.set_workers(w)
    ctx.set_slice(s)
    ctx.set_profiling(gpsense.KERNEL_CLASSES)
    ctx.reset_stats()
    t0 = time.perf_counter()
    outs = ctx.match_batch(G, qs)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    del outs
    st = ctx.stats()
    print(f"== profile workers={w} slice={s}: wall {wall * 1e3:.2f} ms for {len(qs)} queries, "
          f"launches {st['launches']}, syncs {st['host_syncs']}")
    tot = 0
    for k, v in st["kernels"].items():
        if v["launches"]:
            tot += v["ms"]
            print(f"   {k:12s} launches {v['launches']:5d}  ms {v['ms']:8.3f}  avg us {1e3 * v['ms'] / max(v['timed'], 1):8.2f}"
                  f"  GB/s {v['bytes'] / max(v['ms'], 1e-9) / 1e6:8.1f}")
    print(f"   sum kernel ms {tot:.3f}")


if __name__ == "__main__":
    main()
