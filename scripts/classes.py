"""Per-kernel-class breakdown of one config's step (diagnostic; event-timed, one stream).

  python scripts/classes.py CONFIG [count|match]
Config 2/3/5: the stored queries through gps_match_batch (one worker stream, bench slices);
config 4: the stored cyclic queries one at a time.  Prints ms / launches / algorithmic
GB/s per class, the largest table, and the step time without profiling.
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
    mode = sys.argv[2] if len(sys.argv) > 2 else "match"
    data = json.load(open(os.path.join(ROOT, "synth", "data", f"cfg{cfg}_queries.json")))
    qs = [Query.from_json(d["query"]) for d in data["queries"]]
    ctx = gpsense.Context(0)
    G = ctx.load_graph(config_graph(4 if cfg == 4 else 2))
    qb = gpsense.QueryBatch(qs)

    def step():
        if cfg == 4 or os.environ.get("ONE_AT_A_TIME"):
            for q in qs:
                if mode == "count":
                    ctx.count(G, q)
                else:
                    ctx.match_batch_raw(G, [q]).free()
        elif mode == "count":
            ctx.count_batch(G, qb)
        else:
            ctx.match_batch_raw(G, qb).free()
        torch.cuda.synchronize()

    ctx.set_workers(1)
    ctx.set_slice(34)
    step()
    ctx.set_profiling(gpsense.KERNEL_CLASSES)
    ctx.reset_stats()
    step()
    st = ctx.stats()
    tot = 0.0
    print(f"== cfg{cfg} {mode}: launches/step {st['launches']}, syncs/step {st['host_syncs']}, "
          f"join_rows_max {st['join_rows_max']}, join_rows_total {st['join_rows_total']}, "
          f"embeddings {st['embeddings']}")
    for k, v in sorted(st["kernels"].items(), key=lambda kv: -kv[1]["ms"]):
        if v["launches"]:
            tot += v["ms"]
            print(f"   {k:12s} launches {v['launches']:5d}  ms {v['ms']:9.3f}  avg us "
                  f"{1e3 * v['ms'] / max(v['timed'], 1):9.2f}  MB {v['bytes'] / 1e6:10.2f}  "
                  f"GB/s {v['bytes'] / max(v['ms'], 1e-9) / 1e6:8.1f}")
    print(f"   sum of kernel time {tot:.3f} ms/step")
    ctx.set_profiling([])
    ctx.set_workers(3)
    step()
    t0 = time.perf_counter()
    for _ in range(3):
        step()
    print(f"step (3 workers, no profiling): {(time.perf_counter() - t0) / 3 * 1e3:.3f} ms")


if __name__ == "__main__":
    main()
