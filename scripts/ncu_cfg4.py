"""ncu target: the config-4 large joins (20M-vertex / 100M-arc graph), one warm pass + one profiled pass."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from synth import config_graph  # noqa: E402
from synth.large import CFG4  # noqa: E402
from paper_1807_08804_b200 import gpsense  # noqa: E402

ctx = gpsense.Context(0)
G = ctx.load_graph(config_graph(4))
for _ in range(2):
    for name, q, mode in CFG4:
        if mode == "count":
            n = ctx.count(G, q)
        else:
            br = ctx.match_batch_raw(G, [q])
            n = int(br.rows().sum())
            br.free()
        torch.cuda.synchronize()
if os.environ.get("CLASSES"):   # per-class breakdown of one more pass (event-timed, single stream)
    ctx.set_profiling(gpsense.KERNEL_CLASSES)
    ctx.reset_stats()
    for name, q, mode in CFG4:
        if mode == "count":
            ctx.count(G, q)
        else:
            ctx.match_batch_raw(G, [q]).free()
    torch.cuda.synchronize()
    st = ctx.stats()
    for k, v in sorted(st["kernels"].items(), key=lambda kv: -kv[1]["ms"]):
        if v["launches"]:
            print(f"   {k:12s} launches {v['launches']:5d}  ms {v['ms']:.4f}  MB {v['bytes'] / 1e6:9.2f}  "
                  f"GB/s {v['bytes'] / max(v['ms'], 1e-9) / 1e6:8.1f}")
print("ok")
