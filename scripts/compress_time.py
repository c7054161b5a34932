"""Time gps_compress (3 levels, delta = 1) on the config-2 and config-4 graphs."""
import os
import sys
import time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from synth import config_graph  # noqa: E402
from paper_1807_08804_b200 import gpsense  # noqa: E402

ctx = gpsense.Context(0)
for cfg in [int(x) for x in (sys.argv[1:] or ["2", "4"])]:
    g = config_graph(cfg)
    G = ctx.load_graph(g)
    for rep in range(2):
        torch.cuda.synchronize()
        t = time.time()
        cg = ctx.compress(G, [1.0, 1.0, 1.0])
        torch.cuda.synchronize()
        dt = time.time() - t
        print(f"cfg{cfg} n={g.n} arcs={G.arcs} levels(nodes, out-edges, in-edges)="
              f"{[cg.info(l) for l in (1, 2, 3)]} compress {dt:.3f} s")
        cg.free()
    G.free()
