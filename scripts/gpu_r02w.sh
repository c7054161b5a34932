mkdir -p gpurun_out
(timeout 900 python -m pytest tests/test_gpu_compress.py -m gpu -x -q > gpurun_out/w_tests.log 2>&1; echo exit $? >> gpurun_out/w_tests.log)
tail -30 gpurun_out/w_tests.log
timeout 600 python - <<'PY' 2>&1 | tail -5
import time, torch
from synth import config_graph
from paper_1807_08804_b200 import gpsense
ctx = gpsense.Context(0)
for cfg in (2, 4):
    g = config_graph(cfg); G = ctx.load_graph(g)
    torch.cuda.synchronize(); t = time.time()
    cg = ctx.compress(G, [1.0, 1.0, 1.0]); torch.cuda.synchronize()
    print("cfg", cfg, "n", g.n, "levels", [cg.level(l)["nodes"] for l in (1, 2, 3)], "s %.3f" % (time.time() - t))
    cg.free(); G.free()
PY
