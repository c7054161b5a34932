"""N > 1 host logic of bench.py on CPU with the gloo backend (world_size 2, 127.0.0.1).

The cfg2 bench shards independent queries across ranks (weak scaling, no data-path
collective); its timing is the max over ranks.  These tests run that host logic in
two real processes over gloo."""
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


WORKER = r"""
import os, sys
sys.path.insert(0, {root!r})
import torch, torch.distributed as dist
import bench
dist.init_process_group("gloo")
r, w = dist.get_rank(), dist.get_world_size()
vals = bench.max_over_ranks([10.0 * (r + 1), 1.0 + r], dist, "cpu")
assert vals == [10.0 * w, float(w)], vals
qs, cs = bench.rank_batch(list(range(100)), list(range(100)), r)
assert sorted(qs) == list(range(100)) and qs[0] == (r * 37) % 100
# every rank holds the same batch size (weak scaling)
n = torch.tensor([len(qs)])
dist.all_reduce(n)
assert int(n) == 100 * w
dist.destroy_process_group()
open(os.path.join({tmp!r}, "ok%d" % r), "w").write("ok")
"""


def test_bench_multirank_gloo(tmp_path):
    script = tmp_path / "w.py"
    script.write_text(WORKER.format(root=ROOT, tmp=str(tmp_path)))
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(script)]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=240, cwd=ROOT)
    assert p.returncode == 0, p.stdout + p.stderr
    # one marker file per rank (the two ranks' stdout can interleave)
    assert (tmp_path / "ok0").exists() and (tmp_path / "ok1").exists()


def test_reference_arm_rank1_exits_quietly(tmp_path):
    """--impl reference under torchrun: rank 0 alone prints; other ranks exit 0 without work."""
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=120, cwd=ROOT, env=env)
    assert p.returncode == 0 and p.stdout.strip() == ""


def test_reference_arm_json_line():
    """--impl reference (the CPU oracle arm) prints one JSON line with the contract's keys."""
    import json
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0",
                        "--ref-queries-per-step", "1"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert p.returncode == 0, p.stderr
    line = json.loads(p.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0 and line["cpu_baseline"]["kind"] == "oracle"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
