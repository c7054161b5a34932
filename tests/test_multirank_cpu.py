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
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--steps", "1",
                        "--warmup", "0"], capture_output=True, text=True, timeout=120, cwd=ROOT, env=env)
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


SHARD_WORKER = r"""
import os, sys
sys.path.insert(0, {root!r})
import numpy as np
import torch, torch.distributed as dist
from paper_1807_08804_b200 import gpsense as gps
dist.init_process_group("gloo")
r, w = dist.get_rank(), dist.get_world_size()
for trial in range(20):
    rng = np.random.default_rng(100 * trial + r)
    # this rank's local table: R rows (ids = global position) with skewed segment lengths
    R = int(rng.integers(0, 400)) if trial % 5 else (0 if r == 0 else 300)
    seg = rng.zipf(1.6, size=R).clip(max=500).astype(np.uint64) * (rng.random(R) > 0.1)
    base = [None] * w
    dist.all_gather_object(base, R)
    rows = np.arange(sum(base[:r]), sum(base[:r]) + R, dtype=np.int64)
    poff = np.concatenate([[0], np.cumsum(seg)]).astype(np.uint64)
    pall = [None] * w
    dist.all_gather_object(pall, int(poff[-1]))
    lt, reb, total = gps.shard_plan(w, r, np.array(pall, np.uint64), 0.0 if trial % 2 else 1.10)
    assert total == sum(pall)
    mean = total / w
    assert reb == (total > 0 and max(pall) > (0.0 if trial % 2 else 1.10) * mean)
    # rows whose first pair lies in [lt[t], lt[t+1]) go to rank t (lower bound on poff)
    cuts = np.minimum(np.searchsorted(poff, lt, side="left"), R).astype(np.int64)
    cuts[0], cuts[w] = 0, R
    cnt = np.maximum(cuts[1:] - cuts[:-1], 0)
    mat = [None] * w
    dist.all_gather_object(mat, cnt.tolist())
    at, got = gps.shard_recv(w, r, np.array(mat, np.uint64).reshape(w, w))
    assert got == sum(mat[s][r] for s in range(w))
    # the exchange (rows and their segment lengths), blocks placed at `at`
    parts = [None] * w
    dist.all_gather_object(parts, [(rows[cuts[t]:cuts[t + 1]].tolist(), seg[cuts[t]:cuts[t + 1]].tolist())
                                   for t in range(w)])
    new_rows = np.full(got, -1, np.int64)
    new_seg = np.zeros(got, np.int64)
    for s in range(w):
        blk, sg = parts[s][r]
        new_rows[int(at[s]):int(at[s]) + len(blk)] = blk
        new_seg[int(at[s]):int(at[s]) + len(blk)] = sg
    assert (new_rows >= 0).all()
    # global order preserved: the new shards in rank order are the old global table
    allnew = [None] * w
    dist.all_gather_object(allnew, new_rows.tolist())
    assert sum(allnew, []) == list(range(sum(base)))
    # balance: every rank's pairs are within one row of its exact share
    mine = int(new_seg.sum())
    q, rem = divmod(total, w)
    share = q + (1 if r < rem else 0)
    assert abs(mine - share) <= max(500, 0) + 1 or total == 0, (mine, share)
dist.destroy_process_group()
open(os.path.join({tmp!r}, "shard%d" % r), "w").write("ok")
"""


@pytest.mark.parametrize("world", [2, 3])
def test_shard_arithmetic_gloo(tmp_path, world):
    """Row-sharded join host arithmetic (gps_shard_plan / gps_shard_recv, the library's own
    functions) driven through a real all-gather / exchange protocol over gloo: the
    rebalanced shards in rank order are the old global table, every rank ends within one
    row of its pair share, receive offsets match the all-gathered send matrix."""
    script = tmp_path / "s.py"
    script.write_text(SHARD_WORKER.format(root=ROOT, tmp=str(tmp_path)))
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(script)]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    for r in range(world):
        assert (tmp_path / f"shard{r}").exists()


def test_bench_gpus_mismatch_fails_loudly():
    """A torchrun environment whose world size differs from --gpus is an error, never a
    silent single-rank run."""
    env = dict(os.environ, RANK="0", WORLD_SIZE="2", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, "bench.py", "--gpus", "4", "--steps", "1"], capture_output=True,
                       text=True, timeout=120, cwd=ROOT, env=env)
    assert p.returncode == 2 and "WORLD_SIZE" in p.stderr
