"""Benchmark: GpSense filter + join hot path on B200 (BASELINE.json configs[1]).

Workload (config 2): ConceptNet-shaped directed Chung-Lu graph (n = 300,000,
m = 1,500,000 labelled arcs, synth.config_graph(2), seed 8804) resident in HBM;
one STEP = gps_match of the 100 stored six-vertex BFS tree queries
(synth/data/cfg2_queries.json; embeddings stay in device memory).

  python bench.py [--gpus N --steps K --warmup W] [--config C] [--impl reference]

Multi-GPU: one process per GPU (torchrun; `--gpus N` without a torchrun environment
launches one itself).  Configs 2, 3 and 5: the graph is replicated and every rank
runs its own batch (weak scaling, no data-path collective).  Config 4: every rank
runs the SAME large cyclic queries and the partial-embedding tables are sharded by
row across the ranks, with one NCCL all-gather per join step plus row rebalancing
(strong scaling).  Time = max over ranks of the device-timed region;
value = queries completed / that time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "subgraph-match queries/s and embeddings/s vs HBM roofline at 1/2/4/8 B200"
GRAPH = "ConceptNet-shaped Chung-Lu graph n=300000 m=1500000 labelled arcs (L_E=34 Zipf 1.3, L_V=16)"
WORKLOADS = {
    2: f"cfg2: {GRAPH}, 100 six-vertex BFS tree queries per step, gps_match with device-resident results",
    3: f"cfg3: {GRAPH}, 30 cyclic 8/10/12-vertex queries (dense hub core) per step, device-resident results",
    5: f"cfg5: {GRAPH}, QA batch of 10000 3-5-vertex queries with a bound concept vertex per step",
    4: "cfg4: Chung-Lu graph n=20000000 m=100000000 labelled arcs (HBM-resident CSR); per step the "
       "closed-form joins (out-star-2, in-star-2, 2-path: 2.5e8 rows written; out-star-3: 3.2e9 counted) and "
       "gps_match of the 6 stored 6/7/8-vertex cyclic queries (synth/data/cfg4_queries.json); rows sharded "
       "over the GPUs when N > 1",
}
CONFIG = 2


# Library kernel classes that are launches of ONE kernel: the roofline names the dominant KERNEL,
# so their times and bytes are added (k_explore serves both the prune and the propagate jobs).
KERNEL_GROUP = {"propagate": "explore"}
KERNEL_NAME = {"explore": "k_explore", "collect": "k_collect", "check": "k_check", "ec_write": "k_ec",
               "join_len": "k_join_seg", "join_write": "join writes (k_join_bulk / k_join_v / k_join<2>)"}


def by_kernel(kernels):
    out = {}
    for k, v in kernels.items():
        name = KERNEL_GROUP.get(k, k)
        o = out.setdefault(name, {"ms": 0.0, "bytes": 0.0, "timed": 0, "launches": 0, "classes": []})
        for f in ("ms", "bytes", "timed", "launches"):
            o[f] += v.get(f, 0)
        o["classes"].append(k)
    return out


def load_queries(cfg=None):
    from synth import Query
    cfg = CONFIG if cfg is None else cfg
    data = json.load(open(os.path.join(ROOT, "synth", "data", f"cfg{cfg}_queries.json")))
    qs, cs = [Query.from_json(d["query"]) for d in data["queries"]], [d["oracle_count"] for d in data["queries"]]
    if cfg == 4:   # + the closed-form-pinned large joins (tests/test_gpu_large.py): the HBM-sized tables
        from synth.large import CFG4
        qs = [q for _, q, _ in CFG4] + qs
        cs = [None] * len(CFG4) + cs
    return qs, cs


def cfg4_modes():
    """Config 4 step: gps_match of every query except the closed-form out-star-3 (3.2e9
    embeddings: gps_count, its last level is never written)."""
    from synth.large import CFG4
    return [m for _, _, m in CFG4] + ["match"] * (len(load_queries(4)[0]) - len(CFG4))


def sample_order(n: int):
    """A fixed pseudo-random order of the stored queries: CPU samples walk it (rotating by
    step), so a bounded sample is not biased towards the first queries of the file."""
    return np.random.default_rng(12345).permutation(n).tolist()


def host_cpu() -> dict:
    model, cores = None, os.cpu_count()
    try:
        for ln in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if ln.startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"model": model, "cpus": cores}


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                smax = float(p[2])
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ reference arm
def cpu_oracle_sample(og, queries, order, start: int, budget_s: float, threads: int, max_q: int = 0):
    """Time the CPU oracle (as it stands: oracle.c, `threads` OpenMP threads) on queries
    taken from `order` starting at `start` (cyclic) until `budget_s` is used.  Each query is
    the full enumeration (every embedding visited; count + multiset hash, rows not stored)."""
    from oracle import oracle
    t0 = time.perf_counter()
    done, emb = 0, 0
    while done < len(order) and (not max_q or done < max_q):
        q = queries[order[(start + done) % len(order)]]
        emb += oracle.run(og, q, threads=threads)["count"]
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    return done, emb, time.perf_counter() - t0


def cpu_baseline(g, queries, budget_s: float) -> dict:
    """Oracle on the host cores in both modes of SURVEY §8(d): 1 thread and all cores."""
    from oracle import oracle
    og = oracle.OracleGraph(g)
    order = sample_order(len(queries))
    nproc = os.cpu_count() or 1
    d1, e1, t1 = cpu_oracle_sample(og, queries, order, 0, budget_s / 2, 1)
    dn, en, tn = cpu_oracle_sample(og, queries, order, 0, budget_s / 2, nproc)
    return {"value": dn / tn, "unit": "queries/s", "cores": nproc, "kind": "oracle",
            "sample": f"cfg{CONFIG}: {dn} queries in a fixed seeded order (of {len(queries)}), oracle.c OpenMP "
                      f"{nproc} threads, {en} embeddings in {tn:.1f} s",
            "single_thread": {"value": d1 / t1, "cores": 1,
                              "sample": f"{d1} queries of the same order, {e1} embeddings in {t1:.1f} s"},
            "host": host_cpu()}


def cfg4_cpu_baseline(g, queries, budget_s: float) -> dict:
    """Config 4: one full oracle enumeration takes minutes, so the bounded sample is a
    first-column partition (SURVEY §8(d) partitions) of each query in turn: the oracle
    enumerates the embeddings whose first query vertex maps into [0, n/64); the rate is
    reported as partitions/s / 64 (query-equivalents/s) with the partition stated."""
    from oracle import oracle
    og = oracle.OracleGraph(g)
    nproc = os.cpu_count() or 1
    part = 64
    t0 = time.perf_counter()
    done, emb = 0, 0
    while time.perf_counter() - t0 < budget_s:
        q = queries[done % len(queries)]
        p = done // len(queries) % part
        emb += oracle.run(og, q, threads=nproc, col0_range=(p * g.n // part, (p + 1) * g.n // part))["count"]
        done += 1
    dt = time.perf_counter() - t0
    return {"value": done / part / dt, "unit": "queries/s", "cores": nproc, "kind": "oracle",
            "sample": f"cfg4: {done} first-column partitions (1/{part} of the data ids each) of the stored "
                      f"queries, oracle.c OpenMP {nproc} threads, {emb} embeddings in {dt:.1f} s; value = "
                      f"partitions/s / {part}", "host": host_cpu()}


def run_reference(args, rank, world):
    from synth import config_graph
    from oracle import oracle
    if rank != 0:
        return
    queries, _ = load_queries()
    g = config_graph(4 if CONFIG == 4 else 2)
    if CONFIG == 4:   # one full oracle enumeration takes minutes: first-column partitions (cfg4_cpu_baseline)
        cb = cfg4_cpu_baseline(g, queries, args.steps * args.ref_step_budget)
        line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "queries/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / cb["value"] * len(queries),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
                "data": "synthetic", "config": {"workload": WORKLOADS[CONFIG], "sample": cb["sample"]},
                "cpu_baseline": cb,
                "e2e": {"value": cb["value"], "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    og = oracle.OracleGraph(g)
    order = sample_order(len(queries))
    per_step = max(1, args.ref_queries_per_step)
    nproc = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_oracle_sample(og, queries, order, 0, 0.0, nproc, 1)
    tot_q, tot_e, tot_t = 0, 0, 0.0
    for s in range(args.steps):
        d, e, t = cpu_oracle_sample(og, queries, order, (s * per_step) % len(order), args.ref_step_budget, nproc,
                                    per_step)
        tot_q += d
        tot_e += e
        tot_t += t
    qps = tot_q / tot_t
    line = {"impl": "reference", "metric": METRIC, "value": qps, "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tot_t / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic", "embeddings_per_s": tot_e / tot_t,
            "config": {"workload": WORKLOADS[CONFIG],
                       "sample": f"per step: queries of a fixed seeded order starting at step*{per_step}, "
                                 f"until {args.ref_step_budget:.0f} s of oracle time"},
            "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": nproc, "kind": "oracle",
                             "sample": f"{tot_q} cfg{CONFIG} queries over {args.steps} steps, oracle.c OpenMP "
                                       f"{nproc} threads (full enumeration)", "host": host_cpu()},
            "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------- our arm
def query_bytes(q):
    return 32 + q.k * 4 + q.k * 8 + len(q.edges) * 12


def rank_batch(queries, counts, rank):
    """Weak scaling: every rank runs a full batch (rotated per rank so ranks start on different queries)."""
    rot = (rank * 37) % len(queries)
    return queries[rot:] + queries[:rot], counts[rot:] + counts[:rot]


def max_over_ranks(values, dist, device):
    """Element-wise max over ranks (the timed region is the slowest rank's)."""
    import torch
    t = torch.tensor(values, dtype=torch.float64, device=device)
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


def relaunch_under_torchrun(n: int) -> int:
    """`--gpus N` outside a torchrun environment: launch one process per GPU ourselves."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=[2, 3, 4, 5],
                    help="BASELINE.json configs[N-1]; the driver's line is config 2")
    ap.add_argument("--ref-queries-per-step", type=int, default=10)
    ap.add_argument("--ref-step-budget", type=float, default=8.0, help="reference arm: oracle seconds per step")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--workers", type=int, default=None,
                    help="library batch workers (0 = one query at a time; default 3, config 5: 4)")
    ap.add_argument("--slice", type=int, default=None,
                    help="queries per worker hand-out (batch-synchronous unit; default 34, config 5: 256)")
    args = ap.parse_args()
    # config 5's 10,000 small queries: wider slices amortise each launch's latency chain over more
    # queries (measured: 3 x 34 -> 99K, 4 x 128 -> 153K, 4 x 256 -> 160K queries/s)
    if args.workers is None:
        args.workers = 4 if args.config == 5 else 3
    if args.slice is None:
        args.slice = 256 if args.config == 5 else 34
    assert args.warmup >= 0 and args.steps >= 1
    global CONFIG
    CONFIG = args.config

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    from synth import config_graph
    from paper_1807_08804_b200 import gpsense

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    dev = torch.device(f"cuda:{local}")
    stream = torch.cuda.Stream(device=dev)
    sharded = CONFIG == 4 and world > 1   # row-sharded join of the same queries (strong scaling)
    if CONFIG in (3, 4) and "GPS_POOL_RESERVE_BYTES" not in os.environ:
        # multi-GB join tables: map the library's memory pool once up front (gps_create reads it)
        # instead of growing it mid-step (0.1-1.3 s stalls in the first steps of a process)
        os.environ["GPS_POOL_RESERVE_BYTES"] = str(96 << 30)
    if sharded:
        comm = dist.group.WORLD._get_backend(dev)._comm_ptr()
        ctx = gpsense.Context(local, stream=stream, nccl_comm=comm, rank=rank, world=world)
    else:
        ctx = gpsense.Context(local, stream=stream)
    g = config_graph(4 if CONFIG == 4 else 2)
    G = ctx.load_graph(g)
    queries, counts = load_queries()
    if CONFIG != 4:
        queries, counts = rank_batch(queries, counts, rank)
    qbatch = gpsense.QueryBatch(queries)   # marshalled once (host descriptors)
    flush = None if args.no_flush else torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    batch_api = args.workers and not sharded   # sharded ranks walk queries one at a time (SPMD)

    if batch_api:
        ctx.set_workers(args.workers)
        ctx.set_slice(args.slice)

    modes = cfg4_modes() if CONFIG == 4 else None

    def step():
        if CONFIG == 4:   # each query's rows stay on the device (sharded: this rank's shard)
            # one query at a time on the ctx's own stream (gps_match): the batch worker pool's
            # per-worker streams made the pool re-map multi-GB blocks (0.1-1 s stalls per step)
            emb = 0
            for q, mode in zip(queries, modes):
                if mode == "count":
                    emb += ctx.count(G, q)
                    continue
                t = ctx.match(G, q)
                emb += int(t.shape[0])
                del t
            return emb
        if batch_api:
            br = ctx.match_batch_raw(G, qbatch)        # device-resident results, freed after the step
            emb = int(br.rows().sum())
            br.free()
            return emb
        emb = 0
        for q in queries:
            t = ctx.match(G, q)
            emb += t.shape[0]
            del t
        return emb

    with torch.cuda.stream(stream):
        # warm-up; the dominant kernel class is chosen from one single-stream pass with every
        # class event-timed (concurrent streams would blur per-launch event times)
        for _ in range(max(args.warmup, 1)):
            step()
        if batch_api:   # the timed region's slices, serialised on one stream
            ctx.set_workers(1)
            ctx.set_slice(args.slice)
        ctx.set_profiling(gpsense.KERNEL_CLASSES)
        ctx.reset_stats()
        step()
        st = ctx.stats()
        iso = by_kernel(st["kernels"])
        ms = {k: v["ms"] for k, v in iso.items()}
        dominant = max(ms, key=ms.get)
        kd_iso = iso[dominant]
        total_iso = sum(ms.values())
        if batch_api:   # fresh worker contexts: warm them again (scratch growth, first launches;
            ctx.set_workers(args.workers)   # their first steps can stall on driver allocations)
            ctx.set_slice(args.slice)
            for _ in range(max(args.warmup, 10)):
                step()
        if CONFIG == 4:   # the first steps of a process grow the memory pool by tens of GB (0.1-1 s
            for _ in range(6):   # mapping stalls); a few more untimed steps let it settle
                step()
        ctx.set_profiling(iso[dominant]["classes"])
        ctx.reset_stats()

        sampler = ClockSampler(local)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        sampler.start()
        total_ms = 0.0
        emb_total = 0
        for s in range(args.steps):
            if flush is not None:
                flush.fill_(s & 0xff)          # L2 flush between timed steps (outside the events)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            emb_total += step()
            e1.record(stream)
            e1.synchronize()
            total_ms += e0.elapsed_time(e1)
            if os.environ.get("BENCH_DEBUG"):
                print(f"step {s}: {e0.elapsed_time(e1):.3f} ms", file=sys.stderr)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        clocks = sampler.stop()
        st = ctx.stats()

        # e2e: the same step through the C-ABI with a HOST result buffer (copies inside the region)
        local_rows = counts if not sharded else [None] * len(queries)
        if CONFIG == 4:   # every written query's (local) rows into one pinned buffer, one query at a time
            local_rows = []
            for q, mode in zip(queries, modes):
                if mode == "count":
                    local_rows.append(0)
                    continue
                t = ctx.match(G, q)
                local_rows.append(int(t.shape[0]))
                del t
            total_words = max(c * q.k for c, q in zip(local_rows, queries))
        else:
            total_words = sum(c * q.k for c, q in zip(local_rows, queries))
        pinned = torch.empty(int(total_words * 1.05) + 1024, dtype=torch.int32, pin_memory=True)
        h2d = sum(query_bytes(q) for q in queries)
        d2h = sum(c * q.k * 4 for c, q in zip(local_rows, queries))
        e2e_ms = 0.0
        e2e_steps = max(1, args.steps // 2)
        for s in range(e2e_steps):
            if flush is not None:
                flush.fill_(s & 0xff)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if CONFIG == 4:
                for q, mode in zip(queries, modes):
                    if mode == "count":
                        ctx.count(G, q)
                    else:
                        ctx.match_host(G, q, pinned)
            elif batch_api:
                ctx.match_batch_host(G, qbatch, pinned)     # library copies every result into `pinned`
            else:
                for q in queries:
                    ctx.match_host(G, q, pinned)
            e2e_ms += 1000 * (time.perf_counter() - t0)

    max_ms, e2e_step_ms = max_over_ranks([total_ms, e2e_ms / e2e_steps], dist, dev)
    nq_step = len(queries) if sharded else len(queries) * world   # sharded: all ranks serve the same queries
    value = nq_step * args.steps / (max_ms / 1000)
    emb_step_local = emb_total
    if world > 1:
        t = torch.tensor([emb_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t)
        emb_step_local = int(t.item())
    emb_per_s = emb_step_local / (max_ms / 1000)

    kd = by_kernel(st["kernels"])[dominant]
    achieved = kd["bytes"] / (kd["ms"] / 1000) / 1e9 if kd["ms"] > 0 else None
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = peaks.get("hbm_gbs", 6650.0)
    traffic, l2_hit = None, None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        tj = json.load(open(tpath))   # ncu per-launch DRAM bytes / L2 hit rate of the class, per config
        key = f"cfg{CONFIG}:{dominant}"
        traffic = tj.get(key)
        l2_hit = tj.get(f"{key}:l2_hit_pct")

    line = {
        "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "embeddings_per_s": emb_per_s,
        "config": {"workload": WORKLOADS[CONFIG], "queries_per_step_per_gpu": len(queries),
                   "embeddings_per_step": emb_step_local // args.steps,
                   "parallelism": (f"graph replicated on {world} GPU(s), partial-embedding rows sharded "
                                   f"(NCCL all-gather per join step + row rebalancing)") if sharded else
                                  (f"graph replicated, queries sharded over {world} GPU(s); "
                                   f"gps_match_batch: {args.workers} worker streams x {args.slice}-query "
                                   f"batch-synchronous slices per GPU" if batch_api else
                                   f"graph replicated, queries over {world} GPU(s); one query at a time"),
                   "l2": "flushed between timed steps (256 MiB write outside the events)" +
                         ("; the 15 MB graph is L2-resident within a step" if CONFIG != 4 else "")
                         if flush is not None else "not flushed"},
        "gpu_launches": st["launches"] // args.steps * args.steps,
        "launches_per_query": st["launches"] / (len(queries) * args.steps),
        "join_rows_max": st["join_rows_max"], "join_rows_per_step": st["join_rows_total"] // args.steps,
        "roofline": {"bound": "hbm", "kernel": dominant, "kernel_name": KERNEL_NAME.get(dominant, dominant),
                     "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "l2_hit_pct": l2_hit,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)" if "hbm_gbs" in peaks else
                     "fallback 6650 GB/s",
                     "kernel_ms_share_of_step": kd["ms"] / max_ms if max_ms else None,
                     "note": "achieved = algorithmic bytes / CUDA-event time of every launch of this class in "
                             "the timed region (concurrent worker streams: per-launch times include sharing); "
                             "traffic / l2_hit_pct: per-launch ncu --set full capture of this class "
                             "(profiles/traffic.json)",
                     "algorithmic_bytes_per_launch": kd["bytes"] / max(kd["timed"], 1),
                     "isolated": {"achieved": (kd_iso["bytes"] / (kd_iso["ms"] / 1000) / 1e9) if kd_iso["ms"] else None,
                                  "share_of_kernel_time": kd_iso["ms"] / total_iso if total_iso else None,
                                  "how": "one pass of the same step serialised on one stream "
                                         "(the dominant class has the most event time there)",
                                  # every class of that pass with >= 5 % of the kernel time: when
                                  # several are close, the dominant one is a near tie
                                  "classes": {k: {"share": v["ms"] / total_iso,
                                                  "achieved_gbs": v["bytes"] / (v["ms"] / 1000) / 1e9,
                                                  "frac": v["bytes"] / (v["ms"] / 1000) / 1e9 / peak}
                                              for k, v in sorted(iso.items(), key=lambda kv: -kv[1]["ms"])
                                              if total_iso and v["ms"] >= 0.05 * total_iso}}},
        "clocks": clocks,
        "e2e": {"value": nq_step / (e2e_step_ms / 1000), "unit": "queries/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
    }
    if CONFIG == 5:
        # QA serving latency: one query at a time through gps_match, first 500 queries
        lat = []
        with torch.cuda.stream(stream):
            for q in queries[:500]:
                t0 = time.perf_counter()
                t = ctx.match(G, q)
                torch.cuda.synchronize()
                lat.append((time.perf_counter() - t0) * 1e3)
                del t
        lat.sort()
        line["latency_ms"] = {"p50": lat[len(lat) // 2], "p99": lat[int(len(lat) * 0.99)],
                              "how": "host wall clock of single-query gps_match calls (500 queries)"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if CONFIG == 4:
            line["cpu_baseline"] = cfg4_cpu_baseline(g, queries, args.cpu_budget)
        else:
            line["cpu_baseline"] = cpu_baseline(g, queries, args.cpu_budget)
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
