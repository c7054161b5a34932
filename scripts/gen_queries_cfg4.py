"""Generate the config-4 cyclic query set (calls only synth/ and oracle/).

BASELINE configs[3] / SURVEY §8(d): on the 20M-vertex / 100M-arc graph, 6/7/8-vertex
CYCLIC queries (BFS from a top-10% seed expanding the highest-degree neighbours first,
every induced arc with its relation label) whose intermediate tables are large: starting
from the fully labelled query, vertex labels are replaced by '*' one at a time in a
seeded order (a replacement that makes the oracle exceed its limits is undone; the
fully labelled query is tried first) until
the oracle's largest BFS-prefix table (#embeddings of the sub-query induced on a BFS
prefix of >= 2 vertices, oracle.run levels[1:]) reaches PEAK rows; accepted iff that happens with
#Emb <= 10^8.  Every oracle run uses the OpenMP variant on all host cores.  Stored with
the oracle's count, multiset hash and per-depth table sizes; the file is rewritten
after every acceptance, so a run cut short keeps what it found.

Usage: python scripts/gen_queries_cfg4.py OUT.json [n_queries] [seconds] [peak]
(writes synth/data/cfg4_queries.json when OUT.json is that path).  The peak used for the
stored set is 10^8: with wildcard edge labels (or a 10^9 peak) no hub-core query of this
graph finished within the oracle's work limit.  Never touches the CUDA path.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from synth import Query, bfs_query, config_graph  # noqa: E402
from oracle import oracle  # noqa: E402

RECIPE = dict(cfg=4, k=(6, 7, 8), seed0=4000, induced=True, max_children=2, keep_elabels=True,
              prefer_hubs=True, top_fraction=0.1, hi=10**8, work_per_thread=200_000_000)


def peak_of(res) -> int:
    """Largest BFS-prefix table of 2+ vertices (the first level is just the root's candidates:
    all n data vertices when the root is a wildcard)."""
    return max(res["levels"][1:]) if len(res["levels"]) > 1 else 0


def main():
    out_path = sys.argv[1]
    want = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    budget_s = float(sys.argv[3]) if len(sys.argv) > 3 else 2400
    peak = int(float(sys.argv[4])) if len(sys.argv) > 4 else 10**9
    scale = float(os.environ.get("CFG4_SCALE", "1"))
    r = dict(RECIPE, peak=peak, scale=scale)
    threads = os.cpu_count() or 1
    t0 = time.time()
    g = config_graph(4, scale)
    og = oracle.OracleGraph(g)
    print(f"graph + oracle adjacency: {time.time() - t0:.0f} s, {threads} threads", flush=True)
    oracle.set_work_limit(r["work_per_thread"])
    out = []
    seed = r["seed0"]
    while len(out) < want and time.time() - t0 < budget_s:
        k = r["k"][seed % len(r["k"])]
        q = bfs_query(g, k, seed, induced=True, max_children=r["max_children"], p_wild_v=0.0,
                      keep_elabels=r["keep_elabels"], prefer_hubs=r["prefer_hubs"], top_fraction=r["top_fraction"])
        perm = np.random.default_rng(seed + 777).permutation(k)
        vl = list(q.vlabels)
        ts = time.time()
        got = None
        trace = []
        res = oracle.run(og, q, threads=threads, limit=r["hi"])   # the fully labelled query first
        trace.append((-1, res["count"], peak_of(res) if res["count"] >= 0 else -1))
        if res["count"] >= 0 and peak_of(res) >= r["peak"]:
            got = (q, res)
            perm = []
        elif res["count"] < 0:
            perm = []
        for u in perm:
            trial = list(vl)
            trial[int(u)] = -1
            qt = Query(q.k, trial, q.bound, q.edges)
            res = oracle.run(og, qt, threads=threads, limit=r["hi"])
            trace.append((int(u), res["count"], peak_of(res) if res["count"] >= 0 else -1))
            if res["count"] < 0:
                continue
            vl = trial
            if peak_of(res) >= r["peak"]:
                got = (qt, res)
                break
            if time.time() - t0 > budget_s:
                break
        dt = time.time() - ts
        print(f"seed {seed} k={k} arcs={len(q.edges)} {'ACCEPT' if got else 'reject'} {dt:.0f} s {trace}",
              flush=True)
        if got:
            qt, res = got
            out.append({"seed": seed, "query": qt.to_json(), "oracle_count": res["count"],
                        "oracle_hash": str(res["hash"]), "oracle_levels": res["levels"],
                        "oracle_order": res["order"], "oracle_threads": res["threads"],
                        "oracle_seconds": round(dt, 1)})
            with open(out_path, "w") as fh:
                json.dump({"recipe": r, "generator": "scripts/gen_queries_cfg4.py",
                           "counts_from": "oracle/oracle.c (CPU backtracking oracle, OpenMP variant)",
                           "queries": out}, fh)
        seed += 1
    print("accepted", len(out), "in", round(time.time() - t0), "s", flush=True)


if __name__ == "__main__":
    main()
