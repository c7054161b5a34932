"""Generate the stored benchmark query sets (calls only synth/ and oracle/).

cfg2: 6-vertex BFS *tree* queries from top-decile seeds, max 2 children
per BFS expansion, vertex labels kept with prob 0.5 (else '*'), edge labels kept;
accepted iff 10^3 <= #Emb <= 10^6 by the CPU oracle (count with a limit).
Seeds 2000+i in order; the first 100 accepted are stored with their oracle counts.

cfg3: 8/10/12-vertex CYCLIC queries (all induced arcs among the chosen
vertices, wildcard edge labels) from the dense hub core, whose intermediate tables are
large: starting from the fully labelled query, vertex labels are replaced by '*' one
at a time in a seeded order (a replacement that makes the oracle exceed its limits is
undone) until the oracle's largest BFS-prefix table (#embeddings of the sub-query
induced on a BFS prefix, oracle.run levels) reaches 10^7 rows; accepted iff that
happens with #Emb <= 10^8.  10 queries per size.  Stored with the oracle's count,
multiset hash and per-depth table sizes.

Usage: python scripts/gen_queries.py cfg2 [n_queries]
Writes synth/data/<cfg>_queries.json.  Never touches the CUDA path.
"""
import json
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from synth import bfs_query, config_graph  # noqa: E402
from oracle import oracle  # noqa: E402

RECIPES = {
    # configs[1]: 6-vertex BFS trees from top-decile seeds
    "cfg2": dict(cfg=2, k=6, seed0=2000, induced=False, max_children=2, p_wild_v=0.5,
                 lo=10**3, hi=10**6, n=100),
    # configs[2]: 8/10/12-vertex CYCLIC queries from the dense hub core (top 1% seeds, highest-degree
    # neighbours first, induced arcs -- one per vertex pair, wildcard edge labels, vertex labels kept)
    "cfg3": dict(cfg=2, k=(8, 10, 12), seed0=3000, induced=True, max_children=2, p_wild_v=0.0,
                 keep_elabels=False, prefer_hubs=True, top_fraction=0.01, lo=1, hi=10**8, n=30,
                 dial=True, peak=10**7, work=600_000_000, per_size=10),
    # configs[4]: QA batch -- 3..5 vertices, BFS seed bound as a concept node, induced arcs with
    # relation labels, non-bound vertex labels '*' with p = 0.5; every query accepted
    "cfg5": dict(cfg=2, k=(3, 4, 5), seed0=5000, induced=True, max_children=0, p_wild_v=0.5,
                 bind_seed=True, lo=0, hi=10**7, n=10000),
}

_G = None
_OG = None


def _init(cfg):
    global _G, _OG
    _G = config_graph(cfg)
    _OG = oracle.OracleGraph(_G)
    oracle.set_work_limit(300_000_000)   # give up on searches that would take minutes


def _dial(seed, r, k):
    """cfg3: wildcard vertex labels one at a time until the oracle's peak table >= r['peak']."""
    import numpy as np
    from synth import Query
    q = bfs_query(_G, k, seed, induced=r["induced"], max_children=r["max_children"], p_wild_v=0.0,
                  keep_elabels=r.get("keep_elabels", True), prefer_hubs=r.get("prefer_hubs", False),
                  top_fraction=r.get("top_fraction", 0.1))
    oracle.set_work_limit(r["work"])
    perm = np.random.default_rng(seed + 777).permutation(k)
    vl = list(q.vlabels)
    t = time.time()
    for u in perm:
        trial = list(vl)
        trial[int(u)] = -1
        qt = Query(q.k, trial, q.bound, q.edges)
        res = oracle.run(_OG, qt, threads=1, limit=r["hi"])
        if res["count"] < 0:
            continue   # too large for the oracle / over the final bound: keep this label
        vl = trial
        if max(res["levels"]) >= r["peak"]:
            return seed, qt.to_json(), res, time.time() - t
    return seed, None, None, time.time() - t


def _try(args):
    seed, r = args
    k = r["k"] if isinstance(r["k"], int) else r["k"][seed % len(r["k"])]
    if r.get("dial"):
        return _dial(seed, r, k)
    q = bfs_query(_G, k, seed, induced=r["induced"], max_children=r["max_children"],
                  p_wild_v=r["p_wild_v"], keep_elabels=r.get("keep_elabels", True),
                  prefer_hubs=r.get("prefer_hubs", False), top_fraction=r.get("top_fraction", 0.1),
                  bind_seed=r.get("bind_seed", False))
    t = time.time()
    c = oracle.count(_OG, q, limit=r["hi"])
    return seed, q.to_json(), c, time.time() - t


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    r = RECIPES[name]
    want = int(sys.argv[2]) if len(sys.argv) > 2 else r["n"]
    out = []
    seed = r["seed0"]
    if r.get("dial"):   # seeds in order, evaluated in parallel; the first per_size accepted per size
        with mp.Pool(min(8, os.cpu_count() or 1), initializer=_init, initargs=(r["cfg"],)) as pool:
            it = pool.imap(_try, ((s, r) for s in range(seed, seed + 100000)), chunksize=1)
            for s, qj, c, dt in it:
                if qj is not None and sum(1 for x in out if x["query"]["k"] == qj["k"]) < r["per_size"]:
                    out.append({"seed": s, "query": qj, "oracle_count": c["count"], "oracle_hash": str(c["hash"]),
                                "oracle_levels": c["levels"], "oracle_order": c["order"],
                                "oracle_seconds_1thread": round(dt, 2)})
                    print(f"  accept seed {s} k={qj['k']} count={c['count']} peak={max(c['levels'])} "
                          f"({dt:.0f} s)", flush=True)
                elif s % 8 == 0:
                    print(f"  seed {s}: accepted {len(out)}", flush=True)
                if len(out) >= want:
                    pool.terminate()
                    break
    with mp.Pool(min(8, os.cpu_count() or 1), initializer=_init, initargs=(r["cfg"],)) as pool:
        while len(out) < want:
            step = 8 if r.get("dial") else (32 if want <= 1000 else 2048)
            batch = [(s, r) for s in range(seed, seed + step)]
            seed += step
            for s, qj, c, dt in pool.map(_try, batch):
                if r.get("dial"):
                    if qj is None:
                        continue
                    kk = qj["k"]
                    if sum(1 for x in out if x["query"]["k"] == kk) >= r["per_size"]:
                        continue
                    out.append({"seed": s, "query": qj, "oracle_count": c["count"], "oracle_hash": str(c["hash"]),
                                "oracle_levels": c["levels"], "oracle_order": c["order"],
                                "oracle_seconds_1thread": round(dt, 2)})
                    print(f"  accept seed {s} k={kk} count={c['count']} peak={max(c['levels'])}", flush=True)
                    continue
                if r["lo"] <= c <= r["hi"] and len(out) < want:
                    out.append({"seed": s, "query": qj, "oracle_count": c})
            print(f"tried up to seed {seed}, accepted {len(out)}", flush=True)
            if isinstance(r["k"], tuple) and want <= 1000:   # balance sizes: stop a size once it has its share
                pass
    out.sort(key=lambda d: d["seed"])
    path = os.path.join(ROOT, "synth", "data", f"{name}_queries.json")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    with open(path, "w") as fh:
        json.dump({"recipe": {k: v for k, v in r.items()}, "generator": "scripts/gen_queries.py",
                   "counts_from": "oracle/oracle.c (CPU backtracking oracle)", "queries": out}, fh)
    print("wrote", path, len(out))


if __name__ == "__main__":
    main()
