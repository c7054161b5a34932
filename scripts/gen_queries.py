"""Generate the stored benchmark query sets (calls only synth/ and oracle/).

cfg2: 6-vertex BFS *tree* queries from top-decile seeds, max 2 children
per BFS expansion, vertex labels kept with prob 0.5 (else '*'), edge labels kept;
accepted iff 10^3 <= #Emb <= 10^6 by the CPU oracle (count with a limit).
Seeds 2000+i in order; the first 100 accepted are stored with their oracle counts.

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
                 keep_elabels=False, prefer_hubs=True, top_fraction=0.01, lo=10**2, hi=10**7, n=30),
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


def _try(args):
    seed, r = args
    k = r["k"] if isinstance(r["k"], int) else r["k"][seed % len(r["k"])]
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
    with mp.Pool(min(8, os.cpu_count() or 1), initializer=_init, initargs=(r["cfg"],)) as pool:
        while len(out) < want:
            step = 32 if want <= 1000 else 2048
            batch = [(s, r) for s in range(seed, seed + step)]
            seed += step
            for s, qj, c, dt in pool.map(_try, batch):
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
