// planner.h -- host query plan (a1) and join order (a7).
//
// PAPER.md §"Query Plan Generation": ranking f(u) = deg(u)/freq(u.label);
// seed edge (u,v) with f(u) >= f(v) and f(u)+f(v) maximal; u starts the visit
// order O; edges of u whose other endpoint is outside V(T) join the spanning
// tree T; repeat from T until no edge remains.  P:641: "The query plan
// generation is the only step that runs on the CPU."  Refinement (P:786-801,
// P:943): simplified graph without low-connectivity nodes, one round, reversed
// order.  Join order: seed = edge with the fewest candidate edges; then
// an unvisited edge with both endpoints visited, else one endpoint visited;
// ties -> fewest candidates.  Readings R12-R20 in DESIGN.md fix the details the
// text leaves open (tie-breaks by lowest index, exact rationals, ...).
#pragma once
#include <stdint.h>

#include <vector>

#include "../../include/gpsense.h"

namespace gps {

struct QArc {
    int a, b;        // arc a -> b
    int32_t lab;     // label or -1
};

struct Constraint {  // one query arc seen from vertex u
    int arc;         // index into Plan::arcs
    int v;           // the other endpoint
    int dir;         // 0: arc u -> v, 1: arc v -> u
};

struct FilterStep {  // explore(u) (init) or prune(u) (refine)
    int u;
    bool propagate;
    std::vector<Constraint> cons;
};

struct Plan {
    int k = 0;
    std::vector<QArc> arcs;
    int32_t vlab[GPS_MAX_QV];
    int64_t bound[GPS_MAX_QV];
    uint32_t qout[GPS_MAX_QV], qin[GPS_MAX_QV];
    uint32_t deg[GPS_MAX_QV];      // #distinct skeleton neighbours
    uint64_t freq[GPS_MAX_QV];     // freq(u.label); bound vertex -> 1
    bool empty = false;            // some query vertex has no data vertex with its label
    std::vector<int> order;        // visit order O
    std::vector<int> discovery;    // order in which vertices entered V(T)
    std::vector<int> tparent;      // parent in T (-1 for the root)
    std::vector<FilterStep> init_steps;
    std::vector<FilterStep> refine_steps;
    bool until_stable = false;     // refine_steps is ONE round, repeated until no set shrinks
};

// Throws gps::Error (GPS_EINVAL / GPS_EDISCONNECTED).
Plan make_plan(const gps_query* q, uint32_t n, bool undirected, const std::vector<uint64_t>& lab_hist,
               const gps_match_opts& o);

struct JoinStepPlan {
    int arc;                 // extension arc (or the seed arc)
    int key;                 // visited endpoint (EC key)
    int nv;                  // vertex added by this step
    int key_dir;             // 0: EC keyed by arc source (out-adjacency), 1: keyed by arc target (in)
    std::vector<int> closing;  // arcs fused into this step (both endpoints visited after it)
};

// Join order from per-arc candidate-edge counts.  seed_dir[e]: the
// direction the seed arc is keyed by if e becomes the seed (the one already built).
std::vector<JoinStepPlan> make_join_order(const Plan& p, const std::vector<uint64_t>& ec_count,
                                          const std::vector<int>& seed_dir);

}  // namespace gps
