// planner.cpp -- host query plan (a1) and join order (a7); see planner.h.
#include "planner.h"

#include <algorithm>
#include <string>

#include "internal.cuh"

namespace gps {

namespace {
typedef unsigned __int128 u128;

// f(x) + f(y) > f(z) + f(w) on exact rationals deg/freq (reading R14: no float ties)
struct Rat {
    u128 num, den;
};
Rat rat_sum(uint64_t d1, uint64_t f1, uint64_t d2, uint64_t f2) {
    return Rat{(u128)d1 * f2 + (u128)d2 * f1, (u128)f1 * f2};
}
bool rat_gt(const Rat& a, const Rat& b) {
    // a.num / a.den > b.num / b.den ; numerators < 2^71, denominators < 2^64: split to avoid overflow
    // compare a.num * b.den vs b.num * a.den using 256-bit via two 128-bit halves
    auto mul = [](u128 x, u128 y, u128& hi, u128& lo) {
        const u128 M = ((u128)1 << 64) - 1;
        u128 x0 = x & M, x1 = x >> 64, y0 = y & M, y1 = y >> 64;
        u128 p00 = x0 * y0, p01 = x0 * y1, p10 = x1 * y0, p11 = x1 * y1;
        u128 mid = (p00 >> 64) + (p01 & M) + (p10 & M);
        lo = (p00 & M) | (mid << 64);
        hi = p11 + (p01 >> 64) + (p10 >> 64) + (mid >> 64);
    };
    u128 h1, l1, h2, l2;
    mul(a.num, b.den, h1, l1);
    mul(b.num, a.den, h2, l2);
    return h1 != h2 ? h1 > h2 : l1 > l2;
}
bool f_ge(const Plan& p, int u, int v) {  // f(u) >= f(v)
    return (u128)p.deg[u] * p.freq[v] >= (u128)p.deg[v] * p.freq[u];
}
bool f_gt(const Plan& p, int u, int v) {
    return (u128)p.deg[u] * p.freq[v] > (u128)p.deg[v] * p.freq[u];
}
}  // namespace

Plan make_plan(const gps_query* q, uint32_t n, bool undirected, const std::vector<uint64_t>& lab_hist,
               const gps_match_opts& o) {
    if (!q) fail(GPS_EINVAL, "null query");
    Plan p;
    const uint32_t k = q->n_vertices, e = q->n_edges;
    if (k == 0 || k > GPS_MAX_QV) fail(GPS_EINVAL, "query must have 1..32 vertices");
    if (e > GPS_MAX_QE) fail(GPS_EINVAL, "query must have <= 64 arcs");
    if (e > 0 && !q->edges) fail(GPS_EINVAL, "null query edges");
    p.k = (int)k;
    uint32_t adj[GPS_MAX_QV] = {0}, outn[GPS_MAX_QV] = {0}, inn[GPS_MAX_QV] = {0};
    for (uint32_t i = 0; i < e; i++) {
        const gps_qedge& qe = q->edges[i];
        if (qe.src < 0 || qe.dst < 0 || (uint32_t)qe.src >= k || (uint32_t)qe.dst >= k)
            fail(GPS_EINVAL, "query edge endpoint out of range");
        if (qe.src == qe.dst) fail(GPS_EINVAL, "query self-loop");
        if (qe.label < -1) fail(GPS_EINVAL, "query edge label < -1");
        p.arcs.push_back({qe.src, qe.dst, qe.label});
        adj[qe.src] |= 1u << qe.dst;
        adj[qe.dst] |= 1u << qe.src;
        outn[qe.src] |= 1u << qe.dst;
        inn[qe.dst] |= 1u << qe.src;
    }
    for (uint32_t u = 0; u < k; u++) {
        p.vlab[u] = q->vertex_labels ? q->vertex_labels[u] : -1;
        p.bound[u] = q->bound ? q->bound[u] : -1;
        if (p.vlab[u] < -1) fail(GPS_EINVAL, "query vertex label < -1");
        if (p.bound[u] < -1) fail(GPS_EINVAL, "bound id < -1");
        if (p.bound[u] >= (int64_t)n) fail(GPS_EINVAL, "bound data id >= n_vertices");
        p.deg[u] = (uint32_t)__builtin_popcount(adj[u]);
        // Def. 3 degree test, direction-split (reading R12); undirected data is symmetric
        p.qout[u] = undirected ? p.deg[u] : (uint32_t)__builtin_popcount(outn[u]);
        p.qin[u] = undirected ? p.deg[u] : (uint32_t)__builtin_popcount(inn[u]);
        if (p.bound[u] >= 0) p.freq[u] = 1;                      // concept node
        else if (p.vlab[u] < 0) p.freq[u] = n;                   // wildcard: every data vertex
        else p.freq[u] = (uint32_t)p.vlab[u] < lab_hist.size() ? lab_hist[p.vlab[u]] : 0;
        if (p.freq[u] == 0) p.empty = true;
    }
    // connectivity of the undirected skeleton (reading R11)
    if (k > 1) {
        uint32_t seen = 1u, frontier = 1u;
        while (frontier) {
            uint32_t nxt = 0;
            for (uint32_t u = 0; u < k; u++)
                if (frontier >> u & 1u) nxt |= adj[u];
            nxt &= ~seen;
            seen |= nxt;
            frontier = nxt;
        }
        const uint32_t all = k == 32 ? 0xffffffffu : ((1u << k) - 1u);
        if (seen != all) fail(GPS_EDISCONNECTED, "query graph is not connected");
    }
    // ---- spanning tree T and visit order O (reading R13) ----
    p.tparent.assign(k, -1);
    uint32_t inT = 0;
    auto add_vertex_edges = [&](int u) {
        // add u's edges whose other endpoint is not yet in V(T), in increasing id
        for (uint32_t v = 0; v < k; v++)
            if ((adj[u] >> v & 1u) && !(inT >> v & 1u)) {
                inT |= 1u << v;
                p.tparent[v] = u;
                p.discovery.push_back((int)v);
            }
    };
    if (k == 1) {
        p.order.push_back(0);
        p.discovery.push_back(0);
        inT = 1u;
    } else if (o.plan_mode == GPS_PLAN_COMMONSENSE) {
        // P:937-939 (commonsense queries): the concept (bound) node of maximum degree first (no
        // concept node: the vertex of maximum degree); then, among the vertices adjacent to the
        // order, the one with the most neighbours not yet in the order; until the order's edges
        // cover the query graph.  Ties -> lowest id.
        int u = -1;
        for (int x = 0; x < (int)k; x++) {
            const bool cx = p.bound[x] >= 0, cu = u >= 0 && p.bound[u] >= 0;
            if (u < 0 || (cx && !cu) || (cx == cu && p.deg[x] > p.deg[u])) u = x;
        }
        uint32_t inO = 1u << u;
        p.order.push_back(u);
        p.discovery.push_back(u);
        inT |= 1u << u;
        add_vertex_edges(u);
        auto covered = [&]() {
            for (const QArc& a : p.arcs)
                if (!(inO >> a.a & 1u) && !(inO >> a.b & 1u)) return false;
            return true;
        };
        while (!covered()) {
            int pick = -1, best = -1;
            for (int x = 0; x < (int)k; x++) {
                if ((inO >> x & 1u) || !(inT >> x & 1u)) continue;
                const int outside = __builtin_popcount(adj[x] & ~inO);
                if (outside > best) {
                    best = outside;
                    pick = x;
                }
            }
            inO |= 1u << pick;
            p.order.push_back(pick);
            add_vertex_edges(pick);
        }
    } else {
        int best_a = -1, best_b = -1;
        Rat best{0, 1};
        for (int a = 0; a < (int)k; a++)
            for (int b = a + 1; b < (int)k; b++) {
                if (!(adj[a] >> b & 1u)) continue;
                Rat s = rat_sum(p.deg[a], p.freq[a], p.deg[b], p.freq[b]);
                if (best_a < 0 || rat_gt(s, best)) {
                    best = s;
                    best_a = a;
                    best_b = b;
                }
            }
        int u = f_ge(p, best_a, best_b) ? best_a : best_b;
        p.order.push_back(u);
        p.discovery.push_back(u);
        inT |= 1u << u;
        add_vertex_edges(u);
        const uint32_t all = k == 32 ? 0xffffffffu : ((1u << k) - 1u);
        while (inT != all) {
            int pick = -1;
            for (int x = 0; x < (int)k; x++) {
                if (!(inT >> x & 1u)) continue;
                if (!(adj[x] & ~inT)) continue;
                if (pick < 0 || f_gt(p, x, pick)) pick = x;
            }
            p.order.push_back(pick);
            add_vertex_edges(pick);
        }
    }
    // ---- initialisation steps: explore u in O against its T neighbours (Alg. 2) ----
    auto constraints_of = [&](int u, uint32_t nbr_mask) {
        std::vector<Constraint> cs;
        for (int i = 0; i < (int)p.arcs.size(); i++) {
            const QArc& a = p.arcs[i];
            if (a.a == u && (nbr_mask >> a.b & 1u)) cs.push_back({i, a.b, 0});
            else if (a.b == u && (nbr_mask >> a.a & 1u)) cs.push_back({i, a.a, 1});
        }
        return cs;
    };
    for (int u : p.order) {
        uint32_t tn = 0;
        for (uint32_t v = 0; v < k; v++)
            if (p.tparent[v] == u || p.tparent[u] == (int)v) tn |= 1u << v;
        p.init_steps.push_back({u, true, constraints_of(u, tn)});
    }
    // ---- refinement (reading R17) ----
    uint32_t kept = 0;
    for (uint32_t u = 0; u < k; u++)
        if (p.bound[u] >= 0 || p.deg[u] > o.lowconn_threshold) kept |= 1u << u;
    p.until_stable = o.refine_rounds == GPS_REFINE_UNTIL_STABLE;
    const uint32_t rounds = p.until_stable ? 1u : o.refine_rounds;
    for (uint32_t r = 0; r < rounds; r++) {
        std::vector<int> seq = p.discovery;
        if (o.reverse_refine) std::reverse(seq.begin(), seq.end());
        for (int u : seq) {
            if (!(kept >> u & 1u)) continue;
            auto cs = constraints_of(u, kept & adj[u]);
            if (cs.empty()) continue;
            p.refine_steps.push_back({u, false, cs});
        }
    }
    return p;
}

std::vector<JoinStepPlan> make_join_order(const Plan& p, const std::vector<uint64_t>& ec,
                                          const std::vector<int>& seed_dir) {
    std::vector<JoinStepPlan> steps;
    const int E = (int)p.arcs.size();
    if (E == 0) return steps;
    std::vector<char> used(E, 0);
    uint32_t vis = 0;
    auto fuse_closing = [&](JoinStepPlan& st) {
        for (int i = 0; i < E; i++)
            if (!used[i] && (vis >> p.arcs[i].a & 1u) && (vis >> p.arcs[i].b & 1u)) {
                used[i] = 1;
                st.closing.push_back(i);
            }
    };
    int seed = 0;
    for (int i = 1; i < E; i++)
        if (ec[i] < ec[seed]) seed = i;
    {
        JoinStepPlan st;
        st.arc = seed;
        st.key_dir = seed_dir.empty() ? 0 : seed_dir[seed];
        st.key = st.key_dir ? p.arcs[seed].b : p.arcs[seed].a;
        st.nv = st.key_dir ? p.arcs[seed].a : p.arcs[seed].b;
        used[seed] = 1;
        vis |= 1u << p.arcs[seed].a;
        vis |= 1u << p.arcs[seed].b;
        fuse_closing(st);
        steps.push_back(st);
    }
    for (;;) {
        int pick = -1;
        for (int i = 0; i < E; i++) {
            if (used[i]) continue;
            bool va = vis >> p.arcs[i].a & 1u, vb = vis >> p.arcs[i].b & 1u;
            if (va == vb) continue;  // both-visited arcs were fused; unvisited-both not yet reachable
            if (pick < 0 || ec[i] < ec[pick]) pick = i;
        }
        if (pick < 0) break;
        JoinStepPlan st;
        st.arc = pick;
        used[pick] = 1;
        if (vis >> p.arcs[pick].a & 1u) {
            st.key = p.arcs[pick].a;
            st.nv = p.arcs[pick].b;
            st.key_dir = 0;
        } else {
            st.key = p.arcs[pick].b;
            st.nv = p.arcs[pick].a;
            st.key_dir = 1;
        }
        vis |= 1u << st.nv;
        fuse_closing(st);
        steps.push_back(st);
    }
    return steps;
}

}  // namespace gps
