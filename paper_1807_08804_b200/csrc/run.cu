// run.cu -- the batch-synchronous executor of Alg. 1 FilteringAndJoining.
//
// A batch of queries runs phase by phase; every phase is ONE launch for all
// queries (jobs), so launch count and host syncs are per batch, not per query:
//
//   plan (host)            per query: f(u), T, O, refine order (planner.cu)
//   kernel_check                  1 launch                     (a2)
//   filter step s = 0..S-1        collect, prune(+clear), propagate, bit-and (a3-a5)
//   final collect                 1 launch, sync #1 -> |C(u)|   (a3)
//   collect_edge_candidates       count, scan, sync #2 -> #EC(e) -> join order, write (a6, a7)
//   join step s                   seg, count, sync, write      (a8, a9)
//
// Every query's outputs of a phase are concatenated in job order, so one global
// scan / compaction serves the whole batch (two-step output scheme).
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <numeric>

#include "comm.h"
#include "kernels.cuh"
#include "planner.h"
#include "runtime.h"

namespace gps {

namespace {

constexpr size_t kAlign = 256;
constexpr uint32_t kMaxBatch = 512;            // queries per chunk
constexpr size_t kChunkBytes = size_t(6) << 30;  // filter arena budget per chunk
// Output buffer of a single-pass join step: at most this many bytes (and at most the
// step's pairs, an upper bound on its rows); rows past it are produced by a rerun of the
// tail into an exact buffer.  GPS_SINGLE_PASS_BYTES overrides (0 forces count -> write).
double single_pass_bytes() {
    const char* e = std::getenv("GPS_SINGLE_PASS_BYTES");
    return e && *e ? std::atof(e) : 8.0 * (1ull << 30);
}

// Limit on the candidate-edge pairs of one chunk (32-bit value positions); GPS_EC_PAIR_LIMIT
// lowers it (test hook: drives the deferral and per-query overflow paths).
uint64_t ec_pair_limit() {
    const char* e = std::getenv("GPS_EC_PAIR_LIMIT");
    const uint64_t lim = 1ull << 32;
    return e && *e ? std::min<uint64_t>(lim, std::strtoull(e, nullptr, 10)) : lim;
}

// Row budget of a join step (gps_match_opts.row_budget_bytes; 0 = a quarter of the device
// memory, reading R27; a table that fails to allocate below it also goes depth-first).
// The device size is read once per device (cudaMemGetInfo is far too slow per step).
uint64_t step_budget(uint64_t opt) {
    if (opt) return opt;
    static std::mutex mu;
    static std::map<int, uint64_t> total;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    auto it = total.find(dev);
    if (it == total.end()) {
        size_t fr = 0, tot = 0;
        if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
            (void)cudaGetLastError();
            tot = 4ull << 30;
        }
        it = total.emplace(dev, (uint64_t)tot).first;
    }
    return std::max<uint64_t>(it->second / 4, 64ull << 20);
}

struct Carve {
    char* base = nullptr;
    size_t off = 0;
    template <typename T>
    T* take(size_t n) {
        off = (off + kAlign - 1) & ~(kAlign - 1);
        T* p = reinterpret_cast<T*>(base + off);
        off += sizeof(T) * (n ? n : 1);
        return p;
    }
};

// host mirror of pairs_range (pairs.cuh): contiguous share of P items for part b of G
void pairs_range_host(uint64_t P, uint32_t b, uint32_t G, uint64_t& p0, uint64_t& p1) {
    const uint64_t q = P / G, rem = P % G;
    p0 = q * b + (b < rem ? b : rem);
    p1 = p0 + q + (b < rem ? 1 : 0);
}

// Phase tracing: NVTX ranges (visible in any CUDA profiler) and, with GPS_TRACE=1,
// host timestamps of every phase boundary on stderr.
struct Trace {
    bool on = false;
    std::chrono::steady_clock::time_point t0, last;
    explicit Trace(const char* what, size_t nq) {
        const char* e = std::getenv("GPS_TRACE");
        on = e && *e == '1';
        t0 = last = std::chrono::steady_clock::now();
        nvtxRangePushA(what);
        if (on) std::fprintf(stderr, "[gps] %s: %zu queries\n", what, nq);
    }
    void mark(const char* phase) {
        nvtxMarkA(phase);
        if (!on) return;
        auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[gps]   %-28s +%8.1f us  (t=%9.1f us)\n", phase,
                     std::chrono::duration<double, std::micro>(t - last).count(),
                     std::chrono::duration<double, std::micro>(t - t0).count());
        last = t;
    }
    ~Trace() { nvtxRangePop(); }
};

struct QS {                       // one query of a chunk
    uint32_t idx = 0;             // position in the caller's array
    Plan plan;
    int k = 0, E = 0;
    uint32_t cap[GPS_MAX_QV];     // c_array capacity per vertex: min(n, freq(u))
    uint32_t* B = nullptr;
    uint32_t* X = nullptr;
    uint32_t* rp = nullptr;
    uint32_t* carr[GPS_MAX_QV];
    uint32_t* seg[GPS_MAX_QV][2];
    uint32_t* cnt = nullptr;      // k counters, inside the chunk-wide counter array
    uint32_t C[GPS_MAX_QV];
    uint32_t P[GPS_MAX_QV][2];    // out / in pair-space size of C(u) (sum of degrees)
    bool live = true;
    bool stable = false;          // GPS_REFINE_UNTIL_STABLE: the last round removed no candidate
    int ecjob[GPS_MAX_QE][2];
    std::vector<JoinStepPlan> steps;
    int col_of[GPS_MAX_QV];
    uint8_t vert_of_col[GPS_MAX_QV + 1];
    const uint32_t* M = nullptr;
    uint64_t R = 0;
};

struct Chunk {
    gps_ctx* c;
    const gps_graph* g;
    std::vector<QS*> qs;
    Block arena;                  // filter state of every query
    uint32_t* cnt_all = nullptr;  // [Σ k] candidate counts, then [2 Σ k] out/in pair-space sizes
    size_t ncnt = 0;
    std::vector<uint32_t> cnt_base;
    std::vector<DevPtr> keep;     // uploaded job arrays
    float rebalance = 1.10f;      // row-sharded join threshold
    uint64_t budget_opt = 0;      // gps_match_opts.row_budget_bytes
    uint32_t nws = 0, rps = 0;
    uint32_t* Bp(const QS& q, int u) const { return q.B + (size_t)u * nws; }
    uint32_t* Xp(const QS& q, int s) const { return q.X + (size_t)s * nws; }
    uint32_t* rpp(const QS& q, int u) const { return q.rp + (size_t)u * rps; }
};

size_t filter_bytes(const QS& q, uint32_t nws) {
    size_t b = 0;
    b += (size_t)q.k * nws * 4 + (size_t)std::max(q.E, 1) * nws * 4 + (size_t)q.k * (nws + 64) * 4;
    uint32_t maxcap = 1;
    for (int u = 0; u < q.k; u++) {
        b += (size_t)q.cap[u] * 4 + 2 * ((size_t)q.cap[u] + 1) * 4 + 3 * kAlign;
        maxcap = std::max(maxcap, q.cap[u]);
    }
    b += (size_t)maxcap * 8 + 8 * kAlign;
    return b;
}

void carve_all(Chunk& ch, Carve& cv) {
    const uint32_t nws = ch.nws, rps = ch.rps;
    // X first (one memset), then counters (one D2H), then the rest
    for (QS* q : ch.qs) q->X = cv.take<uint32_t>((size_t)std::max(q->E, 1) * nws);
    size_t nc = 0;
    ch.cnt_base.clear();
    for (QS* q : ch.qs) {
        ch.cnt_base.push_back((uint32_t)nc);
        nc += (size_t)q->k;
    }
    ch.cnt_all = cv.take<uint32_t>(3 * nc);   // [counts (nc)][pair-space sizes out/in (2 nc)]
    ch.ncnt = nc;
    for (size_t i = 0; i < ch.qs.size(); i++) ch.qs[i]->cnt = ch.cnt_all + ch.cnt_base[i];
    for (QS* q : ch.qs) {
        q->B = cv.take<uint32_t>((size_t)q->k * nws);
        q->rp = cv.take<uint32_t>((size_t)q->k * rps);
        for (int u = 0; u < q->k; u++) {
            q->carr[u] = cv.take<uint32_t>(q->cap[u]);
            q->seg[u][0] = cv.take<uint32_t>((size_t)q->cap[u] + 1);
            q->seg[u][1] = cv.take<uint32_t>((size_t)q->cap[u] + 1);
        }
    }
}

// kernel_check + initialisation + refinement (stage 0 / 1 / 2).  The end-of-step
// bitmap updates ("posts", B &= AND of a step's X scratch bitmaps) ride on the
// next collect launch of the same vertex (CollectJob.xs); the last step's updates
// are returned in *pending (the caller folds them into its final collect) or, if
// pending is null, applied by a post-only collect launch.
// refine_only: one more refinement round of the queries with mask[qi] != 0 on their current
// bitmaps (every vertex collected by the previous final collect): the fixpoint version of
// P:1008 (GPS_REFINE_UNTIL_STABLE).
void filter_phase(Chunk& ch, int stage, std::vector<CollectJob>* pending = nullptr, bool refine_only = false,
                  const std::vector<char>* mask = nullptr) {
    gps_ctx* c = ch.c;
    const DevGraph& d = ch.g->d;
    if (!refine_only) {
        std::vector<ChkQV> qv;
        for (QS* q : ch.qs)
            for (int u = 0; u < q->k; u++) {
                ChkQV x{};
                x.lab = q->plan.vlab[u];
                x.bound = q->plan.bound[u];
                x.qout = q->plan.qout[u];
                x.qin = q->plan.qin[u];
                x.B = q->B + (size_t)u * d.nws;
                qv.push_back(x);
            }
        const ChkQV* d_qv = upload(c, qv, ch.keep);
        run_check(c, d, d_qv, (uint32_t)qv.size());
        // f3: a graph with an attached compression also applies the weighted candidate test of
        // that level -- never removes a Def. 3 candidate (Theorem 1)
        if (ch.g->cg) run_wcheck(c, ch.g->cg, ch.g->cg_level, d_qv, (uint32_t)qv.size(), false);
        if (stage < 1) return;
    }
    auto in_mask = [&](size_t qi) { return !mask || (*mask)[qi]; };
    auto n_init = [&](const QS* q) { return refine_only ? (size_t)0 : q->plan.init_steps.size(); };
    size_t S = 0;
    for (size_t qi = 0; qi < ch.qs.size(); qi++) {
        if (!in_mask(qi)) continue;
        const QS* q = ch.qs[qi];
        size_t s = n_init(q) + (stage >= 2 ? q->plan.refine_steps.size() : 0);
        S = std::max(S, s);
    }
    // vertices whose candidate array exists (collected by an earlier step: a superset of
    // the current set); a side without one cannot be walked
    std::vector<uint32_t> have(ch.qs.size(), refine_only ? 0xffffffffu : 0u);
    auto job = [&](size_t qi, int A, int Sv, const Constraint& cs, int dir, uint32_t* X) {
        QS* q = ch.qs[qi];
        ExploreJob e{};
        if (have[qi] >> A & 1u) {
            e.candA = q->carr[A];
            e.cntA = q->cnt + A;
            e.segA = q->seg[A][dir];
        }
        if (have[qi] >> Sv & 1u) {
            e.candS = q->carr[Sv];
            e.cntS = q->cnt + Sv;
            e.segS = q->seg[Sv][1 - dir];
        }
        e.BA = ch.Bp(*q, A);
        e.BS = ch.Bp(*q, Sv);
        e.X = X;
        e.lab = q->plan.arcs[cs.arc].lab;
        e.dir = (uint32_t)dir;
        return e;
    };
    struct Staged {
        const CollectJob *cj = nullptr, *cp = nullptr;
        const ExploreJob *ej = nullptr, *pj = nullptr;
        uint32_t* const* xs = nullptr;
        uint32_t ncj = 0, ncp = 0, nej = 0, npj = 0;
    };
    // a post waiting for the next collect launch: B of query qi's vertex v &= AND xs[x0..x1)
    struct Pend {
        size_t qi;
        int v;
        CollectJob job;   // post_only form (B, xs, x0, x1)
    };
    auto post_only = [](uint32_t* B, uint32_t* const* xs, uint32_t x0, uint32_t x1) {
        CollectJob j{B, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
        j.xs = xs;
        j.x0 = x0;
        j.x1 = x1;
        j.post_only = 1;
        return j;
    };
    // fold the pending posts of matching (query, vertex) into jobs; the rest become post-only jobs
    auto fold = [](std::vector<Pend>& pend, std::vector<CollectJob>& jobs, const std::vector<size_t>& job_q,
                   const std::vector<int>& job_u) {
        for (const Pend& p : pend) {
            bool done = false;
            for (size_t i = 0; i < jobs.size() && !done; i++)
                if (!jobs[i].post_only && job_q[i] == p.qi && job_u[i] == p.v && jobs[i].x1 == jobs[i].x0) {
                    jobs[i].xs = p.job.xs;
                    jobs[i].x0 = p.job.x0;
                    jobs[i].x1 = p.job.x1;
                    done = true;
                }
            if (!done) jobs.push_back(p.job);
        }
        pend.clear();
    };
    std::vector<Staged> staged;
    std::vector<Pend> pend;   // posts of the previous step
    for (size_t s = 0; s < S; s++) {
        std::vector<CollectJob> cj;
        std::vector<size_t> cj_q;
        std::vector<int> cj_u;
        std::vector<ExploreJob> ej, pj;
        struct P {
            size_t qi;
            int v;
            uint32_t* B;
            uint32_t x0, x1;
        };
        std::vector<P> post1, post2;
        std::vector<uint32_t*> xs;
        for (size_t qi = 0; qi < ch.qs.size(); qi++) {
            if (!in_mask(qi)) continue;
            QS* q = ch.qs[qi];
            const Plan& p = q->plan;
            const size_t ni = n_init(q);
            const size_t nr = stage >= 2 ? p.refine_steps.size() : 0;
            if (s >= ni + nr) continue;
            const FilterStep& st = s < ni ? p.init_steps[s] : p.refine_steps[s - ni];
            const int u = st.u;
            const uint32_t nc = (uint32_t)st.cons.size();
            if (nc == 0) continue;
            have[qi] |= 1u << u;
            cj.push_back(CollectJob{ch.Bp(*q, u), ch.rpp(*q, u), q->carr[u], q->cnt + u, q->seg[u][0], q->seg[u][1],
                                    nullptr});
            cj_q.push_back(qi);
            cj_u.push_back(u);
            // prune (Alg. 2 lines 14-18): A = u, S = v; X_i = members of C(u) meeting constraint i
            const uint32_t x0 = (uint32_t)xs.size();
            for (uint32_t i = 0; i < nc; i++) {
                const Constraint& cs = st.cons[i];
                ej.push_back(job(qi, u, cs.v, cs, cs.dir, ch.Xp(*q, (int)i)));
                ej.back().freshA = 1;   // u was collected by this step
                xs.push_back(ch.Xp(*q, (int)i));
            }
            post1.push_back(P{qi, u, ch.Bp(*q, u), x0, (uint32_t)xs.size()});
            if (!st.propagate) continue;
            // propagation (lines 19-22, reading R15): A = v, S = u (arcs seen from v: direction flipped)
            std::vector<int> targets;
            for (const Constraint& cs : st.cons)
                if (std::find(targets.begin(), targets.end(), cs.v) == targets.end()) targets.push_back(cs.v);
            for (int v : targets) {
                const uint32_t y0 = (uint32_t)xs.size();
                for (uint32_t i = 0; i < nc; i++) {
                    const Constraint& cs = st.cons[i];
                    if (cs.v != v) continue;
                    pj.push_back(job(qi, v, u, cs, 1 - cs.dir, ch.Xp(*q, (int)i)));
                    pj.back().freshS = 1;   // u is re-collected after its prune
                    xs.push_back(ch.Xp(*q, (int)i));
                }
                post2.push_back(P{qi, v, ch.Bp(*q, v), y0, (uint32_t)xs.size()});
            }
        }
        if (cj.empty()) continue;
        // stage every job array of the step now; the launches below all run after the loop
        // (one host->device copy covers the whole filter phase)
        Staged x;
        x.xs = upload(c, xs, ch.keep);
        fold(pend, cj, cj_q, cj_u);   // the previous step's posts ride on this step's collect
        x.cj = upload(c, cj, ch.keep);
        x.ncj = (uint32_t)cj.size();
        x.ej = upload(c, ej, ch.keep);
        x.nej = (uint32_t)ej.size();
        if (!pj.empty()) {
            // re-collect the pruned vertices (propagation walks only the survivors); their prune
            // posts ride on this re-collect, the other queries' prune posts go with it post-only
            std::vector<CollectJob> cp;
            std::vector<size_t> cp_q;
            std::vector<int> cp_u;
            for (size_t i = 0; i < x.ncj; i++) {
                const CollectJob& y = cj[i];
                if (y.post_only) continue;
                if (std::any_of(pj.begin(), pj.end(), [&](const ExploreJob& e) { return e.candS == y.carr; })) {
                    CollectJob z = y;
                    z.xs = nullptr;
                    z.x0 = z.x1 = 0;
                    cp.push_back(z);
                    cp_q.push_back(cj_q[i]);
                    cp_u.push_back(cj_u[i]);
                }
            }
            std::vector<Pend> p1;
            for (const P& e : post1) p1.push_back(Pend{e.qi, e.v, post_only(e.B, x.xs, e.x0, e.x1)});
            fold(p1, cp, cp_q, cp_u);
            x.cp = upload(c, cp, ch.keep);
            x.ncp = (uint32_t)cp.size();
            x.pj = upload(c, pj, ch.keep);
            x.npj = (uint32_t)pj.size();
            for (const P& e : post2) pend.push_back(Pend{e.qi, e.v, post_only(e.B, x.xs, e.x0, e.x1)});
        } else {   // no propagation: the prune updates ride on the next collect launch
            for (const P& e : post1) pend.push_back(Pend{e.qi, e.v, post_only(e.B, x.xs, e.x0, e.x1)});
        }
        staged.push_back(x);
    }
    const CollectJob* tail = nullptr;
    uint32_t ntail = 0;
    if (!pend.empty()) {
        if (pending) {
            for (const Pend& p : pend) pending->push_back(p.job);
        } else {
            std::vector<CollectJob> t;
            for (const Pend& p : pend) t.push_back(p.job);
            tail = upload(c, t, ch.keep);
            ntail = (uint32_t)t.size();
        }
    }
    for (const Staged& x : staged) {
        run_collect(c, d, x.cj, x.ncj);
        run_explore(c, d, x.ej, x.nej, GPS_K_EXPLORE);
        if (!x.npj) continue;
        run_collect(c, d, x.cp, x.ncp);
        run_explore(c, d, x.pj, x.npj, GPS_K_PROPAGATE);
    }
    if (ntail) run_collect(c, d, tail, ntail);
}

void setup_chunk(Chunk& ch) {
    gps_ctx* c = ch.c;
    ch.nws = ch.g->d.nws;
    ch.rps = ch.g->d.nws + 64;
    Carve sz;
    carve_all(ch, sz);
    const size_t need = sz.off + kAlign;
    if (c->arena_cache && c->arena_cache_bytes >= need && c->arena_cache.use_count() == 1) {
        ch.arena = c->arena_cache;   // the last run is over (arena_reset synced the stream)
    } else {
        c->arena_cache.reset();
        const size_t cap = need + need / 4;
        ch.arena = make_block(c, cap);
        c->arena_cache = ch.arena;
        c->arena_cache_bytes = cap;
    }
    Carve cv;
    cv.base = static_cast<char*>(ch.arena->p);
    carve_all(ch, cv);
    size_t xbytes = 0;
    for (QS* q : ch.qs) xbytes += (size_t)std::max(q->E, 1) * ch.nws * 4;
    // X regions are carved first and back to back (modulo alignment): clear the whole span
    const char* x0 = reinterpret_cast<const char*>(ch.qs.front()->X);
    const char* x1 = reinterpret_cast<const char*>(ch.qs.back()->X) + (size_t)std::max(ch.qs.back()->E, 1) * ch.nws * 4;
    GPS_CK(cudaMemsetAsync((void*)x0, 0, (size_t)(x1 - x0), c->stream));
    (void)xbytes;
}

// Final collect of every query vertex of the chunk (+ the pending posts of the last filter
// step), then one sync: |C(u)| and the out/in pair-space sizes of every vertex to the host.
void final_collect(Chunk& ch, const std::vector<CollectJob>& pend) {
    gps_ctx* c = ch.c;
    const DevGraph& d = ch.g->d;
    std::vector<CollectJob> cj;
    for (size_t i = 0; i < ch.qs.size(); i++) {
        QS* q = ch.qs[i];
        for (int u = 0; u < q->k; u++)
            cj.push_back(CollectJob{ch.Bp(*q, u), ch.rpp(*q, u), q->carr[u], q->cnt + u, q->seg[u][0],
                                    q->seg[u][1], ch.cnt_all + ch.ncnt + 2 * (ch.cnt_base[i] + u)});
    }
    for (const CollectJob& p : pend) {   // every vertex is collected here: each post finds its job
        auto it = std::find_if(cj.begin(), cj.end(), [&](const CollectJob& y) { return y.B == p.B && y.x1 == y.x0; });
        if (it == cj.end()) {
            cj.push_back(p);
        } else {
            it->xs = p.xs;
            it->x0 = p.x0;
            it->x1 = p.x1;
        }
    }
    run_collect(c, d, upload(c, cj, ch.keep), (uint32_t)cj.size());
    const size_t nc = ch.ncnt;
    size_t got = 0;
    uint32_t* h = static_cast<uint32_t*>(pinned_alloc(c, nc * 12, &got));
    GPS_CK(cudaMemcpyAsync(h, ch.cnt_all, nc * 12, cudaMemcpyDeviceToHost, c->stream));
    ctx_sync(c);
    for (size_t i = 0; i < ch.qs.size(); i++) {
        QS* q = ch.qs[i];
        for (int u = 0; u < q->k; u++) {
            const size_t x = ch.cnt_base[i] + u;
            q->C[u] = h[x];
            q->P[u][0] = h[nc + 2 * x];
            q->P[u][1] = h[nc + 2 * x + 1];
        }
    }
    pinned_release(c, h, got);
}

// GPS_REFINE_UNTIL_STABLE (the first two versions): further refinement rounds of the
// queries whose candidate sets still shrank, until none does.
// stop_on_empty: a query with an empty candidate set has no match -- stop refining it (the
// debug entry point refines on, to show the sets the fixpoint reaches).
void refine_to_fixpoint(Chunk& ch, bool stop_on_empty = true) {
    for (int round = 0; round < 1024; round++) {
        std::vector<char> m(ch.qs.size(), 0);
        std::vector<std::vector<uint32_t>> prev(ch.qs.size());
        bool any = false;
        for (size_t i = 0; i < ch.qs.size(); i++) {
            QS* q = ch.qs[i];
            if (!q->plan.until_stable || q->stable || q->plan.refine_steps.empty()) continue;
            bool empty = false;
            for (int u = 0; u < q->k; u++) empty |= q->C[u] == 0;
            if (empty && stop_on_empty) continue;
            m[i] = 1;
            prev[i].assign(q->C, q->C + q->k);
            any = true;
        }
        if (!any) break;
        std::vector<CollectJob> pend2;
        filter_phase(ch, 2, &pend2, true, &m);
        final_collect(ch, pend2);
        for (size_t i = 0; i < ch.qs.size(); i++)
            if (m[i]) ch.qs[i]->stable = std::equal(prev[i].begin(), prev[i].end(), ch.qs[i]->C);
    }
}

// Host copy of n u64 that a collective left in device memory (stream-ordered + sync).
std::vector<uint64_t> d2h_u64(gps_ctx* c, const uint64_t* d, size_t n) {
    size_t got = 0;
    uint64_t* h = static_cast<uint64_t*>(pinned_alloc(c, n * 8 + 8, &got));
    GPS_CK(cudaMemcpyAsync(h, d, n * 8, cudaMemcpyDeviceToHost, c->stream));
    ctx_sync(c);
    std::vector<uint64_t> v(h, h + n);
    pinned_release(c, h, got);
    return v;
}

// A fused closing arc a -> b checks value(tgt) in EC[value(key)] through whichever
// direction of the arc was materialised (dir 0: keyed by a, dir 1: keyed by b).
CloseChk make_close(const Chunk& ch, const QS& q, int ci, int nv,
                    const std::function<const uint32_t*(int)>& ec_off_of) {
    const QArc& a = q.plan.arcs[ci];
    // prefer the direction keyed by the endpoint visited before this step (its segment is a
    // per-row constant the join kernels look up once per row)
    const int pref = a.a == nv ? 1 : 0;
    const int dir = q.ecjob[ci][pref] >= 0 ? pref : 1 - pref;
    const int key = dir ? a.b : a.a, tgt = dir ? a.a : a.b;
    CloseChk x{};
    x.key_new = key == nv;
    x.key_col = x.key_new ? 0u : (uint32_t)q.col_of[key];
    x.tgt_new = tgt == nv;
    x.tgt_col = x.tgt_new ? 0u : (uint32_t)q.col_of[tgt];
    x.Bk = ch.Bp(q, key);
    x.rpk = ch.rpp(q, key);
    x.off = ec_off_of(q.ecjob[ci][dir]);
    return x;
}

// Depth-first join of ONE query from step s on (reading R27): the step's
// pair space is cut into ranges whose output fits the row budget; each range is
// counted, written and carried through the remaining steps before the next range
// starts, so at most one piece per level is alive.  The result set is the same as the
// breadth-first batch path (pieces partition the pair space; the last level's pieces
// are concatenated in pair order).  Used when a step of the batch path would exceed
// the budget or its allocation fails.
struct DeepOut {
    uint64_t count = 0;
    std::vector<std::pair<Block, uint64_t>> pieces;   // final rows (match mode), in pair order
};

void join_deep(Chunk& ch, QS* q, size_t s, const uint32_t* M, uint64_t R, const uint32_t* ec_val,
               const std::function<const uint32_t*(int)>& ec_off_of, uint64_t* blk, bool count_only,
               DeepOut& acc) {
    gps_ctx* c = ch.c;
    const JoinStepPlan& st = q->steps[s];
    const uint32_t w = (uint32_t)s + 1;
    const bool last = s + 1 == q->steps.size();
    const uint32_t G = (uint32_t)c->nsm * 4;
    if (R == 0) return;
    DevPtr jt(c, sizeof(unsigned long long));
    JoinJob j{};
    j.row0 = 0;
    j.M = M;
    j.Bx = ch.Bp(*q, st.key);
    j.rpx = ch.rpp(*q, st.key);
    j.ec_off = ec_off_of(q->ecjob[st.arc][st.key_dir]);
    j.Bn = ch.Bp(*q, st.nv);
    j.total = jt.as<unsigned long long>();
    j.x_col = (uint32_t)q->col_of[st.key];
    std::vector<CloseChk> cl;
    for (int ci : st.closing) cl.push_back(make_close(ch, *q, ci, st.nv, ec_off_of));
    j.nclose = (uint32_t)cl.size();
    j.final_ = last ? 1u : 0u;
    j.nowrite = (last && count_only) ? 1u : 0u;
    if (last) {
        for (uint32_t col = 0; col < w; col++) j.perm[col] = q->vert_of_col[col];
        j.perm[w] = (uint8_t)st.nv;
    }
    for (uint32_t col = 0; col <= w && col < kJoinStageCols; col++)
        j.perm_packed |= (last ? (uint32_t)j.perm[col] : col) << (4 * col);
    DevPtr s0(c, sizeof(uint32_t) * (R + 1));
    DevPtr poff(c, sizeof(uint64_t) * (R + 1));
    JoinStep js{};
    js.w = w;
    js.wout = w + 1;
    js.R = R;
    js.jobs = upload(c, std::vector<JoinJob>{j}, ch.keep);
    js.nj = 1;
    js.cl = cl.empty() ? nullptr : upload(c, cl, ch.keep);
    js.ec_val = ec_val;
    js.s0 = s0.as<uint32_t>();
    js.poff = poff.as<uint64_t>();
    js.ctl = PassCtl{blk, c->d_done, c->d_info};
    run_join_seg(c, js);
    const uint64_t P = d2h_u64(c, js.poff + R, 1)[0];
    if (P == 0) return;
    const int nv = st.nv;
    // one pair range: count -> (split if over budget) -> write -> descend
    std::function<void(uint64_t, uint64_t)> range = [&](uint64_t lo, uint64_t hi) {
        GPS_CK(cudaMemsetAsync(jt.p, 0, sizeof(unsigned long long), c->stream));
        js.plo = lo;
        js.phi = hi;
        run_join_count(c, js, G);
        const uint64_t valid = d2h_u64(c, (const uint64_t*)j.total, 1)[0];
        const uint64_t writes = d2h_u64(c, c->d_info + 1, 1)[0];
        c->stats.k_bytes[GPS_K_JOIN_COUNT] += 4.0 * (double)(hi - lo);
        if (last && count_only) {
            acc.count += valid;
            return;
        }
        if (writes == 0) return;
        const double bytes = 4.0 * (w + 1) * (double)writes;
        const uint64_t budget = step_budget(ch.budget_opt);
        const bool final_rows = last;   // the final rows are the result: never split for the budget
        if (!final_rows && bytes > (double)budget && hi - lo > 1) {
            const uint64_t parts = std::min<uint64_t>(hi - lo, (uint64_t)(bytes / (double)budget) + 1);
            for (uint64_t t = 0; t < parts; t++) {
                uint64_t a, b;
                pairs_range_host(hi - lo, (uint32_t)t, (uint32_t)parts, a, b);
                if (b > a) range(lo + a, lo + b);
            }
            return;
        }
        Block ob;
        try {
            ob = make_block(c, sizeof(uint32_t) * writes * (w + 1));
        } catch (const Error& e) {
            if (e.status != GPS_ENOMEM || final_rows || hi - lo < 2) throw;
            const uint64_t mid = lo + (hi - lo) / 2;   // the table does not fit now: halve it
            range(lo, mid);
            range(mid, hi);
            return;
        }
        // the count pass left this range's per-block offsets in blk: the write pass uses them
        GPS_CK(cudaMemsetAsync(jt.p, 0, sizeof(unsigned long long), c->stream));
        js.out = static_cast<uint32_t*>(ob->p);
        run_join_write(c, js, G);
        c->stats.k_bytes[GPS_K_JOIN_WRITE] += 4.0 * (double)(hi - lo) + 4.0 * (w + 1) * (double)writes;
        if (last) {
            acc.pieces.emplace_back(ob, writes);
            return;
        }
        c->stats.join_rows_max = std::max<uint64_t>(c->stats.join_rows_max, writes);
        c->stats.join_rows_total += writes;
        q->col_of[nv] = (int)w;
        q->vert_of_col[w] = (uint8_t)nv;
        join_deep(ch, q, s + 1, static_cast<const uint32_t*>(ob->p), writes, ec_val, ec_off_of, blk, count_only,
                  acc);
    };
    range(0, P);
}

// Finish a query with join_deep from step s (its input table q->M, q->R).
void finish_deep(Chunk& ch, QS* q, size_t s, const uint32_t* ec_val,
                 const std::function<const uint32_t*(int)>& ec_off_of, uint64_t* blk, bool count_only,
                 QueryResult& r) {
    gps_ctx* c = ch.c;
    DeepOut acc;
    join_deep(ch, q, s, q->M, q->R, ec_val, ec_off_of, blk, count_only, acc);
    q->live = false;
    if (count_only) {
        r.rows = acc.count;
        return;
    }
    uint64_t total = 0;
    for (auto& pc : acc.pieces) total += pc.second;
    r.rows = total;
    if (total == 0) return;
    if (acc.pieces.size() == 1) {
        r.block = acc.pieces[0].first;
    } else {
        const size_t k = (size_t)q->k;
        if (total > (~0ull) / (4ull * k)) fail(GPS_EOVERFLOW, "result size overflows");
        r.block = make_block(c, sizeof(uint32_t) * total * k);   // GPS_ENOMEM: the final rows do not fit
        uint64_t at = 0;
        for (auto& pc : acc.pieces) {
            GPS_CK(cudaMemcpyAsync(static_cast<uint32_t*>(r.block->p) + at * k, pc.first->p,
                                   sizeof(uint32_t) * pc.second * k, cudaMemcpyDeviceToDevice, c->stream));
            at += pc.second;
        }
        acc.pieces.clear();
    }
    r.data = static_cast<const uint32_t*>(r.block->p);
}

// deferred: queries of this chunk whose candidate-edge tables do not fit next to the others'
// (32-bit value positions / tile numbers); the caller runs them in a later chunk.
void run_chunk(gps_ctx* c, const gps_graph* g, std::vector<QS*>& qsv, bool count_only, float thr,
               uint64_t budget_opt, std::vector<QueryResult>& out, std::vector<QS*>& deferred) {
    Trace tr("gps chunk", qsv.size());
    arena_reset(c);   // previous chunks' kernels are complete (their last step synced)
    Chunk ch;
    ch.c = c;
    ch.g = g;
    ch.qs = qsv;
    ch.rebalance = thr;
    ch.budget_opt = budget_opt;
    const DevGraph& d = g->d;
    setup_chunk(ch);
    tr.mark("setup (arena)");
    std::vector<CollectJob> pend;
    filter_phase(ch, 2, &pend);
    tr.mark("filter enqueued");

    // ---- final collect of every query vertex (+ the last filter step's posts), sync #1 ----
    final_collect(ch, pend);
    refine_to_fixpoint(ch);
    tr.mark("sync1 (|C(u)|)");
    for (QS* q : ch.qs) {
        QueryResult& r = out[q->idx];
        r.cols = (uint32_t)q->k;
        for (int u = 0; u < q->k; u++)
            if (q->C[u] == 0) q->live = false;
        if (!q->live) continue;
        if (q->k == 1) {   // single-vertex query: the candidate set is the answer (reading R11)
            r.rows = q->C[0];
            r.global_rows = r.rows;
            if (c->comm && c->comm->rank != 0) r.rows = 0;   // one shard holds it
            if (!count_only) {
                r.block = make_block(c, (size_t)r.rows * 4);
                GPS_CK(cudaMemcpyAsync(r.block->p, q->carr[0], (size_t)r.rows * 4, cudaMemcpyDeviceToDevice,
                                       c->stream));
                r.data = static_cast<const uint32_t*>(r.block->p);
            }
            q->live = false;
        }
    }

    // ---- collect_edge_candidates, sync #2 ----
    // Pass 1 materialises every arc in its cheaper direction (smaller pair space); the
    // count is the same in both, so the join order can be planned from it.  Pass 2
    // adds the other direction only for arcs the join extends from their target.
    std::vector<ECJob> ej;
    std::vector<uint64_t> kc_off;
    uint64_t kc_total = 0, ec_pairs = 0;
    uint32_t ntiles = 0;
    auto add_ec = [&](QS* q, int e, int dir) {
        const QArc& a = q->plan.arcs[e];
        const int key = dir ? a.b : a.a, other = dir ? a.a : a.b;
        q->ecjob[e][dir] = (int)ej.size();
        ECJob j{};
        j.keys = q->carr[key];
        j.nkeys = q->cnt + key;
        j.seg = q->seg[key][dir];
        j.Bq = ch.Bp(*q, other);
        j.lab = a.lab;
        j.dir = (uint32_t)dir;
        j.tile0 = ntiles;
        j.P = q->P[key][dir];
        j.C = q->C[key];
        ec_pairs += j.P;
        const uint64_t nt = (j.P + kEcPairTile - 1) / kEcPairTile;
        if ((uint64_t)ntiles + nt > 0x7fffffffull) fail(GPS_EOVERFLOW, "EC pair space too large");
        ntiles += (uint32_t)nt;
        ej.push_back(j);
        kc_off.push_back(kc_total);
        kc_total += (uint64_t)q->C[key] + 1;
    };
    // the candidate-edge values of the chunk share one array with 32-bit positions and one
    // 31-bit tile numbering: a query that would push either over its limit waits for a later
    // chunk (or, first in its chunk, fails alone with GPS_EOVERFLOW)
    {
        uint64_t pairs = 0, tiles = 0;
        bool first = true;
        for (QS* q : ch.qs) {
            if (!q->live) continue;
            uint64_t qp = 0, qt = 0;
            for (int e = 0; e < q->E; e++) {
                const QArc& a = q->plan.arcs[e];
                const uint64_t p0 = q->P[a.a][0], p1 = q->P[a.b][1];
                qp += p0 + p1;
                qt += (p0 + kEcPairTile - 1) / kEcPairTile + (p1 + kEcPairTile - 1) / kEcPairTile;
            }
            if (pairs + qp >= ec_pair_limit() || tiles + qt > 0x7fffffffull) {
                q->live = false;
                if (first) {
                    out[q->idx].status = GPS_EOVERFLOW;
                    out[q->idx].error = "more than 2^32 candidate-edge pairs in one query";
                } else {
                    deferred.push_back(q);
                }
                continue;
            }
            first = false;
            pairs += qp;
            tiles += qt;
        }
    }
    uint64_t both_dirs = 0;   // value capacity: every pair of both directions (upper bound)
    for (QS* q : ch.qs) {
        if (!q->live) continue;
        for (int e = 0; e < q->E; e++) {
            const QArc& a = q->plan.arcs[e];
            q->ecjob[e][0] = q->ecjob[e][1] = -1;
            add_ec(q, e, q->P[a.b][1] < q->P[a.a][0] ? 1 : 0);
            both_dirs += (uint64_t)q->P[a.a][0] + q->P[a.b][1];
        }
    }
    if (ej.empty()) return;
    if (both_dirs >= (1ull << 32)) fail(GPS_EOVERFLOW, "more than 2^32 candidate-edge pairs in one batch");
    const uint32_t G = (uint32_t)c->nsm * 4;
    // key offsets: capacity for both directions of every arc
    uint64_t kc_cap = 0;
    for (QS* q : ch.qs)
        if (q->live)
            for (int e = 0; e < q->E; e++) kc_cap += (uint64_t)q->C[q->plan.arcs[e].a] + q->C[q->plan.arcs[e].b] + 2;
    DevPtr ecoff(c, sizeof(uint32_t) * (kc_cap + 2));
    DevPtr span(c, sizeof(unsigned long long) * 2 * (2 * ej.size()));
    DevPtr blk(c, sizeof(uint64_t) * (G + 1));
    DevPtr val(c, sizeof(uint32_t) * (both_dirs + 1));
    auto launch_ec = [&](size_t j0, uint64_t base) {
        const uint32_t nj = (uint32_t)(ej.size() - j0);
        if (nj > kMaxJobsPerLaunch) fail(GPS_EINVAL, "internal: EC job list too long");
        for (size_t j = j0; j < ej.size(); j++) {
            ej[j].off = ecoff.as<uint32_t>() + kc_off[j];
            ej[j].span = span.as<unsigned long long>() + 2 * j;
        }
        std::vector<ECJob> part(ej.begin() + j0, ej.end());
        run_ec(c, d, upload(c, part, ch.keep), nj, ntiles, val.as<uint32_t>(), base);
    };
    launch_ec(0, 0);
    const size_t nj1 = ej.size();
    uint64_t ec_values = 0;
    std::vector<uint64_t> ectot(nj1);
    {
        size_t got = 0;
        uint64_t* h = static_cast<uint64_t*>(pinned_alloc(c, 2 * nj1 * 8, &got));
        GPS_CK(cudaMemcpyAsync(h, span.p, 2 * nj1 * 8, cudaMemcpyDeviceToHost, c->stream));
        ctx_sync(c);
        for (size_t j = 0; j < nj1; j++) {
            ectot[j] = h[2 * j + 1] - h[2 * j];
            ec_values = std::max<uint64_t>(ec_values, h[2 * j + 1]);
        }
        pinned_release(c, h, got);
    }
    tr.mark("sync2 (#EC)");
    ntiles = 0;
    for (QS* q : ch.qs) {
        if (!q->live) continue;
        std::vector<uint64_t> cnts(q->E);
        std::vector<int> mdir(q->E);
        for (int e = 0; e < q->E; e++) {
            mdir[e] = q->ecjob[e][0] >= 0 ? 0 : 1;
            cnts[e] = ectot[q->ecjob[e][mdir[e]]];
            if (cnts[e] == 0) q->live = false;   // an edge with no candidate edge: no match
        }
        if (!q->live) continue;
        q->steps = make_join_order(q->plan, cnts, mdir);
        for (const JoinStepPlan& st : q->steps) {
            if (q->ecjob[st.arc][st.key_dir] < 0) add_ec(q, st.arc, st.key_dir);
            // a closing arc is checked fastest keyed by its endpoint visited earlier (one segment
            // per input row instead of a rank lookup per pair): build that direction too unless
            // it costs much more than the one built
            for (int ci : st.closing) {
                const QArc& a = q->plan.arcs[ci];
                const int dir = a.a == st.nv ? 1 : 0;
                if (q->ecjob[ci][dir] >= 0 || std::getenv("GPS_NO_CLOSE_DIR")) continue;
                const int key = dir ? a.b : a.a, okey = dir ? a.a : a.b;
                if ((uint64_t)q->P[key][dir] <= 2ull * q->P[okey][1 - dir] + 65536) add_ec(q, ci, dir);
            }
        }
    }
    if (ej.size() > nj1) launch_ec(nj1, ec_values);
    auto ec_off_of = [&](int job) { return ecoff.as<uint32_t>() + kc_off[job]; };
    tr.mark("join order");

    // ---- combine_edge_candidates: one join step for all queries at a time ----
    for (QS* q : ch.qs) {
        if (!q->live) continue;
        for (int u = 0; u < GPS_MAX_QV; u++) q->col_of[u] = -1;
        const JoinStepPlan& s0 = q->steps[0];
        q->col_of[s0.key] = 0;
        q->vert_of_col[0] = (uint8_t)s0.key;
        q->M = q->carr[s0.key];
        q->R = q->C[s0.key];
    }
    Comm* cm = c->comm;   // row-sharded join (one query)
    DevPtr coll;
    if (cm) coll = DevPtr(c, sizeof(uint64_t) * (4 * (size_t)cm->world * cm->world + 8 * cm->world + 16));
    Block cur;   // holds the previous step's output while its rows are read
    Block recv;  // sharded: rows received by a rebalance
    bool replicated = cm != nullptr;   // sharded: the seed table is the same on every rank
    for (size_t s = 0;; s++) {
        std::vector<QS*> act;
        for (QS* q : ch.qs)
            if (q->live && q->steps.size() > s) act.push_back(q);
        if (act.empty()) break;
        const uint32_t w = (uint32_t)s + 1;
        std::vector<JoinJob> jj;
        std::vector<CloseChk> cl;
        uint64_t R = 0;
        DevPtr jt(c, sizeof(unsigned long long) * act.size());
        JoinStep js{};
        DevPtr s0, poff, imask, woff;
        bool any_write = false, fast = false;
        // job table + seg pass of the queries' current tables (q->M, q->R)
        auto prepare = [&]() {
            jj.clear();
            cl.clear();
            R = 0;
            GPS_CK(cudaMemsetAsync(jt.p, 0, sizeof(unsigned long long) * act.size(), c->stream));
            for (size_t i = 0; i < act.size(); i++) {
                QS* q = act[i];
                const JoinStepPlan& st = q->steps[s];
                JoinJob j{};
                j.row0 = R;
                j.M = q->M;
                j.Bx = ch.Bp(*q, st.key);
                j.rpx = ch.rpp(*q, st.key);
                j.ec_off = ec_off_of(q->ecjob[st.arc][st.key_dir]);
                j.Bn = ch.Bp(*q, st.nv);
                j.total = jt.as<unsigned long long>() + i;
                j.x_col = (uint32_t)q->col_of[st.key];
                j.close0 = (uint32_t)cl.size();
                for (int ci : st.closing) cl.push_back(make_close(ch, *q, ci, st.nv, ec_off_of));
                j.nclose = (uint32_t)st.closing.size();
                const bool last = s + 1 == q->steps.size();
                j.final_ = last ? 1u : 0u;
                j.nowrite = (last && count_only) ? 1u : 0u;
                if (last) {
                    for (uint32_t col = 0; col < w; col++) j.perm[col] = q->vert_of_col[col];
                    j.perm[w] = (uint8_t)st.nv;
                }
                for (uint32_t col = 0; col <= w && col < kJoinStageCols; col++)
                    j.perm_packed |= (last ? (uint32_t)j.perm[col] : col) << (4 * col);
                jj.push_back(j);
                R += q->R;
            }
            if (jj.size() > kMaxJobsPerLaunch) fail(GPS_EINVAL, "internal: join job list too long");
            s0 = DevPtr(c, sizeof(uint32_t) * (R + 1));
            poff = DevPtr(c, sizeof(uint64_t) * (R + 1));
            js = JoinStep{};
            js.w = w;
            js.wout = w + 1;
            js.R = R;
            js.jobs = upload(c, jj, ch.keep);
            js.nj = (uint32_t)jj.size();
            js.cl = cl.empty() ? nullptr : upload(c, cl, ch.keep);
            js.ec_val = val.as<uint32_t>();
            js.s0 = s0.as<uint32_t>();
            js.poff = poff.as<uint64_t>();
            js.ctl = PassCtl{blk.as<uint64_t>(), c->d_done, c->d_info};
            any_write = false;
            for (const JoinJob& x : jj) any_write |= !x.nowrite;
            // closing-free step with narrow rows: the seg pass finds each row's own values in its
            // segment, which fixes every output position -- no count pass, one sync
            fast = cl.empty() && w + 1 <= kJoinStageCols && std::getenv("GPS_NO_FAST_JOIN") == nullptr;
            imask = DevPtr();
            woff = DevPtr();
            if (fast) {
                imask = DevPtr(c, sizeof(uint32_t) * (R + 1));
                woff = DevPtr(c, sizeof(uint64_t) * (R + 1));
                js.fast = 1;
                js.imask = imask.as<uint32_t>();
                js.woff = woff.as<uint64_t>();
            }
            if (R == 0) {   // a rank's share can be empty: the step's totals are 0
                GPS_CK(cudaMemsetAsync(poff.p, 0, sizeof(uint64_t), c->stream));
                if (fast) GPS_CK(cudaMemsetAsync(woff.p, 0, sizeof(uint64_t), c->stream));
            }
            run_join_seg(c, js);
        };
        prepare();
        if (cm) {   // ---- row-sharded join: this rank's share of the step ----
            QS* q = act[0];
            if (replicated) {
                // the seed table is replicated: rank r keeps the rows whose first pair lies in
                // [r*P/N, (r+1)*P/N) (whole rows, so every local path applies unchanged)
                const uint64_t P = d2h_u64(c, js.poff + R, 1)[0];
                uint64_t lo, hi;
                pairs_range_host(P, (uint32_t)cm->rank, (uint32_t)cm->world, lo, hi);
                const uint64_t tg[2] = {lo, hi};
                uint64_t* d_cut = coll.as<uint64_t>();
                run_lower_bound(c, js.poff, R, upload(c, std::vector<uint64_t>(tg, tg + 2), ch.keep), 2, d_cut);
                const std::vector<uint64_t> cut = d2h_u64(c, d_cut, 2);
                const uint64_t i0 = cm->rank == 0 ? 0 : cut[0];
                const uint64_t i1 = cm->rank + 1 == cm->world ? R : cut[1];
                q->M = q->M + i0 * w;
                q->R = i1 > i0 ? i1 - i0 : 0;
                replicated = false;
                prepare();
            } else {
                uint64_t* d_send = coll.as<uint64_t>();
                uint64_t* d_all = d_send + 4 * cm->world;
                cm->allgather_u64(js.poff + R, d_all, 1, c->stream);
                const std::vector<uint64_t> Pall = d2h_u64(c, d_all, cm->world);
                ShardPlan sp = shard_plan(cm->world, cm->rank, Pall.data(), ch.rebalance);
                if (sp.rebalance) {
                    // cut the local rows at the targets' pair boundaries (whole rows), all-gather
                    // the send counts, then one grouped send/recv; received blocks in source-rank
                    // order keep the global row order
                    run_lower_bound(c, js.poff, R, upload(c, sp.local_targets, ch.keep), (uint32_t)cm->world + 1,
                                    d_send);
                    std::vector<uint64_t> cuts = d2h_u64(c, d_send, cm->world + 1);
                    cuts[0] = 0;
                    cuts[cm->world] = R;
                    std::vector<uint64_t> cnt(cm->world);
                    for (int t = 0; t < cm->world; t++) cnt[t] = cuts[t + 1] > cuts[t] ? cuts[t + 1] - cuts[t] : 0;
                    const uint64_t* dc = upload(c, cnt, ch.keep);
                    flush_uploads(c);
                    GPS_CK(cudaMemcpyAsync(d_send, dc, sizeof(uint64_t) * cm->world, cudaMemcpyDeviceToDevice,
                                           c->stream));
                    cm->allgather_u64(d_send, d_all, cm->world, c->stream);
                    const std::vector<uint64_t> mat = d2h_u64(c, d_all, (size_t)cm->world * cm->world);
                    const ShardRecv rv = shard_recv(cm->world, cm->rank, mat.data());
                    Block nb = make_block(c, sizeof(uint32_t) * (rv.total * w + 1));
                    uint32_t* NBp = static_cast<uint32_t*>(nb->p);
                    std::vector<P2POp> ops;
                    for (int t = 0; t < cm->world; t++) {
                        const uint64_t ns = cnt[t], nr = mat[(size_t)t * cm->world + cm->rank];
                        const uint32_t* src = q->M + cuts[t] * w;
                        if (t == cm->rank) {
                            if (ns)
                                GPS_CK(cudaMemcpyAsync(NBp + rv.at[t] * w, src, ns * w * 4, cudaMemcpyDeviceToDevice,
                                                       c->stream));
                            continue;
                        }
                        if (ns || nr) ops.push_back(P2POp{t, src, ns * w * 4, NBp + rv.at[t] * w, nr * w * 4});
                    }
                    cm->exchange(ops, c->stream);
                    recv = nb;   // keeps the received rows; the old table (cur) may go
                    q->M = NBp;
                    q->R = rv.total;
                    prepare();
                }
            }
        }
        const uint64_t budget = cm ? ~0ull : step_budget(ch.budget_opt);   // sharded: no depth-first split
        // the step's tables exceed the row budget (or cannot be allocated): every query of the
        // step finishes depth-first, one pair range at a time (join_deep)
        auto go_deep = [&]() {
            for (QS* q : act)
                finish_deep(ch, q, s, val.as<uint32_t>(), ec_off_of, blk.as<uint64_t>(), count_only, out[q->idx]);
        };
        Block ob;
        bool single = false;
        uint64_t P0 = 0;
        if (fast) {
            GPS_CK(cudaMemcpyAsync(c->d_info, js.poff + R, 8, cudaMemcpyDeviceToDevice, c->stream));
            GPS_CK(cudaMemcpyAsync(c->d_info + 1, js.woff + R, 8, cudaMemcpyDeviceToDevice, c->stream));
        } else {
            P0 = d2h_u64(c, js.poff + R, 1)[0];
            // single pass (no count pass) into a buffer of min(P0 rows (an upper bound), the
            // single-pass byte cap): a step whose rows overflow it reruns only its tail
            const double rowb = 4.0 * (w + 1);
            const double cap_bytes = std::min<double>(single_pass_bytes(), (double)budget);
            single = !any_write || cap_bytes > 0;
            if (single) {
                js.cap = any_write ? std::min<uint64_t>(P0, (uint64_t)(cap_bytes / rowb)) : 0;
                if (js.cap) {
                    try {
                        ob = make_block(c, sizeof(uint32_t) * js.cap * (w + 1));
                    } catch (const Error& e) {
                        if (e.status != GPS_ENOMEM) throw;
                        single = false;   // no room for the buffer: count first
                    }
                    if (ob) js.out = static_cast<uint32_t*>(ob->p);
                }
            }
            if (single) {
                if (P0) run_join_tiles(c, js, P0);
                else GPS_CK(cudaMemsetAsync(c->d_info, 0, 16, c->stream));
            } else {
                js.cap = ~0ull;
                run_join_count(c, js, G);
            }
        }
        std::vector<uint64_t> tot(act.size());
        uint64_t P = 0, writes = 0;
        {
            size_t got = 0;
            uint64_t* h = static_cast<uint64_t*>(pinned_alloc(c, (act.size() + 2) * 8, &got));
            GPS_CK(cudaMemcpyAsync(h, jt.p, act.size() * 8, cudaMemcpyDeviceToHost, c->stream));
            GPS_CK(cudaMemcpyAsync(h + act.size(), c->d_info, 16, cudaMemcpyDeviceToHost, c->stream));
            ctx_sync(c);
            for (size_t i = 0; i < act.size(); i++) tot[i] = h[i];
            P = h[act.size()];
            writes = h[act.size() + 1];
            pinned_release(c, h, got);
        }
        tr.mark(fast ? "join step synced (fast)" : single ? "join step synced (single pass)" : "join step synced");
        if (tr.on)
            std::fprintf(stderr, "[gps]     step %zu: %zu queries, w=%u, rows %llu, pairs %llu, written %llu, closing %zu\n",
                         s, act.size(), w, (unsigned long long)R, (unsigned long long)P, (unsigned long long)writes,
                         cl.size());
        if (writes && (double)writes * 4.0 * (w + 1) > (double)budget && (!single || writes > js.cap)) {
            bool fin = true;   // a step whose written rows are all final results is never split
            for (QS* q : act) fin = fin && s + 1 == q->steps.size();
            if (!fin) {
                go_deep();
                break;
            }
        }
        if (single && writes > js.cap) {
            // the rows overflowed the single-pass buffer: keep the first cap rows, rerun the
            // tail (from the first tile not fully written) into an exact buffer
            Block nb = make_block(c, sizeof(uint32_t) * writes * (w + 1));
            if (js.cap)
                GPS_CK(cudaMemcpyAsync(nb->p, ob->p, sizeof(uint32_t) * js.cap * (w + 1), cudaMemcpyDeviceToDevice,
                                       c->stream));
            run_cap_tile(c, P0, js.cap, c->d_info + 2);
            const std::vector<uint64_t> tp = d2h_u64(c, c->d_info + 2, 2);
            JoinStep rt = js;
            rt.plo = tp[0] * kJoinTilePairs;
            rt.out = static_cast<uint32_t*>(nb->p);
            rt.out_base = tp[1];
            rt.cap = ~0ull;
            run_join_tiles(c, rt, P0 - rt.plo);   // per-job totals are already on the host
            ob = nb;
            c->stats.k_bytes[GPS_K_JOIN_WRITE] += 4.0 * (double)(P0 - rt.plo) + 4.0 * (w + 1) * (double)(writes - tp[1]);
        }
        if (single) {
            c->stats.k_bytes[GPS_K_JOIN_WRITE] += 4.0 * w * (double)R + 4.0 * (double)P + 4.0 * (w + 1) * (double)writes;
        } else {
            if (!fast) c->stats.k_bytes[GPS_K_JOIN_COUNT] += 4.0 * w * (double)R + 4.0 * (double)P;
            if (writes) {
                if (writes > (~0ull) / (4ull * (w + 1))) fail(GPS_EOVERFLOW, "result size overflows");
                bool all_final = true;
                for (QS* q : act) all_final = all_final && s + 1 == q->steps.size();
                try {
                    ob = make_block(c, sizeof(uint32_t) * writes * (w + 1));
                } catch (const Error& e) {
                    if (e.status != GPS_ENOMEM || all_final || cm) throw;
                    go_deep();
                    break;
                }
                js.out = static_cast<uint32_t*>(ob->p);
                if (fast) run_join_fast_write(c, js, P);
                else run_join_write(c, js, G);
                c->stats.k_bytes[GPS_K_JOIN_WRITE] += 4.0 * w * (double)R + 4.0 * (double)P +
                                                      4.0 * (w + 1) * (double)writes;
            }
        }
        // sharded: every rank learns the step's global size (one all-gather of the local total)
        uint64_t global = tot.empty() ? 0 : tot[0];
        if (cm) {
            uint64_t* d_send = coll.as<uint64_t>();
            uint64_t* d_all = d_send + 4 * cm->world;
            GPS_CK(cudaMemcpyAsync(d_send, jt.p, sizeof(uint64_t), cudaMemcpyDeviceToDevice, c->stream));
            cm->allgather_u64(d_send, d_all, 1, c->stream);
            global = 0;
            for (uint64_t x : d2h_u64(c, d_all, cm->world)) global += x;
        }
        uint64_t off = 0;
        for (size_t i = 0; i < act.size(); i++) {
            QS* q = act[i];
            const JoinStepPlan& st = q->steps[s];
            QueryResult& r = out[q->idx];
            const uint64_t t = tot[i];
            const uint64_t gt = cm ? global : t;
            const bool last = s + 1 == q->steps.size();
            const bool wrote = !(last && count_only);
            if (last) {
                r.rows = t;
                r.global_rows = gt;
                if (wrote && t) {
                    r.block = ob;
                    r.data = static_cast<const uint32_t*>(ob->p) + off * (w + 1);
                }
                q->live = false;
            } else if (gt == 0) {
                r.rows = 0;
                r.global_rows = 0;
                q->live = false;
            } else {
                q->M = t ? static_cast<const uint32_t*>(ob->p) + off * (w + 1) : nullptr;
                q->R = t;
                c->stats.join_rows_max = std::max<uint64_t>(c->stats.join_rows_max, gt);
                c->stats.join_rows_total += t;
                q->col_of[st.nv] = (int)w;
                q->vert_of_col[w] = (uint8_t)st.nv;
            }
            if (wrote) off += t;
        }
        cur = ob;   // the previous output block is released once no query reads it
        recv.reset();
    }
}

}  // namespace

void run_queries(gps_ctx* c, const gps_graph* g, const gps_query* qs, uint32_t nq, const gps_match_opts& o,
                 bool count_only, std::vector<QueryResult>& out) {
    out.assign(nq, QueryResult{});
    std::vector<QS> all(nq);
    std::vector<QS*> todo;
    const uint32_t n = g->d.n;
    for (uint32_t i = 0; i < nq; i++) {
        QS& q = all[i];
        q.idx = i;
        out[i].cols = qs[i].n_vertices;
        try {
            q.plan = make_plan(&qs[i], n, g->undirected, g->lab_hist, o);
        } catch (const Error& e) {
            out[i].status = e.status;
            out[i].error = e.msg;
            continue;
        }
        q.k = q.plan.k;
        q.E = (int)q.plan.arcs.size();
        if (q.plan.empty) continue;   // a label no data vertex carries: no candidates
        for (int u = 0; u < q.k; u++) q.cap[u] = (uint32_t)std::min<uint64_t>(n, q.plan.freq[u]);
        todo.push_back(&q);
    }
    // chunk: bounded queries, EC jobs and filter-arena bytes per chunk
    size_t i = 0;
    while (i < todo.size()) {
        std::vector<QS*> chunk;
        size_t bytes = 0, ecj = 0, vtx = 0;
        while (i < todo.size()) {
            QS* q = todo[i];
            size_t b = filter_bytes(*q, g->d.nws);
            const size_t maxb = c->comm ? 1 : kMaxBatch;   // sharded: one query at a time
            if (!chunk.empty() && (chunk.size() >= maxb || bytes + b > kChunkBytes ||
                                   ecj + 2 * (size_t)std::max(q->E, 1) > kMaxJobsPerLaunch || vtx + q->k > kMaxJobsPerLaunch))
                break;
            chunk.push_back(q);
            bytes += b;
            ecj += 2 * (size_t)q->E;
            vtx += (size_t)q->k;
            i++;
        }
        std::vector<QS*> deferred;
        run_chunk(c, g, chunk, count_only, o.rebalance_threshold, o.row_budget_bytes, out, deferred);
        // a deferred query starts the next chunk (where it is first, so it never defers again)
        todo.insert(todo.begin() + (std::ptrdiff_t)i, deferred.begin(), deferred.end());
        for (QS* q : deferred) {
            q->live = true;
            q->stable = false;
        }
    }
    const bool sharded = c->comm != nullptr;
    for (uint32_t j = 0; j < nq; j++)
        if (out[j].status == GPS_OK) {
            if (!sharded) out[j].global_rows = out[j].rows;
            c->stats.queries++;
            c->stats.embeddings += out[j].rows;
        }
}

void run_filter_debug(gps_ctx* c, const gps_graph* g, const gps_query* q, const gps_match_opts& o, int stage,
                      uint32_t* host_bitmaps) {
    QS one;
    one.plan = make_plan(q, g->d.n, g->undirected, g->lab_hist, o);
    one.k = one.plan.k;
    one.E = (int)one.plan.arcs.size();
    for (int u = 0; u < one.k; u++) one.cap[u] = (uint32_t)std::min<uint64_t>(g->d.n, std::max<uint64_t>(1, one.plan.freq[u]));
    arena_reset(c);
    Chunk ch;
    ch.c = c;
    ch.g = g;
    ch.qs = {&one};
    setup_chunk(ch);
    if (stage == 2 && one.plan.until_stable) {
        std::vector<CollectJob> pend;
        filter_phase(ch, stage, &pend);
        final_collect(ch, pend);
        refine_to_fixpoint(ch, false);
    } else {
        filter_phase(ch, stage);
    }
    GPS_CK(cudaMemcpy2DAsync(host_bitmaps, sizeof(uint32_t) * g->d.nw, one.B, sizeof(uint32_t) * ch.nws,
                             sizeof(uint32_t) * g->d.nw, one.k, cudaMemcpyDeviceToHost, c->stream));
    ctx_sync(c);
}

}  // namespace gps
