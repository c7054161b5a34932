// api.cu -- the C-ABI (include/gpsense.h) and the per-query pipeline of Alg. 1
// FilteringAndJoining:
//   P := generate_query_plan(q, g)          host            planner.cu
//   c_set := initialize_node_candidates      k_check/collect/explore  filter.cu
//   refine_node_candidates                   collect + explore(prune)  filter.cu
//   EC(e) := collect_edge_candidates (all e) k_ec count/scan/write    join.cu
//   M := combine_edge_candidates             join order (host) + k_join_* steps
// Host syncs per query: 1 (candidate counts) + 1 (EC totals -> join order)
// + 1 per join step (output size, two-step scheme P:809).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "planner.h"
#include "prims.cuh"

namespace gps {

static thread_local std::string g_err;
void set_last_error(const std::string& m) { g_err = m; }
void fail(gps_status s, const std::string& m) { throw Error{s, m}; }
void check_cuda(cudaError_t e, const char* what, const char* file, int line) {
    if (e == cudaSuccess) return;
    gps_status s = (e == cudaErrorMemoryAllocation) ? GPS_ENOMEM : GPS_ECUDA;
    (void)cudaGetLastError();
    throw Error{s, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" + std::to_string(line) + ")"};
}

cudaEvent_t ctx_event(gps_ctx* c) {
    if (c->event_pool.empty()) {
        cudaEvent_t e;
        GPS_CK(cudaEventCreate(&e));
        return e;
    }
    cudaEvent_t e = c->event_pool.back();
    c->event_pool.pop_back();
    return e;
}
void ctx_harvest(gps_ctx* c) {
    for (auto& t : c->pending) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, t.e0, t.e1) == cudaSuccess) {
            c->stats.k_ms[t.cls] += ms;
            c->stats.k_timed[t.cls]++;
        }
        c->event_pool.push_back(t.e0);
        c->event_pool.push_back(t.e1);
    }
    c->pending.clear();
}
void ctx_sync(gps_ctx* c) {
    GPS_CK(cudaStreamSynchronize(c->stream));
    c->stats.host_syncs++;
    ctx_harvest(c);
}
void* dmalloc(gps_ctx* c, size_t bytes) {
    void* p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, bytes ? bytes : 16, c->stream);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        fail(GPS_ENOMEM, "device allocation of " + std::to_string(bytes) + " bytes failed");
    }
    return p;
}
void dfree(gps_ctx* c, void* p) {
    if (p) (void)cudaFreeAsync(p, c->stream);
}

struct DeviceGuard {
    int prev = -1, want;
    explicit DeviceGuard(int d) : want(d) {
        cudaGetDevice(&prev);
        if (prev != d) GPS_CK(cudaSetDevice(d));
    }
    ~DeviceGuard() {
        if (prev >= 0 && prev != want) cudaSetDevice(prev);
    }
};

template <typename F>
static gps_status guarded(F&& f) {
    try {
        f();
        return GPS_OK;
    } catch (const Error& e) {
        set_last_error(e.msg);
        return e.status;
    } catch (const std::bad_alloc&) {
        set_last_error("host allocation failed");
        return GPS_ENOMEM;
    } catch (...) {
        set_last_error("unexpected internal error");
        return GPS_ECUDA;
    }
}

struct GatherArgs {
    int n;
    const uint32_t* p[GPS_MAX_QE];
};
__global__ void k_gather(GatherArgs a, uint64_t* out) {
    int i = threadIdx.x;
    if (i < a.n) out[i] = *a.p[i];
}

// ------------------------------------------------------------------ filter
struct Filtered {
    Plan plan;
    DevPtr B, X, rp, carr, cnt;
    uint32_t nws = 0, rps = 0, n = 0;
    uint32_t C[GPS_MAX_QV] = {0};
    uint32_t* Bp(int u) const { return B.as<uint32_t>() + (size_t)u * nws; }
    uint32_t* Xp(int s) const { return X.as<uint32_t>() + (size_t)s * nws; }
    uint32_t* rpp(int u) const { return rp.as<uint32_t>() + (size_t)u * rps; }
    uint32_t* carrp(int u) const { return carr.as<uint32_t>() + (size_t)u * n; }
    uint32_t* cntp(int u) const { return cnt.as<uint32_t>() + u; }
};

static void filter_step(gps_ctx* c, const gps_graph* g, Filtered& F, const FilterStep& st) {
    const Plan& p = F.plan;
    CollectArgs ca{};
    ca.nu = 1;
    ca.B[0] = F.Bp(st.u);
    ca.rp[0] = F.rpp(st.u);
    ca.carr[0] = F.carrp(st.u);
    ca.cnt[0] = F.cntp(st.u);
    run_collect(c, g->d, ca);
    ExploreArgs ea{};
    ea.nc = (int)st.cons.size();
    for (int i = 0; i < ea.nc; i++) {
        const Constraint& cs = st.cons[i];
        ea.c[i] = Cons{F.Bp(cs.v), st.propagate ? F.Xp(i) : nullptr, p.arcs[cs.arc].lab, cs.dir};
    }
    ea.cands = F.carrp(st.u);
    ea.cnt = F.cntp(st.u);
    ea.Bu = F.Bp(st.u);
    run_explore(c, g->d, ea, g->d.n);
    if (st.propagate && ea.nc) {
        AndArgs aa{};
        std::vector<int> targets;
        for (const Constraint& cs : st.cons)
            if (std::find(targets.begin(), targets.end(), cs.v) == targets.end()) targets.push_back(cs.v);
        int nx = 0;
        for (int t = 0; t < (int)targets.size(); t++) {
            aa.B[t] = F.Bp(targets[t]);
            aa.xbeg[t] = nx;
            for (int i = 0; i < ea.nc; i++)
                if (st.cons[i].v == targets[t]) aa.X[nx++] = F.Xp(i);
        }
        aa.nt = (int)targets.size();
        aa.xbeg[aa.nt] = nx;
        run_bitand(c, g->d, aa);
    }
}

// stage: 0 = after check, 1 = after initialisation, 2 = after refinement, 3 = + final collect & counts
static void run_filter(gps_ctx* c, const gps_graph* g, Filtered& F, int stage) {
    const Plan& p = F.plan;
    const int k = p.k;
    F.n = g->d.n;
    F.nws = g->d.nws;
    F.rps = g->d.nws + 64;
    F.B = DevPtr(c, sizeof(uint32_t) * (size_t)k * F.nws);
    const size_t nx = std::max<size_t>(p.arcs.size(), 1);
    F.X = DevPtr(c, sizeof(uint32_t) * nx * F.nws);
    F.rp = DevPtr(c, sizeof(uint32_t) * (size_t)k * F.rps);
    F.carr = DevPtr(c, sizeof(uint32_t) * (size_t)k * F.n);
    F.cnt = DevPtr(c, sizeof(uint32_t) * 64);
    GPS_CK(cudaMemsetAsync(F.X.p, 0, sizeof(uint32_t) * nx * F.nws, c->stream));
    QDesc qd{};
    qd.k = k;
    for (int u = 0; u < k; u++) {
        qd.lab[u] = p.vlab[u];
        qd.bound[u] = p.bound[u];
        qd.qout[u] = p.qout[u];
        qd.qin[u] = p.qin[u];
    }
    run_check(c, g->d, qd, F.B.as<uint32_t>());
    if (stage >= 1)
        for (const FilterStep& st : p.init_steps) filter_step(c, g, F, st);
    if (stage >= 2)
        for (const FilterStep& st : p.refine_steps) filter_step(c, g, F, st);
    if (stage >= 3) {
        CollectArgs ca{};
        ca.nu = k;
        for (int u = 0; u < k; u++) {
            ca.B[u] = F.Bp(u);
            ca.rp[u] = F.rpp(u);
            ca.carr[u] = F.carrp(u);
            ca.cnt[u] = F.cntp(u);
        }
        run_collect(c, g->d, ca);
        GPS_CK(cudaMemcpyAsync(c->h_info, F.cnt.p, sizeof(uint32_t) * k, cudaMemcpyDeviceToHost, c->stream));
        ctx_sync(c);
        const uint32_t* h = reinterpret_cast<const uint32_t*>(c->h_info);
        for (int u = 0; u < k; u++) F.C[u] = h[u];
    }
}

// -------------------------------------------------------------- EC tables
struct ECTab {
    DevPtr cnt, off, val;
    uint64_t total = 0;
    int dir = 0;   // 0: keyed by arc source, 1: keyed by arc target
};

static void ec_count(gps_ctx* c, const gps_graph* g, const Filtered& F, std::vector<ECTab>& T,
                     const std::vector<int>& arcs, bool need_totals) {
    const Plan& p = F.plan;
    ECArgs ea{};
    ScanBatch<uint32_t, uint32_t> sb{};
    uint32_t maxk = 0;
    for (int i : arcs) {
        ECTab& t = T[i];
        const QArc& a = p.arcs[i];
        const int key = t.dir ? a.b : a.a, other = t.dir ? a.a : a.b;
        const uint32_t nk = F.C[key];
        t.cnt = DevPtr(c, sizeof(uint32_t) * ((size_t)nk + 1));
        t.off = DevPtr(c, sizeof(uint32_t) * ((size_t)nk + 1));
        ea.a[ea.na++] = ECArc{F.carrp(key), nk, t.dir, a.lab, F.Bp(other), t.cnt.as<uint32_t>(), nullptr, nullptr};
        sb.in[sb.nseg] = t.cnt.as<uint32_t>();
        sb.out[sb.nseg] = t.off.as<uint32_t>();
        sb.n[sb.nseg++] = nk;
        maxk = std::max(maxk, nk);
    }
    run_ec(c, g->d, ea, false, maxk);
    scan_exclusive(c, sb);
    if (need_totals) {
        GatherArgs ga{};
        for (int i : arcs) {
            const QArc& a = p.arcs[i];
            ga.p[ga.n++] = T[i].off.as<uint32_t>() + F.C[T[i].dir ? a.b : a.a];
        }
        launch(c, GPS_K_SCAN, dim3(1), dim3(64), 0, k_gather, ga, c->d_info);
        GPS_CK(cudaMemcpyAsync(c->h_info, c->d_info, sizeof(uint64_t) * ga.n, cudaMemcpyDeviceToHost, c->stream));
        ctx_sync(c);
        for (int j = 0; j < (int)arcs.size(); j++) T[arcs[j]].total = c->h_info[j];
    }
}

static void ec_write(gps_ctx* c, const gps_graph* g, const Filtered& F, std::vector<ECTab>& T) {
    const Plan& p = F.plan;
    ECArgs ea{};
    uint32_t maxk = 0;
    for (int i = 0; i < (int)p.arcs.size(); i++) {
        ECTab& t = T[i];
        const QArc& a = p.arcs[i];
        const int key = t.dir ? a.b : a.a, other = t.dir ? a.a : a.b;
        t.val = DevPtr(c, sizeof(uint32_t) * (t.total + 1));
        ea.a[ea.na++] = ECArc{F.carrp(key), F.C[key], t.dir, a.lab, F.Bp(other), nullptr, t.off.as<uint32_t>(),
                              t.val.as<uint32_t>()};
        maxk = std::max(maxk, F.C[key]);
    }
    run_ec(c, g->d, ea, true, maxk);
}

// ------------------------------------------------------------------- query
struct QueryOut {
    uint64_t rows = 0;
    DevPtr table;                      // R x k, query-vertex order (match mode)
    const uint32_t* borrowed = nullptr;  // k == 1: points into the filter workspace
};

static gps_match_opts resolve_opts(const gps_match_opts* o) {
    gps_match_opts d;
    gps_default_opts(&d);
    return o ? *o : d;
}

// count_only: the last join level is counted, never written (gps_count).
static void run_query(gps_ctx* c, const gps_graph* g, const gps_query* q, const gps_match_opts* opts,
                      bool count_only, Filtered& F, QueryOut& out) {
    const gps_match_opts o = resolve_opts(opts);
    F.plan = make_plan(q, g->d.n, g->undirected, g->lab_hist, o);
    const Plan& p = F.plan;
    out.rows = 0;
    if (p.empty) return;
    run_filter(c, g, F, 3);
    for (int u = 0; u < p.k; u++)
        if (F.C[u] == 0) return;
    if (p.k == 1) {
        out.rows = F.C[0];
        out.borrowed = F.carrp(0);
        return;
    }
    const int E = (int)p.arcs.size();
    std::vector<ECTab> T(E);
    std::vector<int> all(E);
    for (int i = 0; i < E; i++) all[i] = i;
    ec_count(c, g, F, T, all, true);
    std::vector<uint64_t> ecn(E);
    for (int i = 0; i < E; i++) {
        ecn[i] = T[i].total;
        if (ecn[i] == 0) return;   // an edge without candidate edges: no match
    }
    std::vector<JoinStepPlan> steps = make_join_order(p, ecn);
    std::vector<int> redo;
    for (const JoinStepPlan& st : steps)
        if (st.key_dir == 1) {
            T[st.arc].dir = 1;
            redo.push_back(st.arc);
        }
    if (!redo.empty()) ec_count(c, g, F, T, redo, false);  // totals are direction independent
    ec_write(c, g, F, T);

    const uint32_t G = (uint32_t)c->nsm * 8;
    DevPtr blk(c, sizeof(uint64_t) * (G + 1));
    int col_of[GPS_MAX_QV];
    uint8_t vert_of_col[GPS_MAX_QV + 1];
    for (int u = 0; u < GPS_MAX_QV; u++) col_of[u] = -1;
    const JoinStepPlan& s0p = steps[0];
    col_of[s0p.key] = 0;
    vert_of_col[0] = (uint8_t)s0p.key;
    const uint32_t* M = F.carrp(s0p.key);
    DevPtr Mbuf;
    uint64_t R = F.C[s0p.key];
    uint32_t w = 1;
    for (size_t si = 0; si < steps.size(); si++) {
        const JoinStepPlan& st = steps[si];
        const bool last = si + 1 == steps.size();
        StepArgs sa{};
        sa.M = M;
        sa.w = w;
        sa.R = R;
        sa.x_col = (uint32_t)col_of[st.key];
        sa.Bx = F.Bp(st.key);
        sa.rpx = F.rpp(st.key);
        sa.ec_off = T[st.arc].off.as<uint32_t>();
        sa.ec_val = T[st.arc].val.as<uint32_t>();
        sa.nclose = 0;
        for (int ci : st.closing) {
            const QArc& a = p.arcs[ci];   // closing arcs use their source-keyed table (dir 0)
            CloseChk& cl = sa.cl[sa.nclose++];
            cl.key_new = a.a == st.nv;
            cl.key_col = cl.key_new ? 0u : (uint32_t)col_of[a.a];
            cl.tgt_new = a.b == st.nv;
            cl.tgt_col = cl.tgt_new ? 0u : (uint32_t)col_of[a.b];
            cl.Bk = F.Bp(a.a);
            cl.rpk = F.rpp(a.a);
            cl.off = T[ci].off.as<uint32_t>();
            cl.val = T[ci].val.as<uint32_t>();
        }
        DevPtr s0(c, sizeof(uint32_t) * (R + 1));
        DevPtr len(c, sizeof(uint32_t) * (R + 1));
        DevPtr poff(c, sizeof(uint64_t) * (R + 1));
        sa.s0 = s0.as<uint32_t>();
        run_join_len(c, sa, len.as<uint32_t>());
        scan_exclusive1<uint32_t, uint64_t>(c, len.as<uint32_t>(), poff.as<uint64_t>(), R);
        sa.poff = poff.as<uint64_t>();
        sa.blk = blk.as<uint64_t>();
        sa.info = c->d_info;
        sa.done = c->d_done;
        run_join_count(c, sa, G);
        GPS_CK(cudaMemcpyAsync(c->h_info, c->d_info, sizeof(uint64_t) * 2, cudaMemcpyDeviceToHost, c->stream));
        ctx_sync(c);
        const uint64_t P = c->h_info[0], total = c->h_info[1];
        c->stats.k_bytes[GPS_K_JOIN_COUNT] += 4.0 * w * R + 4.0 * P;
        if (total == 0) return;
        if (last && count_only) {
            out.rows = total;
            return;
        }
        const uint32_t wout = w + 1;
        if (total > (~0ull) / (4ull * wout)) fail(GPS_EOVERFLOW, "result size overflows");
        DevPtr tab(c, sizeof(uint32_t) * total * wout);
        sa.out = tab.as<uint32_t>();
        sa.wout = wout;
        sa.final_ = last ? 1 : 0;
        vert_of_col[w] = (uint8_t)st.nv;
        for (uint32_t j = 0; j <= w; j++) sa.perm[j] = vert_of_col[j];
        run_join_write(c, sa, G);
        c->stats.k_bytes[GPS_K_JOIN_WRITE] += 4.0 * w * R + 4.0 * P + 4.0 * wout * total;
        col_of[st.nv] = (int)w;
        w = wout;
        R = total;
        Mbuf = std::move(tab);
        M = Mbuf.as<uint32_t>();
    }
    out.rows = R;
    out.table = std::move(Mbuf);
}

}  // namespace gps

using namespace gps;

extern "C" {

gps_status gps_default_opts(gps_match_opts* o) {
    if (!o) return GPS_EINVAL;
    o->refine_rounds = 1;
    o->reverse_refine = 1;
    o->lowconn_threshold = 1;
    o->result_on_device = 1;
    return GPS_OK;
}

const char* gps_last_error(void) { return g_err.c_str(); }

gps_status gps_create(const gps_ctx_opts* opts, gps_ctx** out) {
    return guarded([&] {
        if (!out) fail(GPS_EINVAL, "null out");
        int dev = opts ? opts->device : 0;
        if (opts && (opts->nccl_comm || opts->world > 1)) fail(GPS_EUNSUPPORTED, "row-sharded join not built yet");
        int ndev = 0;
        GPS_CK(cudaGetDeviceCount(&ndev));
        if (dev < 0 || dev >= ndev) fail(GPS_EINVAL, "bad device ordinal");
        DeviceGuard dg(dev);
        gps_ctx* c = new gps_ctx();
        c->device = dev;
        GPS_CK(cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, dev));
        if (opts && opts->stream) {
            c->stream = (cudaStream_t)opts->stream;
        } else {
            GPS_CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
            c->own_stream = true;
        }
        cudaMemPool_t pool;
        GPS_CK(cudaDeviceGetDefaultMemPool(&pool, dev));
        uint64_t thr = ~0ull;
        GPS_CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
        GPS_CK(cudaMalloc(&c->d_bytes, sizeof(unsigned long long) * GPS_K_NCLASSES));
        GPS_CK(cudaMemset(c->d_bytes, 0, sizeof(unsigned long long) * GPS_K_NCLASSES));
        GPS_CK(cudaMalloc(&c->d_info, sizeof(uint64_t) * 128));
        GPS_CK(cudaMallocHost(&c->h_info, sizeof(uint64_t) * 128));
        GPS_CK(cudaMalloc(&c->d_done, sizeof(unsigned int) * 4));
        GPS_CK(cudaMemset(c->d_done, 0, sizeof(unsigned int) * 4));
        GPS_CK(cudaDeviceSynchronize());
        *out = c;
    });
}

gps_status gps_destroy(gps_ctx* c) {
    if (!c) return GPS_OK;
    return guarded([&] {
        DeviceGuard dg(c->device);
        cudaStreamSynchronize(c->stream);
        for (gps_result* r : c->results) {
            if (r->data && r->on_device) cudaFreeAsync(r->data, c->stream);
            r->data = nullptr;
            r->rows = 0;
            r->ctx = nullptr;
        }
        c->results.clear();
        cudaStreamSynchronize(c->stream);
        for (auto& t : c->pending) {
            c->event_pool.push_back(t.e0);
            c->event_pool.push_back(t.e1);
        }
        for (cudaEvent_t e : c->event_pool) cudaEventDestroy(e);
        cudaFree(c->d_bytes);
        cudaFree(c->d_info);
        cudaFreeHost(c->h_info);
        cudaFree(c->d_done);
        if (c->own_stream) cudaStreamDestroy(c->stream);
        delete c;
    });
}

gps_status gps_load_data_graph(gps_ctx* c, const gps_csr_desc* d, gps_graph** out) {
    return guarded([&] {
        if (!c || !out) fail(GPS_EINVAL, "null ctx/out");
        DeviceGuard dg(c->device);
        gps_graph* g = new gps_graph();
        g->device = c->device;
        try {
            load_graph(c, d, g);
        } catch (...) {
            cudaStreamSynchronize(c->stream);
            free_graph_mem(g);
            delete g;
            throw;
        }
        *out = g;
    });
}

gps_status gps_free_graph(gps_graph* g) {
    if (!g) return GPS_OK;
    return guarded([&] {
        DeviceGuard dg(g->device);
        cudaDeviceSynchronize();
        free_graph_mem(g);
        delete g;
    });
}

gps_status gps_graph_info(const gps_graph* g, uint32_t* n, uint64_t* arcs, uint32_t* nvl, uint32_t* lbits) {
    if (!g) return GPS_EINVAL;
    if (n) *n = g->d.n;
    if (arcs) *arcs = g->m;
    if (nvl) *nvl = g->n_vlabels;
    if (lbits) *lbits = g->d.lbits;
    return GPS_OK;
}

static void check_args(gps_ctx* c, const gps_graph* g, const gps_query* q) {
    if (!c || !g || !q) fail(GPS_EINVAL, "null ctx/graph/query");
    if (g->device != c->device) fail(GPS_EINVAL, "graph and ctx on different devices");
}

gps_status gps_match(gps_ctx* c, const gps_graph* g, const gps_query* q, const gps_match_opts* opts,
                     gps_result** out) {
    return guarded([&] {
        check_args(c, g, q);
        if (!out) fail(GPS_EINVAL, "null out");
        DeviceGuard dg(c->device);
        Filtered F;
        QueryOut qo;
        run_query(c, g, q, opts, false, F, qo);
        const gps_match_opts o = resolve_opts(opts);
        gps_result* r = new gps_result();
        r->rows = qo.rows;
        r->cols = (uint32_t)F.plan.k;
        r->ctx = c;
        const size_t bytes = sizeof(uint32_t) * qo.rows * r->cols;
        if (o.result_on_device) {
            r->on_device = 1;
            if (qo.borrowed) {
                DevPtr cp(c, bytes);
                GPS_CK(cudaMemcpyAsync(cp.p, qo.borrowed, bytes, cudaMemcpyDeviceToDevice, c->stream));
                r->data = static_cast<uint32_t*>(cp.release());
            } else {
                r->data = static_cast<uint32_t*>(qo.table.release());
            }
            if (!r->data) r->data = static_cast<uint32_t*>(dmalloc(c, 16));
            c->results.push_back(r);
            ctx_sync(c);
        } else {
            r->on_device = 0;
            r->data = static_cast<uint32_t*>(std::malloc(bytes ? bytes : 16));
            if (!r->data) {
                delete r;
                fail(GPS_ENOMEM, "host result allocation failed");
            }
            const void* src = qo.borrowed ? (const void*)qo.borrowed : qo.table.p;
            if (bytes) GPS_CK(cudaMemcpyAsync(r->data, src, bytes, cudaMemcpyDeviceToHost, c->stream));
            ctx_sync(c);
        }
        c->stats.queries++;
        c->stats.embeddings += qo.rows;
        *out = r;
    });
}

gps_status gps_match_host(gps_ctx* c, const gps_graph* g, const gps_query* q, const gps_match_opts* opts,
                          uint32_t* host_out, uint64_t cap_rows, uint64_t* rows) {
    return guarded([&] {
        check_args(c, g, q);
        if (!rows) fail(GPS_EINVAL, "null rows");
        DeviceGuard dg(c->device);
        Filtered F;
        QueryOut qo;
        run_query(c, g, q, opts, false, F, qo);
        *rows = qo.rows;
        if (qo.rows > cap_rows) {
            ctx_sync(c);
            fail(GPS_EOVERFLOW, "result has more rows than cap_rows");
        }
        if (qo.rows && !host_out) fail(GPS_EINVAL, "null host_out");
        const size_t bytes = sizeof(uint32_t) * qo.rows * (size_t)F.plan.k;
        const void* src = qo.borrowed ? (const void*)qo.borrowed : qo.table.p;
        if (bytes) GPS_CK(cudaMemcpyAsync(host_out, src, bytes, cudaMemcpyDeviceToHost, c->stream));
        ctx_sync(c);
        c->stats.queries++;
        c->stats.embeddings += qo.rows;
    });
}

gps_status gps_count(gps_ctx* c, const gps_graph* g, const gps_query* q, const gps_match_opts* opts,
                     uint64_t* count) {
    return guarded([&] {
        check_args(c, g, q);
        if (!count) fail(GPS_EINVAL, "null count");
        DeviceGuard dg(c->device);
        Filtered F;
        QueryOut qo;
        run_query(c, g, q, opts, true, F, qo);
        ctx_sync(c);
        c->stats.queries++;
        c->stats.embeddings += qo.rows;
        *count = qo.rows;
    });
}

gps_status gps_result_info(const gps_result* r, uint64_t* rows, uint32_t* cols, const uint32_t** data,
                           int* on_device) {
    if (!r) return GPS_EINVAL;
    if (rows) *rows = r->rows;
    if (cols) *cols = r->cols;
    if (data) *data = r->data;
    if (on_device) *on_device = r->on_device;
    return GPS_OK;
}

void gps_result_free(gps_result* r) {
    if (!r) return;
    if (r->on_device) {
        if (r->ctx) {
            gps_ctx* c = r->ctx;
            DeviceGuard dg(c->device);
            if (r->data) cudaFreeAsync(r->data, c->stream);
            c->results.erase(std::remove(c->results.begin(), c->results.end(), r), c->results.end());
        }
    } else {
        std::free(r->data);
    }
    delete r;
}

gps_status gps_get_stats(gps_ctx* c, gps_stats* out) {
    return guarded([&] {
        if (!c || !out) fail(GPS_EINVAL, "null ctx/out");
        DeviceGuard dg(c->device);
        ctx_sync(c);
        unsigned long long hb[GPS_K_NCLASSES];
        GPS_CK(cudaMemcpy(hb, c->d_bytes, sizeof(hb), cudaMemcpyDeviceToHost));
        *out = c->stats;
        for (int i = 0; i < GPS_K_NCLASSES; i++) out->k_bytes[i] += (double)hb[i];
    });
}

gps_status gps_reset_stats(gps_ctx* c) {
    return guarded([&] {
        if (!c) fail(GPS_EINVAL, "null ctx");
        DeviceGuard dg(c->device);
        ctx_sync(c);
        c->stats = gps_stats{};
        GPS_CK(cudaMemset(c->d_bytes, 0, sizeof(unsigned long long) * GPS_K_NCLASSES));
    });
}

gps_status gps_set_profiling(gps_ctx* c, uint32_t mask) {
    if (!c) return GPS_EINVAL;
    c->prof_mask = mask;
    return GPS_OK;
}

gps_status gps_debug_plan(gps_ctx* c, const gps_graph* g, const gps_query* q, const gps_match_opts* opts,
                          int32_t* order_out, uint32_t* n_order, uint64_t* rank_out) {
    return guarded([&] {
        check_args(c, g, q);
        const gps_match_opts o = resolve_opts(opts);
        Plan p = make_plan(q, g->d.n, g->undirected, g->lab_hist, o);
        if (n_order) *n_order = (uint32_t)p.order.size();
        if (order_out)
            for (size_t i = 0; i < p.order.size(); i++) order_out[i] = p.order[i];
        if (rank_out)
            for (int u = 0; u < p.k; u++) {
                rank_out[2 * u] = p.deg[u];
                rank_out[2 * u + 1] = p.freq[u];
            }
    });
}

gps_status gps_debug_candidates(gps_ctx* c, const gps_graph* g, const gps_query* q, const gps_match_opts* opts,
                                int stage, uint32_t* bitmaps_out) {
    return guarded([&] {
        check_args(c, g, q);
        if (!bitmaps_out) fail(GPS_EINVAL, "null bitmaps_out");
        if (stage < 0 || stage > 2) fail(GPS_EINVAL, "stage must be 0, 1 or 2");
        DeviceGuard dg(c->device);
        const gps_match_opts o = resolve_opts(opts);
        Filtered F;
        F.plan = make_plan(q, g->d.n, g->undirected, g->lab_hist, o);
        run_filter(c, g, F, stage);
        GPS_CK(cudaMemcpy2DAsync(bitmaps_out, sizeof(uint32_t) * g->d.nw, F.B.p, sizeof(uint32_t) * F.nws,
                                 sizeof(uint32_t) * g->d.nw, F.plan.k, cudaMemcpyDeviceToHost, c->stream));
        ctx_sync(c);
    });
}

}  // extern "C"
