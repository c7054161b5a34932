// api.cu -- the C-ABI of include/gpsense.h.  Argument checks and result
// ownership only; the pipeline is run.cu, the runtime ctx.cu.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "comm.h"
#include "kernels.cuh"
#include "planner.h"
#include "runtime.h"

namespace gps {

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

static gps_match_opts resolve_opts(const gps_match_opts* o) {
    gps_match_opts d;
    gps_default_opts(&d);
    return o ? *o : d;
}

static void check_args(gps_ctx* c, const gps_graph* g) {
    if (!c || !g) fail(GPS_EINVAL, "null ctx/graph");
    if (g->device != c->device) fail(GPS_EINVAL, "graph and ctx on different devices");
}

// Wrap one query's outcome as a gps_result owned by ctx c (device rows or pinned host rows).
// owner: the ctx the caller holds (a batch's worker results are re-homed to it, so they
// outlive gps_set_workers and are released on the caller's ctx stream, which the batch
// call ordered after every worker stream).
static gps_result* wrap_result(gps_ctx* c, QueryResult& qr, bool on_device, gps_ctx* owner = nullptr) {
    gps_result* r = new gps_result();
    r->rows = qr.rows;
    r->cols = qr.cols;
    r->ctx = c;
    r->global_rows = qr.global_rows;
    const size_t bytes = sizeof(uint32_t) * qr.rows * qr.cols;
    if (on_device) {
        r->on_device = 1;
        if (qr.block) {
            r->hold = qr.block;
            r->data = const_cast<uint32_t*>(qr.data);
        } else {
            r->hold = make_block(c, 16);
            r->data = static_cast<uint32_t*>(r->hold->p);
        }
    } else {
        r->on_device = 0;
        size_t got = 0;
        r->data = static_cast<uint32_t*>(pinned_alloc(c, bytes ? bytes : 16, &got));
        r->host_bytes = got;
        if (bytes) GPS_CK(cudaMemcpyAsync(r->data, qr.data, bytes, cudaMemcpyDeviceToHost, c->stream));
    }
    if (owner && owner != c) {
        if (r->hold) r->hold->c = owner;   // freed on the owner's stream from now on
        r->ctx = owner;
        std::lock_guard<std::mutex> lk(owner->results_mu);
        owner->results.push_back(r);
    } else {
        std::lock_guard<std::mutex> lk(c->results_mu);
        c->results.push_back(r);
    }
    return r;
}

static void ensure_workers(gps_ctx* c) {
    const uint32_t n = c->nworkers_req ? c->nworkers_req : 2;
    if (c->pool && c->workers.size() == n) return;
    for (uint32_t w = (uint32_t)c->workers.size(); w < n; w++) {
        gps_ctx* sc = new gps_ctx();
        ctx_init(sc, c->device, nullptr);
        sc->prof_mask = c->prof_mask;
        sc->dev_alloc = c->dev_alloc;
        sc->dev_free = c->dev_free;
        sc->alloc_user = c->alloc_user;
        c->workers.push_back(sc);
    }
    c->pool = new WorkerPool((int)n);
}

static void drop_workers(gps_ctx* c) {
    if (c->pool) {
        delete c->pool;
        c->pool = nullptr;
    }
    for (gps_ctx* w : c->workers) {
        ctx_release(w);
        delete w;
    }
    c->workers.clear();
}

// Split the batch into contiguous slices handed out dynamically to the workers;
// each worker runs its slice batch-synchronously on its own stream
// (run_queries).  body(worker ctx, first query, count) fills the outputs.
// A slice whose worker threw reports the error as the status of each of its queries
// (on_fail(lo, cnt, status)); the other slices are unaffected.
static void run_sliced(gps_ctx* c, uint32_t nq, const std::function<void(gps_ctx*, uint32_t, uint32_t)>& body,
                       const std::function<void(uint32_t, uint32_t, gps_status)>& on_fail) {
    if (c->comm) {   // SPMD ranks: every rank walks the batch in the same order
        body(c, 0, nq);
        return;
    }
    ensure_workers(c);
    const uint32_t W = (uint32_t)c->workers.size();
    const uint32_t slice = std::max<uint32_t>(1, std::min<uint32_t>(c->slice ? c->slice : 64, (nq + W - 1) / W));
    if (nq <= slice) {
        // one slice: run it on the caller's ctx and stream.  Handing it to whichever worker is
        // free put consecutive large single-query batches on different streams, and the memory
        // pool then mapped fresh multi-GB blocks instead of reusing the freed ones (0.1-1 s stalls)
        try {
            body(c, 0, nq);
        } catch (const Error& e) {
            on_fail(0, nq, e.status);
            set_last_error(e.msg);
        }
        return;
    }
    cudaEvent_t start;
    GPS_CK(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
    GPS_CK(cudaEventRecord(start, c->stream));
    std::vector<cudaEvent_t> fin(W, nullptr);
    std::vector<Error> errs;
    std::mutex emu;
    std::atomic<uint32_t> next{0};
    c->pool->run([&](int w) {
        gps_ctx* sc = c->workers[w];
        cudaSetDevice(sc->device);
        cudaStreamWaitEvent(sc->stream, start, 0);
        for (;;) {
            const uint32_t lo = next.fetch_add(slice);
            if (lo >= nq) break;
            const uint32_t cnt = std::min(slice, nq - lo);
            try {
                body(sc, lo, cnt);
            } catch (const Error& e) {
                std::lock_guard<std::mutex> lk(emu);
                errs.push_back(e);
                on_fail(lo, cnt, e.status);
            } catch (...) {
                std::lock_guard<std::mutex> lk(emu);
                errs.push_back(Error{GPS_ECUDA, "unexpected internal error in a batch worker"});
                on_fail(lo, cnt, GPS_ECUDA);
            }
        }
        cudaEventCreateWithFlags(&fin[w], cudaEventDisableTiming);
        cudaEventRecord(fin[w], sc->stream);
    });
    for (cudaEvent_t e : fin)
        if (e) {
            cudaStreamWaitEvent(c->stream, e, 0);
            cudaEventDestroy(e);
        }
    cudaEventDestroy(start);
    if (!errs.empty()) set_last_error(errs.front().msg);
}

static std::vector<gps_ctx*> all_ctx(gps_ctx* c) {
    std::vector<gps_ctx*> v{c};
    v.insert(v.end(), c->workers.begin(), c->workers.end());
    return v;
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
    o->rebalance_threshold = 1.10f;
    o->row_budget_bytes = 0;
    o->plan_mode = GPS_PLAN_RANKING;
    return GPS_OK;
}

const char* gps_last_error(void) { return last_error(); }

gps_status gps_create(const gps_ctx_opts* opts, gps_ctx** out) {
    return guarded([&] {
        if (!out) fail(GPS_EINVAL, "null out");
        int dev = opts ? opts->device : 0;
        if (opts && opts->world > 1 && !opts->nccl_comm) fail(GPS_EINVAL, "world > 1 needs an nccl_comm");
        if (opts && opts->nccl_comm && (opts->world < 1 || opts->rank < 0 || opts->rank >= opts->world))
            fail(GPS_EINVAL, "an nccl_comm needs world >= 1 and 0 <= rank < world");
        int ndev = 0;
        GPS_CK(cudaGetDeviceCount(&ndev));
        if (dev < 0 || dev >= ndev) fail(GPS_EINVAL, "bad device ordinal");
        DeviceGuard dg(dev);
        gps_ctx* c = new gps_ctx();
        try {
            ctx_init(c, dev, opts ? (cudaStream_t)opts->stream : nullptr);
            if (opts && (!opts->dev_alloc) != (!opts->dev_free)) fail(GPS_EINVAL, "dev_alloc and dev_free go together");
            if (opts) {
                c->dev_alloc = opts->dev_alloc;
                c->dev_free = opts->dev_free;
                c->alloc_user = opts->alloc_user;
            }
            if (opts && opts->nccl_comm) c->comm = make_nccl_comm(opts->nccl_comm, opts->rank, opts->world);
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

gps_status gps_destroy(gps_ctx* c) {
    if (!c) return GPS_OK;
    return guarded([&] {
        DeviceGuard dg(c->device);
        drop_workers(c);
        ctx_release(c);
        delete c->comm;
        delete c;
    });
}

gps_status gps_result_global_rows(const gps_result* r, uint64_t* g) {
    if (!r || !g) return GPS_EINVAL;
    *g = r->global_rows;
    return GPS_OK;
}

gps_status gps_shard_plan(int world, int rank, const uint64_t* pairs_all, float threshold,
                          uint64_t* local_targets, int* rebalance, uint64_t* total) {
    return guarded([&] {
        if (world < 1 || rank < 0 || rank >= world || !pairs_all) fail(GPS_EINVAL, "bad shard plan arguments");
        const ShardPlan sp = shard_plan(world, rank, pairs_all, threshold);
        if (local_targets) std::copy(sp.local_targets.begin(), sp.local_targets.end(), local_targets);
        if (rebalance) *rebalance = sp.rebalance ? 1 : 0;
        if (total) *total = sp.total;
    });
}

gps_status gps_shard_recv(int world, int rank, const uint64_t* send_matrix, uint64_t* at, uint64_t* total) {
    return guarded([&] {
        if (world < 1 || rank < 0 || rank >= world || !send_matrix) fail(GPS_EINVAL, "bad shard recv arguments");
        const ShardRecv r = shard_recv(world, rank, send_matrix);
        if (at) std::copy(r.at.begin(), r.at.end(), at);
        if (total) *total = r.total;
    });
}

gps_status gps_local_comm_create(int world, gps_local_comm** out) {
    return guarded([&] {
        if (world < 1 || !out) fail(GPS_EINVAL, "world >= 1 and out required");
        *out = new gps_local_comm(world);
    });
}

gps_status gps_local_comm_destroy(gps_local_comm* comm) {
    delete comm;
    return GPS_OK;
}

gps_status gps_create_local_rank(const gps_ctx_opts* opts, gps_local_comm* comm, int rank, gps_ctx** out) {
    return guarded([&] {
        if (!comm || !out || rank < 0 || rank >= comm->hub.world) fail(GPS_EINVAL, "bad local rank");
        int dev = opts ? opts->device : 0;
        DeviceGuard dg(dev);
        gps_ctx* c = new gps_ctx();
        try {
            ctx_init(c, dev, opts ? (cudaStream_t)opts->stream : nullptr);
            c->comm = make_local_comm(&comm->hub, rank);
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

gps_status gps_set_workers(gps_ctx* c, uint32_t n) {
    return guarded([&] {
        if (!c) fail(GPS_EINVAL, "null ctx");
        if (n > 64) fail(GPS_EINVAL, "at most 64 workers");
        if (n == c->nworkers_req && c->pool) return;
        DeviceGuard dg(c->device);
        drop_workers(c);
        c->nworkers_req = n;
    });
}

gps_status gps_set_slice(gps_ctx* c, uint32_t n) {
    if (!c) return GPS_EINVAL;
    c->slice = n;
    return GPS_OK;
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

gps_status gps_match(gps_ctx* c, const gps_graph* g, const gps_query* q, const gps_match_opts* opts,
                     gps_result** out) {
    return guarded([&] {
        check_args(c, g);
        if (!q || !out) fail(GPS_EINVAL, "null query/out");
        DeviceGuard dg(c->device);
        const gps_match_opts o = resolve_opts(opts);
        std::vector<QueryResult> qr;
        run_queries(c, g, q, 1, o, false, qr);
        if (qr[0].status != GPS_OK) fail(qr[0].status, qr[0].error);
        gps_result* r = wrap_result(c, qr[0], o.result_on_device != 0);
        ctx_sync(c);
        *out = r;
    });
}

gps_status gps_match_host(gps_ctx* c, const gps_graph* g, const gps_query* q, const gps_match_opts* opts,
                          uint32_t* host_out, uint64_t cap_rows, uint64_t* rows) {
    return guarded([&] {
        check_args(c, g);
        if (!q || !rows) fail(GPS_EINVAL, "null query/rows");
        DeviceGuard dg(c->device);
        const gps_match_opts o = resolve_opts(opts);
        std::vector<QueryResult> qr;
        run_queries(c, g, q, 1, o, false, qr);
        if (qr[0].status != GPS_OK) fail(qr[0].status, qr[0].error);
        *rows = qr[0].rows;
        if (qr[0].rows > cap_rows) {
            ctx_sync(c);
            fail(GPS_EOVERFLOW, "result has more rows than cap_rows");
        }
        if (qr[0].rows && !host_out) fail(GPS_EINVAL, "null host_out");
        const size_t bytes = sizeof(uint32_t) * qr[0].rows * qr[0].cols;
        if (bytes) GPS_CK(cudaMemcpyAsync(host_out, qr[0].data, bytes, cudaMemcpyDeviceToHost, c->stream));
        ctx_sync(c);
    });
}

gps_status gps_count(gps_ctx* c, const gps_graph* g, const gps_query* q, const gps_match_opts* opts,
                     uint64_t* count) {
    return guarded([&] {
        check_args(c, g);
        if (!q || !count) fail(GPS_EINVAL, "null query/count");
        DeviceGuard dg(c->device);
        const gps_match_opts o = resolve_opts(opts);
        std::vector<QueryResult> qr;
        run_queries(c, g, q, 1, o, true, qr);
        ctx_sync(c);
        if (qr[0].status != GPS_OK) fail(qr[0].status, qr[0].error);
        *count = qr[0].global_rows;   // = rows on one GPU; the sum over ranks when sharded
    });
}

gps_status gps_match_batch(gps_ctx* c, const gps_graph* g, const gps_query* qs, uint32_t nq,
                           const gps_match_opts* opts, gps_result** results, gps_status* statuses) {
    return guarded([&] {
        check_args(c, g);
        if (nq && (!qs || !results)) fail(GPS_EINVAL, "null queries/results");
        DeviceGuard dg(c->device);
        const gps_match_opts o = resolve_opts(opts);
        for (uint32_t i = 0; i < nq; i++) results[i] = nullptr;
        std::vector<gps_status> st(nq, GPS_OK);
        run_sliced(c, nq, [&](gps_ctx* sc, uint32_t lo, uint32_t cnt) {
            std::vector<QueryResult> qr;
            run_queries(sc, g, qs + lo, cnt, o, false, qr);
            for (uint32_t i = 0; i < cnt; i++) {
                st[lo + i] = qr[i].status;
                if (qr[i].status == GPS_OK) results[lo + i] = wrap_result(sc, qr[i], o.result_on_device != 0, c);
            }
            ctx_sync(sc);
        }, [&](uint32_t lo, uint32_t cnt, gps_status e) {
            for (uint32_t i = lo; i < lo + cnt; i++)
                if (!results[i]) st[i] = e;
        });
        gps_status first = GPS_OK;
        for (uint32_t i = 0; i < nq; i++) {
            if (statuses) statuses[i] = st[i];
            if (st[i] != GPS_OK && first == GPS_OK) first = st[i];
        }
        if (first != GPS_OK) fail(first, "some queries of the batch failed (see statuses)");
    });
}

gps_status gps_match_batch_host(gps_ctx* c, const gps_graph* g, const gps_query* qs, uint32_t nq,
                                const gps_match_opts* opts, uint32_t* host_out, uint64_t cap_words,
                                uint64_t* offsets, uint64_t* rows, gps_status* statuses) {
    return guarded([&] {
        check_args(c, g);
        if (nq && (!qs || !offsets || !rows)) fail(GPS_EINVAL, "null queries/offsets/rows");
        DeviceGuard dg(c->device);
        const gps_match_opts o = resolve_opts(opts);
        std::vector<gps_status> st(nq, GPS_OK);
        std::atomic<uint64_t> bump{0};
        std::atomic<bool> overflow{false};
        run_sliced(c, nq, [&](gps_ctx* sc, uint32_t lo, uint32_t cnt) {
            std::vector<QueryResult> qr;
            run_queries(sc, g, qs + lo, cnt, o, false, qr);
            for (uint32_t i = 0; i < cnt; i++) {
                st[lo + i] = qr[i].status;
                const uint64_t words = qr[i].rows * qr[i].cols;
                rows[lo + i] = qr[i].rows;
                const uint64_t at = bump.fetch_add(words);
                offsets[lo + i] = at;
                if (at + words > cap_words) {
                    overflow = true;
                    continue;
                }
                if (words && host_out)
                    GPS_CK(cudaMemcpyAsync(host_out + at, qr[i].data, words * 4, cudaMemcpyDeviceToHost, sc->stream));
            }
            ctx_sync(sc);
        }, [&](uint32_t lo, uint32_t cnt, gps_status e) {
            for (uint32_t i = lo; i < lo + cnt; i++) st[i] = e;
        });
        gps_status first = GPS_OK;
        for (uint32_t i = 0; i < nq; i++) {
            if (statuses) statuses[i] = st[i];
            if (st[i] != GPS_OK && first == GPS_OK) first = st[i];
        }
        if (first != GPS_OK) fail(first, "some queries of the batch failed (see statuses)");
        if (overflow) fail(GPS_EOVERFLOW, "results exceed cap_words");
    });
}

gps_status gps_count_batch(gps_ctx* c, const gps_graph* g, const gps_query* qs, uint32_t nq,
                           const gps_match_opts* opts, uint64_t* counts, gps_status* statuses) {
    return guarded([&] {
        check_args(c, g);
        if (nq && (!qs || !counts)) fail(GPS_EINVAL, "null queries/counts");
        DeviceGuard dg(c->device);
        const gps_match_opts o = resolve_opts(opts);
        std::vector<gps_status> st(nq, GPS_OK);
        run_sliced(c, nq, [&](gps_ctx* sc, uint32_t lo, uint32_t cnt) {
            std::vector<QueryResult> qr;
            run_queries(sc, g, qs + lo, cnt, o, true, qr);
            ctx_sync(sc);
            for (uint32_t i = 0; i < cnt; i++) {
                st[lo + i] = qr[i].status;
                counts[lo + i] = qr[i].global_rows;
            }
        }, [&](uint32_t lo, uint32_t cnt, gps_status e) {
            for (uint32_t i = lo; i < lo + cnt; i++) {
                st[i] = e;
                counts[i] = 0;
            }
        });
        gps_status first = GPS_OK;
        for (uint32_t i = 0; i < nq; i++) {
            if (statuses) statuses[i] = st[i];
            if (st[i] != GPS_OK && first == GPS_OK) first = st[i];
        }
        if (first != GPS_OK) fail(first, "some queries of the batch failed (see statuses)");
    });
}

gps_status gps_load_triples(gps_ctx* c, uint32_t n, uint64_t m, const uint32_t* subj, const uint16_t* rel,
                            const uint32_t* obj, const uint16_t* vlab, uint32_t flags, gps_graph** out) {
    return guarded([&] {
        if (!c || !out) fail(GPS_EINVAL, "null ctx/out");
        if (m && (!subj || !obj)) fail(GPS_EINVAL, "null subject/object");
        // counting sort by subject on the host (input marshalling; the device load sorts and
        // de-duplicates every row)
        std::vector<uint64_t> off((size_t)n + 1, 0);
        for (uint64_t i = 0; i < m; i++) {
            if (subj[i] >= n || obj[i] >= n) fail(GPS_EINVAL, "triple endpoint >= n_vertices");
            off[subj[i] + 1]++;
        }
        for (uint32_t v = 0; v < n; v++) off[v + 1] += off[v];
        std::vector<uint32_t> tgt(m);
        std::vector<uint16_t> lab(rel ? m : 0);
        std::vector<uint64_t> at(off.begin(), off.end() - 1);
        for (uint64_t i = 0; i < m; i++) {
            const uint64_t j = at[subj[i]]++;
            tgt[j] = obj[i];
            if (rel) lab[j] = rel[i];
        }
        gps_csr_desc d{n, m, off.data(), tgt.data(), rel ? lab.data() : nullptr, vlab, flags};
        const gps_status st = gps_load_data_graph(c, &d, out);
        if (st != GPS_OK) fail(st, last_error());
    });
}

static void project_call(gps_ctx* c, const gps_graph* g, const gps_query* q, const gps_match_opts* opts, uint32_t kp,
                         const int32_t* cols, gps_result** out, uint64_t* count) {
    check_args(c, g);
    if (!q) fail(GPS_EINVAL, "null query");
    if (kp && !cols) fail(GPS_EINVAL, "null projection");
    if (c->comm) fail(GPS_EUNSUPPORTED, "projection with a row-sharded ctx");
    DeviceGuard dg(c->device);
    const gps_match_opts o = resolve_opts(opts);
    std::vector<QueryResult> qr;
    run_queries(c, g, q, 1, o, false, qr);
    if (qr[0].status != GPS_OK) fail(qr[0].status, qr[0].error);
    QueryResult pr;
    pr.cols = kp;
    pr.rows = project_unique(c, qr[0].data, qr[0].rows, qr[0].cols, cols, kp, g->d.n ? g->d.n - 1 : 0,
                             out ? &pr.block : nullptr);
    pr.global_rows = pr.rows;
    if (pr.block) pr.data = static_cast<const uint32_t*>(pr.block->p);
    qr.clear();
    if (count) *count = pr.rows;
    if (out) *out = wrap_result(c, pr, o.result_on_device != 0);
    ctx_sync(c);
}

gps_status gps_match_project(gps_ctx* c, const gps_graph* g, const gps_query* q, const gps_match_opts* opts,
                             uint32_t kp, const int32_t* cols, gps_result** out) {
    return guarded([&] {
        if (!out) fail(GPS_EINVAL, "null out");
        project_call(c, g, q, opts, kp, cols, out, nullptr);
    });
}

gps_status gps_count_project(gps_ctx* c, const gps_graph* g, const gps_query* q, const gps_match_opts* opts,
                             uint32_t kp, const int32_t* cols, uint64_t* count) {
    return guarded([&] {
        if (!count) fail(GPS_EINVAL, "null count");
        project_call(c, g, q, opts, kp, cols, nullptr, count);
    });
}

static void named_call(gps_ctx* c, const gps_graph* g, const gps_query* q, const gps_match_opts* opts,
                       const int32_t* edge_var, uint32_t kp, const int32_t* cols, gps_result** out, uint64_t* count) {
    check_args(c, g);
    if (!q) fail(GPS_EINVAL, "null query");
    if (kp && !cols) fail(GPS_EINVAL, "null projection");
    if (c->comm) fail(GPS_EUNSUPPORTED, "named edges with a row-sharded ctx");
    DeviceGuard dg(c->device);
    const gps_match_opts o = resolve_opts(opts);
    QueryResult pr;
    uint32_t V = 0;
    {
        std::vector<int32_t> ids;
        for (uint32_t e = 0; e < q->n_edges && edge_var; e++)
            if (edge_var[e] >= 0) ids.push_back(edge_var[e]);
        std::sort(ids.begin(), ids.end());
        V = (uint32_t)(std::unique(ids.begin(), ids.end()) - ids.begin());
    }
    pr.cols = (kp ? kp : q->n_vertices) + V;
    pr.rows = named_unique(c, g, q, o, edge_var, kp, cols, out ? &pr.block : nullptr);
    pr.global_rows = pr.rows;
    if (pr.block) pr.data = static_cast<const uint32_t*>(pr.block->p);
    if (count) *count = pr.rows;
    if (out) *out = wrap_result(c, pr, o.result_on_device != 0);
    ctx_sync(c);
}

gps_status gps_match_named(gps_ctx* c, const gps_graph* g, const gps_query* q, const gps_match_opts* opts,
                           const int32_t* edge_var, uint32_t kp, const int32_t* cols, gps_result** out) {
    return guarded([&] {
        if (!out) fail(GPS_EINVAL, "null out");
        named_call(c, g, q, opts, edge_var, kp, cols, out, nullptr);
    });
}

gps_status gps_count_named(gps_ctx* c, const gps_graph* g, const gps_query* q, const gps_match_opts* opts,
                           const int32_t* edge_var, uint32_t kp, const int32_t* cols, uint64_t* count) {
    return guarded([&] {
        if (!count) fail(GPS_EINVAL, "null count");
        named_call(c, g, q, opts, edge_var, kp, cols, nullptr, count);
    });
}

// ---- f3 multi-level graph compression --------------------------------------
gps_status gps_compress(gps_ctx* c, const gps_graph* g, uint32_t n_levels, const float* deltas, gps_compressed** out) {
    return guarded([&] {
        check_args(c, g);
        if (!out || (n_levels && !deltas)) fail(GPS_EINVAL, "null argument");
        if (n_levels == 0 || n_levels > 16) fail(GPS_EINVAL, "1..16 compression levels");
        DeviceGuard dg(c->device);
        *out = compress_graph(c, g, n_levels, deltas);
    });
}

gps_status gps_free_compressed(gps_compressed* cg) {
    if (!cg) return GPS_OK;
    free_compressed(cg);
    return GPS_OK;
}

gps_status gps_compressed_info(const gps_compressed* cg, uint32_t level, uint32_t* n_nodes, uint64_t* n_edges_out,
                               uint64_t* n_edges_in) {
    return guarded([&] {
        if (!cg) fail(GPS_EINVAL, "null compression");
        compressed_level_info(cg, level, n_nodes, n_edges_out, n_edges_in);
    });
}

gps_status gps_compressed_fetch(gps_ctx* c, const gps_compressed* cg, uint32_t level, uint32_t* group,
                                uint32_t* label, uint32_t* w_out, uint32_t* w_in, uint64_t* edge_out,
                                uint32_t* weight_out, uint64_t* edge_in, uint32_t* weight_in) {
    return guarded([&] {
        if (!c || !cg) fail(GPS_EINVAL, "null argument");
        DeviceGuard dg(c->device);
        compressed_fetch(c, cg, level, group, label, w_out, w_in, edge_out, weight_out, edge_in, weight_in);
    });
}

gps_status gps_compressed_candidates(gps_ctx* c, const gps_compressed* cg, uint32_t level, const gps_query* q,
                                     uint32_t* bitmaps_out) {
    return guarded([&] {
        if (!c || !cg || !q || !bitmaps_out) fail(GPS_EINVAL, "null argument");
        const gps_graph* g = compressed_graph(cg);
        DeviceGuard dg(c->device);
        const uint32_t k = q->n_vertices;
        if (k == 0 || k > GPS_MAX_QV) fail(GPS_EINVAL, "query size");
        std::vector<std::vector<uint32_t>> outs(k), ins(k);
        for (uint32_t e = 0; e < q->n_edges; e++) {
            const gps_qedge& x = q->edges[e];
            if (x.src < 0 || x.dst < 0 || (uint32_t)x.src >= k || (uint32_t)x.dst >= k) fail(GPS_EINVAL, "edge");
            outs[x.src].push_back((uint32_t)x.dst);
            ins[x.dst].push_back((uint32_t)x.src);
        }
        const uint32_t nws = g->d.nws;
        DevPtr B(c, sizeof(uint32_t) * (size_t)k * nws);
        std::vector<ChkQV> qv(k);
        for (uint32_t u = 0; u < k; u++) {
            auto uniq = [](std::vector<uint32_t> v) {
                std::sort(v.begin(), v.end());
                return (uint32_t)(std::unique(v.begin(), v.end()) - v.begin());
            };
            qv[u].lab = q->vertex_labels ? q->vertex_labels[u] : GPS_ANY;
            qv[u].bound = q->bound ? q->bound[u] : GPS_FREE;
            if (qv[u].bound >= (int64_t)g->d.n) fail(GPS_EINVAL, "bound id out of range");
            qv[u].qout = uniq(outs[u]);
            qv[u].qin = uniq(ins[u]);
            qv[u].B = B.as<uint32_t>() + (size_t)u * nws;
        }
        std::vector<DevPtr> keep;
        run_wcheck(c, cg, level, upload(c, qv, keep), k, true);
        GPS_CK(cudaMemcpy2DAsync(bitmaps_out, sizeof(uint32_t) * g->d.nw, B.p, sizeof(uint32_t) * nws,
                                 sizeof(uint32_t) * g->d.nw, k, cudaMemcpyDeviceToHost, c->stream));
        ctx_sync(c);
    });
}

gps_status gps_graph_attach_compressed(gps_graph* g, const gps_compressed* cg, uint32_t level) {
    return guarded([&] {
        if (!g) fail(GPS_EINVAL, "null graph");
        if (!cg || level == 0) {
            g->cg = nullptr;
            g->cg_level = 0;
            return;
        }
        if (compressed_graph(cg) != g) fail(GPS_EINVAL, "the compression was built from another graph");
        if (level > compressed_levels(cg)) fail(GPS_EINVAL, "compression level out of range");
        g->cg = cg;
        g->cg_level = level;
    });
}

// ---- f4: gSparql relation primitives -------------------------------------
static gps_status rel_call(gps_ctx* c, int op, const uint32_t* as, const uint32_t* ad, uint64_t na, const uint32_t* bs,
                           const uint32_t* bd, uint64_t nb, gps_result** out) {
    return guarded([&] {
        if (!c || !out) fail(GPS_EINVAL, "null argument");
        DeviceGuard dg(c->device);
        QueryResult qr;
        relation_op(c, op, as, ad, na, bs, bd, nb, qr);
        *out = wrap_result(c, qr, true);
    });
}
gps_status gps_rel_join(gps_ctx* c, const uint32_t* r_src, const uint32_t* r_dst, uint64_t nr, const uint32_t* s_src,
                        const uint32_t* s_dst, uint64_t ns, gps_result** out) {
    return rel_call(c, 0, r_src, r_dst, nr, s_src, s_dst, ns, out);
}
gps_status gps_rel_union(gps_ctx* c, const uint32_t* a_src, const uint32_t* a_dst, uint64_t na, const uint32_t* b_src,
                         const uint32_t* b_dst, uint64_t nb, gps_result** out) {
    return rel_call(c, 1, a_src, a_dst, na, b_src, b_dst, nb, out);
}
gps_status gps_rel_difference(gps_ctx* c, const uint32_t* a_src, const uint32_t* a_dst, uint64_t na,
                              const uint32_t* b_src, const uint32_t* b_dst, uint64_t nb, gps_result** out) {
    return rel_call(c, 2, a_src, a_dst, na, b_src, b_dst, nb, out);
}
gps_status gps_rel_closure(gps_ctx* c, const uint32_t* src, const uint32_t* dst, uint64_t n, uint32_t max_rounds,
                           gps_result** out, uint32_t* rounds) {
    return guarded([&] {
        if (!c || !out) fail(GPS_EINVAL, "null argument");
        DeviceGuard dg(c->device);
        QueryResult qr;
        relation_closure(c, src, dst, n, max_rounds, qr, rounds);
        *out = wrap_result(c, qr, true);
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

void gps_result_free_after(gps_result* r, void* stream) {
    if (!r) return;
    if (r->ctx) {
        gps_ctx* c = r->ctx;
        int prev = -1;
        cudaGetDevice(&prev);
        if (prev != c->device) cudaSetDevice(c->device);
        if (r->on_device && stream && (cudaStream_t)stream != c->stream) {
            // the consumer's stream may still be reading the rows: order the release after it
            cudaEvent_t e;
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess) {
                cudaEventRecord(e, (cudaStream_t)stream);
                cudaStreamWaitEvent(c->stream, e, 0);
                cudaEventDestroy(e);
            } else {
                (void)cudaGetLastError();
                cudaStreamSynchronize((cudaStream_t)stream);
            }
        }
        if (r->on_device) r->hold.reset();
        else pinned_release(c, r->data, r->host_bytes);
        {
            std::lock_guard<std::mutex> lk(c->results_mu);
            c->results.erase(std::remove(c->results.begin(), c->results.end(), r), c->results.end());
        }
        if (prev >= 0 && prev != c->device) cudaSetDevice(prev);
    }
    delete r;
}

void gps_result_free(gps_result* r) { gps_result_free_after(r, nullptr); }

gps_status gps_get_stats(gps_ctx* c, gps_stats* out) {
    return guarded([&] {
        if (!c || !out) fail(GPS_EINVAL, "null ctx/out");
        DeviceGuard dg(c->device);
        *out = gps_stats{};
        for (gps_ctx* x : all_ctx(c)) {
            ctx_sync(x);
            unsigned long long hb[GPS_K_NCLASSES];
            GPS_CK(cudaMemcpy(hb, x->d_bytes, sizeof(hb), cudaMemcpyDeviceToHost));
            out->queries += x->stats.queries;
            out->embeddings += x->stats.embeddings;
            out->launches += x->stats.launches;
            out->host_syncs += x->stats.host_syncs;
            out->join_rows_max = std::max(out->join_rows_max, x->stats.join_rows_max);
            out->join_rows_total += x->stats.join_rows_total;
            for (int i = 0; i < GPS_K_NCLASSES; i++) {
                out->k_launches[i] += x->stats.k_launches[i];
                out->k_bytes[i] += x->stats.k_bytes[i] + (double)hb[i];
                out->k_ms[i] += x->stats.k_ms[i];
                out->k_timed[i] += x->stats.k_timed[i];
            }
        }
    });
}

gps_status gps_reset_stats(gps_ctx* c) {
    return guarded([&] {
        if (!c) fail(GPS_EINVAL, "null ctx");
        DeviceGuard dg(c->device);
        for (gps_ctx* x : all_ctx(c)) {
            ctx_sync(x);
            x->stats = gps_stats{};
            GPS_CK(cudaMemset(x->d_bytes, 0, sizeof(unsigned long long) * GPS_K_NCLASSES));
        }
    });
}

gps_status gps_set_profiling(gps_ctx* c, uint32_t mask) {
    if (!c) return GPS_EINVAL;
    c->prof_mask = mask;
    for (gps_ctx* w : c->workers) w->prof_mask = mask;
    return GPS_OK;
}

gps_status gps_debug_plan(gps_ctx* c, const gps_graph* g, const gps_query* q, const gps_match_opts* opts,
                          int32_t* order_out, uint32_t* n_order, uint64_t* rank_out) {
    return guarded([&] {
        check_args(c, g);
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
        check_args(c, g);
        if (!q || !bitmaps_out) fail(GPS_EINVAL, "null query/bitmaps_out");
        if (stage < 0 || stage > 2) fail(GPS_EINVAL, "stage must be 0, 1 or 2");
        DeviceGuard dg(c->device);
        run_filter_debug(c, g, q, resolve_opts(opts), stage, bitmaps_out);
    });
}

}  // extern "C"
