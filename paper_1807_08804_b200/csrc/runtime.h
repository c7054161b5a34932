// runtime.h -- host runtime of libgpsense: ctx lifecycle, worker pool, and the
// batch-synchronous query executor (run.cu).
#pragma once
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "internal.cuh"

namespace gps {

const char* last_error();
void ctx_init(gps_ctx* c, int dev, cudaStream_t stream);
void ctx_release(gps_ctx* c);

// Persistent host worker pool: run(f) calls f(w) once on every worker and waits.
struct WorkerPool {
    std::vector<std::thread> th;
    std::mutex mu;
    std::condition_variable cv, done_cv;
    std::function<void(int)> job;
    uint64_t gen = 0;
    int remaining = 0;
    bool stop = false;
    explicit WorkerPool(int n);
    void run(std::function<void(int)> f);
    ~WorkerPool();
};

// Outcome of one query of a batch.
struct QueryResult {
    gps_status status = GPS_OK;
    std::string error;
    uint64_t rows = 0;
    uint32_t cols = 0;
    Block block;                 // device rows (match mode), row-major rows x cols at data
    const uint32_t* data = nullptr;
    uint64_t global_rows = 0;    // over all ranks (row-sharded join)
};

// Run queries qs[0..nq) on ctx c (its stream), batch-synchronously: every phase
// of Alg. 1 is one launch for the whole batch.  count_only: gps_count semantics
// (the last join level is counted, never written).
void run_queries(gps_ctx* c, const gps_graph* g, const gps_query* qs, uint32_t nq, const gps_match_opts& o,
                 bool count_only, std::vector<QueryResult>& out);

// f2: distinct projections of R device rows (k columns) onto cols[0..kp), lexicographic
// order, into *out (nullptr: count only); returns their number (project.cu).
uint64_t project_unique(gps_ctx* c, const uint32_t* rows, uint64_t R, uint32_t k, const int32_t* cols, uint32_t kp,
                        uint32_t vmax, Block* out);

// f2 named variable edges: the distinct (projection, label bindings) tuples (project.cu).
uint64_t named_unique(gps_ctx* c, const gps_graph* g, const gps_query* q, const gps_match_opts& o,
                      const int32_t* edge_var, uint32_t kp, const int32_t* cols, Block* out);

// f3 multi-level compression (compress.cu)
struct ChkQV;
gps_compressed* compress_graph(gps_ctx* c, const gps_graph* g, uint32_t nlev, const float* deltas);
void free_compressed(gps_compressed* cg);
uint32_t compressed_levels(const gps_compressed* cg);
const gps_graph* compressed_graph(const gps_compressed* cg);
void compressed_level_info(const gps_compressed* cg, uint32_t level, uint32_t* N, uint64_t* ne_out, uint64_t* ne_in);
void compressed_fetch(gps_ctx* c, const gps_compressed* cg, uint32_t level, uint32_t* grp, uint32_t* label,
                      uint32_t* wout, uint32_t* win, uint64_t* ekey_out, uint32_t* ew_out, uint64_t* ekey_in,
                      uint32_t* ew_in);
void run_wcheck(gps_ctx* c, const gps_compressed* cg, uint32_t level, const ChkQV* d_qv, uint32_t nf, bool fresh);

// f4 gSparql relation primitives (relate.cu): op 0 join, 1 union, 2 difference; the
// recursive-rule loop (transitive closure).  Results: rows x 2 (a, b), sorted, distinct.
void relation_op(gps_ctx* c, int op, const uint32_t* a_src, const uint32_t* a_dst, uint64_t na, const uint32_t* b_src,
                 const uint32_t* b_dst, uint64_t nb, QueryResult& qr);
void relation_closure(gps_ctx* c, const uint32_t* src, const uint32_t* dst, uint64_t n, uint32_t max_rounds,
                      QueryResult& qr, uint32_t* rounds);

// Filter only (debug entry point): candidate bitmaps after stage 0/1/2 to host.
void run_filter_debug(gps_ctx* c, const gps_graph* g, const gps_query* q, const gps_match_opts& o, int stage,
                      uint32_t* host_bitmaps);

}  // namespace gps
