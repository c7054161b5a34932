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

// Filter only (debug entry point): candidate bitmaps after stage 0/1/2 to host.
void run_filter_debug(gps_ctx* c, const gps_graph* g, const gps_query* q, const gps_match_opts& o, int stage,
                      uint32_t* host_bitmaps);

}  // namespace gps
