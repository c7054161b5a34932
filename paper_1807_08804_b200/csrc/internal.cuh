// internal.cuh -- shared declarations of libgpsense (CUDA path).  Never included by oracle/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/gpsense.h"

namespace gps {
struct WorkerPool;
struct Comm;
}

namespace gps {

constexpr int kWarp = 32;
constexpr uint32_t kFull = 0xffffffffu;

// ---- errors ---------------------------------------------------------------
struct Error {
    gps_status status;
    std::string msg;
};
void set_last_error(const std::string& m);
[[noreturn]] void fail(gps_status s, const std::string& m);
void check_cuda(cudaError_t e, const char* what, const char* file, int line);
#define GPS_CK(x) ::gps::check_cuda((x), #x, __FILE__, __LINE__)

// ---- device views (POD, passed by value to kernels) ----------------------
// Packed arc word: (dst << lbits) | elabel; rows sorted
// ascending by the word = by (dst, label), de-duplicated.
struct DevGraph {
    uint32_t n;       // #vertices
    uint32_t nw;      // ceil(n / 32) bitmap words actually used
    uint32_t nws;     // bitmap row stride in words (nw rounded up to 64)
    uint32_t lbits;   // bits of the edge label in an arc word
    uint32_t lmask;   // (1 << lbits) - 1
    const uint32_t* off_out;  // [n+1]
    const uint32_t* arc_out;  // [m]
    const uint32_t* off_in;   // [n+1]
    const uint32_t* arc_in;   // [m]
    const uint16_t* vlab;     // [n]
    const uint2* deg;         // [n] (out-degree, in-degree): one 8-byte load per candidate
};

__device__ __forceinline__ bool bit_test(const uint32_t* __restrict__ B, uint32_t v) {
    return (__ldg(B + (v >> 5)) >> (v & 31)) & 1u;
}
// Rank of v among the set bits of bitmap B (v must be set): rp = per-word exclusive prefix.
__device__ __forceinline__ uint32_t bit_rank(const uint32_t* __restrict__ B, const uint32_t* __restrict__ rp,
                                             uint32_t v) {
    uint32_t w = v >> 5;
    return __ldg(rp + w) + __popc(__ldg(B + w) & ((1u << (v & 31)) - 1u));
}
__device__ __forceinline__ bool lab_ok(uint32_t arc, uint32_t lmask, int32_t lab) {
    return lab < 0 || (arc & lmask) == (uint32_t)lab;
}

// ---- context ----------------------------------------------------------------
struct PendingTiming {
    int cls;
    cudaEvent_t e0, e1;
};

}  // namespace gps

namespace gps {
struct DevBlock;
}

struct gps_ctx {
    int device = 0;
    int nsm = 148;
    cudaStream_t stream = nullptr;
    cudaMemPool_t pool_mem = nullptr;        // the library's memory pool of this device (ctx.cu device_pool)
    // optional caller allocator (gps_ctx_opts.dev_alloc / dev_free), inherited by batch workers
    void* (*dev_alloc)(size_t, void*, void*) = nullptr;
    void (*dev_free)(void*, void*, void*) = nullptr;
    void* alloc_user = nullptr;
    bool own_stream = false;
    uint32_t prof_mask = 0;
    gps_stats stats{};
    std::vector<gps::PendingTiming> pending;
    std::vector<cudaEvent_t> event_pool;
    unsigned long long* d_bytes = nullptr;   // [GPS_K_NCLASSES] device-accumulated algorithmic bytes
    uint64_t* d_info = nullptr;              // small device scratch (counts, totals)
    uint64_t* h_info = nullptr;              // pinned mirror
    unsigned int* d_done = nullptr;          // last-block counters [1 + GPS_MAX_QE], self-resetting
    uint64_t* lb_status = nullptr;           // decoupled look-back status words [lb_slots * lb_tiles]
    unsigned int* lb_ctr = nullptr;          // look-back tickets [lb_slots], self-resetting
    uint32_t lb_tiles = 0;                   // tiles per slot currently allocated
    uint32_t lb_slots = 0;                   // slots currently allocated
    uint32_t lb_epoch = 0;                   // launch epoch (never 0 once used)
    // job-array staging: pinned segments with device twins (same offsets), bump allocated,
    // rewound only by arena_reset() at the start of a run (never while arrays are in use)
    struct ArenaSeg {
        char* h;
        char* d;
        size_t cap;
    };
    std::vector<ArenaSeg> arena;
    size_t arena_seg = 0, h_arena_off = 0;
    size_t h_flushed = 0;                    // [h_flushed, h_arena_off) of the current segment not yet copied
    std::multimap<size_t, void*> pinned_free;  // pinned host buffers for host results (reused)
    std::vector<gps_result*> results;        // live results (freed at destroy)
    std::mutex results_mu;                   // batch workers register results concurrently
    // batch execution: worker sub-contexts (own stream + scratch) driven by a host thread pool
    std::vector<gps_ctx*> workers;
    gps::WorkerPool* pool = nullptr;
    uint32_t nworkers_req = 0;               // 0 = default (2)
    uint32_t slice = 0;                      // queries per worker hand-out (0 = default 64)
    gps::Comm* comm = nullptr;               // row-sharded join across the ranks of a communicator
    // the previous run's filter-state arena, reused by the next run when large enough and no
    // result holds it (saves an allocation per batch slice)
    std::shared_ptr<gps::DevBlock> arena_cache;
    size_t arena_cache_bytes = 0;
};

struct gps_compressed;   // f3 (compress.cu)
struct gps_graph {
    int device = 0;
    gps::DevGraph d{};
    uint64_t m = 0;              // stored arcs (per direction)
    bool undirected = false;
    uint32_t n_vlabels = 1;
    std::vector<uint64_t> lab_hist;   // freq(label)
    std::vector<uint32_t> elabels;    // edge labels carried by at least one stored arc, ascending
    const gps_compressed* cg = nullptr;   // f3: attached compression (filters start from its level cg_level)
    uint32_t cg_level = 0;
    void* mem[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
};

namespace gps {
// A stream-ordered device allocation shared by several results (a batch writes
// the final rows of many queries into one buffer).
struct DevBlock {
    gps_ctx* c = nullptr;
    void* p = nullptr;
    ~DevBlock();
};
using Block = std::shared_ptr<DevBlock>;
}  // namespace gps

struct gps_result {
    uint64_t rows = 0;
    uint32_t cols = 0;
    uint32_t* data = nullptr;
    int on_device = 0;
    gps_ctx* ctx = nullptr;       // owner (device rows / pinned host rows)
    gps::Block hold;              // device rows live in this block
    uint64_t global_rows = 0;     // rows over all ranks (row-sharded join); = rows otherwise
    size_t host_bytes = 0;        // pinned host buffer size (on_device == 0)
};

namespace gps {

// ---- launch helper: stats, optional CUDA-event timing --------------------
cudaEvent_t ctx_event(gps_ctx* c);
void ctx_harvest(gps_ctx* c);          // after a stream sync: fold finished event pairs into stats
void ctx_sync(gps_ctx* c);             // stream sync + harvest

void flush_uploads(gps_ctx* c);         // one H2D copy of every job array staged since the last launch
void arena_reset(gps_ctx* c);           // rewind the staging arena (no staged array may still be in use)

template <typename Kernel, typename... Args>
inline void launch(gps_ctx* c, int cls, dim3 grid, dim3 block, size_t smem, Kernel k, Args... args) {
    if (grid.x == 0 || grid.y == 0 || grid.z == 0) return;
    if (c->h_arena_off > c->h_flushed) flush_uploads(c);
    bool timed = (c->prof_mask >> cls) & 1u;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (timed) {
        e0 = ctx_event(c);
        e1 = ctx_event(c);
        GPS_CK(cudaEventRecord(e0, c->stream));
    }
    (void)cudaGetLastError();   // a non-sticky error left by another caller's API call is not ours
    k<<<grid, block, smem, c->stream>>>(args...);
    GPS_CK(cudaGetLastError());
    if (timed) {
        GPS_CK(cudaEventRecord(e1, c->stream));
        c->pending.push_back({cls, e0, e1});
    }
    c->stats.launches++;
    c->stats.k_launches[cls]++;
}

// ---- stream-ordered device memory -----------------------------------------
cudaMemPool_t device_pool(int dev);
// opt a kernel in to `bytes` of dynamic shared memory on the current device (idempotent, thread-safe)
void allow_smem(const void* func, int bytes);
void* dmalloc(gps_ctx* c, size_t bytes);
void dfree(gps_ctx* c, void* p);
template <typename T>
T* dalloc(gps_ctx* c, size_t count) {
    return static_cast<T*>(dmalloc(c, count * sizeof(T) + 16));
}
struct DevPtr {  // RAII stream-ordered buffer
    gps_ctx* c = nullptr;
    void* p = nullptr;
    DevPtr() = default;
    DevPtr(gps_ctx* ctx, size_t bytes) : c(ctx), p(dmalloc(ctx, bytes)) {}
    DevPtr(const DevPtr&) = delete;
    DevPtr& operator=(const DevPtr&) = delete;
    DevPtr(DevPtr&& o) noexcept : c(o.c), p(o.p) { o.p = nullptr; }
    DevPtr& operator=(DevPtr&& o) noexcept {
        reset();
        c = o.c;
        p = o.p;
        o.p = nullptr;
        return *this;
    }
    ~DevPtr() { reset(); }
    void reset() {
        if (p) dfree(c, p);
        p = nullptr;
    }
    void* release() {
        void* q = p;
        p = nullptr;
        return q;
    }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

// ---- primitives (scan.cu, sort.cu) ------------------------------------------
// Exclusive scan of nseg independent arrays: out[s][0..n[s]] (n[s]+1 entries,
// out[s][n[s]] = total).  TI/TO in {u32->u32, u32->u64, u64->u64}.
constexpr int kMaxScanSeg = 64;
template <typename TI, typename TO>
struct ScanBatch {
    int nseg;
    const TI* in[kMaxScanSeg];
    TO* out[kMaxScanSeg];
    uint64_t n[kMaxScanSeg];
};
template <typename TI, typename TO>
void scan_exclusive(gps_ctx* c, const ScanBatch<TI, TO>& b);
template <typename TI, typename TO>
inline void scan_exclusive1(gps_ctx* c, const TI* in, TO* out, uint64_t n) {
    ScanBatch<TI, TO> b{};
    b.nseg = 1;
    b.in[0] = in;
    b.out[0] = out;
    b.n[0] = n;
    scan_exclusive(c, b);
}
// LSD radix sort of u64 keys on bits [0, nbits); result in *keys (ping-pong with tmp).
void radix_sort_u64(gps_ctx* c, uint64_t* keys, uint64_t* tmp, uint64_t n, int nbits);

// ---- pinned host memory (ctx.cu) --------------------------------------------
void* pinned_alloc(gps_ctx* c, size_t bytes, size_t* got);
void pinned_release(gps_ctx* c, void* p, size_t bytes);
// Copy a host array into device memory via the pinned arena (stream-ordered).
void* upload_bytes(gps_ctx* c, const void* src, size_t bytes, std::vector<DevPtr>& keep);
template <typename T>
T* upload(gps_ctx* c, const std::vector<T>& v, std::vector<DevPtr>& keep) {
    return static_cast<T*>(upload_bytes(c, v.data(), sizeof(T) * v.size(), keep));
}
Block make_block(gps_ctx* c, size_t bytes);

// ---- graph load (load.cu) ---------------------------------------------------
void load_graph(gps_ctx* c, const gps_csr_desc* desc, gps_graph* g);
void free_graph_mem(gps_graph* g);

}  // namespace gps
