// ctx.cu -- runtime plumbing of a gps_ctx: errors, stream-ordered device memory,
// pinned staging for job uploads, pinned host results, decoupled look-back
// scratch, event timing, and the host worker pool of the batch API.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <mutex>
#include <utility>

#include "kernels.cuh"
#include "runtime.h"

namespace gps {

static thread_local std::string g_err;
void set_last_error(const std::string& m) { g_err = m; }
const char* last_error() { return g_err.c_str(); }
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

// Test hook: GPS_FAULT_ALLOC=N makes the N-th device allocation after the variable
// (re)takes that value fail with GPS_ENOMEM, so tests can drive every failure path.
static void fault_injection() {
    static std::mutex mu;
    static std::string last;
    static long count = 0;
    const char* e = std::getenv("GPS_FAULT_ALLOC");
    if (!e || !*e) return;
    std::lock_guard<std::mutex> lk(mu);
    if (last != e) {
        last = e;
        count = 0;
    }
    if (++count == std::atol(e)) fail(GPS_ENOMEM, "injected device allocation failure");
}

// The library's own stream-ordered memory pool per device (never the device's default
// pool, whose attributes other users of the process own).  Freed blocks stay cached
// up to GPS_POOL_KEEP_BYTES (default three quarters of the device memory) across
// synchronisations, so a steady stream of queries reuses memory without driver calls;
// anything above is returned to the driver at the next synchronisation, and all of it
// when the process ends.
cudaMemPool_t device_pool(int dev) {
    static std::mutex mu;
    static std::map<int, cudaMemPool_t> pools;
    std::lock_guard<std::mutex> lk(mu);
    auto it = pools.find(dev);
    if (it != pools.end()) return it->second;
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool;
    GPS_CK(cudaMemPoolCreate(&pool, &props));
    const char* e = std::getenv("GPS_POOL_KEEP_BYTES");
    uint64_t keep = 64ull << 30;
    if (e && *e) {
        keep = std::strtoull(e, nullptr, 10);
    } else {   // three quarters of the device: trimming below the working set of a large join
        size_t fr = 0, tot = 0;   // re-maps tens of GB on the next step (0.3-0.7 s stalls, config 3)
        int prev = -1;
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
        if (cudaMemGetInfo(&fr, &tot) == cudaSuccess) keep = (uint64_t)tot / 4 * 3;
        else (void)cudaGetLastError();
        if (prev >= 0 && prev != dev) cudaSetDevice(prev);
    }
    GPS_CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    // GPS_POOL_RESERVE_BYTES: map that much physical memory into the pool once, up front (one
    // allocation, freed at once and kept below the release threshold), so large joins later
    // sub-allocate instead of mapping fresh blocks mid-step (0.1-1 s stalls in a fresh process)
    if (const char* r = std::getenv("GPS_POOL_RESERVE_BYTES")) {
        const uint64_t want = std::min<uint64_t>(std::strtoull(r, nullptr, 10), keep);
        if (want) {
            int prev = -1;
            cudaGetDevice(&prev);
            if (prev != dev) cudaSetDevice(dev);
            void* p = nullptr;
            if (cudaMallocFromPoolAsync(&p, want, pool, 0) == cudaSuccess) {
                (void)cudaFreeAsync(p, 0);
                (void)cudaStreamSynchronize(0);
            } else {
                (void)cudaGetLastError();
            }
            if (prev >= 0 && prev != dev) cudaSetDevice(prev);
        }
    }
    pools[dev] = pool;
    return pool;
}

// Dynamic shared memory opt-in of a kernel on the CURRENT device (the attribute is per
// function per device context), once per (device, kernel, size).
void allow_smem(const void* func, int bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, int> done;
    int dev = 0;
    GPS_CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    auto& have = done[{dev, func}];
    if (have >= bytes) return;
    GPS_CK(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    have = bytes;
}

void* dmalloc(gps_ctx* c, size_t bytes) {
    fault_injection();
    void* p = nullptr;
    // +16 bytes: bulk copies (bulk.cuh) round staged ranges out to 16-byte boundaries
    const size_t padded = ((bytes + 15) & ~size_t(15)) + 16;
    if (c->dev_alloc) {
        p = c->dev_alloc(padded, (void*)c->stream, c->alloc_user);
        if (!p) fail(GPS_ENOMEM, "caller allocator: device allocation of " + std::to_string(bytes) + " bytes failed");
        return p;
    }
    cudaError_t e = cudaMallocFromPoolAsync(&p, padded, c->pool_mem, c->stream);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        fail(GPS_ENOMEM, "device allocation of " + std::to_string(bytes) + " bytes failed");
    }
    return p;
}
void dfree(gps_ctx* c, void* p) {
    if (!p) return;
    if (c->dev_free) c->dev_free(p, (void*)c->stream, c->alloc_user);
    else (void)cudaFreeAsync(p, c->stream);
}

DevBlock::~DevBlock() {
    if (p && c) dfree(c, p);
}
Block make_block(gps_ctx* c, size_t bytes) {
    auto b = std::make_shared<DevBlock>();
    b->c = c;
    b->p = dmalloc(c, bytes ? bytes : 16);
    return b;
}

// Job arrays go through a pinned arena and its device twin (same offsets, bump
// allocated): no device allocation per upload, and all the arrays staged for one
// launch travel in ONE H2D copy (flush_uploads, called by launch()).  The arena
// grows by whole segments and is rewound only at the start of a run.
void* upload_bytes(gps_ctx* c, const void* src, size_t bytes, std::vector<DevPtr>& keep) {
    (void)keep;
    const size_t need = (bytes + 255) & ~size_t(255);
    if (c->arena.empty() || c->h_arena_off + need > c->arena[c->arena_seg].cap) {
        if (!c->arena.empty()) {
            flush_uploads(c);
            c->arena_seg++;
        }
        if (c->arena_seg >= c->arena.size() || c->arena[c->arena_seg].cap < need) {
            const size_t prev = c->arena.empty() ? 0 : c->arena.back().cap;
            gps_ctx::ArenaSeg sg{nullptr, nullptr, std::max<size_t>(need, std::max<size_t>(2 * prev, 4u << 20))};
            GPS_CK(cudaMallocHost(&sg.h, sg.cap));
            GPS_CK(cudaMalloc(&sg.d, sg.cap));
            c->arena.insert(c->arena.begin() + c->arena_seg, sg);
        }
        c->h_arena_off = 0;
        c->h_flushed = 0;
    }
    gps_ctx::ArenaSeg& sg = c->arena[c->arena_seg];
    char* h = sg.h + c->h_arena_off;
    void* d = sg.d + c->h_arena_off;
    c->h_arena_off += need;
    if (bytes) std::memcpy(h, src, bytes);
    return d;
}

void flush_uploads(gps_ctx* c) {
    if (c->arena.empty()) return;
    gps_ctx::ArenaSeg& sg = c->arena[c->arena_seg];
    const size_t a = c->h_flushed, b = c->h_arena_off;
    if (b > a) GPS_CK(cudaMemcpyAsync(sg.d + a, sg.h + a, b - a, cudaMemcpyHostToDevice, c->stream));
    c->h_flushed = b;
}

void arena_reset(gps_ctx* c) {
    flush_uploads(c);
    GPS_CK(cudaStreamSynchronize(c->stream));   // earlier staged copies / kernels are done with the arena
    c->arena_seg = 0;
    c->h_arena_off = 0;
    c->h_flushed = 0;
}

void* pinned_alloc(gps_ctx* c, size_t bytes, size_t* got) {
    size_t want = std::max<size_t>(bytes, 4096);
    auto it = c->pinned_free.lower_bound(want);
    if (it != c->pinned_free.end() && it->first <= 2 * want + (1u << 20)) {
        void* p = it->second;
        *got = it->first;
        c->pinned_free.erase(it);
        return p;
    }
    size_t cap = 4096;
    while (cap < want) cap <<= 1;
    void* p = nullptr;
    GPS_CK(cudaMallocHost(&p, cap));
    *got = cap;
    return p;
}
void pinned_release(gps_ctx* c, void* p, size_t bytes) {
    if (p) c->pinned_free.emplace(bytes, p);
}

LbScratch lb_scratch(gps_ctx* c, uint32_t slots, uint32_t tiles) {
    if (tiles == 0) tiles = 1;
    if (slots == 0) slots = 1;
    if (tiles > c->lb_tiles || slots > c->lb_slots) {
        const uint32_t tcap = std::max<uint32_t>(std::max(tiles, c->lb_tiles), 64);
        const uint32_t scap = std::max<uint32_t>(std::max(slots, c->lb_slots), 192);
        // drop the old buffers first and forget them, so a failed allocation leaves no dangling state
        if (c->lb_status) dfree(c, c->lb_status);
        if (c->lb_ctr) dfree(c, c->lb_ctr);
        c->lb_status = nullptr;
        c->lb_ctr = nullptr;
        c->lb_tiles = c->lb_slots = 0;
        c->lb_status = static_cast<uint64_t*>(dmalloc(c, sizeof(uint64_t) * (size_t)tcap * scap));
        c->lb_ctr = static_cast<unsigned int*>(dmalloc(c, sizeof(unsigned int) * scap));
        GPS_CK(cudaMemsetAsync(c->lb_status, 0, sizeof(uint64_t) * (size_t)tcap * scap, c->stream));
        GPS_CK(cudaMemsetAsync(c->lb_ctr, 0, sizeof(unsigned int) * scap, c->stream));
        c->lb_tiles = tcap;
        c->lb_slots = scap;
    }
    return LbScratch{c->lb_status, c->lb_ctr, c->lb_tiles};
}
uint32_t resident_grid(gps_ctx* c, const void* func, int threads, size_t smem) {
    static std::mutex mu;
    static std::map<std::pair<const void*, size_t>, int> cache;   // (kernel, smem rounded to 1 KB) -> blocks/SM
    const size_t key_smem = (smem + 1023) & ~size_t(1023);
    int occ = 0;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find({func, key_smem});
        if (it != cache.end()) occ = it->second;
    }
    if (occ == 0) {
        GPS_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, func, threads, key_smem));
        if (occ < 1) occ = 1;
        std::lock_guard<std::mutex> lk(mu);
        cache[{func, key_smem}] = occ;
    }
    return (uint32_t)(c->nsm * occ);
}

uint32_t lb_next_epoch(gps_ctx* c) {
    c->lb_epoch++;
    if (c->lb_epoch >= (1u << 20)) {   // wrap: clear stale words so old epochs cannot alias
        GPS_CK(cudaMemsetAsync(c->lb_status, 0, sizeof(uint64_t) * (size_t)c->lb_tiles * c->lb_slots, c->stream));
        c->lb_epoch = 1;
    }
    return c->lb_epoch;
}

void ctx_init(gps_ctx* c, int dev, cudaStream_t stream) {
    c->device = dev;
    GPS_CK(cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, dev));
    if (stream) {
        c->stream = stream;
    } else {
        GPS_CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
    }
    c->pool_mem = device_pool(dev);
    GPS_CK(cudaMalloc(&c->d_bytes, sizeof(unsigned long long) * GPS_K_NCLASSES));
    GPS_CK(cudaMemset(c->d_bytes, 0, sizeof(unsigned long long) * GPS_K_NCLASSES));
    GPS_CK(cudaMalloc(&c->d_info, sizeof(uint64_t) * 128));
    GPS_CK(cudaMemset(c->d_info, 0, sizeof(uint64_t) * 128));
    GPS_CK(cudaMallocHost(&c->h_info, sizeof(uint64_t) * 128));
    GPS_CK(cudaMalloc(&c->d_done, sizeof(unsigned int) * 64));
    GPS_CK(cudaMemset(c->d_done, 0, sizeof(unsigned int) * 64));
    GPS_CK(cudaDeviceSynchronize());
}

void ctx_release(gps_ctx* c) {
    cudaStreamSynchronize(c->stream);
    c->arena_cache.reset();
    if (std::getenv("GPS_EXPLORE_STATS") && c->d_info) {
        uint64_t h[8];
        if (cudaMemcpy(h, c->d_info + 96, sizeof(h), cudaMemcpyDeviceToHost) == cudaSuccess && h[0] + h[4])
            std::fprintf(stderr, "[gps] explore pairs %llu live %llu fit %llu s-side %llu | propagate pairs %llu live %llu "
                         "fit %llu s-side %llu\n", (unsigned long long)h[0], (unsigned long long)h[1],
                         (unsigned long long)h[2], (unsigned long long)h[3], (unsigned long long)h[4],
                         (unsigned long long)h[5], (unsigned long long)h[6], (unsigned long long)h[7]);
    }
    for (gps_result* r : c->results) {
        if (r->on_device) {
            r->hold.reset();
        } else if (r->data) {
            cudaFreeHost(r->data);
        }
        r->data = nullptr;
        r->rows = 0;
        r->ctx = nullptr;
    }
    c->results.clear();
    dfree(c, c->lb_status);   // dmalloc'd: the caller's allocator when one is set
    dfree(c, c->lb_ctr);
    c->lb_status = nullptr;
    c->lb_ctr = nullptr;
    cudaStreamSynchronize(c->stream);
    for (auto& t : c->pending) {
        c->event_pool.push_back(t.e0);
        c->event_pool.push_back(t.e1);
    }
    c->pending.clear();
    for (cudaEvent_t e : c->event_pool) cudaEventDestroy(e);
    c->event_pool.clear();
    for (auto& kv : c->pinned_free) cudaFreeHost(kv.second);
    c->pinned_free.clear();
    for (auto& sg : c->arena) {
        cudaFreeHost(sg.h);
        cudaFree(sg.d);
    }
    c->arena.clear();
    cudaFree(c->d_bytes);
    cudaFree(c->d_info);
    cudaFreeHost(c->h_info);
    cudaFree(c->d_done);
    if (c->own_stream) cudaStreamDestroy(c->stream);
}

WorkerPool::WorkerPool(int n) {
    for (int w = 0; w < n; w++)
        th.emplace_back([this, w] {
            uint64_t seen = 0;
            for (;;) {
                std::function<void(int)> f;
                {
                    std::unique_lock<std::mutex> lk(mu);
                    cv.wait(lk, [&] { return stop || gen != seen; });
                    if (stop) return;
                    seen = gen;
                    f = job;
                }
                f(w);
                {
                    std::lock_guard<std::mutex> lk(mu);
                    if (--remaining == 0) done_cv.notify_all();
                }
            }
        });
}
void WorkerPool::run(std::function<void(int)> f) {
    std::unique_lock<std::mutex> lk(mu);
    job = std::move(f);
    remaining = (int)th.size();
    gen++;
    cv.notify_all();
    done_cv.wait(lk, [&] { return remaining == 0; });
}
WorkerPool::~WorkerPool() {
    {
        std::lock_guard<std::mutex> lk(mu);
        stop = true;
    }
    cv.notify_all();
    for (auto& t : th) t.join();
}

}  // namespace gps
