// lookback.cuh -- single-pass decoupled look-back prefix scan building blocks.
//
// Each tile publishes (epoch | flag | value) in one 64-bit status word; the
// epoch (a per-ctx launch counter) makes stale words from earlier launches
// invalid, so status arrays never need clearing.  Tiles are numbered in
// scheduling order through an atomic ticket (self-resetting), so a tile only
// ever waits on tiles that are already resident -- no deadlock.
#pragma once
#include "prims.cuh"

namespace gps {

constexpr uint64_t kLbValueBits = 42;
constexpr uint64_t kLbValueMask = (1ull << kLbValueBits) - 1;
constexpr uint64_t kLbAgg = 1ull << kLbValueBits;
constexpr uint64_t kLbIncl = 2ull << kLbValueBits;
constexpr uint64_t kLbFlagMask = 3ull << kLbValueBits;
constexpr int kLbEpochShift = 44;

__device__ __forceinline__ uint64_t lb_pack(uint32_t epoch, uint64_t flag, uint64_t v) {
    return ((uint64_t)epoch << kLbEpochShift) | flag | (v & kLbValueMask);
}
__device__ __forceinline__ void lb_store(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t lb_load(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Ticket for this block (call from every thread; uses one shared slot).
__device__ __forceinline__ uint32_t lb_ticket(unsigned int* counter, uint32_t ntiles) {
    __shared__ uint32_t s_t;
    if (threadIdx.x == 0) {
        uint32_t t = atomicAdd(counter, 1u);
        if (t == ntiles - 1) atomicExch(counter, 0u);   // every block has its ticket: reset for the next launch
        s_t = t;
    }
    __syncthreads();
    uint32_t t = s_t;
    __syncthreads();
    return t;
}

// Warp-0 look-back: returns the exclusive prefix of `tile` and publishes its
// inclusive prefix.  `status` holds one word per tile.  Call with all 32 lanes
// of warp 0 (aggregate must be the same in every lane).
__device__ __forceinline__ uint64_t lb_warp_lookback(uint64_t* status, uint32_t tile, uint64_t aggregate,
                                                     uint32_t epoch) {
    const uint32_t lane = threadIdx.x & 31u;
    if (tile == 0) {
        if (lane == 0) lb_store(status, lb_pack(epoch, kLbIncl, aggregate));
        return 0;
    }
    if (lane == 0) lb_store(status + tile, lb_pack(epoch, kLbAgg, aggregate));
    uint64_t prefix = 0;
    int64_t j = (int64_t)tile - 1;
    while (true) {
        const int64_t idx = j - (int64_t)lane;
        uint64_t s;
        uint64_t flag;
        if (idx >= 0) {
            do {
                s = lb_load(status + idx);
                flag = ((uint32_t)(s >> kLbEpochShift) == epoch) ? (s & kLbFlagMask) : 0ull;
            } while (flag == 0);
        } else {
            s = 0;
            flag = kLbIncl;
        }
        const uint64_t val = idx >= 0 ? (s & kLbValueMask) : 0ull;
        const uint32_t incl = __ballot_sync(kFull, flag == kLbIncl);
        const uint32_t first = incl ? (uint32_t)(__ffs(incl) - 1) : 32u;  // closest inclusive predecessor
        uint64_t mine = lane <= first ? val : 0ull;
        mine = warp_sum(mine);
        prefix += mine;
        if (incl) break;
        j -= 32;
    }
    if (lane == 0) lb_store(status + tile, lb_pack(epoch, kLbIncl, prefix + aggregate));
    return prefix;
}

}  // namespace gps
