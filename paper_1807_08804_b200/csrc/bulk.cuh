// bulk.cuh -- TMA bulk copies (cp.async.bulk, SASS UBLKCP) global -> shared with
// mbarrier transaction counting: one elected thread arms the barrier with the byte
// count and issues the copies; the copy engine completes the transaction when the
// bytes land, and consumer threads wait on the barrier's phase parity.
//
// Contract of bulk_stage(): the copy covers [floor16(src), ceil16(src + bytes)) --
// up to 15 bytes either side of the requested range -- so every device array staged
// this way must be a library allocation (dmalloc pads every allocation by 16 bytes
// and the pool hands out 16-byte-aligned blocks); the data lands at the same
// address offset mod 16 inside the destination slot (dst must be 16-byte aligned).
#pragma once
#include <cstdint>

namespace gps {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

// Make barrier inits visible to the async proxy (the copy engine).
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Order this thread's earlier generic-proxy shared-memory accesses before later
// async-proxy (bulk copy) accesses of the same buffer.
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    }
}

// One bulk copy of `bytes` (multiple of 16) from 16-byte-aligned global src to
// 16-byte-aligned shared dst, completing `bytes` transactions on bar.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Bulk store shared -> global (16-byte aligned both sides, bytes a multiple of 16), in the
// issuing thread's current bulk group.
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// At most one of this thread's bulk groups may still be READING shared memory.
__device__ __forceinline__ void bulk_wait_read_le1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
// None of this thread's bulk groups is still reading shared memory.
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// Every bulk group of this thread has completed (writes performed).
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Stage [src, src + bytes) into the slot at dst (16-byte aligned).  Returns the byte
// shift of src inside the slot (the element at src lands at dst + shift) and adds the
// copied size to *tx.  Bulk copies are limited to < 2^20 bytes per instruction here;
// larger ranges are split.
__device__ __forceinline__ uint32_t bulk_stage(char* dst, const void* src, uint64_t bytes, uint64_t* bar,
                                               uint32_t* tx) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(src);
    const uintptr_t lo = a & ~uintptr_t(15);
    const uintptr_t hi = (a + bytes + 15) & ~uintptr_t(15);
    if (bytes == 0) return (uint32_t)(a - lo);
    uint64_t n = hi - lo;
    uint64_t o = 0;
    while (n) {
        const uint32_t part = n > (1u << 19) ? (1u << 19) : (uint32_t)n;
        bulk_g2s(dst + o, reinterpret_cast<const void*>(lo + o), part, bar);
        o += part;
        n -= part;
    }
    *tx += (uint32_t)(hi - lo);
    return (uint32_t)(a - lo);
}

// Bytes a staged range can occupy in its slot (the 16-byte rounding of both ends).
__host__ __device__ constexpr uint64_t bulk_slot(uint64_t bytes) { return ((bytes + 15) & ~uint64_t(15)) + 16; }

}  // namespace gps
