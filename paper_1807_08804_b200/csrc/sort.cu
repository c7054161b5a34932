// sort.cu -- stable LSD radix sort of u64 keys (4-bit digits), used only at graph
// load (a0) to sort + de-duplicate adjacency rows and to build the incoming CSR
// (P:941).  Not on the per-query path.
#include "prims.cuh"

namespace gps {

constexpr int kRsThreads = 256;
constexpr int kRsItems = 16;
constexpr int kRsTile = kRsThreads * kRsItems;
constexpr int kRsBins = 16;

// Per-block digit histogram, digit-major layout: hist[d * nblocks + b].
__global__ void __launch_bounds__(kRsThreads) k_rs_hist(const uint64_t* __restrict__ keys, uint64_t n, int shift,
                                                        uint32_t* __restrict__ hist, uint32_t nblocks) {
    __shared__ uint32_t s_h[kRsBins];
    if (threadIdx.x < kRsBins) s_h[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t base = (uint64_t)blockIdx.x * kRsTile;
#pragma unroll 4
    for (int i = 0; i < kRsItems; i++) {
        uint64_t idx = base + (uint64_t)i * kRsThreads + threadIdx.x;
        if (idx < n) atomicAdd(&s_h[(keys[idx] >> shift) & 15u], 1u);
    }
    __syncthreads();
    if (threadIdx.x < kRsBins) hist[(uint64_t)threadIdx.x * nblocks + blockIdx.x] = s_h[threadIdx.x];
}

// Stable scatter: thread t owns the kRsItems consecutive keys t*kRsItems.. of the tile.
__global__ void __launch_bounds__(kRsThreads) k_rs_scatter(const uint64_t* __restrict__ keys, uint64_t* __restrict__ out,
                                                           uint64_t n, int shift, const uint32_t* __restrict__ offs,
                                                           uint32_t nblocks) {
    __shared__ uint64_t s_k[kRsTile];
    __shared__ uint16_t s_c[kRsBins * kRsThreads];  // [digit][thread]
    __shared__ uint32_t s_dstart[kRsBins];
    const uint64_t base = (uint64_t)blockIdx.x * kRsTile;
    const uint32_t t = threadIdx.x;
#pragma unroll 4
    for (int i = 0; i < kRsItems; i++) {
        uint64_t idx = base + (uint64_t)i * kRsThreads + t;
        s_k[i * kRsThreads + t] = idx < n ? keys[idx] : ~0ull;
    }
    __syncthreads();
    uint64_t k[kRsItems];
    uint32_t cnt[kRsBins];
#pragma unroll
    for (int d = 0; d < kRsBins; d++) cnt[d] = 0;
    uint8_t local[kRsItems];
#pragma unroll
    for (int i = 0; i < kRsItems; i++) {
        k[i] = s_k[t * kRsItems + i];
        uint32_t d = (k[i] >> shift) & 15u;
        uint32_t r = 0;
#pragma unroll
        for (int dd = 0; dd < kRsBins; dd++)
            if (dd == (int)d) { r = cnt[dd]; cnt[dd]++; }
        local[i] = (uint8_t)r;
    }
#pragma unroll
    for (int d = 0; d < kRsBins; d++) s_c[d * kRsThreads + t] = (uint16_t)cnt[d];
    __syncthreads();
    // exclusive scan over s_c in linear (digit-major) order: thread t owns entries [t*16, t*16+16)
    uint32_t v[kRsBins];
    uint32_t sum = 0;
#pragma unroll
    for (int j = 0; j < kRsBins; j++) {
        v[j] = sum;
        sum += s_c[t * kRsBins + j];
    }
    uint32_t tot;
    uint32_t pre = block_excl_scan(sum, &tot);
    // block_excl_scan ended with a barrier: every thread has read its own s_c entries
#pragma unroll
    for (int j = 0; j < kRsBins; j++) s_c[t * kRsBins + j] = (uint16_t)(pre + v[j]);
    __syncthreads();
    if (t < kRsBins) s_dstart[t] = s_c[t * kRsThreads];
    __syncthreads();
    const uint64_t valid = n - base < (uint64_t)kRsTile ? n - base : (uint64_t)kRsTile;
#pragma unroll
    for (int i = 0; i < kRsItems; i++) {
        uint64_t tile_pos = (uint64_t)t * kRsItems + i;
        if (tile_pos >= valid) break;
        uint32_t d = (k[i] >> shift) & 15u;
        uint32_t rank = s_c[d * kRsThreads + t] + local[i];
        uint64_t dst = (uint64_t)offs[(uint64_t)d * nblocks + blockIdx.x] + (rank - s_dstart[d]);
        out[dst] = k[i];
    }
}

void radix_sort_u64(gps_ctx* c, uint64_t* keys, uint64_t* tmp, uint64_t n, int nbits) {
    if (n <= 1) return;
    if (n >= (1ull << 32)) fail(GPS_EUNSUPPORTED, "sort larger than 2^32 keys");
    const uint32_t nblocks = (uint32_t)((n + kRsTile - 1) / kRsTile);
    DevPtr hist(c, sizeof(uint32_t) * ((uint64_t)kRsBins * nblocks + 1));
    DevPtr offs(c, sizeof(uint32_t) * ((uint64_t)kRsBins * nblocks + 1));
    uint64_t* src = keys;
    uint64_t* dst = tmp;
    int passes = (nbits + 3) / 4;
    for (int p = 0; p < passes; p++) {
        int shift = 4 * p;
        launch(c, GPS_K_LOAD, dim3(nblocks), dim3(kRsThreads), 0, k_rs_hist, (const uint64_t*)src, n, shift,
               hist.as<uint32_t>(), nblocks);
        scan_exclusive1<uint32_t, uint32_t>(c, hist.as<uint32_t>(), offs.as<uint32_t>(),
                                            (uint64_t)kRsBins * nblocks);
        launch(c, GPS_K_LOAD, dim3(nblocks), dim3(kRsThreads), 0, k_rs_scatter, (const uint64_t*)src, dst, n, shift,
               (const uint32_t*)offs.as<uint32_t>(), nblocks);
        uint64_t* t = src;
        src = dst;
        dst = t;
    }
    if (src != keys) GPS_CK(cudaMemcpyAsync(keys, src, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, c->stream));
}

}  // namespace gps
