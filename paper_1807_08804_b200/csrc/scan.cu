// scan.cu -- device-wide exclusive prefix scan, batched over independent
// segments, single pass (decoupled look-back, lookback.cuh).  This is the
// "prefix scan to calculate the output addresses" of kernel_collect (P:773,
// citing Harris) and of the two-step output scheme: counts ->
// exclusive offsets, out[n] = total.
#include "kernels.cuh"
#include "lookback.cuh"

namespace gps {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

template <typename TI, typename TO>
__global__ void __launch_bounds__(kScanThreads) k_scan(const __grid_constant__ ScanBatch<TI, TO> b, LbScratch lb,
                                                       uint32_t epoch) {
    __shared__ TI s_in[kScanTile];
    __shared__ TO s_out[kScanTile];
    __shared__ uint64_t s_pre;
    const int s = blockIdx.y;
    const uint32_t tile = lb_ticket(lb.ctr + s, gridDim.x);
    const uint64_t n = b.n[s];
    TO* out = b.out[s];
    const uint64_t ntiles = (n + kScanTile - 1) / kScanTile;
    if (n == 0) {
        if (tile == 0 && threadIdx.x == 0) out[0] = 0;
        return;
    }
    if (tile >= ntiles) return;
    const uint64_t base = (uint64_t)tile * kScanTile;
    const TI* in = b.in[s];
#pragma unroll
    for (int i = 0; i < kScanItems; i++) {
        uint64_t idx = base + (uint64_t)i * kScanThreads + threadIdx.x;
        s_in[i * kScanThreads + threadIdx.x] = idx < n ? in[idx] : TI(0);
    }
    __syncthreads();
    TO v[kScanItems];
    TO tsum = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; i++) {
        v[i] = tsum;
        tsum += (TO)s_in[threadIdx.x * kScanItems + i];
    }
    TO tot;
    const TO pre = block_excl_scan(tsum, &tot);
    if (threadIdx.x < 32) {
        uint64_t p = lb_warp_lookback(lb.status + (size_t)s * lb.max_tiles, tile, (uint64_t)tot, epoch);
        if (threadIdx.x == 0) s_pre = p;
    }
    __syncthreads();
    const TO bpre = (TO)s_pre;
#pragma unroll
    for (int i = 0; i < kScanItems; i++) s_out[threadIdx.x * kScanItems + i] = bpre + pre + v[i];
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kScanItems; i++) {
        uint64_t idx = base + (uint64_t)i * kScanThreads + threadIdx.x;
        if (idx < n) out[idx] = s_out[i * kScanThreads + threadIdx.x];
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) out[n] = bpre + tot;
}

template <typename TI, typename TO>
void scan_exclusive(gps_ctx* c, const ScanBatch<TI, TO>& b) {
    if (b.nseg <= 0) return;
    uint64_t maxn = 0;
    for (int s = 0; s < b.nseg; s++) maxn = b.n[s] > maxn ? b.n[s] : maxn;
    uint64_t nt = (maxn + kScanTile - 1) / kScanTile;
    if (nt == 0) nt = 1;
    if (nt > 0x7fffffffull) fail(GPS_EOVERFLOW, "scan too large");
    LbScratch lb = lb_scratch(c, (uint32_t)b.nseg, (uint32_t)nt);
    launch(c, GPS_K_SCAN, dim3((uint32_t)nt, b.nseg), dim3(kScanThreads), 0, k_scan<TI, TO>, b, lb,
           lb_next_epoch(c));
}

template void scan_exclusive<uint32_t, uint32_t>(gps_ctx*, const ScanBatch<uint32_t, uint32_t>&);
template void scan_exclusive<uint32_t, uint64_t>(gps_ctx*, const ScanBatch<uint32_t, uint64_t>&);
template void scan_exclusive<uint64_t, uint64_t>(gps_ctx*, const ScanBatch<uint64_t, uint64_t>&);

}  // namespace gps
