// scan.cu -- device-wide exclusive prefix scan (reduce-then-scan), batched over
// independent segments.  This is the "prefix scan to calculate the output
// addresses" of kernel_collect (citing Harris) and of the two-step output
// scheme: counts -> exclusive offsets, out[n] = total.
#include "prims.cuh"

namespace gps {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

template <typename TI, typename TO>
__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(ScanBatch<TI, TO> b, TO* part, uint32_t nbmax) {
    const int s = blockIdx.y;
    const uint64_t n = b.n[s];
    const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
    if (base >= n) return;
    const TI* in = b.in[s];
    TO sum = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; i++) {
        uint64_t idx = base + (uint64_t)i * kScanThreads + threadIdx.x;
        if (idx < n) sum += (TO)in[idx];
    }
    sum = block_sum(sum);
    if (threadIdx.x == 0) part[(uint64_t)s * nbmax + blockIdx.x] = sum;
}

// One block per segment: exclusive scan of that segment's block partials, in place.
template <typename TI, typename TO>
__global__ void __launch_bounds__(1024) k_scan_partials(ScanBatch<TI, TO> b, TO* part, uint32_t nbmax) {
    const int s = blockIdx.y;
    const uint64_t nb = (b.n[s] + kScanTile - 1) / kScanTile;
    TO* p = part + (uint64_t)s * nbmax;
    TO carry = 0;
    for (uint64_t base = 0; base < nb; base += blockDim.x) {
        uint64_t i = base + threadIdx.x;
        TO v = i < nb ? p[i] : TO(0);
        TO tot;
        TO ex = block_excl_scan(v, &tot);
        if (i < nb) p[i] = carry + ex;
        carry += tot;
    }
}

template <typename TI, typename TO>
__global__ void __launch_bounds__(kScanThreads) k_scan_down(ScanBatch<TI, TO> b, const TO* part, uint32_t nbmax) {
    __shared__ TI s_in[kScanTile];
    __shared__ TO s_out[kScanTile];
    const int s = blockIdx.y;
    const uint64_t n = b.n[s];
    const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
    TO* out = b.out[s];
    if (n == 0) {
        if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = 0;
        return;
    }
    if (base >= n) return;
    const TI* in = b.in[s];
    // coalesced load into shared memory, then thread-contiguous scan
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
    TO pre = block_excl_scan(tsum, &tot);
    const TO bpre = part ? part[(uint64_t)s * nbmax + blockIdx.x] : TO(0);
#pragma unroll
    for (int i = 0; i < kScanItems; i++) s_out[threadIdx.x * kScanItems + i] = bpre + pre + v[i];
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kScanItems; i++) {
        uint64_t idx = base + (uint64_t)i * kScanThreads + threadIdx.x;
        if (idx < n) out[idx] = s_out[i * kScanThreads + threadIdx.x];
    }
    if (base + kScanTile >= n && threadIdx.x == 0) out[n] = bpre + tot;
}

template <typename TI, typename TO>
void scan_exclusive(gps_ctx* c, const ScanBatch<TI, TO>& b) {
    if (b.nseg <= 0) return;
    uint64_t maxn = 0;
    for (int s = 0; s < b.nseg; s++) maxn = b.n[s] > maxn ? b.n[s] : maxn;
    uint64_t nbmax = (maxn + kScanTile - 1) / kScanTile;
    if (nbmax == 0) nbmax = 1;
    if (nbmax > 0x7fffffffull) fail(GPS_EOVERFLOW, "scan too large");
    if (nbmax == 1) {
        launch(c, GPS_K_SCAN, dim3(1, b.nseg), dim3(kScanThreads), 0, k_scan_down<TI, TO>, b,
               (const TO*)nullptr, (uint32_t)1);
        return;
    }
    DevPtr part(c, sizeof(TO) * nbmax * b.nseg);
    launch(c, GPS_K_SCAN, dim3((uint32_t)nbmax, b.nseg), dim3(kScanThreads), 0, k_scan_reduce<TI, TO>, b,
           part.as<TO>(), (uint32_t)nbmax);
    launch(c, GPS_K_SCAN, dim3(1, b.nseg), dim3(1024), 0, k_scan_partials<TI, TO>, b, part.as<TO>(),
           (uint32_t)nbmax);
    launch(c, GPS_K_SCAN, dim3((uint32_t)nbmax, b.nseg), dim3(kScanThreads), 0, k_scan_down<TI, TO>, b,
           (const TO*)part.as<TO>(), (uint32_t)nbmax);
}

template void scan_exclusive<uint32_t, uint32_t>(gps_ctx*, const ScanBatch<uint32_t, uint32_t>&);
template void scan_exclusive<uint32_t, uint64_t>(gps_ctx*, const ScanBatch<uint32_t, uint64_t>&);
template void scan_exclusive<uint64_t, uint64_t>(gps_ctx*, const ScanBatch<uint64_t, uint64_t>&);

}  // namespace gps
