// project.cu -- f2 commonsense query semantics: projection of the
// embeddings onto a subset of the query vertices and deduplication of the projected rows
// ("we only need to find the matches of ... projection", "We only need to find
// the matches of nodes in a subset of variable nodes, termed projection").  The result is
// the SET of projected tuples, in lexicographic order.
//
//   k_project      gather the projected columns of every embedding (row-major R x kp)
//   LSD sort       for each column from the last: keys = (value << 32 | position), device
//                  radix sort (sort.cu), positions composed into a permutation -- a stable
//                  sort by column, so after kp passes the rows are in lexicographic order
//   k_gather       rows in sorted order; k_mark: first row of each run of equal rows;
//                  exclusive scan; k_compact: one row per run.
#include <algorithm>

#include "kernels.cuh"
#include "runtime.h"

namespace gps {

namespace {

constexpr uint32_t kProjMax = GPS_MAX_QV;

struct ProjCols {
    uint32_t n;
    uint8_t col[kProjMax];
};

__global__ void k_project(const uint32_t* __restrict__ in, uint64_t R, uint32_t k, ProjCols pc,
                          uint32_t* __restrict__ out) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= R) return;
    for (uint32_t j = 0; j < pc.n; j++) out[i * pc.n + j] = __ldg(in + i * k + pc.col[j]);
}

// key = value << pbits | position (position < 2^pbits): sorting the key sorts by value,
// ties kept in the current order (a stable sort by this column)
__global__ void k_sort_keys(const uint32_t* __restrict__ P, const uint32_t* __restrict__ perm, uint64_t R,
                            uint32_t kp, uint32_t col, uint32_t pbits, uint64_t* __restrict__ keys) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= R) return;
    const uint32_t r = perm ? perm[i] : (uint32_t)i;
    keys[i] = ((uint64_t)__ldg(P + (uint64_t)r * kp + col) << pbits) | i;
}

__global__ void k_compose(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ perm, uint64_t R,
                          uint32_t pbits, uint32_t* __restrict__ nperm) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= R) return;
    const uint32_t pos = (uint32_t)(keys[i] & ((1ull << pbits) - 1));
    nperm[i] = perm ? perm[pos] : pos;
}

// flags[t] = 1 iff sorted row t differs from sorted row t-1 (rows P[perm[t]])
__global__ void k_mark(const uint32_t* __restrict__ P, const uint32_t* __restrict__ perm, uint64_t R, uint32_t kp,
                       uint32_t* __restrict__ flags) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= R) return;
    uint32_t f = 1;
    if (t > 0) {
        const uint32_t* a = P + (uint64_t)perm[t] * kp;
        const uint32_t* b = P + (uint64_t)perm[t - 1] * kp;
        f = 0;
        for (uint32_t j = 0; j < kp; j++) f |= __ldg(a + j) != __ldg(b + j);
    }
    flags[t] = f;
}

__global__ void k_compact(const uint32_t* __restrict__ P, const uint32_t* __restrict__ perm,
                          const uint32_t* __restrict__ flags, const uint64_t* __restrict__ pos, uint64_t R,
                          uint32_t kp, uint32_t* __restrict__ out) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= R || !flags[t]) return;
    const uint32_t* a = P + (uint64_t)perm[t] * kp;
    uint32_t* o = out + pos[t] * kp;
    for (uint32_t j = 0; j < kp; j++) o[j] = __ldg(a + j);
}

uint32_t bits_for(uint64_t x) {
    uint32_t b = 0;
    while (b < 64 && (x >> b)) b++;
    return b;
}

}  // namespace

// Distinct projections of R rows of k columns (device, row-major) onto cols[0..kp); the
// result rows (row-major R' x kp, lexicographic order) go to *out (nullptr: count only).
uint64_t project_unique(gps_ctx* c, const uint32_t* rows, uint64_t R, uint32_t k, const int32_t* cols, uint32_t kp,
                        uint32_t vmax, Block* out) {
    if (kp == 0 || kp > kProjMax) fail(GPS_EINVAL, "projection must name 1..32 query vertices");
    ProjCols pc{};
    pc.n = kp;
    for (uint32_t j = 0; j < kp; j++) {
        if (cols[j] < 0 || (uint32_t)cols[j] >= k) fail(GPS_EINVAL, "projected vertex out of range");
        pc.col[j] = (uint8_t)cols[j];
    }
    if (R == 0) return 0;
    if (R >= (1ull << 32)) fail(GPS_EUNSUPPORTED, "projection of more than 2^32 embeddings");
    if (bits_for(R - 1) + bits_for(vmax) > 64) fail(GPS_EUNSUPPORTED, "projection sort key wider than 64 bits");
    const uint32_t T = 256;
    const dim3 g((uint32_t)((R + T - 1) / T));
    DevPtr P(c, sizeof(uint32_t) * R * kp);
    launch(c, GPS_K_JOIN_WRITE, g, dim3(T), 0, k_project, rows, R, k, pc, P.as<uint32_t>());
    DevPtr keys(c, sizeof(uint64_t) * R), tmp(c, sizeof(uint64_t) * R);
    DevPtr pa(c, sizeof(uint32_t) * R), pb(c, sizeof(uint32_t) * R);
    uint32_t* perm = nullptr;
    uint32_t* next = pa.as<uint32_t>();
    const uint32_t pbits = std::max<uint32_t>(1, bits_for(R - 1));            // positions
    const int nbits = (int)(pbits + bits_for(vmax));                            // + vertex ids
    for (int j = (int)kp - 1; j >= 0; j--) {   // LSD: stable sort by each column from the last
        launch(c, GPS_K_JOIN_WRITE, g, dim3(T), 0, k_sort_keys, (const uint32_t*)P.as<uint32_t>(), (const uint32_t*)perm,
               R, kp, (uint32_t)j, pbits, keys.as<uint64_t>());
        radix_sort_u64(c, keys.as<uint64_t>(), tmp.as<uint64_t>(), R, nbits);
        launch(c, GPS_K_JOIN_WRITE, g, dim3(T), 0, k_compose, (const uint64_t*)keys.as<uint64_t>(),
               (const uint32_t*)perm, R, pbits, next);
        perm = next;
        next = perm == pa.as<uint32_t>() ? pb.as<uint32_t>() : pa.as<uint32_t>();
    }
    DevPtr flags(c, sizeof(uint32_t) * (R + 1)), pos(c, sizeof(uint64_t) * (R + 1));
    launch(c, GPS_K_JOIN_WRITE, g, dim3(T), 0, k_mark, (const uint32_t*)P.as<uint32_t>(), (const uint32_t*)perm, R, kp,
           flags.as<uint32_t>());
    scan_exclusive1<uint32_t, uint64_t>(c, flags.as<uint32_t>(), pos.as<uint64_t>(), R);
    uint64_t total = 0;
    {
        size_t got = 0;
        uint64_t* h = static_cast<uint64_t*>(pinned_alloc(c, 16, &got));
        GPS_CK(cudaMemcpyAsync(h, pos.as<uint64_t>() + R, 8, cudaMemcpyDeviceToHost, c->stream));
        ctx_sync(c);
        total = h[0];
        pinned_release(c, h, got);
    }
    if (out) {
        *out = make_block(c, sizeof(uint32_t) * total * kp + 16);
        launch(c, GPS_K_JOIN_WRITE, g, dim3(T), 0, k_compact, (const uint32_t*)P.as<uint32_t>(), (const uint32_t*)perm,
               (const uint32_t*)flags.as<uint32_t>(), (const uint64_t*)pos.as<uint64_t>(), R, kp,
               static_cast<uint32_t*>((*out)->p));
    }
    return total;
}

}  // namespace gps
