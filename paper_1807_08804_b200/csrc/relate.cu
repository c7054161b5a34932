// relate.cu -- f4 gSparql primitives (PAPER.md Ch. 4 §"Backward-Chaining Inference",
// P:1222-1262) on binary relations of u32 terms.
//
// A relation (a property table's (subject, object) pairs) lives on the device
// as sorted, de-duplicated u64 keys a << 32 | b.  The primitives of P:1226-1238 map to:
//   sort            LSD radix sort of the keys (sort.cu) + run-head compaction (dedup, the
//                   "sorting and then removing duplications" of P:1264)
//   sort-merge join R(x, y) |x| S(y, z): R re-keyed by y (y << 32 | x) and sorted; per R row
//                   the equal range of y in S by binary search (S sorted by its first term),
//                   lengths -> exclusive scan -> write (x, z) at the row's offset (the two-step
//                   output scheme), then sort + dedup
//   merge / union   concatenation + sort + dedup
//   difference      per key of A a binary search in B, flags -> scan -> compaction
//   recursive rule  Algorithm P:1247-1262 (reading R37): NewT := T; while NewT: InferT :=
//                   join(NewT, T) u join(T, NewT); NewT := InferT \ T; T := T u NewT
#include <algorithm>
#include <vector>

#include "kernels.cuh"
#include "runtime.h"

namespace gps {

namespace {

dim3 grid1(uint64_t n) { return dim3((uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 1u << 30))); }

__global__ void k_pack(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b, uint64_t n,
                       uint64_t* __restrict__ out) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = ((uint64_t)a[i] << 32) | b[i];
}
__global__ void k_swap(const uint64_t* __restrict__ in, uint64_t n, uint64_t* __restrict__ out) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (in[i] << 32) | (in[i] >> 32);
}
__global__ void k_runheads(const uint64_t* __restrict__ k, uint64_t n, uint32_t* __restrict__ flag) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flag[i] = (i == 0 || k[i] != k[i - 1]) ? 1u : 0u;
}
__global__ void k_select(const uint64_t* __restrict__ k, const uint32_t* __restrict__ flag,
                         const uint64_t* __restrict__ pos, uint64_t n, uint64_t* __restrict__ out) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && flag[i]) out[pos[i]] = k[i];
}

__device__ __forceinline__ uint64_t lower_hi(const uint64_t* __restrict__ s, uint64_t n, uint32_t y) {
    uint64_t lo = 0, hi = n;   // first index with (s >> 32) >= y
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if ((uint32_t)(s[mid] >> 32) < y) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// per row (y << 32 | x) of R': the equal range of y in S, as a length
__global__ void k_join_len(const uint64_t* __restrict__ r, uint64_t nr, const uint64_t* __restrict__ s, uint64_t ns,
                           uint64_t* __restrict__ lo, uint32_t* __restrict__ len) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nr) return;
    const uint32_t y = (uint32_t)(r[i] >> 32);
    const uint64_t a = lower_hi(s, ns, y), b = y == 0xffffffffu ? ns : lower_hi(s, ns, y + 1);
    lo[i] = a;
    len[i] = (uint32_t)(b - a);
}
__global__ void k_join_emit(const uint64_t* __restrict__ r, uint64_t nr, const uint64_t* __restrict__ s,
                            const uint64_t* __restrict__ lo, const uint32_t* __restrict__ len,
                            const uint64_t* __restrict__ off, uint64_t* __restrict__ out) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nr) return;
    const uint64_t x = r[i] & 0xffffffffull;
    uint64_t o = off[i];
    for (uint32_t j = 0; j < len[i]; j++) out[o++] = (x << 32) | (s[lo[i] + j] & 0xffffffffull);
}

__global__ void k_absent(const uint64_t* __restrict__ a, uint64_t na, const uint64_t* __restrict__ b, uint64_t nb,
                         uint32_t* __restrict__ flag) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= na) return;
    const uint64_t t = a[i];
    uint64_t lo = 0, hi = nb;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (b[mid] < t) lo = mid + 1; else hi = mid;
    }
    flag[i] = (lo < nb && b[lo] == t) ? 0u : 1u;
}

__global__ void k_rows(const uint64_t* __restrict__ k, uint64_t n, uint32_t* __restrict__ out) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[2 * i] = (uint32_t)(k[i] >> 32);
    out[2 * i + 1] = (uint32_t)k[i];
}

uint64_t d2h_1(gps_ctx* c, const uint64_t* p) {
    uint64_t h = 0;
    GPS_CK(cudaMemcpyAsync(&h, p, 8, cudaMemcpyDeviceToHost, c->stream));
    ctx_sync(c);
    return h;
}

}  // namespace

// A device relation: n sorted unique keys.
struct Rel {
    Block b;
    uint64_t n = 0;
    const uint64_t* k() const { return b ? static_cast<const uint64_t*>(b->p) : nullptr; }
};

// keys[0..n) (device, may be unsorted / duplicated) -> sorted unique relation (keys are clobbered)
static Rel make_rel(gps_ctx* c, uint64_t* keys, uint64_t n) {
    Rel r;
    if (n == 0) return r;
    DevPtr tmp(c, sizeof(uint64_t) * n);
    radix_sort_u64(c, keys, tmp.as<uint64_t>(), n, 64);
    DevPtr flag(c, sizeof(uint32_t) * (n + 1)), pos(c, sizeof(uint64_t) * (n + 1));
    launch(c, GPS_K_JOIN_WRITE, grid1(n), dim3(256), 0, k_runheads, (const uint64_t*)keys, n, flag.as<uint32_t>());
    scan_exclusive1<uint32_t, uint64_t>(c, flag.as<uint32_t>(), pos.as<uint64_t>(), n);
    r.n = d2h_1(c, pos.as<uint64_t>() + n);
    r.b = make_block(c, sizeof(uint64_t) * r.n);
    launch(c, GPS_K_JOIN_WRITE, grid1(n), dim3(256), 0, k_select, (const uint64_t*)keys,
           (const uint32_t*)flag.as<uint32_t>(), (const uint64_t*)pos.as<uint64_t>(), n, static_cast<uint64_t*>(r.b->p));
    return r;
}

static Rel rel_upload(gps_ctx* c, const uint32_t* a, const uint32_t* b, uint64_t n) {
    if (n == 0) return Rel{};
    if (!a || !b) fail(GPS_EINVAL, "null relation column");
    DevPtr da(c, sizeof(uint32_t) * n), db(c, sizeof(uint32_t) * n), k(c, sizeof(uint64_t) * n);
    GPS_CK(cudaMemcpyAsync(da.p, a, sizeof(uint32_t) * n, cudaMemcpyHostToDevice, c->stream));
    GPS_CK(cudaMemcpyAsync(db.p, b, sizeof(uint32_t) * n, cudaMemcpyHostToDevice, c->stream));
    launch(c, GPS_K_JOIN_WRITE, grid1(n), dim3(256), 0, k_pack, (const uint32_t*)da.as<uint32_t>(),
           (const uint32_t*)db.as<uint32_t>(), n, k.as<uint64_t>());
    return make_rel(c, k.as<uint64_t>(), n);
}

// R(x, y) |x| S(y, z) -> (x, z)
static Rel rel_join(gps_ctx* c, const Rel& R, const Rel& S) {
    if (R.n == 0 || S.n == 0) return Rel{};
    DevPtr rs(c, sizeof(uint64_t) * R.n), tmp(c, sizeof(uint64_t) * R.n);
    launch(c, GPS_K_JOIN_WRITE, grid1(R.n), dim3(256), 0, k_swap, R.k(), R.n, rs.as<uint64_t>());
    radix_sort_u64(c, rs.as<uint64_t>(), tmp.as<uint64_t>(), R.n, 64);
    DevPtr lo(c, sizeof(uint64_t) * R.n), len(c, sizeof(uint32_t) * (R.n + 1)), off(c, sizeof(uint64_t) * (R.n + 1));
    launch(c, GPS_K_JOIN_LEN, grid1(R.n), dim3(256), 0, k_join_len, (const uint64_t*)rs.as<uint64_t>(), R.n, S.k(), S.n,
           lo.as<uint64_t>(), len.as<uint32_t>());
    scan_exclusive1<uint32_t, uint64_t>(c, len.as<uint32_t>(), off.as<uint64_t>(), R.n);
    const uint64_t total = d2h_1(c, off.as<uint64_t>() + R.n);
    if (total == 0) return Rel{};
    if (total >= (1ull << 32)) fail(GPS_EUNSUPPORTED, "join of more than 2^32 pairs");
    DevPtr out(c, sizeof(uint64_t) * total);
    launch(c, GPS_K_JOIN_WRITE, grid1(R.n), dim3(256), 0, k_join_emit, (const uint64_t*)rs.as<uint64_t>(), R.n, S.k(),
           (const uint64_t*)lo.as<uint64_t>(), (const uint32_t*)len.as<uint32_t>(), (const uint64_t*)off.as<uint64_t>(),
           out.as<uint64_t>());
    return make_rel(c, out.as<uint64_t>(), total);
}

static Rel rel_union(gps_ctx* c, const Rel& A, const Rel& B) {
    const uint64_t n = A.n + B.n;
    if (n == 0) return Rel{};
    DevPtr k(c, sizeof(uint64_t) * n);
    if (A.n) GPS_CK(cudaMemcpyAsync(k.p, A.k(), sizeof(uint64_t) * A.n, cudaMemcpyDeviceToDevice, c->stream));
    if (B.n)
        GPS_CK(cudaMemcpyAsync(k.as<uint64_t>() + A.n, B.k(), sizeof(uint64_t) * B.n, cudaMemcpyDeviceToDevice,
                               c->stream));
    return make_rel(c, k.as<uint64_t>(), n);
}

static Rel rel_diff(gps_ctx* c, const Rel& A, const Rel& B) {
    if (A.n == 0) return Rel{};
    if (B.n == 0) return A;
    DevPtr flag(c, sizeof(uint32_t) * (A.n + 1)), pos(c, sizeof(uint64_t) * (A.n + 1));
    launch(c, GPS_K_JOIN_WRITE, grid1(A.n), dim3(256), 0, k_absent, A.k(), A.n, B.k(), B.n, flag.as<uint32_t>());
    scan_exclusive1<uint32_t, uint64_t>(c, flag.as<uint32_t>(), pos.as<uint64_t>(), A.n);
    Rel r;
    r.n = d2h_1(c, pos.as<uint64_t>() + A.n);
    if (r.n == 0) return Rel{};
    r.b = make_block(c, sizeof(uint64_t) * r.n);
    launch(c, GPS_K_JOIN_WRITE, grid1(A.n), dim3(256), 0, k_select, A.k(), (const uint32_t*)flag.as<uint32_t>(),
           (const uint64_t*)pos.as<uint64_t>(), A.n, static_cast<uint64_t*>(r.b->p));
    return r;
}

static void rel_result(gps_ctx* c, const Rel& r, QueryResult& qr) {
    qr.cols = 2;
    qr.rows = r.n;
    qr.global_rows = r.n;
    if (r.n == 0) return;
    qr.block = make_block(c, sizeof(uint32_t) * 2 * r.n);
    launch(c, GPS_K_JOIN_WRITE, grid1(r.n), dim3(256), 0, k_rows, r.k(), r.n, static_cast<uint32_t*>(qr.block->p));
    qr.data = static_cast<const uint32_t*>(qr.block->p);
}

// op: 0 join, 1 union, 2 difference
void relation_op(gps_ctx* c, int op, const uint32_t* a_src, const uint32_t* a_dst, uint64_t na, const uint32_t* b_src,
                 const uint32_t* b_dst, uint64_t nb, QueryResult& qr) {
    const Rel A = rel_upload(c, a_src, a_dst, na), B = rel_upload(c, b_src, b_dst, nb);
    Rel r = op == 0 ? rel_join(c, A, B) : (op == 1 ? rel_union(c, A, B) : rel_diff(c, A, B));
    rel_result(c, r, qr);
    ctx_sync(c);
}

void relation_closure(gps_ctx* c, const uint32_t* src, const uint32_t* dst, uint64_t n, uint32_t max_rounds,
                      QueryResult& qr, uint32_t* rounds) {
    Rel T = rel_upload(c, src, dst, n);
    Rel nw = T;
    uint32_t it = 0;
    while (nw.n) {
        if (max_rounds && it >= max_rounds) fail(GPS_EOVERFLOW, "recursive rule did not converge within max_rounds");
        const Rel inf = rel_union(c, rel_join(c, nw, T), rel_join(c, T, nw));
        nw = rel_diff(c, inf, T);
        T = rel_union(c, T, nw);
        it++;
    }
    if (rounds) *rounds = it;
    rel_result(c, T, qr);
    ctx_sync(c);
}

}  // namespace gps
