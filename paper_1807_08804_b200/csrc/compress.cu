// compress.cu -- f3 multi-level graph compression (PAPER.md §"Multi-level Graph
// Compression") on the device, and the weighted candidate
// test that lets the filter of gps_match start from the compressed graph.
//
// Level i combines SIMILAR nodes of level i-1 pairwise into weighted nodes (P:836,
// P:846).  With the readings of DESIGN R33-R36 and delta = 1, similar = same vertex
// label and the same set of labelled edge ends (direction, edge label, neighbour node);
// that relation is an equivalence, so the greedy pairing of R34 (in id order, each
// unpaired node takes the smallest unpaired similar node) pairs consecutive members of
// each class.  The device finds the classes by hashing each node's deduplicated edge-end
// set (a sum of 64-bit mixes: a set hash), sorting the nodes by (hash, id) and checking
// every candidate pair for exact equality of label and edge-end list.
//
//   k_adj_keys     per stored arc (x, l, y): edge ends (grp x, out, l, grp y) and
//                  (grp y, in, l, grp x) as u64 keys -> radix sort -> unique
//   k_set_hash     per unique edge end: node hash += mix(end), count++
//   k_pair         per sorted position: pair with the next one when both are in the
//                  same hash run at an even offset and exactly equal
//   k_new_ids      leaders (unpaired or first of a pair) numbered in id order
//   k_edge_slots   edge-weight recursion (R35): each weighted edge (U', V', w) of
//                  level i-1 lands in slot (U' second part?, V' second part?) of its
//                  level-i edge (U, V); w(U, V) = max(s00, s10) + max(s01, s11)
//   k_node_weight  w(U) = max over members x of arcs x -> M(U)
//   k_wcheck       the weighted candidate test (R36) of every data vertex through
//                  its node, ANDed into the query's candidate bitmaps (filter start)
#include <algorithm>
#include <vector>

#include "kernels.cuh"
#include "runtime.h"

namespace gps {

namespace {

constexpr uint32_t kNone = 0xffffffffu;

__device__ __forceinline__ uint64_t mix64(uint64_t x) {   // splitmix64 finaliser
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

__device__ __forceinline__ uint32_t src_of(const uint32_t* __restrict__ off, uint32_t n, uint64_t i) {
    uint32_t lo = 0, hi = n;   // largest s with off[s] <= i
    while (hi - lo > 1) {
        const uint32_t mid = lo + (hi - lo) / 2;
        if (off[mid] <= i) lo = mid; else hi = mid;
    }
    return lo;
}

__global__ void k_iota(uint32_t* __restrict__ a, uint32_t n) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = i;
}

__global__ void k_label_u32(const uint16_t* __restrict__ vlab, uint32_t n, uint32_t* __restrict__ out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = vlab[i];
}

// Level-0 weighted edges of one CSR direction: one per (x, y) with weight = #labelled arcs.
// flag[i] = 1 at the first arc of each (x, y) run.
__global__ void k_edge0_flags(const uint32_t* __restrict__ off, const uint32_t* __restrict__ arc, uint32_t n,
                              uint64_t m, uint32_t lbits, uint32_t* __restrict__ flag) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const uint32_t x = src_of(off, n, i);
    flag[i] = (i == off[x] || (arc[i - 1] >> lbits) != (arc[i] >> lbits)) ? 1u : 0u;
}
__global__ void k_edge0_emit(const uint32_t* __restrict__ off, const uint32_t* __restrict__ arc, uint32_t n,
                             uint64_t m, uint32_t lbits, const uint32_t* __restrict__ flag,
                             const uint32_t* __restrict__ pos, uint64_t* __restrict__ key, uint32_t* __restrict__ w) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m || !flag[i]) return;
    const uint32_t x = src_of(off, n, i), y = arc[i] >> lbits;
    uint64_t e = i + 1;
    while (e < off[x + 1] && (arc[e] >> lbits) == y) e++;
    key[pos[i]] = ((uint64_t)x << 32) | y;
    w[pos[i]] = (uint32_t)(e - i);
}

// Edge ends of every stored out-arc at the current level.
__global__ void k_adj_keys(const uint32_t* __restrict__ off, const uint32_t* __restrict__ arc, uint32_t n, uint64_t m,
                           uint32_t lbits, const uint32_t* __restrict__ grp, uint32_t b, uint64_t* __restrict__ keys) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const uint32_t x = src_of(off, n, i), y = arc[i] >> lbits, l = arc[i] & ((1u << lbits) - 1u);
    const uint32_t sh2 = b + lbits, sh1 = sh2 + 1;
    const uint64_t gx = grp[x], gy = grp[y];
    keys[2 * i] = (gx << sh1) | ((uint64_t)l << b) | gy;                       // (gx, out, l, gy)
    keys[2 * i + 1] = (gy << sh1) | (1ull << sh2) | ((uint64_t)l << b) | gx;   // (gy, in, l, gx)
}

__global__ void k_flags(const uint64_t* __restrict__ keys, uint64_t m, uint32_t* __restrict__ flag) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    flag[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1u : 0u;
}
__global__ void k_compact(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ flag,
                          const uint32_t* __restrict__ pos, uint64_t m, uint64_t* __restrict__ out) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m || !flag[i]) return;
    out[pos[i]] = keys[i];
}

__global__ void k_set_hash(const uint64_t* __restrict__ ends, uint64_t u, uint32_t sh1, unsigned long long* hash,
                           uint32_t* cnt, uint32_t* first) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= u) return;
    const uint64_t k = ends[i];
    const uint32_t node = (uint32_t)(k >> sh1);
    atomicAdd(hash + node, (unsigned long long)mix64(k & ((1ull << sh1) - 1)));
    atomicAdd(cnt + node, 1u);
    if (i == 0 || (uint32_t)(ends[i - 1] >> sh1) != node) first[node] = (uint32_t)i;
}

__global__ void k_hash_label(unsigned long long* hash, const uint32_t* __restrict__ label, uint32_t N) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x)
        hash[i] += mix64((1ull << 63) | label[i]);
}

// LSD sort of the nodes by (hash, id): keys (hash half << pb) | position
__global__ void k_hkeys(const unsigned long long* __restrict__ hash, const uint32_t* __restrict__ perm, uint32_t N,
                        int hi, uint32_t pb, uint64_t* __restrict__ keys) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
        const uint32_t p = perm ? perm[i] : i;
        const uint64_t h = hash[p];
        keys[i] = ((hi ? (h >> 32) : (h & 0xffffffffull)) << pb) | i;
    }
}
__global__ void k_hperm(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ perm, uint32_t N, uint32_t pb,
                        uint32_t* __restrict__ out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
        const uint32_t pos = (uint32_t)(keys[i] & ((1ull << pb) - 1));
        out[i] = perm ? perm[pos] : pos;
    }
}

__global__ void k_run_flags(const unsigned long long* __restrict__ hash, const uint32_t* __restrict__ perm, uint32_t N,
                            uint32_t* __restrict__ flag) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x)
        flag[i] = (i == 0 || hash[perm[i]] != hash[perm[i - 1]]) ? 1u : 0u;
}
__global__ void k_sub1(uint32_t* __restrict__ a, uint32_t n) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] -= 1u;
}
__global__ void k_run_start(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ rid, uint32_t N,
                            uint32_t* __restrict__ start) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x)
        if (flag[i]) start[rid[i]] = i;
}

// Pair sorted positions (i, i+1) at an even offset of the same hash run when the two nodes
// have the same label and exactly the same edge-end list (R33 at delta = 1).
__global__ void k_pair(const uint32_t* __restrict__ perm, const uint32_t* __restrict__ flag,
                       const uint32_t* __restrict__ rid, const uint32_t* __restrict__ start, uint32_t N,
                       const uint32_t* __restrict__ label, const uint32_t* __restrict__ cnt,
                       const uint32_t* __restrict__ first, const uint64_t* __restrict__ ends, uint32_t sh1,
                       uint32_t* __restrict__ partner) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i + 1 < N; i += gridDim.x * blockDim.x) {
        if (flag[i + 1] || ((i - start[rid[i]]) & 1u)) continue;
        const uint32_t p = perm[i], q = perm[i + 1];
        if (label[p] != label[q] || cnt[p] != cnt[q]) continue;
        const uint64_t mask = (1ull << sh1) - 1;
        bool eq = true;
        for (uint32_t e = 0; e < cnt[p] && eq; e++) eq = (ends[first[p] + e] & mask) == (ends[first[q] + e] & mask);
        if (!eq) continue;
        partner[p] = q;
        partner[q] = p;
    }
}

__global__ void k_leaders(const uint32_t* __restrict__ partner, uint32_t N, uint32_t* __restrict__ lead) {
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < N; p += gridDim.x * blockDim.x)
        lead[p] = (partner[p] == kNone || partner[p] > p) ? 1u : 0u;
}
__global__ void k_new_ids(const uint32_t* __restrict__ partner, const uint32_t* __restrict__ lead,
                          const uint32_t* __restrict__ pos, const uint32_t* __restrict__ label_prev, uint32_t N,
                          uint32_t* __restrict__ nid, uint32_t* __restrict__ label_new) {
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < N; p += gridDim.x * blockDim.x) {
        const uint32_t leader = lead[p] ? p : partner[p];
        nid[p] = pos[leader];
        if (lead[p]) label_new[pos[p]] = label_prev[p];
    }
}
__global__ void k_regroup(uint32_t* __restrict__ grp_new, const uint32_t* __restrict__ grp_prev,
                          const uint32_t* __restrict__ nid, uint32_t n) {
    for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x)
        grp_new[x] = nid[grp_prev[x]];
}

__global__ void k_edge_newkeys(const uint64_t* __restrict__ ekey, uint64_t ne, const uint32_t* __restrict__ nid,
                               uint64_t* __restrict__ out) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ne) return;
    const uint64_t k = ekey[i];
    out[i] = ((uint64_t)nid[(uint32_t)(k >> 32)] << 32) | nid[(uint32_t)k];
}
__global__ void k_edge_slots(const uint64_t* __restrict__ ekey, const uint32_t* __restrict__ ew, uint64_t ne,
                             const uint32_t* __restrict__ nid, const uint32_t* __restrict__ lead,
                             const uint64_t* __restrict__ nkeys, uint64_t nn, uint32_t* __restrict__ slots) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ne) return;
    const uint64_t k = ekey[i];
    const uint32_t u1 = (uint32_t)(k >> 32), v1 = (uint32_t)k;
    const uint64_t t = ((uint64_t)nid[u1] << 32) | nid[v1];
    uint64_t lo = 0, hi = nn;   // the level-i edge (binary search in the sorted unique keys)
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (nkeys[mid] < t) lo = mid + 1; else hi = mid;
    }
    const uint32_t slot = (lead[u1] ? 0u : 2u) + (lead[v1] ? 0u : 1u);
    atomicMax(slots + 4 * lo + slot, ew[i]);
}
__global__ void k_edge_weights(const uint32_t* __restrict__ slots, uint64_t nn, uint32_t* __restrict__ w) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nn) return;
    const uint32_t* s = slots + 4 * i;   // [U' first/second][V' first/second]
    w[i] = max(s[0], s[2]) + max(s[1], s[3]);
}

__global__ void k_internal_counts(const uint32_t* __restrict__ off, const uint32_t* __restrict__ arc, uint32_t n,
                                  uint64_t m, uint32_t lbits, const uint32_t* __restrict__ grp, uint32_t* co,
                                  uint32_t* ci) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const uint32_t x = src_of(off, n, i), y = arc[i] >> lbits;
    if (grp[x] == grp[y]) {
        atomicAdd(co + x, 1u);
        atomicAdd(ci + y, 1u);
    }
}
__global__ void k_node_weight(const uint32_t* __restrict__ grp, const uint32_t* __restrict__ co,
                              const uint32_t* __restrict__ ci, uint32_t n, uint32_t* wout, uint32_t* win) {
    for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x) {
        if (co[x]) atomicMax(wout + grp[x], co[x]);
        if (ci[x]) atomicMax(win + grp[x], ci[x]);
    }
}
__global__ void k_totals(const uint32_t* __restrict__ w, uint32_t N, unsigned long long* tot) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) tot[i] = w[i];
}
__global__ void k_edge_totals(const uint64_t* __restrict__ ekey, const uint32_t* __restrict__ ew, uint64_t ne,
                              unsigned long long* tot) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ne) return;
    const uint32_t u = (uint32_t)(ekey[i] >> 32), v = (uint32_t)ekey[i];
    if (u != v) atomicAdd(tot + u, (unsigned long long)ew[i]);
}

// Weighted candidate test (R36) of every data vertex through its node, one warp per bitmap
// word, every query vertex of the launch; the result is ANDed into B (or written if fresh).
__global__ void __launch_bounds__(256) k_wcheck(uint32_t n, uint32_t nw, const uint32_t* __restrict__ grp,
                                                const uint32_t* __restrict__ label,
                                                const unsigned long long* __restrict__ tout,
                                                const unsigned long long* __restrict__ tin,
                                                const ChkQV* __restrict__ qv, uint32_t nf, int fresh) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nw; w += nwarps) {
        const uint32_t v = w * 32 + lane;
        const bool in = v < n;
        const uint32_t X = in ? grp[v] : 0u;
        const uint32_t lab = in ? label[X] : 0u;
        const unsigned long long to = in ? tout[X] : 0ull, ti = in ? tin[X] : 0ull;
        for (uint32_t f0 = 0; f0 < nf; f0 += 32) {
            uint32_t mine = 0;
            const uint32_t fe = min(nf - f0, 32u);
            for (uint32_t x = 0; x < fe; x++) {
                const ChkQV q = qv[f0 + x];
                const bool ok = in && (q.lab < 0 || (uint32_t)q.lab == lab) &&
                                (q.bound < 0 || grp[(uint32_t)q.bound] == X) && q.qout <= to && q.qin <= ti;
                const uint32_t m = __ballot_sync(0xffffffffu, ok);
                if (lane == x) mine = m;
            }
            if (lane < fe) {
                uint32_t* B = qv[f0 + lane].B;
                B[w] = fresh ? mine : (B[w] & mine);
            }
        }
    }
}

uint32_t bits_of(uint64_t x) {
    uint32_t b = 0;
    while (b < 64 && (x >> b)) b++;
    return b;
}

}  // namespace

// ---- host side -------------------------------------------------------------
struct CLevel {
    uint32_t N = 0;
    uint32_t *grp = nullptr, *label = nullptr, *wout = nullptr, *win = nullptr;
    unsigned long long *tout = nullptr, *tin = nullptr;
    uint64_t *ekey_out = nullptr, *ekey_in = nullptr;
    uint32_t *ew_out = nullptr, *ew_in = nullptr;
    uint64_t ne_out = 0, ne_in = 0;
};

}  // namespace gps

struct gps_compressed {
    const gps_graph* g = nullptr;
    int device = 0;
    std::vector<gps::CLevel> lv;   // lv[0] = the original graph (level 0), lv[i] = level i
    std::vector<void*> mem;
};

namespace gps {

namespace {

template <typename T>
T* cmalloc(gps_compressed* cg, size_t count) {
    void* p = nullptr;
    GPS_CK(cudaMalloc(&p, sizeof(T) * (count ? count : 1) + 16));
    cg->mem.push_back(p);
    return static_cast<T*>(p);
}

uint64_t d2h1(gps_ctx* c, const uint32_t* p) {
    uint32_t h = 0;
    GPS_CK(cudaMemcpyAsync(&h, p, 4, cudaMemcpyDeviceToHost, c->stream));
    ctx_sync(c);
    return h;
}

dim3 grid_for(uint64_t n, uint32_t T = 256) {
    return dim3((uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((n + T - 1) / T, 1u << 30)));
}

// Level-0 weighted edges of one direction (x -> y with #labelled arcs; in: x <- y).
void edges0(gps_ctx* c, gps_compressed* cg, const DevGraph& d, bool in, uint64_t m, uint64_t** key, uint32_t** w,
            uint64_t* ne) {
    const uint32_t* off = in ? d.off_in : d.off_out;
    const uint32_t* arc = in ? d.arc_in : d.arc_out;
    DevPtr flag(c, sizeof(uint32_t) * (m + 1)), pos(c, sizeof(uint32_t) * (m + 1));
    if (m) launch(c, GPS_K_LOAD, grid_for(m), dim3(256), 0, k_edge0_flags, off, arc, d.n, m, d.lbits, flag.as<uint32_t>());
    scan_exclusive1<uint32_t, uint32_t>(c, flag.as<uint32_t>(), pos.as<uint32_t>(), m);
    *ne = m ? d2h1(c, pos.as<uint32_t>() + m) : 0;
    *key = cmalloc<uint64_t>(cg, *ne);
    *w = cmalloc<uint32_t>(cg, *ne);
    if (m)
        launch(c, GPS_K_LOAD, grid_for(m), dim3(256), 0, k_edge0_emit, off, arc, d.n, m, d.lbits,
               (const uint32_t*)flag.as<uint32_t>(), (const uint32_t*)pos.as<uint32_t>(), *key, *w);
}

// Sort + unique u64 keys in place (keys[0..m)), returns the unique count (compacted to out).
uint64_t sort_unique(gps_ctx* c, uint64_t* keys, uint64_t m, int nbits, uint64_t* out) {
    if (m == 0) return 0;
    DevPtr tmp(c, sizeof(uint64_t) * m);
    radix_sort_u64(c, keys, tmp.as<uint64_t>(), m, nbits);
    DevPtr flag(c, sizeof(uint32_t) * (m + 1)), pos(c, sizeof(uint32_t) * (m + 1));
    launch(c, GPS_K_LOAD, grid_for(m), dim3(256), 0, k_flags, (const uint64_t*)keys, m, flag.as<uint32_t>());
    scan_exclusive1<uint32_t, uint32_t>(c, flag.as<uint32_t>(), pos.as<uint32_t>(), m);
    const uint64_t u = d2h1(c, pos.as<uint32_t>() + m);
    launch(c, GPS_K_LOAD, grid_for(m), dim3(256), 0, k_compact, (const uint64_t*)keys,
           (const uint32_t*)flag.as<uint32_t>(), (const uint32_t*)pos.as<uint32_t>(), m, out);
    return u;
}

// Weighted edges of level i from level i-1 (R35).
void edges_next(gps_ctx* c, gps_compressed* cg, const uint64_t* ekey, const uint32_t* ew, uint64_t ne,
                const uint32_t* nid, const uint32_t* lead, uint32_t Nn, uint64_t** okey, uint32_t** ow, uint64_t* one) {
    DevPtr nk(c, sizeof(uint64_t) * (ne + 1)), uk(c, sizeof(uint64_t) * (ne + 1));
    if (ne) launch(c, GPS_K_LOAD, grid_for(ne), dim3(256), 0, k_edge_newkeys, ekey, ne, nid, nk.as<uint64_t>());
    const uint64_t nn = sort_unique(c, nk.as<uint64_t>(), ne, (int)(32 + bits_of(Nn ? Nn - 1 : 0)), uk.as<uint64_t>());
    *okey = cmalloc<uint64_t>(cg, nn);
    *ow = cmalloc<uint32_t>(cg, nn);
    *one = nn;
    if (!nn) return;
    GPS_CK(cudaMemcpyAsync(*okey, uk.p, sizeof(uint64_t) * nn, cudaMemcpyDeviceToDevice, c->stream));
    DevPtr slots(c, sizeof(uint32_t) * 4 * nn);
    GPS_CK(cudaMemsetAsync(slots.p, 0, sizeof(uint32_t) * 4 * nn, c->stream));
    launch(c, GPS_K_LOAD, grid_for(ne), dim3(256), 0, k_edge_slots, ekey, ew, ne, nid, lead, (const uint64_t*)*okey, nn,
           slots.as<uint32_t>());
    launch(c, GPS_K_LOAD, grid_for(nn), dim3(256), 0, k_edge_weights, (const uint32_t*)slots.as<uint32_t>(), nn, *ow);
}

void build_level(gps_ctx* c, gps_compressed* cg, const gps_graph* g, const CLevel& P, CLevel& L) {
    const DevGraph& d = g->d;
    const uint32_t n = d.n, Np = P.N;
    const uint64_t m = g->m;   // stored out-arcs
    const uint32_t b = std::max<uint32_t>(1, bits_of(Np ? Np - 1 : 0));
    const uint32_t sh1 = b + d.lbits + 1;
    if (sh1 + b > 64) fail(GPS_EUNSUPPORTED, "compression keys wider than 64 bits");
    if (2 * m >= (1ull << 32)) fail(GPS_EUNSUPPORTED, "compression of more than 2^31 arcs");
    // 1. edge ends of the level-(i-1) nodes, sorted + unique
    DevPtr keys(c, sizeof(uint64_t) * (2 * m + 1)), ends(c, sizeof(uint64_t) * (2 * m + 1));
    if (m) launch(c, GPS_K_LOAD, grid_for(m), dim3(256), 0, k_adj_keys, d.off_out, d.arc_out, n, m, d.lbits, P.grp, b,
                  keys.as<uint64_t>());
    const uint64_t ue = sort_unique(c, keys.as<uint64_t>(), 2 * m, (int)(sh1 + b), ends.as<uint64_t>());
    keys.reset();
    // 2. set hash, count and first edge end of every node
    DevPtr hash(c, sizeof(unsigned long long) * (Np + 1)), cnt(c, sizeof(uint32_t) * (Np + 1)),
        first(c, sizeof(uint32_t) * (Np + 1));
    GPS_CK(cudaMemsetAsync(hash.p, 0, sizeof(unsigned long long) * Np, c->stream));
    GPS_CK(cudaMemsetAsync(cnt.p, 0, sizeof(uint32_t) * Np, c->stream));
    GPS_CK(cudaMemsetAsync(first.p, 0, sizeof(uint32_t) * Np, c->stream));
    if (ue)
        launch(c, GPS_K_LOAD, grid_for(ue), dim3(256), 0, k_set_hash, (const uint64_t*)ends.as<uint64_t>(), ue, sh1,
               hash.as<unsigned long long>(), cnt.as<uint32_t>(), first.as<uint32_t>());
    launch(c, GPS_K_LOAD, grid_for(Np), dim3(256), 0, k_hash_label, hash.as<unsigned long long>(), P.label, Np);
    // 3. nodes sorted by (hash, id): LSD over the two 32-bit halves, positions composed
    const uint32_t pb = std::max<uint32_t>(1, bits_of(Np ? Np - 1 : 0));
    DevPtr hk(c, sizeof(uint64_t) * (Np + 1)), tmp(c, sizeof(uint64_t) * (Np + 1));
    DevPtr pa(c, sizeof(uint32_t) * (Np + 1)), pbuf(c, sizeof(uint32_t) * (Np + 1));
    launch(c, GPS_K_LOAD, grid_for(Np), dim3(256), 0, k_hkeys, (const unsigned long long*)hash.as<unsigned long long>(),
           (const uint32_t*)nullptr, Np, 0, pb, hk.as<uint64_t>());
    radix_sort_u64(c, hk.as<uint64_t>(), tmp.as<uint64_t>(), Np, (int)(32 + pb));
    launch(c, GPS_K_LOAD, grid_for(Np), dim3(256), 0, k_hperm, (const uint64_t*)hk.as<uint64_t>(), (const uint32_t*)nullptr,
           Np, pb, pa.as<uint32_t>());
    launch(c, GPS_K_LOAD, grid_for(Np), dim3(256), 0, k_hkeys, (const unsigned long long*)hash.as<unsigned long long>(),
           (const uint32_t*)pa.as<uint32_t>(), Np, 1, pb, hk.as<uint64_t>());
    radix_sort_u64(c, hk.as<uint64_t>(), tmp.as<uint64_t>(), Np, (int)(32 + pb));
    launch(c, GPS_K_LOAD, grid_for(Np), dim3(256), 0, k_hperm, (const uint64_t*)hk.as<uint64_t>(),
           (const uint32_t*)pa.as<uint32_t>(), Np, pb, pbuf.as<uint32_t>());
    const uint32_t* perm = pbuf.as<uint32_t>();
    // 4. hash runs and pairs
    DevPtr flag(c, sizeof(uint32_t) * (Np + 1)), rpos(c, sizeof(uint32_t) * (Np + 1)), start(c, sizeof(uint32_t) * (Np + 1));
    DevPtr rid(c, sizeof(uint32_t) * (Np + 1));
    launch(c, GPS_K_LOAD, grid_for(Np), dim3(256), 0, k_run_flags, (const unsigned long long*)hash.as<unsigned long long>(),
           perm, Np, flag.as<uint32_t>());
    scan_exclusive1<uint32_t, uint32_t>(c, flag.as<uint32_t>(), rpos.as<uint32_t>(), Np);
    // run id of position i = (#flags in [0, i]) - 1 = rpos[i + 1] - 1: shift by one
    GPS_CK(cudaMemcpyAsync(rid.p, rpos.as<uint32_t>() + 1, sizeof(uint32_t) * Np, cudaMemcpyDeviceToDevice, c->stream));
    launch(c, GPS_K_LOAD, grid_for(Np), dim3(256), 0, k_sub1, rid.as<uint32_t>(), Np);
    launch(c, GPS_K_LOAD, grid_for(Np), dim3(256), 0, k_run_start, (const uint32_t*)flag.as<uint32_t>(),
           (const uint32_t*)rid.as<uint32_t>(), Np, start.as<uint32_t>());
    DevPtr partner(c, sizeof(uint32_t) * (Np + 1));
    GPS_CK(cudaMemsetAsync(partner.p, 0xff, sizeof(uint32_t) * Np, c->stream));
    launch(c, GPS_K_LOAD, grid_for(Np), dim3(256), 0, k_pair, perm, (const uint32_t*)flag.as<uint32_t>(),
           (const uint32_t*)rid.as<uint32_t>(), (const uint32_t*)start.as<uint32_t>(), Np, (const uint32_t*)P.label,
           (const uint32_t*)cnt.as<uint32_t>(), (const uint32_t*)first.as<uint32_t>(),
           (const uint64_t*)ends.as<uint64_t>(), sh1, partner.as<uint32_t>());
    // 5. new ids (leaders in id order), groups, labels
    DevPtr lead(c, sizeof(uint32_t) * (Np + 1)), lpos(c, sizeof(uint32_t) * (Np + 1)), nid(c, sizeof(uint32_t) * (Np + 1));
    launch(c, GPS_K_LOAD, grid_for(Np), dim3(256), 0, k_leaders, (const uint32_t*)partner.as<uint32_t>(), Np,
           lead.as<uint32_t>());
    scan_exclusive1<uint32_t, uint32_t>(c, lead.as<uint32_t>(), lpos.as<uint32_t>(), Np);
    L.N = (uint32_t)d2h1(c, lpos.as<uint32_t>() + Np);
    L.grp = cmalloc<uint32_t>(cg, n);
    L.label = cmalloc<uint32_t>(cg, L.N);
    launch(c, GPS_K_LOAD, grid_for(Np), dim3(256), 0, k_new_ids, (const uint32_t*)partner.as<uint32_t>(),
           (const uint32_t*)lead.as<uint32_t>(), (const uint32_t*)lpos.as<uint32_t>(), (const uint32_t*)P.label, Np,
           nid.as<uint32_t>(), L.label);
    launch(c, GPS_K_LOAD, grid_for(n), dim3(256), 0, k_regroup, L.grp, (const uint32_t*)P.grp,
           (const uint32_t*)nid.as<uint32_t>(), n);
    // 6. weighted edges (recursion) and node weights
    edges_next(c, cg, P.ekey_out, P.ew_out, P.ne_out, nid.as<uint32_t>(), lead.as<uint32_t>(), L.N, &L.ekey_out,
               &L.ew_out, &L.ne_out);
    edges_next(c, cg, P.ekey_in, P.ew_in, P.ne_in, nid.as<uint32_t>(), lead.as<uint32_t>(), L.N, &L.ekey_in, &L.ew_in,
               &L.ne_in);
    L.wout = cmalloc<uint32_t>(cg, L.N);
    L.win = cmalloc<uint32_t>(cg, L.N);
    GPS_CK(cudaMemsetAsync(L.wout, 0, sizeof(uint32_t) * L.N, c->stream));
    GPS_CK(cudaMemsetAsync(L.win, 0, sizeof(uint32_t) * L.N, c->stream));
    {
        DevPtr co(c, sizeof(uint32_t) * (n + 1)), ci(c, sizeof(uint32_t) * (n + 1));
        GPS_CK(cudaMemsetAsync(co.p, 0, sizeof(uint32_t) * n, c->stream));
        GPS_CK(cudaMemsetAsync(ci.p, 0, sizeof(uint32_t) * n, c->stream));
        if (m)
            launch(c, GPS_K_LOAD, grid_for(m), dim3(256), 0, k_internal_counts, d.off_out, d.arc_out, n, m, d.lbits,
                   (const uint32_t*)L.grp, co.as<uint32_t>(), ci.as<uint32_t>());
        launch(c, GPS_K_LOAD, grid_for(n), dim3(256), 0, k_node_weight, (const uint32_t*)L.grp,
               (const uint32_t*)co.as<uint32_t>(), (const uint32_t*)ci.as<uint32_t>(), n, L.wout, L.win);
    }
    L.tout = cmalloc<unsigned long long>(cg, L.N);
    L.tin = cmalloc<unsigned long long>(cg, L.N);
    launch(c, GPS_K_LOAD, grid_for(L.N), dim3(256), 0, k_totals, (const uint32_t*)L.wout, L.N, L.tout);
    launch(c, GPS_K_LOAD, grid_for(L.N), dim3(256), 0, k_totals, (const uint32_t*)L.win, L.N, L.tin);
    if (L.ne_out)
        launch(c, GPS_K_LOAD, grid_for(L.ne_out), dim3(256), 0, k_edge_totals, (const uint64_t*)L.ekey_out,
               (const uint32_t*)L.ew_out, L.ne_out, L.tout);
    if (L.ne_in)
        launch(c, GPS_K_LOAD, grid_for(L.ne_in), dim3(256), 0, k_edge_totals, (const uint64_t*)L.ekey_in,
               (const uint32_t*)L.ew_in, L.ne_in, L.tin);
    ctx_sync(c);
}

}  // namespace

gps_compressed* compress_graph(gps_ctx* c, const gps_graph* g, uint32_t nlev, const float* deltas) {
    for (uint32_t i = 0; i < nlev; i++)
        if (!(deltas[i] > 0.0f && deltas[i] <= 1.0f)) fail(GPS_EINVAL, "delta must be in (0, 1]");
    for (uint32_t i = 0; i < nlev; i++)
        if (deltas[i] != 1.0f)
            fail(GPS_EUNSUPPORTED, "delta < 1 (a similarity join) is not built on the device; delta = 1 only");
    auto* cg = new gps_compressed();
    cg->g = g;
    cg->device = c->device;
    try {
        const DevGraph& d = g->d;
        CLevel L0;
        L0.N = d.n;
        L0.grp = cmalloc<uint32_t>(cg, d.n);
        L0.label = cmalloc<uint32_t>(cg, d.n);
        launch(c, GPS_K_LOAD, grid_for(d.n), dim3(256), 0, k_iota, L0.grp, d.n);
        launch(c, GPS_K_LOAD, grid_for(d.n), dim3(256), 0, k_label_u32, (const uint16_t*)d.vlab, d.n, L0.label);
        edges0(c, cg, d, false, g->m, &L0.ekey_out, &L0.ew_out, &L0.ne_out);
        edges0(c, cg, d, true, g->m, &L0.ekey_in, &L0.ew_in, &L0.ne_in);
        cg->lv.push_back(L0);
        for (uint32_t i = 0; i < nlev; i++) {
            CLevel L;
            build_level(c, cg, g, cg->lv.back(), L);
            cg->lv.push_back(L);
        }
        ctx_sync(c);
    } catch (...) {
        free_compressed(cg);
        throw;
    }
    return cg;
}

void free_compressed(gps_compressed* cg) {
    if (!cg) return;
    if (cg->g && cg->g->cg == cg) {   // still attached: detach so the graph never points at freed levels
        gps_graph* g = const_cast<gps_graph*>(cg->g);
        g->cg = nullptr;
        g->cg_level = 0;
    }
    for (void* p : cg->mem) cudaFree(p);
    delete cg;
}

uint32_t compressed_levels(const gps_compressed* cg) { return (uint32_t)cg->lv.size() - 1; }
const gps_graph* compressed_graph(const gps_compressed* cg) { return cg->g; }

void compressed_level_info(const gps_compressed* cg, uint32_t level, uint32_t* N, uint64_t* ne_out, uint64_t* ne_in) {
    if (level == 0 || level >= cg->lv.size()) fail(GPS_EINVAL, "compression level out of range");
    const CLevel& L = cg->lv[level];
    if (N) *N = L.N;
    if (ne_out) *ne_out = L.ne_out;
    if (ne_in) *ne_in = L.ne_in;
}

void compressed_fetch(gps_ctx* c, const gps_compressed* cg, uint32_t level, uint32_t* grp, uint32_t* label,
                      uint32_t* wout, uint32_t* win, uint64_t* ekey_out, uint32_t* ew_out, uint64_t* ekey_in,
                      uint32_t* ew_in) {
    if (level == 0 || level >= cg->lv.size()) fail(GPS_EINVAL, "compression level out of range");
    const CLevel& L = cg->lv[level];
    const uint32_t n = cg->g->d.n;
    auto cp = [&](void* dst, const void* src, size_t bytes) {
        if (dst && bytes) GPS_CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
    };
    cp(grp, L.grp, sizeof(uint32_t) * n);
    cp(label, L.label, sizeof(uint32_t) * L.N);
    cp(wout, L.wout, sizeof(uint32_t) * L.N);
    cp(win, L.win, sizeof(uint32_t) * L.N);
    cp(ekey_out, L.ekey_out, sizeof(uint64_t) * L.ne_out);
    cp(ew_out, L.ew_out, sizeof(uint32_t) * L.ne_out);
    cp(ekey_in, L.ekey_in, sizeof(uint64_t) * L.ne_in);
    cp(ew_in, L.ew_in, sizeof(uint32_t) * L.ne_in);
    ctx_sync(c);
}

// The weighted candidate test of compression level `level`, for the query vertices qv
// (their bitmaps B over the original vertices): fresh = write, else AND into B.
void run_wcheck(gps_ctx* c, const gps_compressed* cg, uint32_t level, const ChkQV* d_qv, uint32_t nf, bool fresh) {
    if (!cg || nf == 0) return;
    if (level == 0 || level >= cg->lv.size()) fail(GPS_EINVAL, "compression level out of range");
    const CLevel& L = cg->lv[level];
    const DevGraph& d = cg->g->d;
    const uint32_t blocks = std::min<uint32_t>((d.nw + 7) / 8, (uint32_t)c->nsm * 8);
    launch(c, GPS_K_CHECK, dim3(std::max<uint32_t>(1, blocks)), dim3(256), 0, k_wcheck, d.n, d.nw,
           (const uint32_t*)L.grp, (const uint32_t*)L.label, (const unsigned long long*)L.tout,
           (const unsigned long long*)L.tin, d_qv, nf, fresh ? 1 : 0);
}

}  // namespace gps
