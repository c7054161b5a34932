// pairs.cuh -- load-balanced iteration over a "pair space".
//
// Rows (candidate keys, partial embeddings) own segments of work (adjacency
// arcs, EC values) given by a non-decreasing offset function offs(i), i in
// [0, nrows], offs(nrows) = P.  G persistent blocks each take an equal,
// contiguous range of pairs -- so a hub row with 10^4 arcs is shared by many
// blocks instead of stalling one warp (the imbalance P:784 addresses with
// "an entire block instead of a warp").  Within a block, consecutive threads
// get consecutive pairs (coalesced segment reads); the row of each pair is
// found by binary search in a shared-memory window of offsets.
#pragma once
#include "prims.cuh"

namespace gps {

template <typename OffF>
__device__ __forceinline__ uint64_t pairs_find_global(OffF offs, uint64_t lo, uint64_t hi, uint64_t p) {
    // largest r in [lo, hi) with offs(r) <= p   (requires offs(lo) <= p)
    while (hi - lo > 1) {
        uint64_t mid = lo + (hi - lo) / 2;
        if (offs(mid) <= p) lo = mid; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ uint32_t pairs_find_smem(const uint64_t* s, uint32_t n, uint64_t p) {
    uint32_t lo = 0, hi = n;
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (s[mid] <= p) lo = mid; else hi = mid;
    }
    return lo;
}

// Contiguous share [p0, p1) of P pairs for block b of G.
__device__ __forceinline__ void pairs_range(uint64_t P, uint32_t b, uint32_t G, uint64_t& p0, uint64_t& p1) {
    const uint64_t q = P / G, rem = P % G;
    p0 = q * b + (b < rem ? b : rem);
    p1 = p0 + q + (b < rem ? 1 : 0);
}

// Calls body(valid, p, row, j) for every item slot of the block's range, T*IPT
// slots per chunk, all threads together (body may use block-wide barriers).
// s_off must hold W+1 uint64 in shared memory.
template <int T, int IPT, int W, typename OffF, typename Body>
__device__ __forceinline__ void for_pairs(uint64_t p0, uint64_t p1, uint64_t nrows, OffF offs, uint64_t* s_off,
                                          uint64_t* s_row, Body&& body) {
    if (p0 >= p1) return;
    const uint32_t tid = threadIdx.x;
    if (tid == 0) *s_row = pairs_find_global(offs, 0, nrows, p0);
    __syncthreads();
    uint64_t r0 = *s_row;
    for (uint64_t cp = p0; cp < p1; cp += (uint64_t)T * IPT) {
        const uint64_t cend = cp + (uint64_t)T * IPT < p1 ? cp + (uint64_t)T * IPT : p1;
        const uint32_t wn = (uint32_t)((nrows - r0) < (uint64_t)W ? (nrows - r0) : (uint64_t)W);
        for (uint32_t i = tid; i <= wn; i += T) s_off[i] = offs(r0 + i);
        __syncthreads();
        const uint64_t wend = s_off[wn];
#pragma unroll 1
        for (int it = 0; it < IPT; it++) {
            const uint64_t p = cp + (uint64_t)it * T + tid;
            const bool v = p < cend;
            uint64_t row = 0, base = 0;
            if (v) {
                if (p < wend) {
                    const uint32_t i = pairs_find_smem(s_off, wn, p);
                    row = r0 + i;
                    base = s_off[i];
                } else {
                    row = pairs_find_global(offs, r0 + wn, nrows, p);
                    base = offs(row);
                }
            }
            body(v, p, row, p - base);
        }
        __syncthreads();
        if (cend < p1) {
            if (tid == 0)
                *s_row = (cend < wend) ? r0 + pairs_find_smem(s_off, wn, cend)
                                       : pairs_find_global(offs, r0 + wn, nrows, cend);
            __syncthreads();
            r0 = *s_row;
        }
    }
}

// Warp-segmented reduction for lanes holding consecutive pairs: lanes with the
// same key form one group (keys are non-decreasing across lanes).  Returns the
// group's OR / sum in the group's lowest lane (is_leader), 0 elsewhere.
__device__ __forceinline__ uint32_t warp_group_leader(uint32_t key, uint32_t& peers) {
    peers = __match_any_sync(kFull, key);
    return (uint32_t)(__ffs(peers) - 1);
}

// Last-block pattern: every block stores its count in blk[b]; the last block to
// finish turns blk[0..G) into exclusive offsets, blk[G] = total, info[0] = P,
// info[1] = total, and resets *done.
__device__ __forceinline__ void last_block_scan(uint64_t* blk, uint32_t G, unsigned int* done, uint64_t* info,
                                                uint64_t P, uint64_t my_count) {
    __shared__ bool s_last;
    my_count = block_sum(my_count);
    if (threadIdx.x == 0) {
        blk[blockIdx.x] = my_count;
        __threadfence();
        const unsigned prev = atomicAdd(done, 1u);
        s_last = (prev == G - 1);
    }
    __syncthreads();
    if (s_last) {
        __threadfence();
        uint64_t carry = 0;
        for (uint32_t b = 0; b < G; b += blockDim.x) {
            const uint32_t i = b + threadIdx.x;
            const uint64_t v = i < G ? __ldcg(blk + i) : 0ull;
            uint64_t tot;
            const uint64_t ex = block_excl_scan(v, &tot);
            if (i < G) blk[i] = carry + ex;
            carry += tot;
        }
        if (threadIdx.x == 0) {
            blk[G] = carry;
            info[0] = P;
            info[1] = carry;
            *done = 0u;
        }
    }
}

}  // namespace gps

namespace gps {

// Exclusive prefix of per-job pair counts pj(i), i < nj, into s_jp[0..nj]
// (shared memory).  All threads of the block call it.
template <typename PF>
__device__ __forceinline__ void job_prefix(uint32_t nj, PF pj, uint64_t* s_jp) {
    uint64_t carry = 0;
    for (uint32_t b = 0; b < nj; b += blockDim.x) {
        const uint32_t i = b + threadIdx.x;
        const uint64_t v = i < nj ? pj(i) : 0ull;
        uint64_t tot;
        const uint64_t ex = block_excl_scan(v, &tot);
        if (i < nj) s_jp[i] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) s_jp[nj] = carry;
    __syncthreads();
}

// Calls jb(j, lo, hi) for every job j whose pair range meets [p0, p1), with the
// job-local sub-range [lo, hi).  Uniform across the block.
template <typename JB>
__device__ __forceinline__ void for_job_ranges(const uint64_t* s_jp, uint32_t nj, uint64_t p0, uint64_t p1, JB&& jb) {
    if (p0 >= p1 || nj == 0) return;
    uint32_t lo = 0, hi = nj;   // largest j < nj with s_jp[j] <= p0
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (s_jp[mid] <= p0) lo = mid; else hi = mid;
    }
    for (uint32_t j = lo; j < nj && s_jp[j] < p1; j++) {
        const uint64_t a = p0 > s_jp[j] ? p0 : s_jp[j];
        const uint64_t b = p1 < s_jp[j + 1] ? p1 : s_jp[j + 1];
        if (a < b) jb(j, a - s_jp[j], b - s_jp[j]);
    }
}

}  // namespace gps

namespace gps {

// Chunked pair iteration with per-row metadata staged in shared memory.
//
// Per chunk of T*IPT consecutive pairs: the offsets of a window of W rows are
// staged (coalesced), then load_meta(row) -> Meta is evaluated ONCE per row that
// meets the chunk (in parallel) and kept in s_meta.  Thread t owns the IPT
// CONSECUTIVE pairs cp + t*IPT + [0, IPT): one shared-memory binary search finds
// the row of its first pair, the rest walk forward.  body(v[], m[], j[])
// receives all IPT items at once (rows non-decreasing across the items and
// across the threads of the block), so it can issue their global loads back to
// back and aggregate per row.  Rows outside the window (runs of empty rows) fall
// back to load_meta from global.  body may use block-wide barriers.
template <typename Meta, int T, int IPT, int W, int NB, typename OffF, typename LoadMeta, typename Body>
__device__ __forceinline__ void pair_chunks(uint64_t p0, uint64_t p1, uint64_t nrows, OffF offs, LoadMeta load_meta,
                                            Meta* s_meta, uint64_t* s_off, Body&& body) {
    // s_off holds NB*(W+1) and s_meta NB*W entries.  NB = 2 double-buffers the
    // window, so a chunk needs ONE block barrier (between staging and use); the row
    // of the next chunk is recomputed by every thread from the current window.
    if (p0 >= p1) return;
    const uint32_t tid = threadIdx.x;
    uint64_t r0 = pairs_find_global(offs, 0, nrows, p0);
    int buf = 0;
    for (uint64_t cp = p0; cp < p1; cp += (uint64_t)T * IPT, buf = (NB == 2) ? buf ^ 1 : 0) {
        uint64_t* so = s_off + buf * (W + 1);
        Meta* sm = s_meta + buf * W;
        const uint64_t cend = cp + (uint64_t)T * IPT < p1 ? cp + (uint64_t)T * IPT : p1;
        const uint32_t wn = (uint32_t)((nrows - r0) < (uint64_t)W ? (nrows - r0) : (uint64_t)W);
        for (uint32_t i = tid; i <= wn; i += T) {
            const uint64_t a = offs(r0 + i);
            so[i] = a;
            if (i < wn && a < cend) {
                const uint64_t b = offs(r0 + i + 1);
                if (b > a) sm[i] = load_meta(r0 + i);
            }
        }
        __syncthreads();
        const uint64_t wend = so[wn];
        bool v[IPT];
        Meta m[IPT];
        uint64_t j[IPT];
        const uint64_t pt = cp + (uint64_t)tid * IPT;
        uint32_t i = (pt < cend && pt < wend) ? pairs_find_smem(so, wn, pt) : 0;
#pragma unroll
        for (int it = 0; it < IPT; it++) {
            const uint64_t p = pt + it;
            v[it] = p < cend;
            j[it] = 0;
            if (v[it]) {
                if (p < wend) {
                    while (so[i + 1] <= p) i++;
                    m[it] = sm[i];
                    j[it] = p - so[i];
                } else {
                    const uint64_t row = pairs_find_global(offs, r0 + wn, nrows, p);
                    m[it] = load_meta(row);
                    j[it] = p - offs(row);
                }
            }
        }
        body(v, m, j);
        if (cend < p1)
            r0 = (cend < wend) ? r0 + pairs_find_smem(so, wn, cend) : pairs_find_global(offs, r0 + wn, nrows, cend);
        if (NB == 1) __syncthreads();   // the single window is restaged next
    }
    if (NB == 2) __syncthreads();   // the caller may reuse the shared buffers
}

// Dynamic shared memory of a pair kernel: [job prefix (nj+1)] [offset window
// NB*(W+1)] [row metadata NB*W] [extra].
template <typename Meta, int W, int NB>
struct PairSmem {
    static __host__ __device__ size_t a16(size_t x) { return (x + 15) & ~size_t(15); }
    static __host__ __device__ size_t off_off(uint32_t nj) { return a16(sizeof(uint64_t) * (nj + 1)); }
    static __host__ __device__ size_t meta_off(uint32_t nj) { return off_off(nj) + a16(sizeof(uint64_t) * NB * (W + 1)); }
    static __host__ __device__ size_t extra_off(uint32_t nj) { return meta_off(nj) + a16(sizeof(Meta) * NB * W); }
    static __host__ __device__ size_t bytes(uint32_t nj, size_t extra) { return extra_off(nj) + extra; }
};

// Per-key aggregation of a thread's IPT consecutive items (keys non-decreasing
// across items and lanes): runs wholly inside the thread are emitted directly;
// the thread's first and last runs (which may continue in the neighbouring
// lanes) are combined across the warp with __match_any_sync + redux, so a hub
// row spanning a whole warp costs one emit.  emit(key, agg) is called by one lane.
template <int IPT, typename Emit>
__device__ __forceinline__ void run_sum(const bool (&v)[IPT], const uint32_t (&key)[IPT], const uint32_t (&val)[IPT],
                                        Emit&& emit) {
    const uint32_t NONE = 0xffffffffu;
    uint32_t fk = NONE, fa = 0, ck = NONE, ca = 0;
    int nr = 0;
#pragma unroll
    for (int it = 0; it < IPT; it++) {
        if (!v[it]) continue;
        if (nr == 0) { ck = key[it]; ca = val[it]; nr = 1; }
        else if (key[it] == ck) ca += val[it];
        else {
            if (nr == 1) { fk = ck; fa = ca; } else if (ca) emit(ck, ca);
            ck = key[it]; ca = val[it]; nr++;
        }
    }
    {
        const uint32_t k1 = nr >= 2 ? fk : NONE;
        const uint32_t peers = __match_any_sync(kFull, k1);
        const uint32_t s = __reduce_add_sync(peers, nr >= 2 ? fa : 0u);
        if (k1 != NONE && lane_id() == (uint32_t)(__ffs(peers) - 1) && s) emit(k1, s);
    }
    {
        const uint32_t k2 = nr >= 1 ? ck : NONE;
        const uint32_t peers = __match_any_sync(kFull, k2);
        const uint32_t s = __reduce_add_sync(peers, nr >= 1 ? ca : 0u);
        if (k2 != NONE && lane_id() == (uint32_t)(__ffs(peers) - 1) && s) emit(k2, s);
    }
}

template <int IPT, typename Emit>
__device__ __forceinline__ void run_or64(const bool (&v)[IPT], const uint32_t (&key)[IPT],
                                         const unsigned long long (&val)[IPT], Emit&& emit) {
    const uint32_t NONE = 0xffffffffu;
    uint32_t fk = NONE, ck = NONE;
    unsigned long long fa = 0, ca = 0;
    int nr = 0;
#pragma unroll
    for (int it = 0; it < IPT; it++) {
        if (!v[it]) continue;
        if (nr == 0) { ck = key[it]; ca = val[it]; nr = 1; }
        else if (key[it] == ck) ca |= val[it];
        else {
            if (nr == 1) { fk = ck; fa = ca; } else if (ca) emit(ck, ca);
            ck = key[it]; ca = val[it]; nr++;
        }
    }
#pragma unroll
    for (int pass = 0; pass < 2; pass++) {
        const uint32_t k = pass == 0 ? (nr >= 2 ? fk : NONE) : (nr >= 1 ? ck : NONE);
        const unsigned long long a = pass == 0 ? (nr >= 2 ? fa : 0ull) : (nr >= 1 ? ca : 0ull);
        const uint32_t peers = __match_any_sync(kFull, k);
        const uint32_t lo = __reduce_or_sync(peers, (uint32_t)a);
        const uint32_t hi = __reduce_or_sync(peers, (uint32_t)(a >> 32));
        const unsigned long long agg = ((unsigned long long)hi << 32) | lo;
        if (k != NONE && lane_id() == (uint32_t)(__ffs(peers) - 1) && agg) emit(k, agg);
    }
}

}  // namespace gps
