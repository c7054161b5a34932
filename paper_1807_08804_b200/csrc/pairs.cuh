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
// Per chunk of CH = T*IPT consecutive pairs [cp, cend), one pass over a window
// of W rows starting at r0 (the row containing cp) stages, for every row that
// meets the chunk: its start relative to cp (s_start), load_meta(row) (s_meta,
// evaluated ONCE per row), a row-start mark at its first in-chunk pair (s_mark,
// window index as u16), the row covering each warp's first pair (s_wrow) and the
// row containing cend (s_next, the next chunk's r0).  After ONE block barrier,
// thread t owns the IPT consecutive pairs cp + t*IPT + [0, IPT): the window row
// of each is a running max over the marks, seeded by a warp max-scan and the
// warp's s_wrow -- no per-thread search and no walk over row boundaries.  If
// the window ends before cend the chunk is cut at the window end (every chunk
// covers at least row r0's remainder, so no global fallback exists).
//
// body(v[], wi[], j[], sm, r0) receives all IPT items at once: wi = window index
// of the item's row (row r0 + wi, metadata sm[wi]; rows non-decreasing across
// items and across the threads of the block), j = the pair's index within its row.  body
// may use block-wide barriers.  NB = 2 double-buffers the window so a chunk
// needs a single barrier.  Marks are cleared by the thread that read them, so
// the buffers are clean whenever pair_chunks returns.
template <typename Meta, int T, int IPT, int W, int NB>
struct PairSmem {
    static constexpr int CH = T * IPT;
    static_assert(IPT % 4 == 0, "marks are read as 4 x u16 vectors");
    static_assert(W <= 65535, "marks are u16 window indices");
    static __host__ __device__ constexpr size_t a16(size_t x) { return (x + 15) & ~size_t(15); }
    // one buffer: [start W u32][meta W][mark CH u16][wrow T/32 u32][next u32]
    static constexpr size_t START = 0;
    static constexpr size_t META = a16(sizeof(uint32_t) * W);
    static constexpr size_t MARK = META + a16(sizeof(Meta) * W);
    static constexpr size_t WROW = MARK + a16(sizeof(uint16_t) * CH);
    static constexpr size_t NEXT = WROW + sizeof(uint32_t) * (T / 32);
    static constexpr size_t BUF = a16(NEXT + sizeof(uint32_t));
    static __host__ __device__ size_t buf_off(uint32_t nj) { return a16(sizeof(uint64_t) * (nj + 1)); }
    static __host__ __device__ size_t extra_off(uint32_t nj) { return buf_off(nj) + NB * BUF; }
    static __host__ __device__ size_t bytes(uint32_t nj, size_t extra) { return extra_off(nj) + extra; }
    // zero the marks of every buffer (once per kernel, before the first chunk; needs a barrier after)
    static __device__ void init(char* bufs) {
        for (int b = 0; b < NB; b++) {
            uint2* m = reinterpret_cast<uint2*>(bufs + b * BUF + MARK);
            for (int i = threadIdx.x; i < CH / 4; i += blockDim.x) m[i] = make_uint2(0u, 0u);
        }
    }
};

// Largest r in [lo, hi) with offs(r) <= p (offs(lo) <= p): one warp, 32-ary
// search (about log32 of the range dependent global loads instead of log2).
template <typename OffF>
__device__ __forceinline__ uint64_t pairs_find_warp(OffF offs, uint64_t lo, uint64_t hi, uint64_t p) {
    const uint32_t lane = lane_id();
    while (hi - lo > 32) {
        const uint64_t step = (hi - lo + 31) / 32;   // probes lo + lane*step
        const uint64_t x = lo + lane * step;
        const bool le = x < hi && offs(x) <= p;
        const uint32_t b = __ballot_sync(kFull, le);   // lane 0 always set (offs(lo) <= p)
        const uint32_t last = 31 - __clz(b);
        const uint64_t nlo = lo + last * step;
        hi = (nlo + step < hi) ? nlo + step : hi;
        lo = nlo;
    }
    const uint64_t x = lo + lane;
    const bool le = x < hi && offs(x) <= p;
    return lo + (31 - __clz(__ballot_sync(kFull, le)));
}

template <typename Meta, int T, int IPT, int W, int NB, typename OffF, typename LoadMeta, typename Body>
__device__ __forceinline__ void pair_chunks(uint64_t p0, uint64_t p1, uint64_t nrows, OffF offs, LoadMeta load_meta,
                                            char* bufs, Body&& body) {
    using SM = PairSmem<Meta, T, IPT, W, NB>;
    constexpr uint32_t CH = SM::CH, WSPAN = 32 * IPT;
    if (p0 >= p1) return;
    const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
    uint64_t r0 = pairs_find_warp(offs, 0, nrows, p0);
    int buf = 0;
    for (uint64_t cp = p0; cp < p1; buf = (NB == 2) ? buf ^ 1 : 0) {
        char* B = bufs + buf * SM::BUF;
        uint32_t* s_start = reinterpret_cast<uint32_t*>(B + SM::START);
        Meta* s_meta = reinterpret_cast<Meta*>(B + SM::META);
        uint16_t* s_mark = reinterpret_cast<uint16_t*>(B + SM::MARK);
        uint32_t* s_wrow = reinterpret_cast<uint32_t*>(B + SM::WROW);
        uint32_t* s_next = reinterpret_cast<uint32_t*>(B + SM::NEXT);
        const uint32_t wn = (uint32_t)((nrows - r0) < (uint64_t)W ? (nrows - r0) : (uint64_t)W);
        const uint64_t wend = offs(r0 + wn);
        uint64_t cend = cp + CH < p1 ? cp + CH : p1;
        if (cend > wend) cend = wend;   // window exhausted: cut the chunk (wend > cp: row r0 contains cp)
        const uint32_t n = (uint32_t)(cend - cp);
        // scan the window T rows at a time and stop at the first T-row block starting past
        // cend (uniform: every thread reads the same offset) -- a chunk of long rows costs
        // one block of offsets, not the whole window
        for (uint32_t base = 0; base < wn; base += T) {
            const uint32_t i = base + tid;
            if (i < wn) {
                const uint64_t a = offs(r0 + i), b = offs(r0 + i + 1);
                if (a < cend && b > cp && b > a) {   // a non-empty row meeting the chunk
                    const uint32_t rs = a > cp ? (uint32_t)(a - cp) : 0u;
                    const uint32_t re = (uint32_t)((b < cend ? b : cend) - cp);
                    s_start[i] = (uint32_t)(a - cp);   // mod 2^32: j = pair - start
                    if (rs) s_mark[rs] = (uint16_t)i;
                    for (uint32_t wb = (rs + WSPAN - 1) / WSPAN * WSPAN; wb < re; wb += WSPAN) s_wrow[wb / WSPAN] = i;
                    s_meta[i] = load_meta(r0 + i);
                }
                if (a <= cend && cend < b) *s_next = i;   // the row containing cend (if inside the window)
            }
            // rows from base+T on start after cend: none meets the chunk or contains cend
            if (base + T < wn && offs(r0 + base + T) > cend) break;
        }
        __syncthreads();
        const uint32_t q0 = tid * IPT;
        uint32_t mk[IPT];
#pragma unroll
        for (int x = 0; x < IPT; x += 4) {
            uint2* mp = reinterpret_cast<uint2*>(s_mark + q0 + x);
            const uint2 u = *mp;
            *mp = make_uint2(0u, 0u);   // clean for this buffer's next chunk (after >= 1 barrier)
            mk[x] = u.x & 0xffffu;
            mk[x + 1] = u.x >> 16;
            mk[x + 2] = u.y & 0xffffu;
            mk[x + 3] = u.y >> 16;
        }
        uint32_t tmax = 0;
#pragma unroll
        for (int it = 0; it < IPT; it++) tmax = mk[it] > tmax ? mk[it] : tmax;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {   // inclusive warp max-scan
            const uint32_t o = __shfl_up_sync(kFull, tmax, d);
            if (lane >= (uint32_t)d) tmax = o > tmax ? o : tmax;
        }
        uint32_t run = __shfl_up_sync(kFull, tmax, 1);
        if (lane == 0) run = 0;
        const uint32_t ws = warp * WSPAN < n ? s_wrow[warp] : 0u;
        run = run > ws ? run : ws;
        bool v[IPT];
        uint32_t wi[IPT], j[IPT];
#pragma unroll
        for (int it = 0; it < IPT; it++) {
            run = mk[it] > run ? mk[it] : run;
            v[it] = q0 + it < n;
            wi[it] = v[it] ? run : 0u;
            j[it] = v[it] ? q0 + it - s_start[run] : 0u;
        }
        body(v, wi, j, (const Meta*)s_meta, r0);
        if (cend < p1) r0 = (cend < wend) ? r0 + *s_next : pairs_find_warp(offs, r0 + wn - 1, nrows, cend);
        cp = cend;
        if (NB == 1) __syncthreads();   // the single window is restaged next
    }
    if (NB == 2) __syncthreads();   // the caller may reuse the shared buffers
}

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
