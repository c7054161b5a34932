// filter.cu -- filtering phase kernels (PAPER.md §"Filtering Phase"),
// batched: every launch serves all queries (jobs) of a batch.
//
//   k_check        a2 kernel_check (Alg. 2 line 7; Def. 3): one streaming
//                  pass over vlab / off_out / off_in tests ALL k query vertices of a query
//                  and emits one bitmap word per (query vertex, 32 data vertices) with
//                  __ballot_sync.  HBM bound: (2 + 4 + 4) B per vertex read, k/8 B written.
//   k_collect      a3 kernel_collect: stream compaction of a candidate
//                  bitmap into the sorted c_array with popc + block scan + decoupled
//                  look-back (one pass), also emitting the per-word rank prefix (O(1) key
//                  lookup) and the candidates' degree prefixes (the pair spaces of
//                  explore and EC).
//   k_explore      a4/a5 kernel_explore (Alg. 2 lines 14-22) over the PAIR
//                  space of each constraint job, walked from whichever side (the set being
//                  filtered, or the set it must reach) has fewer pairs; it writes the
//                  satisfying members as a bitmap.  Prune (lines 15-18) and propagation
//                  (lines 19-22) are the same job with the roles swapped.  Equal contiguous
//                  pair ranges per block replace the paper's warp-per-candidate +
//                  block-per-hub split.
//   k_post         word-parallel B &= (AND of the jobs' X bitmaps), scratch reset.
#include <cstdlib>

#include "kernels.cuh"
#include "lookback.cuh"
#include "pairs.cuh"

namespace gps {

// ---------------------------------------------------------------- a2 check
// One warp per bitmap word (32 data vertices): the vertex data (label, out/in
// degree) is read ONCE and tested against every query vertex of every query of
// the launch (all queries flattened), so a batch streams vlab / deg once instead
// of once per query.  A warp loads kChkW words' vertex data up front (kChkW
// independent loads in flight per lane: the pass is HBM-bound on large graphs),
// then for each query vertex f -- parameters packed in one shared-memory vector,
// read as a broadcast -- tests its kChkW words with one __ballot_sync each; lane
// f mod 32 keeps the word and stores it once 32 query vertices are done.
constexpr int kChkF = 1024;   // query vertices staged in shared memory per pass
constexpr int kChkW = 4;      // bitmap words per warp iteration
constexpr uint32_t kChkAny = 0xffffffffu;   // wildcard label / free vertex

__global__ void __launch_bounds__(256) k_check(DevGraph g, const ChkQV* __restrict__ qv, uint32_t nf) {
    __shared__ uint4 s_q[kChkF];        // (label or any, out-degree, in-degree, bound or free)
    __shared__ uint32_t* s_b[kChkF];    // bitmap of query vertex f
    const uint32_t lane = lane_id();
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    for (uint32_t f0 = 0; f0 < nf; f0 += kChkF) {
        const uint32_t fn = min(nf - f0, (uint32_t)kChkF);
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < fn; i += blockDim.x) {
            const ChkQV q = qv[f0 + i];
            s_q[i] = make_uint4(q.lab < 0 ? kChkAny : (uint32_t)q.lab, q.qout, q.qin,
                                q.bound < 0 ? kChkAny : (uint32_t)q.bound);
            s_b[i] = q.B;
        }
        __syncthreads();
        for (uint32_t w0 = gw * kChkW; w0 < g.nw; w0 += nwarps * kChkW) {
            uint32_t lab[kChkW], od[kChkW], id[kChkW];
            bool ok[kChkW];
#pragma unroll
            for (int i = 0; i < kChkW; i++) {
                const uint32_t v = (w0 + i) * 32 + lane;
                ok[i] = v < g.n;
                uint2 dg = make_uint2(0u, 0u);
                lab[i] = 0;
                if (ok[i]) {
                    dg = g.deg[v];
                    lab[i] = g.vlab[v];
                }
                od[i] = dg.x;
                id[i] = dg.y;
            }
            for (uint32_t fb = 0; fb < fn; fb += 32) {
                uint32_t mine[kChkW] = {};
                const uint32_t fe = min(fn - fb, 32u);
                for (uint32_t x = 0; x < fe; x++) {
                    const uint4 q = s_q[fb + x];
#pragma unroll
                    for (int i = 0; i < kChkW; i++) {
                        const uint32_t v = (w0 + i) * 32 + lane;
                        const bool p = ok[i] && (q.x == kChkAny || lab[i] == q.x) && (q.w == kChkAny || v == q.w) &&
                                       od[i] >= q.y && id[i] >= q.z;
                        const uint32_t m = __ballot_sync(kFull, p);
                        if (lane == x) mine[i] = m;
                    }
                }
                if (lane < fe) {
                    uint32_t* B = s_b[fb + lane];
#pragma unroll
                    for (int i = 0; i < kChkW; i++)
                        if (w0 + i < g.nw) B[w0 + i] = mine[i];
                }
            }
        }
    }
}

void run_check(gps_ctx* c, const DevGraph& g, const ChkQV* d_qv, uint32_t nf) {
    if (nf == 0) return;
    const uint32_t blocks = std::min<uint32_t>((g.nw + 8 * kChkW - 1) / (8 * kChkW), (uint32_t)c->nsm * 4);
    launch(c, GPS_K_CHECK, dim3(blocks), dim3(256), 0, k_check, g, d_qv, nf);
    // algorithmic: the vertex data once (2 B label + 8 B degrees) + one bitmap word per 32 vertices
    // and query vertex
    c->stats.k_bytes[GPS_K_CHECK] += (double)g.n * 10.0 + (double)nf * g.nw * 4.0;
}

// -------------------------------------------------------------- a3 collect
constexpr int kColThreads = 256;
constexpr int kColWords = 4;                          // bitmap words (128 vertices) per thread
constexpr int kColTile = kColThreads * kColWords;     // words per tile
constexpr int kColBatch = 8;                          // candidates whose degrees are loaded together

__global__ void __launch_bounds__(kColThreads, 5) k_collect(DevGraph g, const CollectJob* __restrict__ jobs,
                                                         LbScratch lb, uint32_t ntiles, uint32_t epoch,
                                                         unsigned long long* bytes_acc) {
    const uint32_t y = blockIdx.y;
    const CollectJob& J = jobs[y];
    const uint32_t tile = lb_ticket(lb.ctr + 3 * y, ntiles);
    const uint32_t w0 = tile * kColTile + threadIdx.x * kColWords;
    uint32_t word[kColWords];
    if (w0 + 3 < g.nw) {   // one 16-byte load of 4 words
        const uint4 b4 = *reinterpret_cast<const uint4*>(J.B + w0);
        word[0] = b4.x;
        word[1] = b4.y;
        word[2] = b4.z;
        word[3] = b4.w;
    } else if (w0 < g.nw) {   // the last words: never read the (unwritten) row padding
#pragma unroll
        for (int i = 0; i < kColWords; i++) word[i] = w0 + i < g.nw ? J.B[w0 + i] : 0u;
    } else {
        word[0] = word[1] = word[2] = word[3] = 0u;
    }
    if (J.x1 > J.x0 && w0 < g.nw) {   // folded post: B &= AND of the X bitmaps, X cleared
        for (uint32_t x = J.x0; x < J.x1; x++) {
            uint4* xp = reinterpret_cast<uint4*>(J.xs[x] + w0);
            const uint4 v = *xp;
            word[0] &= v.x;
            word[1] &= v.y;
            word[2] &= v.z;
            word[3] &= v.w;
            *xp = make_uint4(0u, 0u, 0u, 0u);
        }
        *reinterpret_cast<uint4*>(J.B + w0) = make_uint4(word[0], word[1], word[2], word[3]);
    }
    if (J.post_only) return;   // uniform per block (one job per grid row)
    // the candidates' degrees, kColBatch independent 8-byte loads per round trip
    uint32_t c = 0, so = 0, si = 0;
#pragma unroll
    for (int i = 0; i < kColWords; i++) {
        c += __popc(word[i]);
        uint32_t bits = word[i];
        while (bits) {
            uint2 d[kColBatch];
#pragma unroll
            for (int k = 0; k < kColBatch; k++) {
                d[k] = bits ? __ldg(g.deg + (w0 + i) * 32 + __ffs(bits) - 1) : make_uint2(0u, 0u);
                bits &= bits - 1;
            }
#pragma unroll
            for (int k = 0; k < kColBatch; k++) {
                so += d[k].x;
                si += d[k].y;
            }
        }
    }
    uint32_t tc, tso, tsi;
    const uint32_t ec = block_excl_scan(c, &tc);
    const uint32_t eso = block_excl_scan(so, &tso);
    const uint32_t esi = block_excl_scan(si, &tsi);
    // the three look-backs (count, out-degree, in-degree prefixes) run in warps 0..2 concurrently
    __shared__ uint64_t s_pre[3];
    const uint32_t wid = threadIdx.x >> 5;
    if (wid < 3) {
        const uint64_t agg = wid == 0 ? tc : (wid == 1 ? tso : tsi);
        const size_t base = (size_t)(3 * y + wid) * lb.max_tiles;
        const uint64_t p = lb_warp_lookback(lb.status + base, tile, agg, epoch);
        if ((threadIdx.x & 31u) == 0) s_pre[wid] = p;
    }
    __syncthreads();
    uint32_t rank = (uint32_t)s_pre[0] + ec;
    uint32_t ro = (uint32_t)s_pre[1] + eso;
    uint32_t ri = (uint32_t)s_pre[2] + esi;
    if (w0 < g.nw) {
        uint32_t r[kColWords], x = rank;
#pragma unroll
        for (int i = 0; i < kColWords; i++) {
            r[i] = x;
            x += __popc(word[i]);
        }
        *reinterpret_cast<uint4*>(J.rp + w0) = make_uint4(r[0], r[1], r[2], r[3]);
    }
#pragma unroll
    for (int i = 0; i < kColWords; i++) {
        uint32_t bits = word[i];
        while (bits) {
            uint32_t v[kColBatch];
            uint2 d[kColBatch];
#pragma unroll
            for (int k = 0; k < kColBatch; k++) {
                v[k] = bits ? (w0 + i) * 32 + __ffs(bits) - 1 : 0xffffffffu;
                d[k] = bits ? __ldg(g.deg + v[k]) : make_uint2(0u, 0u);
                bits &= bits - 1;
            }
#pragma unroll
            for (int k = 0; k < kColBatch; k++) {
                if (v[k] == 0xffffffffu) break;
                J.carr[rank] = v[k];
                J.seg_out[rank] = ro;
                J.seg_in[rank] = ri;
                ro += d[k].x;
                ri += d[k].y;
                rank++;
            }
        }
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) {
        const uint32_t C = (uint32_t)s_pre[0] + tc;
        // algorithmic bytes per candidate: its 8-byte degree word read + id and two prefixes written
        atomicAdd(bytes_acc, 20ull * C);
        J.rp[g.nw] = C;
        *J.cnt = C;
        J.seg_out[C] = (uint32_t)s_pre[1] + tso;
        J.seg_in[C] = (uint32_t)s_pre[2] + tsi;
        if (J.segtot) {
            J.segtot[0] = (uint32_t)s_pre[1] + tso;
            J.segtot[1] = (uint32_t)s_pre[2] + tsi;
        }
    }
}

void run_collect(gps_ctx* c, const DevGraph& g, const CollectJob* d_jobs, uint32_t nj) {
    if (nj == 0) return;
    const uint32_t ntiles = (g.nw + kColTile - 1) / kColTile;
    LbScratch lb = lb_scratch(c, 3 * nj, ntiles);
    launch(c, GPS_K_COLLECT, dim3(ntiles, nj), dim3(kColThreads), 0, k_collect, g, d_jobs, lb, ntiles,
           lb_next_epoch(c), c->d_bytes + GPS_K_COLLECT);
    // algorithmic: read the bitmap, write the rank prefix (+ 20 B per candidate, counted on the device)
    c->stats.k_bytes[GPS_K_COLLECT] += (double)nj * g.nw * 8.0;
}

// -------------------------------------------------------------- a4 explore
constexpr int kET = 128;
constexpr int kEI = 4;   // pairs per thread per chunk (8 measured slower on configs 2 and 4)
constexpr int kEW = 256;

struct ExMeta {             // one row (key vertex) of an explore job, staged per chunk
    uint32_t key, base, skip, pad;
};
using ExSmem = PairSmem<ExMeta, kET, kEI, kEW, 2>;

__device__ __forceinline__ uint64_t ex_pairs(const ExploreJob& J, bool* s_side) {
    const uint64_t pa = J.candA ? (uint64_t)__ldg(J.segA + *J.cntA) : ~0ull;
    const uint64_t ps = J.candS ? (uint64_t)__ldg(J.segS + *J.cntS) : ~0ull;
    *s_side = ps < pa;
    return ps < pa ? ps : pa;
}

__global__ void __launch_bounds__(kET, 10) k_explore(DevGraph g, const ExploreJob* __restrict__ jobs, uint32_t nj,
                                                unsigned long long* bytes_acc, unsigned long long* dbg) {
    extern __shared__ __align__(16) char s_dyn[];
    uint64_t* s_jp = reinterpret_cast<uint64_t*>(s_dyn);          // [nj+1] job pair prefix
    char* s_bufs = s_dyn + ExSmem::buf_off(nj);
    ExSmem::init(s_bufs);
    job_prefix(nj, [&](uint32_t j) -> uint64_t { bool sd; return ex_pairs(jobs[j], &sd); }, s_jp);
    uint64_t p0, p1;
    pairs_range(s_jp[nj], blockIdx.x, gridDim.x, p0, p1);
    uint32_t n_live = 0, n_fit = 0, n_sside = 0;
    for_job_ranges(s_jp, nj, p0, p1, [&](uint32_t jj, uint64_t lo, uint64_t hi) {
        const ExploreJob J = jobs[jj];             // by value: fields stay in registers across atomics
        bool sside;
        ex_pairs(J, &sside);                       // uniform per job
        // rows: keys of the walked side; arcs of direction dir (A-side) or 1 - dir (S-side)
        const bool in = sside ? J.dir == 0 : J.dir != 0;
        const uint32_t* off = in ? g.off_in : g.off_out;
        const uint32_t* arcs = in ? g.arc_in : g.arc_out;
        const uint32_t* cand = sside ? J.candS : J.candA;
        const uint32_t* seg = sside ? J.segS : J.segA;
        const uint32_t* Bkey = sside ? J.BS : J.BA;    // the row key must still be a member
        const uint32_t* Btest = sside ? J.BA : J.BS;   // the arc's other end must be a member
        const uint32_t C = sside ? *J.cntS : *J.cntA;
        const bool fresh = (sside ? J.freshS : J.freshA) != 0;
        auto offs = [&](uint64_t i) -> uint64_t { return (uint64_t)__ldg(seg + i); };
        auto load = [&](uint64_t r) -> ExMeta {
            ExMeta m;
            m.key = __ldg(cand + r);
            m.base = __ldg(off + m.key);
            // skip keys that left the set (stale arrays only); A-side also skips keys an earlier chunk
            // already satisfied
            m.skip = (!fresh && !bit_test(Bkey, m.key)) ||
                     (!sside && ((__ldcg(J.X + (m.key >> 5)) >> (m.key & 31)) & 1u));
            m.pad = 0;
            return m;
        };
        pair_chunks<ExMeta, kET, kEI, kEW, 2>(lo, hi, (uint64_t)C, offs, load, s_bufs,
                                           [&](const bool (&v)[kEI], const uint32_t (&wi)[kEI],
                                               const uint32_t (&j)[kEI], const ExMeta* sm, uint64_t) {
            uint32_t arc[kEI];
            bool live[kEI];
#pragma unroll
            for (int it = 0; it < kEI; it++) {
                const ExMeta& m = sm[wi[it]];
                live[it] = v[it] && !m.skip;
                arc[it] = live[it] ? __ldg(arcs + m.base + j[it]) : 0u;
            }
            bool fits[kEI];
#pragma unroll
            for (int it = 0; it < kEI; it++) {
                const uint32_t d = arc[it] >> g.lbits;
                fits[it] = live[it] && lab_ok(arc[it], g.lmask, J.lab) && d != sm[wi[it]].key && bit_test(Btest, d);
                if (dbg) {
                    n_live += live[it];
                    n_fit += fits[it];
                    n_sside += sside && v[it];
                }
            }
            if (!sside) {   // one X bit per satisfied key: OR over the thread's run of the same row
                uint32_t cur = 0xffffffffu;
                bool any = false;
#pragma unroll
                for (int it = 0; it < kEI; it++) {
                    if (wi[it] != cur) {
                        if (any) {
                            const uint32_t key = sm[cur].key;
                            atomicOr(J.X + (key >> 5), 1u << (key & 31));
                        }
                        cur = wi[it];
                        any = false;
                    }
                    any |= fits[it];
                }
                if (any) {
                    const uint32_t key = sm[cur].key;
                    atomicOr(J.X + (key >> 5), 1u << (key & 31));
                }
            } else {
#pragma unroll
                for (int it = 0; it < kEI; it++)
                    if (fits[it]) {   // fire-and-forget reduction (no return value: RED)
                        const uint32_t d = arc[it] >> g.lbits;
                        atomicOr(J.X + (d >> 5), 1u << (d & 31));
                    }
            }
        });
    });
    if (bytes_acc && threadIdx.x == 0 && p1 > p0) atomicAdd(bytes_acc, (unsigned long long)(p1 - p0) * 4ull);
    if (dbg) {   // GPS_EXPLORE_STATS: pairs / live pairs / fitting pairs / S-side pairs
        const uint32_t a = block_sum(n_live), b = block_sum(n_fit), c = block_sum(n_sside);
        if (threadIdx.x == 0) {
            atomicAdd(dbg, (unsigned long long)(p1 - p0));
            atomicAdd(dbg + 1, (unsigned long long)a);
            atomicAdd(dbg + 2, (unsigned long long)b);
            atomicAdd(dbg + 3, (unsigned long long)c);
        }
    }
}

static size_t ex_smem(uint32_t nj) { return ExSmem::bytes(nj, 0); }

void run_explore(gps_ctx* c, const DevGraph& g, const ExploreJob* d_jobs, uint32_t nj, int cls) {
    if (nj == 0) return;
    if (nj > kMaxJobsPerLaunch) fail(GPS_EINVAL, "too many jobs per launch");
    const uint32_t G = resident_grid(c, (const void*)k_explore, kET, ex_smem(nj));
    static const bool dbg = std::getenv("GPS_EXPLORE_STATS") != nullptr;
    launch(c, cls, dim3(G), dim3(kET), ex_smem(nj), k_explore, g, d_jobs, nj, c->d_bytes + cls,
           dbg ? (unsigned long long*)c->d_info + 96 + (cls == GPS_K_PROPAGATE ? 4 : 0) : nullptr);
}

// ------------------------------------------------------------ step end
constexpr int kPostWords = 4;

__global__ void __launch_bounds__(256) k_post(DevGraph g, const PostJob* __restrict__ jobs,
                                              uint32_t* const* __restrict__ xs) {
    const PostJob J = jobs[blockIdx.y];
    const uint32_t w0 = (blockIdx.x * blockDim.x + threadIdx.x) * kPostWords;
    if (w0 >= g.nw) return;   // nws >= nw rounded up to 64 words: the 4-word vector stays in bounds
    uint4 b = *reinterpret_cast<const uint4*>(J.B + w0);
    for (uint32_t x = J.x0; x < J.x1; x++) {
        uint4* xp = reinterpret_cast<uint4*>(xs[x] + w0);
        const uint4 v = *xp;
        b.x &= v.x;
        b.y &= v.y;
        b.z &= v.z;
        b.w &= v.w;
        *xp = make_uint4(0u, 0u, 0u, 0u);
    }
    *reinterpret_cast<uint4*>(J.B + w0) = b;
}

void run_post(gps_ctx* c, const DevGraph& g, const PostJob* d_jobs, uint32_t* const* d_xs, uint32_t nj) {
    if (nj == 0) return;
    const uint32_t bx = (g.nw + 256 * kPostWords - 1) / (256 * kPostWords);
    launch(c, GPS_K_BITAND, dim3(bx, nj), dim3(256), 0, k_post, g, d_jobs, d_xs);
    c->stats.k_bytes[GPS_K_BITAND] += (double)g.nw * 4.0 * 2.0 * nj;
}

}  // namespace gps
