// join.cu -- joining phase kernels (PAPER.md §"Joining Phase"), batched.
//
//   k_ec         a6 collect_edge_candidates over the pair space (job, key u' in C(p),
//                arc of adj_dir(u')): the distinct v' with a fitting label, v' in B[q],
//                v' != u', in pair order, with the address of each key's first v' (the
//                "hash table" of fig3:hashtable).  The paper's two-step output
//                scheme (citing Mars) becomes ONE pass: tiles compact in shared
//                memory and take their output offset from a decoupled look-back.
//   k_join_seg   a8 per input row: O(1) key lookup (bitmap rank, instead of the paper's
//                logarithmic search P:820) -> EC segment start, and the exclusive scan of
//                segment lengths (pair offsets) in the same single pass.
//   k_join<W>    a8 combine over the pair space (row, segment position):
//                injectivity + every fused closing arc (binary search in the closing arc's
//                sorted EC segment); count (W=false, last block scans the block counts)
//                or write (W=true).
#include <mutex>

#include "kernels.cuh"
#include "lookback.cuh"
#include "pairs.cuh"

namespace gps {

constexpr int kPT = 256;    // threads per block
constexpr int kPI = 4;      // pairs per thread per chunk
constexpr int kPW = 1024;   // EC: rows staged per chunk (keys are never empty: a chunk always fits)
constexpr int kJW = 64;     // join: rows staged (single buffer; a chunk meeting more rows is cut at the window end).
                             // 1024 rows (56 KB of row metadata) held k_join<2> to 2 blocks per SM
constexpr uint32_t kStageW = kJoinStageCols;   // join: stage rows of width <= 8 in shared memory


// ------------------------------------------------------------ a6 EC build
// Single pass over TILES of kTile consecutive pairs of one job (tiles of all jobs
// numbered in job order, taken in ticket order): the tile's passing values are
// compacted in shared memory in pair order, the tile's count goes through a
// decoupled look-back, and the tile then writes its values and the offsets of
// the keys whose first pair it holds.  Values of a key therefore come out sorted
// and contiguous, and the count pass + scan of the two-step scheme disappear.
constexpr uint32_t kTile = kPT * kPI;      // pairs per chunk (and per join tile)
static_assert(kTile == kJoinTilePairs, "host and device join tiling differ");
constexpr uint32_t kEcTile = 4 * kTile;     // pairs per EC tile: a few chunks amortise the tile's set-up latency
static_assert(kEcTile == kEcPairTile, "host and device EC tiling differ");

struct EcMeta {             // one key row of an EC job (row = window base + window index)
    uint32_t key, base;
};
using EcSmem = PairSmem<EcMeta, kPT, kPI, kPW, 1>;

__host__ __device__ inline size_t ec_smem_n(uint32_t nj) {
    // [tile0 of every job (nj+1) u32 -> rounded][pair buffers][values kEcTile u32][first/last key started]
    return EcSmem::bytes(nj, sizeof(uint32_t) * kEcTile + 16);
}

__global__ void __launch_bounds__(kPT, 5) k_ec(DevGraph g, const ECJob* __restrict__ jobs, uint32_t nj, LbScratch lb,
                                           uint32_t ntiles, uint32_t epoch, uint32_t* __restrict__ val,
                                           uint64_t base, unsigned long long* bytes_acc) {
    extern __shared__ __align__(16) char s_dyn[];
    uint32_t* s_t0 = reinterpret_cast<uint32_t*>(s_dyn);   // first tile of every job, s_t0[nj] = ntiles
    char* s_bufs = s_dyn + EcSmem::buf_off(nj);
    uint32_t* s_val = reinterpret_cast<uint32_t*>(s_dyn + EcSmem::extra_off(nj));
    uint32_t* s_rows = s_val + kEcTile;   // [0] = first, [1] = last key whose first pair is in the tile
    __shared__ uint64_t s_prefix;
    const uint32_t t = lb_ticket(lb.ctr, ntiles);
    for (uint32_t i = threadIdx.x; i < nj; i += blockDim.x) s_t0[i] = jobs[i].tile0;
    if (threadIdx.x == 0) {
        s_t0[nj] = ntiles;
        s_rows[0] = 0xffffffffu;
        s_rows[1] = 0u;
    }
    EcSmem::init(s_bufs);
    __syncthreads();
    uint32_t lo = 0, hi = nj;   // job of tile t: largest j with tile0 <= t
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (s_t0[mid] <= t) lo = mid; else hi = mid;
    }
    const ECJob& J = jobs[lo];
    const uint32_t kt = t - s_t0[lo];
    const uint32_t C = J.C;
    const uint64_t P = J.P;
    const uint64_t p0 = (uint64_t)kt * kEcTile, p1 = p0 + kEcTile < P ? p0 + kEcTile : P;
    const uint32_t* off = J.dir ? g.off_in : g.off_out;
    const uint32_t* arcs = J.dir ? g.arc_in : g.arc_out;
    auto offs = [&](uint64_t i) -> uint64_t { return (uint64_t)__ldg(J.seg + i); };
    auto load = [&](uint64_t r) -> EcMeta {
        EcMeta m;
        m.key = __ldg(J.keys + r);
        m.base = __ldg(off + m.key);
        return m;
    };
    uint32_t lc = 0;   // values of the tile so far (uniform)
    pair_chunks<EcMeta, kPT, kPI, kPW, 1>(p0, p1, (uint64_t)C, offs, load, s_bufs,
                                       [&](const bool (&v)[kPI], const uint32_t (&wi)[kPI],
                                           const uint32_t (&j)[kPI], const EcMeta* sm, uint64_t wr0) {
        uint32_t x[kPI], xp[kPI];
#pragma unroll
        for (int it = 0; it < kPI; it++) {
            const uint32_t base = sm[wi[it]].base;
            x[it] = v[it] ? __ldg(arcs + base + j[it]) : 0u;
            xp[it] = (v[it] && j[it] > 0) ? __ldg(arcs + base + j[it] - 1) : 0xffffffffu;
        }
        bool pred[kPI];
        uint32_t mine = 0;
#pragma unroll
        for (int it = 0; it < kPI; it++) {
            const uint32_t d = x[it] >> g.lbits;
            pred[it] = false;
            if (v[it] && lab_ok(x[it], g.lmask, J.lab) && d != sm[wi[it]].key && bit_test(J.Bq, d)) {
                // parallel arcs to the same v' (reading R5): count v' once
                const bool dup = j[it] > 0 && (xp[it] >> g.lbits) == d && lab_ok(xp[it], g.lmask, J.lab);
                pred[it] = !dup;
            }
            mine += pred[it] ? 1u : 0u;
        }
        uint32_t tot;
        uint32_t pos = lc + block_excl_scan(mine, &tot);
#pragma unroll
        for (int it = 0; it < kPI; it++) {
            if (v[it] && j[it] == 0) {   // key starts here: tile-relative offset now, + prefix after the look-back
                const uint32_t row = (uint32_t)wr0 + wi[it];
                J.off[row] = pos;
                atomicMin(s_rows, row);
                atomicMax(s_rows + 1, row);
            }
            if (pred[it]) s_val[pos++] = x[it] >> g.lbits;
        }
        lc += tot;
    });
    __syncthreads();   // s_val / s_rows / J.off writes of the last chunk
    if (threadIdx.x < 32) {
        const uint64_t pre = lb_warp_lookback(lb.status, t, lc, epoch);
        if (threadIdx.x == 0) s_prefix = pre;
    }
    __syncthreads();
    const uint64_t pre = s_prefix + base;
    for (uint32_t i = threadIdx.x; i < lc; i += blockDim.x) val[pre + i] = s_val[i];
    // every key has >= 1 pair (a candidate passed the degree check), so the keys starting in
    // this tile are exactly [first, last]
    const uint32_t r0 = s_rows[0], r1 = s_rows[1];
    for (uint32_t r = r0 + threadIdx.x; r0 <= r1 && r <= r1; r += blockDim.x) J.off[r] += (uint32_t)pre;
    if (threadIdx.x == 0) {
        if (kt == 0) J.span[0] = pre;
        if (p1 == P) {
            J.span[1] = pre + lc;
            J.off[C] = (uint32_t)(pre + lc);
        }
        if (bytes_acc) atomicAdd(bytes_acc, (unsigned long long)(p1 - p0) * 4ull + lc * 4ull);
    }
}

void run_ec(gps_ctx* c, const DevGraph& g, const ECJob* d_jobs, uint32_t nj, uint32_t ntiles, uint32_t* val,
            uint64_t base) {
    if (nj == 0 || ntiles == 0) return;
    if (nj > kMaxJobsPerLaunch) fail(GPS_EINVAL, "too many EC jobs per launch");
    allow_smem((const void*)k_ec, (int)ec_smem_n(kMaxJobsPerLaunch));
    LbScratch lb = lb_scratch(c, 1, ntiles);
    launch(c, GPS_K_EC_WRITE, dim3(ntiles), dim3(kPT), ec_smem_n(nj), k_ec, g, d_jobs, nj, lb, ntiles,
           lb_next_epoch(c), val, base, c->d_bytes + GPS_K_EC_WRITE);
}

// ------------------------------------------------------------ a8 join step
// Closing arcs keyed by a column of the input row (the arc's other endpoint is the new
// vertex) have the SAME candidate segment for every pair of the row: the window staging
// looks up the first kHoist of them once per row (rank + two offsets) and the pairs only
// search their segment.  Arcs keyed by the new vertex need its rank per pair.
constexpr uint32_t kHoist = 3;

__device__ __forceinline__ uint2 close_seg(const CloseChk& cl, uint32_t key) {
    const uint32_t rk = bit_rank(cl.Bk, cl.rpk, key);
    return make_uint2(__ldg(cl.off + rk), __ldg(cl.off + rk + 1));
}

// Per-row part: seg[ci] for the hoisted closing arcs (ci < kHoist, keyed by a row column).
__device__ __forceinline__ void hoist_close(const JoinStep& a, const JoinJob& J, const uint32_t* __restrict__ row,
                                            uint2 (&seg)[kHoist]) {
#pragma unroll
    for (uint32_t ci = 0; ci < kHoist; ci++) {
        seg[ci] = make_uint2(0u, 0u);
        if (ci < J.nclose) {
            const CloseChk& cl = a.cl[J.close0 + ci];
            if (!cl.key_new) seg[ci] = close_seg(cl, __ldg(row + cl.key_col));
        }
    }
}

// The row's DRIVER list: of the extension segment and the hoisted closing segments -- all
// sorted lists the new vertex must belong to -- the shortest (first on ties).  The row's
// pairs walk the driver and test membership in the others, so a row costs min(|S|, |T_i|)
// pairs instead of |S| (sorted-list intersection, "closing edges" + the north star's
// "intersect").  The seg pass and the pair kernels compute it the same way.
struct RowLists {
    uint2 ext;                // extension segment [x, y) in ec_val
    uint2 cseg[kHoist];       // hoisted closing segments (0, 0 when not hoisted)
    uint32_t drv;             // 0: extension, 1 + ci: hoisted closing arc ci
};
__device__ __forceinline__ void row_lists(const JoinStep& a, const JoinJob& J, const uint32_t* __restrict__ row,
                                          RowLists& L) {
    const uint32_t rk = bit_rank(J.Bx, J.rpx, __ldg(row + J.x_col));
    L.ext = make_uint2(__ldg(J.ec_off + rk), __ldg(J.ec_off + rk + 1));
    hoist_close(a, J, row, L.cseg);
    L.drv = 0;
    uint32_t best = L.ext.y - L.ext.x;
#pragma unroll
    for (uint32_t ci = 0; ci < kHoist; ci++) {
        if (ci >= J.nclose || a.cl[J.close0 + ci].key_new) continue;
        const uint32_t n = L.cseg[ci].y - L.cseg[ci].x;
        if (n < best) {
            best = n;
            L.drv = 1 + ci;
        }
    }
}
__device__ __forceinline__ uint2 driver_seg(const RowLists& L) {
    uint2 d = L.ext;
#pragma unroll
    for (uint32_t ci = 0; ci < kHoist; ci++)
        if (L.drv == 1 + ci) d = L.cseg[ci];
    return d;
}

// rows per thread (4 rows amortise the scan; the FAST pass interleaves their searches)
// (FAST: 2 rows per thread on small tables -- more threads, shorter chains; 4 on large ones --
// more searches in flight per thread; measured on configs 2 and 4)
constexpr uint64_t kSegBigRows = 1u << 22;


// Per input row: O(1) key lookup -> EC segment start (s0) and the exclusive scan of
// the segment lengths (poff, the step's pair space), one look-back pass.  FAST
// (closing-free steps): also the row values found in the segment (imask, binary
// searches advanced in lockstep), the per-job output totals, and the scan of the
// rows' written outputs (woff) -- two look-backs in two warps.
template <bool FAST, int kSegRows>
__global__ void __launch_bounds__(256, (FAST && kSegRows == 4) ? 4 : 5) k_join_seg(const __grid_constant__ JoinStep a, LbScratch lb, uint32_t ntiles,
                                                  uint32_t epoch) {
    constexpr int kSegTile = 256 * kSegRows;
    extern __shared__ __align__(16) char s_dyn[];
    uint64_t* s_jr = reinterpret_cast<uint64_t*>(s_dyn);   // [nj+1] first row of every job
    const uint32_t** s_jbn = reinterpret_cast<const uint32_t**>(s_jr + a.nj + 1);   // [nj] FAST: Bn of every job
    __shared__ uint64_t s_pre[3];
    const uint32_t tile = lb_ticket(lb.ctr, ntiles);
    for (uint32_t j = threadIdx.x; j < a.nj; j += blockDim.x) {
        s_jr[j] = a.jobs[j].row0;
        if (FAST) s_jbn[j] = a.jobs[j].Bn;
    }
    if (threadIdx.x == 0) s_jr[a.nj] = a.R;
    __syncthreads();
    const uint64_t r0 = (uint64_t)tile * kSegTile + (uint64_t)threadIdx.x * kSegRows;
    uint32_t len[kSegRows], ac[kSegRows], wc[kSegRows];
    uint64_t tsum = 0, wsum = 0;
    uint32_t jb = r0 < a.R ? pairs_find_smem(s_jr, a.nj, r0) : 0;
    const uint32_t* rowp[kSegRows];
    uint32_t sst[kSegRows], nowr[kSegRows], jrow[kSegRows];
#pragma unroll
    for (int i = 0; i < kSegRows; i++) {   // key -> rank -> segment: the rows' loads are independent
        const uint64_t r = r0 + i;
        len[i] = ac[i] = wc[i] = 0;
        rowp[i] = nullptr;
        sst[i] = nowr[i] = 0;
        jrow[i] = jb;
        if (r < a.R) {
            while (jb + 1 < a.nj && s_jr[jb + 1] <= r) jb++;
            const JoinJob& J = a.jobs[jb];
            rowp[i] = J.M + (r - J.row0) * a.w;
            if (FAST || J.nclose == 0) {
                const uint32_t key = __ldg(rowp[i] + J.x_col);
                const uint32_t rk = bit_rank(J.Bx, J.rpx, key);
                sst[i] = __ldg(J.ec_off + rk);
                len[i] = __ldg(J.ec_off + rk + 1) - sst[i];
            } else {   // closing arcs: the row's pairs walk its shortest list
                RowLists L;
                row_lists(a, J, rowp[i], L);
                const uint2 d = driver_seg(L);
                sst[i] = d.x;
                len[i] = d.y - d.x;
            }
            nowr[i] = J.nowrite;
            jrow[i] = jb;
            a.s0[r] = sst[i];
        }
    }
    if (FAST) {
        // every (row, column) pair of the thread's rows is a binary search of the column's value
        // in the row's segment; all of them run in lockstep, 8 at a time, so a thread keeps up to
        // 8 independent loads in flight whatever the row width
        uint32_t mask[kSegRows] = {};
        const uint32_t nsearch = kSegRows * a.w;
        for (uint32_t q0 = 0; q0 < nsearch; q0 += 8) {
            uint32_t t[8], lo[8], hi[8], found = 0;
#pragma unroll
            for (int x = 0; x < 8; x++) {
                const uint32_t q = q0 + x, qi = q / a.w, qc = q - qi * a.w;
                const uint32_t* rp = nullptr;
                uint32_t ss = 0, ll = 0;
#pragma unroll
                for (int i = 0; i < kSegRows; i++)   // select, not index: the arrays stay in registers
                    if (qi == (uint32_t)i) {
                        rp = rowp[i];
                        ss = sst[i];
                        ll = len[i];
                    }
                const bool on = q < nsearch && rp != nullptr && ll > 0;
                t[x] = on ? __ldg(rp + qc) : 0u;
                lo[x] = ss;
                hi[x] = on ? ss + ll : ss;
            }
            // a row value that is not a candidate of the new vertex cannot be in the segment (every
            // extension segment is a subset of that candidate set): one bitmap probe instead of a
            // binary search for most values
#pragma unroll
            for (int x = 0; x < 8; x++) {
                if (hi[x] - lo[x] <= 16) continue;   // a short search costs no more than the probe
                const uint32_t qi = (q0 + x) / a.w;
                uint32_t job = 0;
#pragma unroll
                for (int i = 0; i < kSegRows; i++)
                    if (qi == (uint32_t)i) job = jrow[i];
                const uint32_t* bn = s_jbn[job];
                if (bn != nullptr && !bit_test(bn, t[x])) hi[x] = lo[x];
            }
            bool more = true;
            while (more) {
                more = false;
#pragma unroll
                for (int x = 0; x < 8; x++) {
                    if (lo[x] >= hi[x]) continue;
                    const uint32_t mid = (lo[x] + hi[x]) >> 1;
                    const uint32_t v = __ldg(a.ec_val + mid);
                    if (v == t[x]) {
                        found |= 1u << x;
                        hi[x] = lo[x];
                    } else if (v < t[x]) {
                        lo[x] = mid + 1;
                    } else {
                        hi[x] = mid;
                    }
                    more |= lo[x] < hi[x];
                }
            }
            while (found) {   // search q0 + x found its value: bit (q mod w) of row q / w
                const uint32_t x = __ffs(found) - 1, q = q0 + x, qi = q / a.w;
                found &= found - 1;
#pragma unroll
                for (int i = 0; i < kSegRows; i++) mask[i] |= qi == (uint32_t)i ? 1u << (q - qi * a.w) : 0u;
            }
        }
        bool live[kSegRows];
#pragma unroll
        for (int i = 0; i < kSegRows; i++) {
            live[i] = rowp[i] != nullptr;
            if (!live[i]) continue;
            a.imask[r0 + i] = mask[i];
            ac[i] = len[i] - __popc(mask[i]);
            wc[i] = nowr[i] ? 0u : ac[i];
        }
        // per-job output totals (the host sizes the output with them): run-length per thread,
        // combined across the warp, one atomic per job run
        run_sum<kSegRows>(live, jrow, ac, [&](uint32_t job, uint32_t n) {
            atomicAdd(a.jobs[job].total, (unsigned long long)n);
        });
    }
#pragma unroll
    for (int i = 0; i < kSegRows; i++) {
        tsum += len[i];
        wsum += wc[i];
    }
    // poff and (FAST) woff: the two scans in one pass of barriers, two look-backs in two warps
    uint64_t tot, wtot = 0, pre, wpre = 0;
    if (FAST) {
        ulonglong2 t2;
        const ulonglong2 p2 = block_excl_scan2(make_ulonglong2(tsum, wsum), &t2);
        pre = p2.x;
        wpre = p2.y;
        tot = t2.x;
        wtot = t2.y;
    } else {
        pre = block_excl_scan(tsum, &tot);
    }
    const uint32_t wid = threadIdx.x >> 5;
    if (wid < (FAST ? 2u : 1u)) {
        const uint64_t agg = wid == 0 ? tot : wtot;
        const uint64_t p = lb_warp_lookback(lb.status + (size_t)wid * lb.max_tiles, tile, agg, epoch);
        if ((threadIdx.x & 31u) == 0) s_pre[wid] = p;
    }
    __syncthreads();
    uint64_t run = s_pre[0] + pre, wrun = FAST ? s_pre[1] + wpre : 0;
#pragma unroll
    for (int i = 0; i < kSegRows; i++) {
        const uint64_t r = r0 + i;
        if (r < a.R) {
            a.poff[r] = run;
            if (FAST) a.woff[r] = wrun;
        }
        run += len[i];
        wrun += wc[i];
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) {
        a.poff[a.R] = s_pre[0] + tot;
        if (FAST) a.woff[a.R] = s_pre[1] + wtot;
    }
}

void run_join_seg(gps_ctx* c, const JoinStep& s) {
    const int rows = (s.fast && s.R < kSegBigRows) ? 2 : 4;
    const uint64_t tile = 256ull * rows;
    const uint64_t nt = (s.R + tile - 1) / tile;
    if (nt > 0x7fffffffull) fail(GPS_EOVERFLOW, "join table too large");
    LbScratch lb = lb_scratch(c, 2, (uint32_t)nt);
    const size_t smem = sizeof(uint64_t) * (s.nj + 1) + sizeof(void*) * s.nj;
    const uint32_t ep = lb_next_epoch(c);
    if (!s.fast)
        launch(c, GPS_K_JOIN_LEN, dim3((uint32_t)nt), dim3(256), smem, k_join_seg<false, 4>, s, lb, (uint32_t)nt, ep);
    else if (rows == 2)
        launch(c, GPS_K_JOIN_LEN, dim3((uint32_t)nt), dim3(256), smem, k_join_seg<true, 2>, s, lb, (uint32_t)nt, ep);
    else
        launch(c, GPS_K_JOIN_LEN, dim3((uint32_t)nt), dim3(256), smem, k_join_seg<true, 4>, s, lb, (uint32_t)nt, ep);
    c->stats.k_bytes[GPS_K_JOIN_LEN] += 4.0 * s.R * (s.w + 3);
}


__device__ __forceinline__ bool seg_contains(const uint32_t* __restrict__ val, uint32_t lo, uint32_t hi, uint32_t t) {
    while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        uint32_t v = __ldg(val + mid);
        if (v == t) return true;
        if (v < t) lo = mid + 1; else hi = mid;
    }
    return false;
}

// First index in [lo, hi) with val[i] >= t (val sorted ascending).
__device__ __forceinline__ uint32_t seg_lower(const uint32_t* __restrict__ val, uint32_t lo, uint32_t hi, uint32_t t) {
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(val + mid) < t) lo = mid + 1; else hi = mid;
    }
    return lo;
}
// Same, knowing val[i] < t for every i < lo: doubling probes from lo, then a binary search
// of the last gap -- O(log distance) when consecutive searches land close together.
__device__ __forceinline__ uint32_t seg_gallop(const uint32_t* __restrict__ val, uint32_t lo, uint32_t hi, uint32_t t) {
    uint32_t step = 1, b = lo;
    while (b < hi && __ldg(val + b) < t) {
        lo = b + 1;
        b = lo + step;
        step <<= 1;
    }
    return seg_lower(val, lo, b < hi ? b : hi, t);
}

// Membership of a thread's candidates in the lists of their rows, list by list: the
// extension segment (when it is not the driver) and the hoisted closing segments.  A
// thread's items are consecutive pairs; items of one row carry increasing candidates (the
// driver is sorted), so each search after the first of a row gallops from the previous
// position instead of restarting (a merge-like intersection of the row's lists).  Closing
// arcs that are not hoisted (keyed by the new vertex, or beyond kHoist) are checked per item
// with their own rank lookup.  ok[] holds the injectivity results on entry.
template <int IPT, typename MetaAt, typename RowVal>
__device__ __forceinline__ void lists_check(const JoinStep& a, const uint32_t (&wi)[IPT], const uint32_t (&cand)[IPT],
                                            bool (&ok)[IPT], MetaAt meta_of, RowVal rowval) {
#pragma unroll 1
    for (uint32_t l = 0; l <= kHoist; l++) {
        uint32_t prow = 0xffffffffu, ppos = 0;
#pragma unroll
        for (int it = 0; it < IPT; it++) {
            if (!ok[it]) continue;
            const auto& m = meta_of(wi[it]);
            const JoinJob& J = a.jobs[m.job];
            if (J.nclose == 0) continue;
            uint2 sg = m.ext;
            bool use = m.drv != 0;
            if (l > 0) {
                const uint32_t ci = l - 1;
                use = ci < J.nclose && m.drv != l && !a.cl[J.close0 + ci].key_new;
#pragma unroll
                for (uint32_t h = 0; h < kHoist; h++)
                    if (h == ci) sg = m.cseg[h];
            }
            if (!use) continue;
            const uint32_t pos = wi[it] == prow ? seg_gallop(a.ec_val, max(ppos, sg.x), sg.y, cand[it])
                                                : seg_lower(a.ec_val, sg.x, sg.y, cand[it]);
            ok[it] = pos < sg.y && __ldg(a.ec_val + pos) == cand[it];
            prow = wi[it];
            ppos = pos;
        }
    }
#pragma unroll
    for (int it = 0; it < IPT; it++) {
        if (!ok[it]) continue;
        const auto& m = meta_of(wi[it]);
        const JoinJob& J = a.jobs[m.job];
        for (uint32_t ci = 0; ci < J.nclose && ok[it]; ci++) {
            const CloseChk& cl = a.cl[J.close0 + ci];
            if (!cl.key_new && ci < kHoist) continue;   // done above
            const uint32_t tgt = cl.tgt_new ? cand[it] : rowval(m, cl.tgt_col);
            const uint2 sg = close_seg(cl, cl.key_new ? cand[it] : rowval(m, cl.key_col));
            ok[it] = seg_contains(a.ec_val, sg.x, sg.y, tgt);
        }
    }
}

struct JMeta {              // one input row of a join step
    const uint32_t* rowp;   // its w values
    uint32_t s0;            // start of its driver list in ec_val
    uint32_t job;
    uint2 cseg[kHoist];     // hoisted closing segments (hoist_close)
    uint2 ext;              // extension segment
    uint32_t drv;           // driver list (RowLists)
};
using JoinSmem = PairSmem<JMeta, kPT, kPI, kJW, 1>;

// Block-wide copy of `words` staged u32 to global memory, 16-byte stores where the
// destination allows.
__device__ __forceinline__ void copy_out(uint32_t* __restrict__ g, const uint32_t* __restrict__ s, uint32_t words) {
    const uint32_t head = min(words, (uint32_t)((16u - ((uintptr_t)g & 15u)) & 15u) >> 2);
    if (threadIdx.x < head) g[threadIdx.x] = s[threadIdx.x];
    const uint32_t body = (words - head) & ~3u;
    uint4* g4 = reinterpret_cast<uint4*>(g + head);
    for (uint32_t x = threadIdx.x; x < body / 4; x += blockDim.x) {
        const uint32_t* q = s + head + 4 * x;
        g4[x] = make_uint4(q[0], q[1], q[2], q[3]);
    }
    for (uint32_t x = head + body + threadIdx.x; x < words; x += blockDim.x) g[x] = s[x];
}

// MODE 0: count pass (per-job totals + per-block counts -> last-block scan);
// MODE 1: write pass at the block offsets of the count pass;
// MODE 2: single pass over tiles of kTile pairs in ticket order: outputs staged in
//         shared memory, the tile's output offset from a decoupled look-back.
template <int MODE>
__global__ void __launch_bounds__(kPT) k_join(const __grid_constant__ JoinStep a, LbScratch lb, uint32_t ntiles,
                                              uint32_t epoch) {
    extern __shared__ __align__(16) char s_dyn[];
    constexpr bool WRITE = MODE != 0;
    uint64_t* s_jr = reinterpret_cast<uint64_t*>(s_dyn);      // [nj+1] first row of every job
    char* s_bufs = s_dyn + JoinSmem::buf_off(a.nj);
    uint32_t* s_out = reinterpret_cast<uint32_t*>(s_dyn + JoinSmem::extra_off(a.nj));   // staged output rows
    __shared__ uint64_t s_prefix;
    const bool stage = MODE == 2 || (MODE == 1 && a.wout <= kStageW);
    const uint32_t t = MODE == 2 ? lb_ticket(lb.ctr, ntiles) : 0u;
    JoinSmem::init(s_bufs);
    for (uint32_t j = threadIdx.x; j < a.nj; j += blockDim.x) s_jr[j] = a.jobs[j].row0;
    if (threadIdx.x == 0) s_jr[a.nj] = a.R;
    __syncthreads();
    auto offs = [&](uint64_t i) -> uint64_t { return __ldg(a.poff + i); };
    auto load = [&](uint64_t r) -> JMeta {
        JMeta m;
        m.job = pairs_find_smem(s_jr, a.nj, r);
        const JoinJob& J = a.jobs[m.job];
        m.rowp = J.M + (r - J.row0) * a.w;
        m.s0 = __ldg(a.s0 + r);
        if (J.nclose) {
            RowLists L;
            row_lists(a, J, m.rowp, L);
#pragma unroll
            for (uint32_t h = 0; h < kHoist; h++) m.cseg[h] = L.cseg[h];
            m.ext = L.ext;
            m.drv = L.drv;
        } else {
            m.drv = 0;
        }
        return m;
    };
    const uint64_t plo = a.plo, phi = a.phi == ~0ull ? offs(a.R) : a.phi;
    const uint64_t P = phi > plo ? phi - plo : 0;
    uint64_t p0, p1;
    if (MODE == 2) {
        p0 = plo + (uint64_t)t * kTile;
        p1 = p0 + kTile < phi ? p0 + kTile : phi;
    } else {
        pairs_range(P, blockIdx.x, gridDim.x, p0, p1);
        p0 += plo;
        p1 += plo;
    }
    uint64_t running = MODE == 1 ? a.ctl.blk[blockIdx.x] : 0ull;
    uint32_t lc = 0;        // MODE 2: output rows staged by the tile so far
    uint64_t count = 0;
    pair_chunks<JMeta, kPT, kPI, kJW, 1>(p0, p1, a.R, offs, load, s_bufs,
                                         [&](const bool (&v)[kPI], const uint32_t (&wi)[kPI],
                                             const uint32_t (&j)[kPI], const JMeta* sm, uint64_t) {
        JMeta m[kPI];
#pragma unroll
        for (int it = 0; it < kPI; it++) m[it] = sm[wi[it]];
        uint32_t cand[kPI];
#pragma unroll
        for (int it = 0; it < kPI; it++) cand[it] = v[it] ? __ldg(a.ec_val + m[it].s0 + j[it]) : 0u;
        bool valid[kPI], writes[kPI];
#pragma unroll
        for (int it = 0; it < kPI; it++) {   // injectivity (Def. 2 "injective")
            valid[it] = v[it];
            for (uint32_t c = 0; c < a.w && valid[it]; c++) valid[it] = __ldg(m[it].rowp + c) != cand[it];
        }
        lists_check<kPI>(a, wi, cand, valid, [&](uint32_t w_) -> const JMeta& { return sm[w_]; },
                         [&](const JMeta& mm, uint32_t col) { return __ldg(mm.rowp + col); });
#pragma unroll
        for (int it = 0; it < kPI; it++) writes[it] = valid[it] && !a.jobs[m[it].job].nowrite;
        if (MODE != 1) {   // per-job output totals
            uint32_t key[kPI], one[kPI];
#pragma unroll
            for (int it = 0; it < kPI; it++) {
                key[it] = m[it].job;
                one[it] = valid[it] ? 1u : 0u;
                count += writes[it] ? 1u : 0u;
            }
            run_sum<kPI>(v, key, one, [&](uint32_t job, uint32_t n) {
                atomicAdd(a.jobs[job].total, (unsigned long long)n);
            });
        }
        if (WRITE) {
            uint32_t mine = 0;
#pragma unroll
            for (int it = 0; it < kPI; it++) mine += writes[it] ? 1u : 0u;
            uint32_t tot;
            const uint32_t ex = block_excl_scan(mine, &tot);
            uint64_t pos = running + ex;                 // MODE 1 unstaged: global output row
            uint32_t lpos = (MODE == 2 ? lc : 0u) + ex;  // staged: row within the tile
#pragma unroll
            for (int it = 0; it < kPI; it++) {
                if (!writes[it]) continue;
                const JoinJob& J = a.jobs[m[it].job];
                const uint32_t* row = m[it].rowp;
                uint32_t* dst = stage ? s_out + (size_t)(lpos++) * a.wout : a.out + (pos++) * a.wout;
                if (J.final_) {
                    for (uint32_t c = 0; c < a.w; c++) dst[J.perm[c]] = __ldg(row + c);
                    dst[J.perm[a.w]] = cand[it];
                } else {
                    for (uint32_t c = 0; c < a.w; c++) dst[c] = __ldg(row + c);
                    dst[a.w] = cand[it];
                }
            }
            if (MODE == 1 && stage) {   // the block's rows are contiguous in the output
                __syncthreads();
                copy_out(a.out + running * a.wout, s_out, tot * a.wout);
            }
            running += tot;
            lc += tot;
        }
    });
    if (MODE == 0) last_block_scan(a.ctl.blk, gridDim.x, a.ctl.done, a.ctl.info, P, count);
    if (MODE == 2) {
        __syncthreads();
        if (threadIdx.x < 32) {
            const uint64_t pre = lb_warp_lookback(lb.status, t, lc, epoch);
            if (threadIdx.x == 0) s_prefix = pre;
        }
        __syncthreads();
        const uint64_t pre = s_prefix;
        const uint64_t n = pre >= a.cap ? 0 : (lc < a.cap - pre ? lc : a.cap - pre);   // rows below the capacity
        copy_out(a.out + (a.out_base + pre) * a.wout, s_out, (uint32_t)n * a.wout);
        if (t == ntiles - 1 && threadIdx.x == 0) {
            a.ctl.info[0] = P;
            a.ctl.info[1] = pre + lc;
        }
    }
}

// Single-pass join step for rows of <= kStageW output columns: the window stages,
// per input row, its values (with the output permutation of a final step packed
// in nibbles), EC segment start and flags, so injectivity, closing checks and the
// output row come from shared memory instead of per-pair global loads.
constexpr int kJVW = 128;   // window rows
struct JVMeta {
    uint32_t s0;            // EC segment start
    uint32_t job;
    uint32_t perm;          // output column of input column c (nibble c), of the new value (nibble w)
    uint32_t flags;         // bit 0: count only, bit 1: has closing arcs
    uint32_t val[kStageW];  // the row's w values, unused slots 0xffffffff (never a vertex id)
    uint2 cseg[kHoist];     // hoisted closing segments (hoist_close)
    uint2 ext;              // extension segment
    uint32_t drv;           // driver list (RowLists)
};
using JVSmem = PairSmem<JVMeta, kPT, kPI, kJVW, 1>;

__global__ void __launch_bounds__(kPT) k_join_v(const __grid_constant__ JoinStep a, LbScratch lb, uint32_t ntiles,
                                                uint32_t epoch) {
    extern __shared__ __align__(16) char s_dyn[];
    uint64_t* s_jr = reinterpret_cast<uint64_t*>(s_dyn);      // [nj+1] first row of every job
    char* s_bufs = s_dyn + JVSmem::buf_off(a.nj);
    uint32_t* s_out = reinterpret_cast<uint32_t*>(s_dyn + JVSmem::extra_off(a.nj));   // staged output rows
    __shared__ uint64_t s_prefix;
    const uint32_t t = lb_ticket(lb.ctr, ntiles);
    JVSmem::init(s_bufs);
    for (uint32_t j = threadIdx.x; j < a.nj; j += blockDim.x) s_jr[j] = a.jobs[j].row0;
    if (threadIdx.x == 0) s_jr[a.nj] = a.R;
    __syncthreads();
    const uint32_t w = a.w, wout = a.wout;
    auto offs = [&](uint64_t i) -> uint64_t { return __ldg(a.poff + i); };
    auto load = [&](uint64_t r) -> JVMeta {
        JVMeta m;
        m.job = pairs_find_smem(s_jr, a.nj, r);
        const JoinJob& J = a.jobs[m.job];
        const uint32_t* rowp = J.M + (r - J.row0) * w;
#pragma unroll
        for (uint32_t c = 0; c < kStageW; c++) m.val[c] = c < w ? __ldg(rowp + c) : 0xffffffffu;
        uint32_t perm = 0;
        for (uint32_t c = 0; c <= w; c++) perm |= (J.final_ ? (uint32_t)J.perm[c] : c) << (4 * c);
        m.perm = perm;
        m.flags = (J.nowrite ? 1u : 0u) | (J.nclose ? 2u : 0u);
        m.s0 = __ldg(a.s0 + r);
        if (J.nclose) {
            RowLists L;
            row_lists(a, J, rowp, L);
#pragma unroll
            for (uint32_t h = 0; h < kHoist; h++) m.cseg[h] = L.cseg[h];
            m.ext = L.ext;
            m.drv = L.drv;
        } else {
            m.drv = 0;
        }
        return m;
    };
    const uint64_t P = a.phi == ~0ull ? offs(a.R) - a.plo : a.phi - a.plo;
    const uint64_t p0 = a.plo + (uint64_t)t * kTile;
    const uint64_t p1 = p0 + kTile < a.plo + P ? p0 + kTile : a.plo + P;
    uint32_t lc = 0;   // output rows staged by the tile so far (uniform)
    pair_chunks<JVMeta, kPT, kPI, kJVW, 1>(p0, p1, a.R, offs, load, s_bufs,
                                           [&](const bool (&v)[kPI], const uint32_t (&wi)[kPI],
                                               const uint32_t (&j)[kPI], const JVMeta* sm, uint64_t) {
        uint32_t cand[kPI];
#pragma unroll
        for (int it = 0; it < kPI; it++) cand[it] = v[it] ? __ldg(a.ec_val + sm[wi[it]].s0 + j[it]) : 0u;
        bool valid[kPI], writes[kPI];
        uint32_t mine = 0;
#pragma unroll
        for (int it = 0; it < kPI; it++) {
            const JVMeta& m = sm[wi[it]];
            bool ok = v[it];
#pragma unroll
            for (uint32_t c = 0; c < kStageW; c++) ok = ok && m.val[c] != cand[it];   // injectivity (Def. 2)
            valid[it] = ok;
        }
        lists_check<kPI>(a, wi, cand, valid, [&](uint32_t w_) -> const JVMeta& { return sm[w_]; },
                         [&](const JVMeta& mm, uint32_t col) { return mm.val[col]; });
#pragma unroll
        for (int it = 0; it < kPI; it++) {
            writes[it] = valid[it] && !(sm[wi[it]].flags & 1u);
            mine += writes[it] ? 1u : 0u;
        }
        {   // per-job output totals: warp-wide when the warp's items share one job, else per run
            const uint32_t lane0 = __shfl_sync(kFull, sm[wi[0]].job, 0);
            uint32_t nv = 0;
            bool same = true;
#pragma unroll
            for (int it = 0; it < kPI; it++) {
                nv += valid[it] ? 1u : 0u;
                same = same && (!v[it] || sm[wi[it]].job == lane0);
            }
            if (__all_sync(kFull, same)) {
                const uint32_t s = __reduce_add_sync(kFull, nv);
                if (lane_id() == 0 && s) atomicAdd(a.jobs[lane0].total, (unsigned long long)s);
            } else {
                uint32_t key[kPI], one[kPI];
#pragma unroll
                for (int it = 0; it < kPI; it++) {
                    key[it] = sm[wi[it]].job;
                    one[it] = valid[it] ? 1u : 0u;
                }
                run_sum<kPI>(v, key, one, [&](uint32_t job, uint32_t n) {
                    atomicAdd(a.jobs[job].total, (unsigned long long)n);
                });
            }
        }
        uint32_t tot;
        uint32_t lpos = lc + block_excl_scan(mine, &tot);
#pragma unroll
        for (int it = 0; it < kPI; it++) {
            if (!writes[it]) continue;
            const JVMeta& m = sm[wi[it]];
            uint32_t* dst = s_out + (size_t)(lpos++) * wout;
            for (uint32_t c = 0; c < w; c++) dst[(m.perm >> (4 * c)) & 15u] = m.val[c];
            dst[(m.perm >> (4 * w)) & 15u] = cand[it];
        }
        lc += tot;
    });
    __syncthreads();
    if (threadIdx.x < 32) {
        const uint64_t pre = lb_warp_lookback(lb.status, t, lc, epoch);
        if (threadIdx.x == 0) s_prefix = pre;
    }
    __syncthreads();
    const uint64_t pre = s_prefix;
    const uint64_t n = pre >= a.cap ? 0 : (lc < a.cap - pre ? lc : a.cap - pre);   // rows below the capacity
    copy_out(a.out + (a.out_base + pre) * wout, s_out, (uint32_t)n * wout);
    if (t == ntiles - 1 && threadIdx.x == 0) {
        a.ctl.info[0] = P;
        a.ctl.info[1] = pre + lc;
    }
}

// Write pass of a closing-free step (no count pass): persistent blocks over
// contiguous pair ranges; a valid pair (cand not among the row's values) goes to
// output row woff[r] + j - #(row values in the segment before it).  The chunk's
// outputs are consecutive rows, so the chunk stages only (new value, window row)
// per output row and the block then writes the rows WORD-parallel: thread x forms
// words 4x..4x+3 of the chunk's output (template word or the new value) and
// stores them as one 16-byte vector -- every warp store is 512 contiguous bytes.
struct __align__(16) JFMeta {
    uint32_t tmpl[kStageW]; // the output row with the new value's column unset (0xffffffff)
    uint64_t woff;          // first output row of this input row
    uint32_t s0;            // EC segment start
    uint32_t imask;         // output columns whose value occurs in the segment
    uint32_t hole;          // output column of the new value; kStageW: count-only job (no output)
};
constexpr int kJFW = 512;   // window rows of the fast write (fan-out < 2 cuts chunks short)
constexpr int kFI = 4;      // pairs per thread per chunk of the fast write (8 measured slower: fewer chunks in flight)
constexpr uint32_t kFTile = kPT * kFI;
using JFSmem = PairSmem<JFMeta, kPT, kFI, kJFW, 1>;
__host__ __device__ constexpr size_t jf_stage(uint32_t) { return sizeof(uint2) * kFTile; }

template <uint32_t WOUT>
__device__ __forceinline__ void jf_tmpl(const JFMeta& m, uint32_t (&t)[WOUT]) {
    const uint4* tp = reinterpret_cast<const uint4*>(m.tmpl);
    const uint4 x0 = tp[0];
    const uint4 x1 = WOUT > 4 ? tp[1] : make_uint4(0u, 0u, 0u, 0u);
    const uint32_t all[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
    for (uint32_t c = 0; c < WOUT; c++) t[c] = all[c];
}

template <uint32_t WOUT>
__global__ void __launch_bounds__(kPT, 4) k_join_fast(const __grid_constant__ JoinStep a) {
    extern __shared__ __align__(16) char s_dyn[];
    uint64_t* s_jr = reinterpret_cast<uint64_t*>(s_dyn);
    char* s_bufs = s_dyn + JFSmem::buf_off(a.nj);
    uint2* s_ri = reinterpret_cast<uint2*>(s_dyn + JFSmem::extra_off(a.nj));   // (new value, window row) per output row
    __shared__ uint64_t s_base;
    JFSmem::init(s_bufs);
    for (uint32_t j = threadIdx.x; j < a.nj; j += blockDim.x) s_jr[j] = a.jobs[j].row0;
    if (threadIdx.x == 0) s_jr[a.nj] = a.R;
    __syncthreads();
    constexpr uint32_t w = WOUT - 1;
    auto offs = [&](uint64_t i) -> uint64_t { return __ldg(a.poff + i); };
    auto load = [&](uint64_t r) -> JFMeta {
        JFMeta m;
        const uint32_t job = pairs_find_smem(s_jr, a.nj, r);
        const JoinJob& J = a.jobs[job];
        const uint32_t* rowp = J.M + (r - J.row0) * w;
        const uint32_t perm = J.perm_packed, found = __ldg(a.imask + r);
        uint32_t val[w];
#pragma unroll
        for (uint32_t c = 0; c < w; c++) val[c] = __ldg(rowp + c);
        uint32_t im = 0;
#pragma unroll
        for (uint32_t oc = 0; oc < kStageW; oc++) {   // select, not a dynamic index: stays in registers
            uint32_t t = 0xffffffffu, f = 0;
#pragma unroll
            for (uint32_t c = 0; c < w; c++)
                if (((perm >> (4 * c)) & 15u) == oc) {
                    t = val[c];
                    f = (found >> c) & 1u;
                }
            m.tmpl[oc] = t;
            im |= f << oc;
        }
        m.imask = im;
        m.hole = J.nowrite ? kStageW : (perm >> (4 * w)) & 15u;
        m.s0 = __ldg(a.s0 + r);
        m.woff = __ldg(a.woff + r);
        return m;
    };
    const uint64_t P = offs(a.R);
    uint64_t p0, p1;
    pairs_range(P, blockIdx.x, gridDim.x, p0, p1);
    pair_chunks<JFMeta, kPT, kFI, kJFW, 1>(p0, p1, a.R, offs, load, s_bufs,
                                           [&](const bool (&v)[kFI], const uint32_t (&wi)[kFI],
                                               const uint32_t (&j)[kFI], const JFMeta* sm, uint64_t) {
        uint32_t cand[kFI];
        bool ok[kFI];
        uint32_t mine = 0;
#pragma unroll
        for (int it = 0; it < kFI; it++) {
            const bool live = v[it] && sm[wi[it]].hole < kStageW;
            cand[it] = live ? __ldg(a.ec_val + sm[wi[it]].s0 + j[it]) : 0u;
        }
#pragma unroll
        for (int it = 0; it < kFI; it++) {
            const JFMeta& m = sm[wi[it]];
            uint32_t t[WOUT];
            jf_tmpl<WOUT>(m, t);
            bool good = v[it] && m.hole < kStageW;
#pragma unroll
            for (uint32_t c = 0; c < WOUT; c++) good = good && t[c] != cand[it];   // injectivity (Def. 2)
            ok[it] = good;
            mine += good ? 1u : 0u;
        }
        uint32_t tot;
        uint32_t lpos = block_excl_scan(mine, &tot);
        if (tot == 0) return;
        if (mine && lpos == 0) {   // the chunk's first output: its global row fixes the chunk's base
            uint32_t fc = 0, fw = 0, fj = 0;   // selected, not indexed (keeps the arrays in registers)
#pragma unroll
            for (int it = kFI - 1; it >= 0; it--)
                if (ok[it]) {
                    fc = cand[it];
                    fw = wi[it];
                    fj = j[it];
                }
            const JFMeta& m = sm[fw];
            uint32_t before = 0;
#pragma unroll
            for (uint32_t c = 0; c < WOUT; c++) before += ((m.imask >> c) & 1u) && m.tmpl[c] < fc;
            s_base = m.woff + fj - before;
        }
#pragma unroll
        for (int it = 0; it < kFI; it++) {
            if (!ok[it]) continue;
            s_ri[lpos++] = make_uint2(cand[it], wi[it]);
        }
        __syncthreads();
        // word-parallel: thread x forms words 4x..4x+3 of the chunk's output (a template
        // word of the row's input row, or the new value) and stores one 16-byte vector
        uint32_t* g = a.out + s_base * WOUT;
        const uint32_t words = tot * WOUT;
        const uint32_t head = min(words, (uint32_t)((16u - ((uintptr_t)g & 15u)) & 15u) >> 2);
        auto word_at = [&](uint32_t row, uint32_t col) -> uint32_t {
            const uint2 ri = s_ri[row];
            const JFMeta& m = sm[ri.y];
            return col == m.hole ? ri.x : m.tmpl[col];
        };
        if (threadIdx.x < head) g[threadIdx.x] = word_at(threadIdx.x / WOUT, threadIdx.x % WOUT);
        const uint32_t nvec = (words - head) >> 2;
        uint4* g4 = reinterpret_cast<uint4*>(g + head);
        for (uint32_t x = threadIdx.x; x < nvec; x += kPT) {
            const uint32_t o = head + 4 * x;
            uint32_t row = o / WOUT, col = o - row * WOUT, wv[4];
            uint2 ri = s_ri[row];
            const JFMeta* m = sm + ri.y;
#pragma unroll
            for (int k = 0; k < 4; k++) {   // 4 consecutive words: one division, row info reloaded per row
                wv[k] = col == m->hole ? ri.x : m->tmpl[col];
                if (++col == WOUT && k < 3) {
                    col = 0;
                    ri = s_ri[++row];
                    m = sm + ri.y;
                }
            }
            g4[x] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        }
        for (uint32_t o = head + 4 * nvec + threadIdx.x; o < words; o += kPT) g[o] = word_at(o / WOUT, o % WOUT);
        __syncthreads();
    });
}


template <uint32_t WOUT>
static void launch_join_fast(gps_ctx* c, const JoinStep& s, uint64_t P) {
    const size_t smax = JFSmem::bytes(kMaxJobsPerLaunch, jf_stage(WOUT));
    allow_smem((const void*)k_join_fast<WOUT>, (int)smax);
    // one resident wave; no more blocks than chunks (a block's fixed cost is a global search)
    const uint64_t chunks = (P + kFTile - 1) / kFTile;
    const uint32_t wave = resident_grid(c, (const void*)k_join_fast<WOUT>, kPT, JFSmem::bytes(64, jf_stage(WOUT)));
    const uint32_t G = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)wave, chunks));
    launch(c, GPS_K_JOIN_WRITE, dim3(G), dim3(kPT), JFSmem::bytes(s.nj, jf_stage(WOUT)), k_join_fast<WOUT>, s);
}

void run_join_fast_write(gps_ctx* c, const JoinStep& s, uint64_t P) {
    if (join_bulk_enabled()) return run_join_bulk_write(c, s, P);
    switch (s.wout) {
        case 2: return launch_join_fast<2>(c, s, P);
        case 3: return launch_join_fast<3>(c, s, P);
        case 4: return launch_join_fast<4>(c, s, P);
        case 5: return launch_join_fast<5>(c, s, P);
        case 6: return launch_join_fast<6>(c, s, P);
        case 7: return launch_join_fast<7>(c, s, P);
        case 8: return launch_join_fast<8>(c, s, P);
        default: fail(GPS_EINVAL, "internal: fast join row width out of range");
    }
}

static size_t join_v_smem(uint32_t nj, uint32_t wout) {
    return JVSmem::bytes(nj, sizeof(uint32_t) * kTile * wout);
}

static size_t join_smem(uint32_t nj, int mode, uint32_t wout) {
    const size_t out = mode == 2 ? sizeof(uint32_t) * kTile * wout
                                 : (mode == 1 ? sizeof(uint32_t) * kTile * kStageW : 0);
    return JoinSmem::bytes(nj, out);
}

// Opt the join kernels in to their largest dynamic shared memory ONCE (the
// attribute is per function; setting it per launch would race between the
// batch worker threads).
static void allow_join_smem() {
    allow_smem((const void*)k_join<0>, (int)join_smem(kMaxJobsPerLaunch, 0, 0));
    allow_smem((const void*)k_join<1>, (int)join_smem(kMaxJobsPerLaunch, 1, 0));
    allow_smem((const void*)k_join<2>, (int)join_smem(kMaxJobsPerLaunch, 2, GPS_MAX_QV));
    allow_smem((const void*)k_join_v, (int)join_v_smem(kMaxJobsPerLaunch, kStageW));
}

// out[i] = first j in [0, R] with poff[j] >= t[i] (poff non-decreasing, R+1 entries): the
// row cuts of the row-sharded join (whole rows per rank).
__global__ void k_lower_bound(const uint64_t* __restrict__ poff, uint64_t R, const uint64_t* __restrict__ t,
                              uint32_t n, uint64_t* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t x = t[i];
    uint64_t lo = 0, hi = R + 1;   // answer in [lo, hi)
    while (lo < hi) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (poff[mid] < x) lo = mid + 1; else hi = mid;
    }
    out[i] = lo > R ? R : lo;
}

void run_lower_bound(gps_ctx* c, const uint64_t* poff, uint64_t R, const uint64_t* d_t, uint32_t n, uint64_t* d_out) {
    launch(c, GPS_K_JOIN_LEN, dim3((n + 63) / 64), dim3(64), 0, k_lower_bound, poff, R, d_t, n, d_out);
}

void run_join_count(gps_ctx* c, const JoinStep& s, uint32_t G) {
    allow_join_smem();
    launch(c, GPS_K_JOIN_COUNT, dim3(G), dim3(kPT), join_smem(s.nj, 0, s.wout), k_join<0>, s, LbScratch{}, 0u, 0u);
}
void run_join_write(gps_ctx* c, const JoinStep& s, uint32_t G) {
    allow_join_smem();
    launch(c, GPS_K_JOIN_WRITE, dim3(G), dim3(kPT), join_smem(s.nj, 1, s.wout), k_join<1>, s, LbScratch{}, 0u, 0u);
}
uint32_t run_join_tiles(gps_ctx* c, const JoinStep& s, uint64_t P) {
    if (P == 0) return 0;
    const uint64_t nt = (P + kTile - 1) / kTile;
    if (nt > 0x7fffffffull) fail(GPS_EOVERFLOW, "join pair space too large");
    if (s.wout > GPS_MAX_QV) fail(GPS_EINVAL, "internal: join row too wide");
    allow_join_smem();
    LbScratch lb = lb_scratch(c, 1, (uint32_t)nt);
    const uint32_t ep = lb_next_epoch(c);
    if (s.wout <= kStageW)
        launch(c, GPS_K_JOIN_WRITE, dim3((uint32_t)nt), dim3(kPT), join_v_smem(s.nj, s.wout), k_join_v, s, lb,
               (uint32_t)nt, ep);
    else
        launch(c, GPS_K_JOIN_WRITE, dim3((uint32_t)nt), dim3(kPT), join_smem(s.nj, 2, s.wout), k_join<2>, s, lb,
               (uint32_t)nt, ep);
    return ep;
}

// After a capped single pass (epoch ep, nt tiles, look-back words in slot 0): the first tile
// whose rows reach past row `cap` and its exclusive output prefix -> out[0], out[1].
__global__ void k_cap_tile(const uint64_t* __restrict__ status, uint32_t nt, uint64_t cap, uint64_t* out) {
    if (threadIdx.x != 0) return;
    auto incl = [&](uint32_t t) { return status[t] & kLbValueMask; };
    uint32_t lo = 0, hi = nt;   // first t with incl(t) > cap
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (incl(mid) > cap) hi = mid; else lo = mid + 1;
    }
    out[0] = lo;
    out[1] = lo == 0 ? 0 : incl(lo - 1);
}

void run_cap_tile(gps_ctx* c, uint64_t P, uint64_t cap, uint64_t* d_out) {
    const uint64_t nt = (P + kTile - 1) / kTile;
    LbScratch lb = lb_scratch(c, 1, (uint32_t)nt);
    launch(c, GPS_K_JOIN_LEN, dim3(1), dim3(32), 0, k_cap_tile, (const uint64_t*)lb.status, (uint32_t)nt, cap, d_out);
}

}  // namespace gps
