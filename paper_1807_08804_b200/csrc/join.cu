// join.cu -- joining phase kernels (PAPER.md §"Joining Phase").
//
//   k_ec<W>      a6 collect_edge_candidates with the two-step output scheme (P:809,
//                citing Mars) over the pair space (key u' in C(p), arc of adj_dir(u')):
//                pass 1 (W=false) counts, per key, the distinct v' with a fitting label,
//                v' in B[q], v' != u' (warp-aggregated atomics) and per block (last block
//                scans the block counts); the per-key counts are scanned into the
//                address of each key's first v' (the "hash table" of fig3:hashtable,
//                P:807); pass 2 (W=true) re-examines and writes, block-scan ranks in
//                pair order, so every key's values come out sorted.
//   k_join_seg   a8 per input row: O(1) key lookup (bitmap rank, instead of the paper's
//                logarithmic search P:820) -> EC segment start, and the exclusive scan
//                of segment lengths (pair offsets) in the same single pass.
//   k_join<W>    a8 combine over the pair space (row, segment position):
//                injectivity + every fused closing arc (binary search in the closing
//                arc's sorted EC segment); count (W=false, last block scans the block
//                counts) or write (W=true).
#include "kernels.cuh"
#include "lookback.cuh"
#include "pairs.cuh"

namespace gps {

constexpr int kPT = 256;    // threads per block
constexpr int kPI = 4;      // pairs per thread per chunk
constexpr int kPW = 1024;   // rows of offsets staged in shared memory

// ------------------------------------------------------------ a6 EC build
template <bool WRITE>
__global__ void __launch_bounds__(kPT) k_ec(DevGraph g, const __grid_constant__ ECArgs A,
                                           unsigned long long* bytes_acc) {
    __shared__ uint64_t s_off[kPW + 1];
    __shared__ uint64_t s_row;
    const ECArc& e = A.a[blockIdx.y];
    const uint32_t* off = e.dir ? g.off_in : g.off_out;
    const uint32_t* arcs = e.dir ? g.arc_in : g.arc_out;
    auto offs = [&](uint64_t i) -> uint64_t { return (uint64_t)__ldg(e.seg + i); };
    const uint64_t P = offs(e.nkeys);
    uint64_t p0, p1;
    pairs_range(P, blockIdx.x, gridDim.x, p0, p1);
    uint64_t running = WRITE ? e.blk[blockIdx.x] : 0ull;
    uint64_t count = 0;
    for_pairs<kPT, kPI, kPW>(p0, p1, (uint64_t)e.nkeys, offs, s_off, &s_row,
                             [&](bool v, uint64_t p, uint64_t row, uint64_t j) {
        bool pred = false;
        uint32_t d = 0;
        if (v) {
            const uint32_t key = __ldg(e.keys + row);
            const uint32_t base = __ldg(off + key);
            const uint32_t x = __ldg(arcs + base + j);
            d = x >> g.lbits;
            if (lab_ok(x, g.lmask, e.lab) && d != key && bit_test(e.Bq, d)) {
                bool dup = false;   // parallel arcs to the same v' (reading R5): count v' once
                if (j > 0) {
                    const uint32_t xp = __ldg(arcs + base + j - 1);
                    dup = (xp >> g.lbits) == d && lab_ok(xp, g.lmask, e.lab);
                }
                pred = !dup;
            }
        }
        if (!WRITE) {
            uint32_t peers;
            const uint32_t leader = warp_group_leader(v ? (uint32_t)row : 0xffffffffu, peers);
            const uint32_t nvalid = __popc(__ballot_sync(kFull, pred) & peers);
            if (v && lane_id() == leader && nvalid) atomicAdd(e.cnt + row, nvalid);
            count += pred ? 1 : 0;
        } else {
            uint32_t tot;
            const uint32_t rank = block_excl_scan((uint32_t)pred, &tot);
            if (pred) e.val[running + rank] = d;
            running += tot;
        }
    });
    if (!WRITE) last_block_scan(e.blk, gridDim.x, e.done, e.info, P, count);
    if (bytes_acc) {
        // algorithmic: 4 B per arc examined (the 4 B per value written are added by the host)
        unsigned long long mine = (p1 - p0) * 4ull;
        if (threadIdx.x == 0 && mine) atomicAdd(bytes_acc, mine);
    }
}

void run_ec(gps_ctx* c, const DevGraph& g, const ECArgs& a, bool write, uint32_t G) {
    if (a.na == 0) return;
    if (write)
        launch(c, GPS_K_EC_WRITE, dim3(G, a.na), dim3(kPT), 0, k_ec<true>, g, a, c->d_bytes + GPS_K_EC_WRITE);
    else
        launch(c, GPS_K_EC_COUNT, dim3(G, a.na), dim3(kPT), 0, k_ec<false>, g, a, c->d_bytes + GPS_K_EC_COUNT);
}

// ------------------------------------------------------------ a8 join step
constexpr int kSegRows = 8;
constexpr int kSegTile = 256 * kSegRows;

__global__ void __launch_bounds__(256) k_join_seg(const __grid_constant__ StepArgs a, LbScratch lb, uint32_t ntiles,
                                                  uint32_t epoch) {
    __shared__ uint64_t s_pre;
    const uint32_t tile = lb_ticket(lb.ctr, ntiles);
    const uint64_t r0 = (uint64_t)tile * kSegTile + (uint64_t)threadIdx.x * kSegRows;
    uint32_t len[kSegRows];
    uint64_t tsum = 0;
#pragma unroll
    for (int i = 0; i < kSegRows; i++) {
        const uint64_t r = r0 + i;
        len[i] = 0;
        if (r < a.R) {
            const uint32_t key = __ldg(a.M + r * a.w + a.x_col);
            const uint32_t rk = bit_rank(a.Bx, a.rpx, key);
            const uint32_t s = __ldg(a.ec_off + rk);
            len[i] = __ldg(a.ec_off + rk + 1) - s;
            a.s0[r] = s;
        }
        tsum += len[i];
    }
    uint64_t tot;
    const uint64_t pre = block_excl_scan(tsum, &tot);
    if (threadIdx.x < 32) {
        uint64_t p = lb_warp_lookback(lb.status, tile, tot, epoch);
        if (threadIdx.x == 0) s_pre = p;
    }
    __syncthreads();
    uint64_t run = s_pre + pre;
#pragma unroll
    for (int i = 0; i < kSegRows; i++) {
        const uint64_t r = r0 + i;
        if (r < a.R) a.poff[r] = run;
        run += len[i];
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) a.poff[a.R] = s_pre + tot;
}

void run_join_seg(gps_ctx* c, const StepArgs& s) {
    const uint64_t nt = (s.R + kSegTile - 1) / kSegTile;
    if (nt > 0x7fffffffull) fail(GPS_EOVERFLOW, "join table too large");
    LbScratch lb = lb_scratch(c, (uint32_t)nt);
    launch(c, GPS_K_JOIN_LEN, dim3((uint32_t)nt), dim3(256), 0, k_join_seg, s, lb, (uint32_t)nt, lb_next_epoch(c));
    c->stats.k_bytes[GPS_K_JOIN_LEN] += 4.0 * s.R + 12.0 * s.R;
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

// Injectivity (Def. 2 "injective") + every fused closing arc (P:818 case 1).
__device__ __forceinline__ bool pair_ok(const StepArgs& a, const uint32_t* __restrict__ row, uint32_t cand) {
    for (uint32_t j = 0; j < a.w; j++)
        if (__ldg(row + j) == cand) return false;
    for (int ci = 0; ci < a.nclose; ci++) {
        const CloseChk& cl = a.cl[ci];
        const uint32_t key = cl.key_new ? cand : __ldg(row + cl.key_col);
        const uint32_t tgt = cl.tgt_new ? cand : __ldg(row + cl.tgt_col);
        const uint32_t rk = bit_rank(cl.Bk, cl.rpk, key);
        if (!seg_contains(cl.val, __ldg(cl.off + rk), __ldg(cl.off + rk + 1), tgt)) return false;
    }
    return true;
}

template <bool WRITE>
__global__ void __launch_bounds__(kPT) k_join(const __grid_constant__ StepArgs a) {
    __shared__ uint64_t s_off[kPW + 1];
    __shared__ uint64_t s_row;
    auto offs = [&](uint64_t i) -> uint64_t { return __ldg(a.poff + i); };
    const uint64_t P = offs(a.R);
    uint64_t p0, p1;
    pairs_range(P, blockIdx.x, gridDim.x, p0, p1);
    uint64_t running = WRITE ? a.blk[blockIdx.x] : 0ull;
    uint64_t count = 0;
    for_pairs<kPT, kPI, kPW>(p0, p1, a.R, offs, s_off, &s_row, [&](bool v, uint64_t p, uint64_t r, uint64_t j) {
        bool valid = false;
        uint32_t cand = 0;
        const uint32_t* row = a.M + r * a.w;
        if (v) {
            cand = __ldg(a.ec_val + __ldg(a.s0 + r) + j);
            valid = pair_ok(a, row, cand);
        }
        if (WRITE) {
            uint32_t tot;
            const uint32_t rank = block_excl_scan((uint32_t)valid, &tot);
            if (valid) {
                uint32_t* dst = a.out + (running + rank) * a.wout;
                if (a.final_) {
                    for (uint32_t c = 0; c < a.w; c++) dst[a.perm[c]] = __ldg(row + c);
                    dst[a.perm[a.w]] = cand;
                } else {
                    for (uint32_t c = 0; c < a.w; c++) dst[c] = __ldg(row + c);
                    dst[a.w] = cand;
                }
            }
            running += tot;
        } else {
            count += valid ? 1 : 0;
        }
    });
    if (!WRITE) last_block_scan(a.blk, gridDim.x, a.done, a.info, P, count);
}

void run_join_count(gps_ctx* c, const StepArgs& s, uint32_t G) {
    launch(c, GPS_K_JOIN_COUNT, dim3(G), dim3(kPT), 0, k_join<false>, s);
}
void run_join_write(gps_ctx* c, const StepArgs& s, uint32_t G) {
    launch(c, GPS_K_JOIN_WRITE, dim3(G), dim3(kPT), 0, k_join<true>, s);
}

}  // namespace gps
