// join.cu -- joining phase kernels (PAPER.md §"Joining Phase").
//
//   k_ec<false/true>  a6 collect_edge_candidates with the two-step output scheme
//                     (citing Mars): pass 1 counts, per key u' in C(p), the
//                     distinct v' in adj_dir(u') with a fitting label, v' in B[q],
//                     v' != u'; an exclusive scan gives the address of the first v'
//                     of every key (the "hash table" of fig3:hashtable);
//                     pass 2 re-examines and writes.  One warp per key, lanes
//                     stride the adjacency (coalesced), ballot/popc compaction keeps
//                     each key's values sorted.
//   k_join_len        a8 per input row: O(1) key lookup (bitmap rank instead of the
//                     paper's logarithmic search) -> EC segment start / length.
//   k_join<W>         a8 combine over the PAIR SPACE (row, segment
//                     position): G persistent blocks take equal contiguous pair
//                     ranges (load balanced whatever the fan-out), verify
//                     injectivity + every fused closing arc (binary search in the
//                     closing arc's sorted EC segment), and -- two-step output --
//                     count (W=false; last block scans the block counts) or write
//                     (W=true; block scan gives each valid pair its output row).
#include "kernels.cuh"
#include "prims.cuh"

namespace gps {

// ------------------------------------------------------------ a6 EC build
template <bool WRITE>
__global__ void __launch_bounds__(256) k_ec(DevGraph g, ECArgs A, unsigned long long* bytes_acc) {
    const ECArc e = A.a[blockIdx.y];
    const uint32_t lane = lane_id();
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t* off = e.dir ? g.off_in : g.off_out;
    const uint32_t* arc = e.dir ? g.arc_in : g.arc_out;
    const uint32_t lt = (1u << lane) - 1u;
    unsigned long long bytes = 0;
    for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < e.nkeys; i += nwarps) {
        const uint32_t key = e.keys[i];
        const uint32_t s = off[key], t = off[key + 1];
        uint32_t running = WRITE ? e.off[i] : 0u;
        const uint32_t start = running;
        for (uint32_t b = s; b < t; b += 32) {
            const uint32_t j = b + lane;
            bool pred = false;
            uint32_t d = 0;
            if (j < t) {
                const uint32_t x = __ldg(arc + j);
                d = x >> g.lbits;
                if (lab_ok(x, g.lmask, e.lab) && d != key && bit_test(e.Bq, d)) {
                    bool dup = false;   // parallel arcs to the same v' (reading R5): count v' once
                    if (j > s) {
                        const uint32_t xp = __ldg(arc + j - 1);
                        dup = (xp >> g.lbits) == d && lab_ok(xp, g.lmask, e.lab);
                    }
                    pred = !dup;
                }
            }
            const uint32_t m = __ballot_sync(kFull, pred);
            if (WRITE && pred) e.val[running + __popc(m & lt)] = d;
            running += __popc(m);
        }
        if (!WRITE && lane == 0) e.cnt[i] = running;
        bytes += 8 + 4ull * (t - s) + (WRITE ? 4ull * (running - start) : 0ull);
    }
    if (bytes_acc) {
        unsigned long long v = lane == 0 ? bytes : 0ull;
        v = block_sum(v);
        if (threadIdx.x == 0 && v) atomicAdd(bytes_acc, v);
    }
}

void run_ec(gps_ctx* c, const DevGraph& g, const ECArgs& a, bool write, uint32_t max_keys) {
    if (a.na == 0 || max_keys == 0) return;
    uint32_t blocks = std::min<uint32_t>((max_keys + 7) / 8, (uint32_t)c->nsm * 8);
    if (write)
        launch(c, GPS_K_EC_WRITE, dim3(blocks, a.na), dim3(256), 0, k_ec<true>, g, a, c->d_bytes + GPS_K_EC_WRITE);
    else
        launch(c, GPS_K_EC_COUNT, dim3(blocks, a.na), dim3(256), 0, k_ec<false>, g, a, c->d_bytes + GPS_K_EC_COUNT);
}

// ------------------------------------------------------------ a8 join step
__global__ void __launch_bounds__(256) k_join_len(const StepArgs a, uint32_t* __restrict__ s0,
                                                  uint32_t* __restrict__ len) {
    for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < a.R; r += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t key = a.M[r * a.w + a.x_col];
        const uint32_t rk = bit_rank(a.Bx, a.rpx, key);
        const uint32_t s = __ldg(a.ec_off + rk), t = __ldg(a.ec_off + rk + 1);
        s0[r] = s;
        len[r] = t - s;
    }
}

void run_join_len(gps_ctx* c, const StepArgs& s, uint32_t* len) {
    uint64_t blocks = (s.R + 255) / 256;
    if (blocks > (uint64_t)c->nsm * 16) blocks = (uint64_t)c->nsm * 16;
    launch(c, GPS_K_JOIN_LEN, dim3((uint32_t)blocks), dim3(256), 0, k_join_len, s, const_cast<uint32_t*>(s.s0), len);
    c->stats.k_bytes[GPS_K_JOIN_LEN] += 4.0 * s.R + 8.0 * s.R;
}

constexpr int kJT = 256;            // threads per block
constexpr int kJI = 4;              // pairs per thread per chunk
constexpr int kJC = kJT * kJI;      // pairs per chunk
constexpr int kJW = 1024;           // rows of pair offsets staged in shared memory

// largest r in [lo, hi) with poff[r] <= p (requires poff[lo] <= p)
__device__ __forceinline__ uint64_t find_row_global(const uint64_t* __restrict__ poff, uint64_t lo, uint64_t hi,
                                                    uint64_t p) {
    while (hi - lo > 1) {
        uint64_t mid = lo + (hi - lo) / 2;
        if (__ldg(poff + mid) <= p) lo = mid; else hi = mid;
    }
    return lo;
}
// largest i in [0, n) with s[i] <= p (requires s[0] <= p)
__device__ __forceinline__ uint32_t find_row_smem(const uint64_t* s, uint32_t n, uint64_t p) {
    uint32_t lo = 0, hi = n;
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (s[mid] <= p) lo = mid; else hi = mid;
    }
    return lo;
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
__global__ void __launch_bounds__(kJT) k_join(const __grid_constant__ StepArgs a, uint32_t G) {
    __shared__ uint64_t s_off[kJW + 1];
    __shared__ uint64_t s_row;
    __shared__ bool s_last;
    const uint32_t tid = threadIdx.x;
    const uint64_t P = a.poff[a.R];
    const uint64_t q = P / G, rem = P % G;
    const uint64_t p0 = q * blockIdx.x + (blockIdx.x < rem ? blockIdx.x : rem);
    const uint64_t p1 = p0 + q + (blockIdx.x < rem ? 1 : 0);
    uint64_t running = WRITE ? a.blk[blockIdx.x] : 0;
    uint64_t count = 0;
    if (p0 < p1) {
        if (tid == 0) s_row = find_row_global(a.poff, 0, a.R, p0);
        __syncthreads();
        uint64_t r0 = s_row;
        for (uint64_t cp = p0; cp < p1; cp += kJC) {
            const uint64_t cend = cp + kJC < p1 ? cp + kJC : p1;
            const uint32_t wn = (uint32_t)((a.R - r0) < (uint64_t)kJW ? (a.R - r0) : (uint64_t)kJW);
            for (uint32_t i = tid; i <= wn; i += kJT) s_off[i] = __ldg(a.poff + r0 + i);
            __syncthreads();
            const uint64_t wend = s_off[wn];
#pragma unroll
            for (int it = 0; it < kJI; it++) {
                const uint64_t p = cp + (uint64_t)it * kJT + tid;
                bool valid = false;
                uint64_t r = 0;
                uint32_t cand = 0;
                if (p < cend) {
                    uint64_t base;
                    if (p < wend) {
                        uint32_t i = find_row_smem(s_off, wn, p);
                        r = r0 + i;
                        base = s_off[i];
                    } else {
                        r = find_row_global(a.poff, r0 + wn, a.R, p);
                        base = __ldg(a.poff + r);
                    }
                    cand = __ldg(a.ec_val + __ldg(a.s0 + r) + (p - base));
                    valid = pair_ok(a, a.M + r * a.w, cand);
                }
                if (WRITE) {
                    uint32_t tot;
                    const uint32_t rank = block_excl_scan((uint32_t)valid, &tot);
                    if (valid) {
                        const uint32_t* row = a.M + r * a.w;
                        uint32_t* dst = a.out + (running + rank) * a.wout;
                        if (a.final_) {
                            for (uint32_t j = 0; j < a.w; j++) dst[a.perm[j]] = __ldg(row + j);
                            dst[a.perm[a.w]] = cand;
                        } else {
                            for (uint32_t j = 0; j < a.w; j++) dst[j] = __ldg(row + j);
                            dst[a.w] = cand;
                        }
                    }
                    running += tot;
                } else {
                    count += valid ? 1 : 0;
                }
            }
            __syncthreads();   // s_off reused by the next chunk
            if (cend < p1) {
                if (tid == 0) s_row = (cend < wend) ? r0 + find_row_smem(s_off, wn, cend)
                                                     : find_row_global(a.poff, r0 + wn, a.R, cend);
                __syncthreads();
                r0 = s_row;
            }
        }
    }
    if (!WRITE) {
        count = block_sum(count);
        if (tid == 0) {
            a.blk[blockIdx.x] = count;
            __threadfence();
            const unsigned prev = atomicAdd(a.done, 1u);
            s_last = (prev == G - 1);
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
            uint64_t carry = 0;
            for (uint32_t b = 0; b < G; b += kJT) {
                const uint32_t i = b + tid;
                const uint64_t v = i < G ? __ldcg(a.blk + i) : 0ull;
                uint64_t tot;
                const uint64_t ex = block_excl_scan(v, &tot);
                if (i < G) a.blk[i] = carry + ex;
                carry += tot;
            }
            if (tid == 0) {
                a.blk[G] = carry;
                a.info[0] = P;
                a.info[1] = carry;
                *a.done = 0u;
            }
        }
    }
}

void run_join_count(gps_ctx* c, const StepArgs& s, uint32_t G) {
    launch(c, GPS_K_JOIN_COUNT, dim3(G), dim3(kJT), 0, k_join<false>, s, G);
}
void run_join_write(gps_ctx* c, const StepArgs& s, uint32_t G) {
    launch(c, GPS_K_JOIN_WRITE, dim3(G), dim3(kJT), 0, k_join<true>, s, G);
}

}  // namespace gps
