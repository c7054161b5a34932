// join.cu -- joining phase kernels (PAPER.md §"Joining Phase"), batched.
//
//   k_ec<W>      a6 collect_edge_candidates with the two-step output scheme (P:809,
//                citing Mars) over the pair space (job, key u' in C(p), arc of
//                adj_dir(u')): pass 1 (W=false) counts, per key, the distinct v' with a
//                fitting label, v' in B[q], v' != u' (warp-aggregated atomics), per job
//                and per block (last block scans the block counts); the per-key counts
//                are scanned into the address of each key's first v' (the "hash table"
//                of fig3:hashtable); pass 2 (W=true) re-examines and writes with
//                block-scan ranks in pair order, so every key's values come out sorted.
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
constexpr int kPW = 512;    // EC: rows of offsets staged in shared memory (double-buffered)
constexpr int kJW = 1024;   // join: rows staged (single buffer; fan-out can be 1)
constexpr uint32_t kStageW = 8;   // join write: stage output rows of width <= 8 in shared memory


// ------------------------------------------------------------ a6 EC build
struct EcMeta {             // one key row of an EC job
    uint32_t row, key, base, pad;
};

template <bool WRITE>
__global__ void __launch_bounds__(kPT) k_ec(DevGraph g, const ECJob* __restrict__ jobs, uint32_t nj, PassCtl ctl,
                                           uint32_t* __restrict__ val, unsigned long long* bytes_acc) {
    extern __shared__ __align__(16) char s_dyn[];
    using SM = PairSmem<EcMeta, kPT, kPI, kPW, 2>;
    uint64_t* s_jp = reinterpret_cast<uint64_t*>(s_dyn);
    char* s_bufs = s_dyn + SM::buf_off(nj);
    SM::init(s_bufs);
    job_prefix(nj, [&](uint32_t j) -> uint64_t { return __ldg(jobs[j].seg + *jobs[j].nkeys); }, s_jp);
    const uint64_t P = s_jp[nj];
    uint64_t p0, p1;
    pairs_range(P, blockIdx.x, gridDim.x, p0, p1);
    uint64_t running = WRITE ? ctl.blk[blockIdx.x] : 0ull;
    uint64_t count = 0;
    for_job_ranges(s_jp, nj, p0, p1, [&](uint32_t jj, uint64_t lo, uint64_t hi) {
        const ECJob& J = jobs[jj];
        const uint32_t* off = J.dir ? g.off_in : g.off_out;
        const uint32_t* arcs = J.dir ? g.arc_in : g.arc_out;
        auto offs = [&](uint64_t i) -> uint64_t { return (uint64_t)__ldg(J.seg + i); };
        auto load = [&](uint64_t r) -> EcMeta {
            EcMeta m;
            m.row = (uint32_t)r;
            m.key = __ldg(J.keys + r);
            m.base = __ldg(off + m.key);
            m.pad = 0;
            return m;
        };
        uint32_t jcount = 0;
        pair_chunks<EcMeta, kPT, kPI, kPW, 2>(lo, hi, (uint64_t)*J.nkeys, offs, load, s_bufs,
                                           [&](const bool (&v)[kPI], const uint32_t (&wi)[kPI],
                                               const uint32_t (&j)[kPI], const EcMeta* sm) {
            uint32_t x[kPI], xp[kPI];
#pragma unroll
            for (int it = 0; it < kPI; it++) {
                const uint32_t base = sm[wi[it]].base;
                x[it] = v[it] ? __ldg(arcs + base + j[it]) : 0u;
                xp[it] = (v[it] && j[it] > 0) ? __ldg(arcs + base + j[it] - 1) : 0xffffffffu;
            }
            bool pred[kPI];
#pragma unroll
            for (int it = 0; it < kPI; it++) {
                const uint32_t d = x[it] >> g.lbits;
                pred[it] = false;
                if (v[it] && lab_ok(x[it], g.lmask, J.lab) && d != sm[wi[it]].key && bit_test(J.Bq, d)) {
                    // parallel arcs to the same v' (reading R5): count v' once
                    const bool dup = j[it] > 0 && (xp[it] >> g.lbits) == d && lab_ok(xp[it], g.lmask, J.lab);
                    pred[it] = !dup;
                }
            }
            if (!WRITE) {
                uint32_t one[kPI];
#pragma unroll
                for (int it = 0; it < kPI; it++) {
                    one[it] = pred[it] ? 1u : 0u;
                    count += one[it];
                    jcount += one[it];
                }
                run_sum<kPI>(v, wi, one, [&](uint32_t w, uint32_t n) { atomicAdd(J.kcnt + sm[w].row, n); });
            } else {
                uint32_t mine = 0;
#pragma unroll
                for (int it = 0; it < kPI; it++) mine += pred[it] ? 1u : 0u;
                uint32_t tot;
                uint64_t pos = running + block_excl_scan(mine, &tot);
#pragma unroll
                for (int it = 0; it < kPI; it++)
                    if (pred[it]) val[pos++] = x[it] >> g.lbits;
                running += tot;
            }
        });
        if (!WRITE) {
            const uint32_t s = block_sum(jcount);
            if (threadIdx.x == 0 && s) atomicAdd(J.total, (unsigned long long)s);
        }
    });
    if (!WRITE) last_block_scan(ctl.blk, gridDim.x, ctl.done, ctl.info, P, count);
    if (bytes_acc && threadIdx.x == 0 && p1 > p0) atomicAdd(bytes_acc, (unsigned long long)(p1 - p0) * 4ull);
}

static size_t ec_smem_n(uint32_t nj) { return PairSmem<EcMeta, kPT, kPI, kPW, 2>::bytes(nj, 0); }

void run_ec(gps_ctx* c, const DevGraph& g, const ECJob* d_jobs, uint32_t nj, bool write, PassCtl ctl,
            uint32_t* val, uint32_t G) {
    if (nj == 0) return;
    if (nj > kMaxJobsPerLaunch) fail(GPS_EINVAL, "too many EC jobs per launch");
    if (write)
        launch(c, GPS_K_EC_WRITE, dim3(G), dim3(kPT), ec_smem_n(nj), k_ec<true>, g, d_jobs, nj, ctl, val,
               c->d_bytes + GPS_K_EC_WRITE);
    else
        launch(c, GPS_K_EC_COUNT, dim3(G), dim3(kPT), ec_smem_n(nj), k_ec<false>, g, d_jobs, nj, ctl, val,
               c->d_bytes + GPS_K_EC_COUNT);
}

// ------------------------------------------------------------ a8 join step
constexpr int kSegRows = 8;
constexpr int kSegTile = 256 * kSegRows;

// largest j < nj with jobs[j].row0 <= r
__device__ __forceinline__ uint32_t job_of_row(const JoinJob* __restrict__ jobs, uint32_t nj, uint64_t r) {
    uint32_t lo = 0, hi = nj;
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (jobs[mid].row0 <= r) lo = mid; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ bool seg_find(const uint32_t* __restrict__ val, uint32_t lo, uint32_t hi, uint32_t t,
                                         uint32_t* pos) {
    while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        uint32_t v = __ldg(val + mid);
        if (v == t) {
            *pos = mid;
            return true;
        }
        if (v < t) lo = mid + 1; else hi = mid;
    }
    return false;
}

template <bool FAST>
__global__ void __launch_bounds__(256) k_join_seg(const __grid_constant__ JoinStep a, LbScratch lb, uint32_t ntiles,
                                                  uint32_t epoch) {
    __shared__ uint64_t s_pre[3];
    const uint32_t tile = lb_ticket(lb.ctr, ntiles);
    const uint64_t r0 = (uint64_t)tile * kSegTile + (uint64_t)threadIdx.x * kSegRows;
    uint32_t len[kSegRows], wc[kSegRows], ac[kSegRows];
    uint64_t tsum = 0, wsum = 0, asum = 0;
    uint32_t jb = r0 < a.R ? job_of_row(a.jobs, a.nj, r0) : 0;
#pragma unroll
    for (int i = 0; i < kSegRows; i++) {
        const uint64_t r = r0 + i;
        len[i] = wc[i] = ac[i] = 0;
        if (r < a.R) {
            while (jb + 1 < a.nj && a.jobs[jb + 1].row0 <= r) jb++;
            const JoinJob& J = a.jobs[jb];
            const uint32_t* row = J.M + (r - J.row0) * a.w;
            const uint32_t key = __ldg(row + J.x_col);
            const uint32_t rk = bit_rank(J.Bx, J.rpx, key);
            const uint32_t s = __ldg(J.ec_off + rk);
            len[i] = __ldg(J.ec_off + rk + 1) - s;
            a.s0[r] = s;
            if (FAST) {
                uint32_t excl = 0, pos;
                for (uint32_t c = 0; c < a.w; c++) excl += seg_find(a.ec_val, s, s + len[i], __ldg(row + c), &pos);
                ac[i] = len[i] - excl;
                wc[i] = J.nowrite ? 0u : ac[i];
            }
        }
        tsum += len[i];
        wsum += wc[i];
        asum += ac[i];
    }
    uint64_t tot, wtot = 0, atot = 0;
    const uint64_t pre = block_excl_scan(tsum, &tot);
    uint64_t wpre = 0, apre = 0;
    if (FAST) {
        wpre = block_excl_scan(wsum, &wtot);
        apre = block_excl_scan(asum, &atot);
    }
    if (threadIdx.x < 32) {
        uint64_t p = lb_warp_lookback(lb.status, tile, tot, epoch);
        uint64_t pw = 0, pa = 0;
        if (FAST) {
            pw = lb_warp_lookback(lb.status + lb.max_tiles, tile, wtot, epoch);
            pa = lb_warp_lookback(lb.status + 2 * (size_t)lb.max_tiles, tile, atot, epoch);
        }
        if (threadIdx.x == 0) {
            s_pre[0] = p;
            s_pre[1] = pw;
            s_pre[2] = pa;
        }
    }
    __syncthreads();
    uint64_t run = s_pre[0] + pre, wrun = s_pre[1] + wpre, arun = s_pre[2] + apre;
#pragma unroll
    for (int i = 0; i < kSegRows; i++) {
        const uint64_t r = r0 + i;
        if (r < a.R) {
            a.poff[r] = run;
            if (FAST) {
                a.woff[r] = wrun;
                a.aoff[r] = arun;
            }
        }
        run += len[i];
        wrun += wc[i];
        arun += ac[i];
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) {
        a.poff[a.R] = s_pre[0] + tot;
        if (FAST) {
            a.woff[a.R] = s_pre[1] + wtot;
            a.aoff[a.R] = s_pre[2] + atot;
        }
    }
}

__global__ void k_join_job_totals(const __grid_constant__ JoinStep a) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= a.nj) return;
    const uint64_t lo = a.jobs[j].row0, hi = j + 1 < a.nj ? a.jobs[j + 1].row0 : a.R;
    *a.jobs[j].total = a.aoff[hi] - a.aoff[lo];
}

void run_join_job_totals(gps_ctx* c, const JoinStep& s) {
    launch(c, GPS_K_JOIN_LEN, dim3((s.nj + 127) / 128), dim3(128), 0, k_join_job_totals, s);
}

void run_join_seg(gps_ctx* c, const JoinStep& s) {
    const uint64_t nt = (s.R + kSegTile - 1) / kSegTile;
    if (nt > 0x7fffffffull) fail(GPS_EOVERFLOW, "join table too large");
    LbScratch lb = lb_scratch(c, 3, (uint32_t)nt);
    if (s.fast)
        launch(c, GPS_K_JOIN_LEN, dim3((uint32_t)nt), dim3(256), 0, k_join_seg<true>, s, lb, (uint32_t)nt,
               lb_next_epoch(c));
    else
        launch(c, GPS_K_JOIN_LEN, dim3((uint32_t)nt), dim3(256), 0, k_join_seg<false>, s, lb, (uint32_t)nt,
               lb_next_epoch(c));
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
__device__ __forceinline__ bool pair_ok(const JoinStep& a, const JoinJob& J, const uint32_t* __restrict__ row,
                                        uint32_t cand) {
    for (uint32_t c = 0; c < a.w; c++)
        if (__ldg(row + c) == cand) return false;
    for (uint32_t ci = 0; ci < J.nclose; ci++) {
        const CloseChk& cl = a.cl[J.close0 + ci];
        const uint32_t key = cl.key_new ? cand : __ldg(row + cl.key_col);
        const uint32_t tgt = cl.tgt_new ? cand : __ldg(row + cl.tgt_col);
        const uint32_t rk = bit_rank(cl.Bk, cl.rpk, key);
        if (!seg_contains(a.ec_val, __ldg(cl.off + rk), __ldg(cl.off + rk + 1), tgt)) return false;
    }
    return true;
}

struct JMeta {              // one input row of a join step
    const uint32_t* rowp;   // its w values
    uint64_t r;             // its index in the step's row space
    uint32_t s0;            // start of its EC segment in ec_val
    uint32_t job;
};

template <bool WRITE>
__global__ void __launch_bounds__(kPT) k_join(const __grid_constant__ JoinStep a) {
    extern __shared__ __align__(16) char s_dyn[];
    using SM = PairSmem<JMeta, kPT, kPI, kJW, 1>;
    uint64_t* s_jr = reinterpret_cast<uint64_t*>(s_dyn);      // [nj+1] first row of every job
    char* s_bufs = s_dyn + SM::buf_off(a.nj);
    uint32_t* s_out = reinterpret_cast<uint32_t*>(s_dyn + SM::extra_off(a.nj));   // staged output tile
    const bool stage = WRITE && a.wout <= kStageW;
    SM::init(s_bufs);
    for (uint32_t j = threadIdx.x; j < a.nj; j += blockDim.x) s_jr[j] = a.jobs[j].row0;
    if (threadIdx.x == 0) s_jr[a.nj] = a.R;
    __syncthreads();
    auto offs = [&](uint64_t i) -> uint64_t { return __ldg(a.poff + i); };
    auto load = [&](uint64_t r) -> JMeta {
        JMeta m;
        m.job = pairs_find_smem(s_jr, a.nj, r);
        const JoinJob& J = a.jobs[m.job];
        m.rowp = J.M + (r - J.row0) * a.w;
        m.r = r;
        m.s0 = __ldg(a.s0 + r);
        return m;
    };
    const uint64_t plo = a.plo, phi = a.phi == ~0ull ? offs(a.R) : a.phi;
    const uint64_t P = phi > plo ? phi - plo : 0;
    uint64_t p0, p1;
    pairs_range(P, blockIdx.x, gridDim.x, p0, p1);
    p0 += plo;
    p1 += plo;
    uint64_t running = (WRITE && !a.fast) ? a.ctl.blk[blockIdx.x] : 0ull;
    bool have_base = false;
    uint64_t count = 0;
    pair_chunks<JMeta, kPT, kPI, kJW, 1>(p0, p1, a.R, offs, load, s_bufs,
                                         [&](const bool (&v)[kPI], const uint32_t (&wi)[kPI],
                                             const uint32_t (&j)[kPI], const JMeta* sm) {
        JMeta m[kPI];
#pragma unroll
        for (int it = 0; it < kPI; it++) m[it] = sm[wi[it]];
        uint32_t cand[kPI];
#pragma unroll
        for (int it = 0; it < kPI; it++) cand[it] = v[it] ? __ldg(a.ec_val + m[it].s0 + j[it]) : 0u;
        bool valid[kPI], writes[kPI];
#pragma unroll
        for (int it = 0; it < kPI; it++) {
            valid[it] = false;
            writes[it] = false;
            if (v[it]) {
                const JoinJob& J = a.jobs[m[it].job];
                valid[it] = pair_ok(a, J, m[it].rowp, cand[it]);
                writes[it] = valid[it] && !J.nowrite;
            }
        }
        if (WRITE && a.fast) {
            // closing-free step (no count pass): the chunk's first output row is
            // woff[row] + (j - #row values in the segment prefix) of its first pair;
            // thread 0 computes it, the staged path below does the rest
            __shared__ uint64_t s_base;
            if (!have_base && threadIdx.x == 0 && v[0]) {
                uint32_t excl = 0, fp;
                const bool nw = a.jobs[m[0].job].nowrite;   // count-only rows contribute no output rows
                if (j[0] > 0 && !nw)
                    for (uint32_t c = 0; c < a.w; c++)
                        excl += seg_find(a.ec_val, m[0].s0, m[0].s0 + (uint32_t)j[0], __ldg(m[0].rowp + c), &fp);
                s_base = __ldg(a.woff + m[0].r) + (nw ? 0 : j[0] - excl);
            }
            if (!have_base) {   // later chunks of the block continue from `running`
                __syncthreads();
                running = s_base;
                have_base = true;
            }
        }
        if (WRITE) {
            uint32_t mine = 0;
#pragma unroll
            for (int it = 0; it < kPI; it++) mine += writes[it] ? 1u : 0u;
            uint32_t tot;
            const uint32_t ex = block_excl_scan(mine, &tot);
            uint64_t pos = running + ex;   // global output row
            uint32_t lpos = ex;            // row within the block's tile
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
            if (stage) {
                // the block's rows are contiguous in the output: coalesced copy of the tile
                __syncthreads();
                uint32_t* g = a.out + running * a.wout;
                const uint32_t words = tot * a.wout;
                for (uint32_t x = threadIdx.x; x < words; x += blockDim.x) g[x] = s_out[x];
            }
            running += tot;
        } else {
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
    });
    if (!WRITE) last_block_scan(a.ctl.blk, gridDim.x, a.ctl.done, a.ctl.info, P, count);
}

static size_t join_smem(uint32_t nj, bool write) {
    return PairSmem<JMeta, kPT, kPI, kJW, 1>::bytes(nj, write ? sizeof(uint32_t) * kPT * kPI * kStageW : 0);
}

// Opt the join kernels in to their largest dynamic shared memory ONCE (the
// attribute is per function; setting it per launch would race between the
// batch worker threads).
static void allow_join_smem() {
    static std::once_flag once;
    std::call_once(once, [] {
        GPS_CK(cudaFuncSetAttribute(k_join<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)join_smem(kMaxJobsPerLaunch, false)));
        GPS_CK(cudaFuncSetAttribute(k_join<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)join_smem(kMaxJobsPerLaunch, true)));
    });
}

__global__ void k_rows_for_ranges(const uint64_t* __restrict__ poff, uint64_t R, const uint64_t* __restrict__ lohi,
                                  uint32_t n, uint64_t* __restrict__ rows) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const uint64_t lo = lohi[2 * t], hi = lohi[2 * t + 1];
    if (lo >= hi || R == 0) {
        rows[3 * t] = rows[3 * t + 1] = rows[3 * t + 2] = 0;
        return;
    }
    // i0 = largest row with poff[i0] <= lo; i1 = 1 + largest row with poff[i] <= hi - 1
    auto find = [&](uint64_t p) {
        uint64_t a = 0, b = R;
        while (b - a > 1) {
            uint64_t m = a + (b - a) / 2;
            if (poff[m] <= p) a = m; else b = m;
        }
        return a;
    };
    const uint64_t i0 = find(lo);
    rows[3 * t] = i0;
    rows[3 * t + 1] = find(hi - 1) + 1;
    rows[3 * t + 2] = poff[i0];
}

void run_rows_for_ranges(gps_ctx* c, const uint64_t* poff, uint64_t R, const uint64_t* d_lohi, uint32_t n,
                         uint64_t* d_rows) {
    launch(c, GPS_K_JOIN_LEN, dim3((n + 63) / 64), dim3(64), 0, k_rows_for_ranges, poff, R, d_lohi, n, d_rows);
}

void run_join_count(gps_ctx* c, const JoinStep& s, uint32_t G) {
    allow_join_smem();
    launch(c, GPS_K_JOIN_COUNT, dim3(G), dim3(kPT), join_smem(s.nj, false), k_join<false>, s);
}
void run_join_write(gps_ctx* c, const JoinStep& s, uint32_t G) {
    allow_join_smem();
    launch(c, GPS_K_JOIN_WRITE, dim3(G), dim3(kPT), join_smem(s.nj, true), k_join<true>, s);
}

}  // namespace gps
