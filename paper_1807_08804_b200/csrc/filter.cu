// filter.cu -- filtering phase kernels (PAPER.md §"Filtering Phase").
//
//   k_check        a2 kernel_check (Alg. 2 line 7; Def. 3): one streaming
//                  pass over vlab / off_out / off_in tests ALL k query vertices and
//                  emits one bitmap word per (query vertex, 32 data vertices) with
//                  __ballot_sync.  HBM bound: (2 + 4 + 4) B per vertex read, k/8 B written.
//   k_collect      a3 kernel_collect: stream compaction of a
//                  candidate bitmap into the sorted c_array with popc + block scan +
//                  decoupled look-back (one pass), also emitting the per-word rank
//                  prefix (O(1) key lookup) and the candidates' degree prefixes (the
//                  pair spaces of explore and EC).
//   k_explore<M>   a4/a5 kernel_explore (Alg. 2 lines 14-22) over the PAIR
//                  space (candidate u', constraint, arc of adj_dir(u')): M=prune marks the
//                  constraints u' satisfies (Alg. 2 lines 15-18), M=propagate sets the
//                  fitting neighbours of surviving candidates in per-neighbour scratch
//                  bitmaps (lines 19-22).  Equal contiguous pair ranges per block replace
//                  the paper's warp-per-candidate + block-per-hub split.
//   k_clear        prune candidates that missed a constraint (atomicAnd on B[u]).
//   k_bitand       reading R15: B[v] &= propagated set, scratch reset.
#include "kernels.cuh"
#include "lookback.cuh"
#include "pairs.cuh"

namespace gps {

// ---------------------------------------------------------------- a2 check
__global__ void __launch_bounds__(256) k_check(DevGraph g, QDesc q, uint32_t* __restrict__ B) {
    const uint32_t lane = lane_id();
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < g.nw; w += nwarps) {
        const uint32_t v = w * 32 + lane;
        const bool valid = v < g.n;
        uint32_t lab = 0, od = 0, id = 0;
        if (valid) {
            lab = g.vlab[v];
            od = g.off_out[v + 1] - g.off_out[v];
            id = g.off_in[v + 1] - g.off_in[v];
        }
        uint32_t mine = 0;
        for (int u = 0; u < q.k; u++) {
            bool p = valid && (q.lab[u] < 0 || lab == (uint32_t)q.lab[u]) &&
                     (q.bound[u] < 0 || (int64_t)v == q.bound[u]) && od >= q.qout[u] && id >= q.qin[u];
            uint32_t m = __ballot_sync(kFull, p);
            if ((int)lane == u) mine = m;
        }
        if ((int)lane < q.k) B[(size_t)lane * g.nws + w] = mine;
    }
}

void run_check(gps_ctx* c, const DevGraph& g, const QDesc& q, uint32_t* B) {
    uint32_t blocks = std::min<uint32_t>((g.nw + 7) / 8, (uint32_t)c->nsm * 8);
    launch(c, GPS_K_CHECK, dim3(blocks), dim3(256), 0, k_check, g, q, B);
    c->stats.k_bytes[GPS_K_CHECK] += (double)g.n * 10.0 + (double)q.k * g.nw * 4.0;
}

// -------------------------------------------------------------- a3 collect
constexpr int kColThreads = 256;   // one bitmap word (32 vertices) per thread

__global__ void __launch_bounds__(kColThreads) k_collect(DevGraph g, CollectArgs a, LbScratch lb, uint32_t ntiles,
                                                         uint32_t epoch) {
    const int y = blockIdx.y;
    const uint32_t tile = lb_ticket(lb.ctr + 3 * y, ntiles);
    const uint32_t w = tile * kColThreads + threadIdx.x;
    const uint32_t word = w < g.nw ? a.B[y][w] : 0u;
    uint32_t c = __popc(word), so = 0, si = 0;
    if (word) {
        const uint32_t v0 = w * 32;
        uint32_t bits = word;
        while (bits) {
            const uint32_t b = __ffs(bits) - 1;
            bits &= bits - 1;
            const uint32_t v = v0 + b;
            so += __ldg(g.off_out + v + 1) - __ldg(g.off_out + v);
            si += __ldg(g.off_in + v + 1) - __ldg(g.off_in + v);
        }
    }
    uint32_t tc, tso, tsi;
    const uint32_t ec = block_excl_scan(c, &tc);
    const uint32_t eso = block_excl_scan(so, &tso);
    const uint32_t esi = block_excl_scan(si, &tsi);
    __shared__ uint64_t s_pre[3];
    if (threadIdx.x < 32) {
        const size_t base = (size_t)(3 * y) * lb.max_tiles;
        uint64_t p0 = lb_warp_lookback(lb.status + base, tile, tc, epoch);
        uint64_t p1 = lb_warp_lookback(lb.status + base + lb.max_tiles, tile, tso, epoch);
        uint64_t p2 = lb_warp_lookback(lb.status + base + 2 * (size_t)lb.max_tiles, tile, tsi, epoch);
        if (threadIdx.x == 0) {
            s_pre[0] = p0;
            s_pre[1] = p1;
            s_pre[2] = p2;
        }
    }
    __syncthreads();
    uint32_t rank = (uint32_t)s_pre[0] + ec;
    uint32_t ro = (uint32_t)s_pre[1] + eso;
    uint32_t ri = (uint32_t)s_pre[2] + esi;
    if (w < g.nw) a.rp[y][w] = rank;
    uint32_t* carr = a.carr[y];
    uint32_t* sgo = a.seg_out[y];
    uint32_t* sgi = a.seg_in[y];
    unsigned long long* mask = a.mask[y];
    uint32_t bits = word;
    while (bits) {
        const uint32_t b = __ffs(bits) - 1;
        bits &= bits - 1;
        const uint32_t v = w * 32 + b;
        carr[rank] = v;
        sgo[rank] = ro;
        sgi[rank] = ri;
        if (mask) mask[rank] = 0ull;
        ro += __ldg(g.off_out + v + 1) - __ldg(g.off_out + v);
        ri += __ldg(g.off_in + v + 1) - __ldg(g.off_in + v);
        rank++;
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) {
        const uint32_t C = (uint32_t)s_pre[0] + tc;
        a.rp[y][g.nw] = C;
        *a.cnt[y] = C;
        sgo[C] = (uint32_t)s_pre[1] + tso;
        sgi[C] = (uint32_t)s_pre[2] + tsi;
    }
}

void run_collect(gps_ctx* c, const DevGraph& g, CollectArgs a) {
    if (a.nu == 0) return;
    const uint32_t ntiles = (g.nw + kColThreads - 1) / kColThreads;
    LbScratch lb = lb_scratch(c, ntiles);
    launch(c, GPS_K_COLLECT, dim3(ntiles, a.nu), dim3(kColThreads), 0, k_collect, g, a, lb, ntiles,
           lb_next_epoch(c));
    // algorithmic: read bitmap + 8 B offsets per vertex window, write rank prefix; ids/segments on the device side
    c->stats.k_bytes[GPS_K_COLLECT] += (double)a.nu * g.nw * 8.0;
}

// -------------------------------------------------------------- a4 explore
constexpr int kET = 256;
constexpr int kEI = 4;
constexpr int kEW = 1024;

template <int MODE>   // 0: prune (mark satisfied constraints), 1: propagate
__global__ void __launch_bounds__(kET) k_explore(DevGraph g, const __grid_constant__ ExploreArgs a,
                                                 unsigned long long* bytes_acc) {
    __shared__ uint64_t s_off[kEW + 1];
    __shared__ uint64_t s_row;
    const uint32_t C = *a.cnt;
    const uint64_t no = (uint64_t)a.no, ni = (uint64_t)a.ni;
    auto offs = [&](uint64_t i) -> uint64_t {
        return no * __ldg(a.seg_out + i) + ni * __ldg(a.seg_in + i);
    };
    const uint64_t P = offs(C);
    uint64_t p0, p1;
    pairs_range(P, blockIdx.x, gridDim.x, p0, p1);
    const int nc = a.no + a.ni;
    const unsigned long long full = nc >= 64 ? ~0ull : ((1ull << nc) - 1ull);
    for_pairs<kET, kEI, kEW>(p0, p1, (uint64_t)C, offs, s_off, &s_row,
                             [&](bool v, uint64_t p, uint64_t row, uint64_t j) {
        uint32_t key = 0xffffffffu;
        unsigned long long bits = 0;
        bool fits = false;
        int ci = 0;
        uint32_t d = 0;
        if (v) {
            key = __ldg(a.cands + row);
            const uint32_t dout = __ldg(a.seg_out + row + 1) - __ldg(a.seg_out + row);
            const uint32_t din = __ldg(a.seg_in + row + 1) - __ldg(a.seg_in + row);
            uint32_t arc;
            if (j < no * dout) {
                ci = (int)(j / dout);
                arc = __ldg(g.arc_out + __ldg(g.off_out + key) + (uint32_t)(j % dout));
            } else {
                const uint64_t jj = j - no * dout;
                ci = a.no + (int)(jj / din);
                arc = __ldg(g.arc_in + __ldg(g.off_in + key) + (uint32_t)(jj % din));
            }
            const Cons& cs = a.c[ci];
            d = arc >> g.lbits;
            fits = lab_ok(arc, g.lmask, cs.lab) && d != key && bit_test(cs.Bv, d);
            if (MODE == 1) fits = fits && __ldg(a.mask + row) == full;
            bits = fits ? (1ull << ci) : 0ull;
        }
        if (MODE == 0) {
            uint32_t peers;
            const uint32_t leader = warp_group_leader((uint32_t)row ^ (v ? 0u : 0x80000000u), peers);
            const uint32_t lo = __reduce_or_sync(peers, (uint32_t)bits);
            const uint32_t hi = __reduce_or_sync(peers, (uint32_t)(bits >> 32));
            const unsigned long long agg = ((unsigned long long)hi << 32) | lo;
            if (v && lane_id() == leader && agg && (__ldcg(a.mask + row) & agg) != agg)
                atomicOr(a.mask + row, agg);
        } else {
            if (fits) atomicOr(a.c[ci].X + (d >> 5), 1u << (d & 31));
        }
    });
    if (bytes_acc) {
        // algorithmic bytes: 4 per arc examined (the 8 B of row offsets per candidate are read by collect)
        unsigned long long mine = (p1 - p0) * 4ull;
        if (threadIdx.x == 0 && mine) atomicAdd(bytes_acc, mine);
    }
}

__global__ void __launch_bounds__(256) k_clear(const __grid_constant__ ExploreArgs a) {
    const uint32_t C = *a.cnt;
    const int nc = a.no + a.ni;
    const unsigned long long full = nc >= 64 ? ~0ull : ((1ull << nc) - 1ull);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < C; i += gridDim.x * blockDim.x) {
        if (a.mask[i] != full) {
            const uint32_t key = a.cands[i];
            atomicAnd(a.Bu + (key >> 5), ~(1u << (key & 31)));
        }
    }
}

void run_explore(gps_ctx* c, const DevGraph& g, const ExploreArgs& a) {
    if (a.no + a.ni == 0) return;
    const uint32_t G = (uint32_t)c->nsm * 4;
    launch(c, GPS_K_EXPLORE, dim3(G), dim3(kET), 0, k_explore<0>, g, a, c->d_bytes + GPS_K_EXPLORE);
    launch(c, GPS_K_EXPLORE, dim3((uint32_t)c->nsm * 2), dim3(256), 0, k_clear, a);
    if (a.propagate) launch(c, GPS_K_EXPLORE, dim3(G), dim3(kET), 0, k_explore<1>, g, a, c->d_bytes + GPS_K_EXPLORE);
}

// --------------------------------------------------------------- bit-and
__global__ void __launch_bounds__(256) k_bitand(DevGraph g, AndArgs a) {
    const int t = blockIdx.y;
    uint32_t* B = a.B[t];
    for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < g.nw; w += gridDim.x * blockDim.x) {
        uint32_t v = B[w];
        for (int x = a.xbeg[t]; x < a.xbeg[t + 1]; x++) {
            v &= a.X[x][w];
            a.X[x][w] = 0u;
        }
        B[w] = v;
    }
}

void run_bitand(gps_ctx* c, const DevGraph& g, const AndArgs& a) {
    if (a.nt == 0) return;
    uint32_t blocks = std::min<uint32_t>((g.nw + 255) / 256, (uint32_t)c->nsm * 4);
    launch(c, GPS_K_BITAND, dim3(blocks, a.nt), dim3(256), 0, k_bitand, g, a);
    c->stats.k_bytes[GPS_K_BITAND] += (double)g.nw * 4.0 * (2.0 * a.nt + 2.0 * a.xbeg[a.nt]);
}

}  // namespace gps
