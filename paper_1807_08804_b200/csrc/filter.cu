// filter.cu -- filtering phase kernels (PAPER.md §"Filtering Phase").
//
//   k_check    a2  kernel_check (Alg. 2 line 7; Def. 3): one streaming
//                  pass over vlab / off_out / off_in tests ALL k query vertices and
//                  emits one bitmap word per (query vertex, 32 data vertices) with
//                  __ballot_sync.  HBM bound: (2 + 4 + 4) B per vertex read,
//                  k/8 B per vertex written.
//   k_collect  a3  kernel_collect: stream compaction of a
//                  candidate bitmap into the sorted c_array via popc + block scan,
//                  also emitting the per-word rank prefix used for O(1) key lookup.
//   k_explore  a4/a5 kernel_explore (Alg. 2 lines 14-22): one warp per
//                  candidate u', lanes stride adj(u') (coalesced); prune u'
//                  if some constraint has no fitting neighbour; else propagate its
//                  fitting neighbours into per-neighbour scratch bitmaps (atomicOr).
//   k_bitand   A15 reading: B[v] &= propagated set, scratch reset.
#include "kernels.cuh"
#include "prims.cuh"

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
    uint32_t warps = g.nw;
    uint32_t blocks = std::min<uint32_t>((warps + 7) / 8, (uint32_t)c->nsm * 8);
    launch(c, GPS_K_CHECK, dim3(blocks), dim3(256), 0, k_check, g, q, B);
    c->stats.k_bytes[GPS_K_CHECK] += (double)g.n * 10.0 + (double)q.k * g.nw * 4.0;
}

// -------------------------------------------------------------- a3 collect
constexpr int kColThreads = 256;
constexpr int kColWords = 8;                       // bitmap words per thread
constexpr int kColTile = kColThreads * kColWords;  // words per block

__global__ void __launch_bounds__(kColThreads) k_collect_count(DevGraph g, CollectArgs a, uint32_t* part,
                                                               uint32_t nblk) {
    const int y = blockIdx.y;
    const uint32_t* B = a.B[y];
    const uint32_t base = blockIdx.x * kColTile;
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < kColWords; i++) {
        uint32_t w = base + i * kColThreads + threadIdx.x;
        if (w < g.nw) s += __popc(B[w]);
    }
    s = block_sum(s);
    if (threadIdx.x == 0) part[y * nblk + blockIdx.x] = s;
}

__global__ void __launch_bounds__(kColThreads) k_collect_write(DevGraph g, CollectArgs a, const uint32_t* part,
                                                               uint32_t nblk) {
    const int y = blockIdx.y;
    const uint32_t* B = a.B[y];
    const uint32_t base = blockIdx.x * kColTile;
    // prefix of the preceding blocks (nblk is small: ceil(n / 65536))
    uint32_t pre = 0;
    if (part) {
        uint32_t s = 0;
        for (uint32_t j = threadIdx.x; j < blockIdx.x; j += blockDim.x) s += part[y * nblk + j];
        pre = block_sum(s);
    }
    uint32_t wv[kColWords];
    uint32_t cnt = 0;
    const uint32_t w0 = base + threadIdx.x * kColWords;
#pragma unroll
    for (int i = 0; i < kColWords; i++) {
        wv[i] = (w0 + i < g.nw) ? B[w0 + i] : 0u;
        cnt += __popc(wv[i]);
    }
    uint32_t tot;
    uint32_t ex = pre + block_excl_scan(cnt, &tot);
    uint32_t* rp = a.rp[y];
    uint32_t* out = a.carr[y];
#pragma unroll
    for (int i = 0; i < kColWords; i++) {
        uint32_t w = w0 + i;
        if (w < g.nw) {
            rp[w] = ex;
            uint32_t bits = wv[i];
            while (bits) {
                uint32_t b = __ffs(bits) - 1;
                out[ex++] = w * 32 + b;
                bits &= bits - 1;
            }
        }
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
        rp[g.nw] = pre + tot;
        *a.cnt[y] = pre + tot;
    }
}

void run_collect(gps_ctx* c, const DevGraph& g, const CollectArgs& a) {
    if (a.nu == 0) return;
    const uint32_t nblk = (g.nw + kColTile - 1) / kColTile;
    if (nblk <= 1) {
        launch(c, GPS_K_COLLECT, dim3(1, a.nu), dim3(kColThreads), 0, k_collect_write, g, a,
               (const uint32_t*)nullptr, 1u);
    } else {
        DevPtr part(c, sizeof(uint32_t) * nblk * a.nu);
        launch(c, GPS_K_COLLECT, dim3(nblk, a.nu), dim3(kColThreads), 0, k_collect_count, g, a, part.as<uint32_t>(),
               nblk);
        launch(c, GPS_K_COLLECT, dim3(nblk, a.nu), dim3(kColThreads), 0, k_collect_write, g, a,
               (const uint32_t*)part.as<uint32_t>(), nblk);
    }
    // algorithmic: read the bitmap, write rank prefix + (<= n) ids; ids counted as written on device
    c->stats.k_bytes[GPS_K_COLLECT] += (double)a.nu * g.nw * 8.0;
}

// -------------------------------------------------------------- a4 explore
__global__ void __launch_bounds__(256) k_explore(DevGraph g, ExploreArgs a, unsigned long long* bytes_acc) {
    const uint32_t lane = lane_id();
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t cnt = *a.cnt;
    unsigned long long bytes = 0;
    for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < cnt; i += nwarps) {
        const uint32_t up = a.cands[i];
        bool alive = true;
        // prune (Alg. 2 lines 15-18): every constraint needs one fitting neighbour
        for (int ci = 0; ci < a.nc && alive; ci++) {
            const Cons cs = a.c[ci];
            const uint32_t* off = cs.dir ? g.off_in : g.off_out;
            const uint32_t* arc = cs.dir ? g.arc_in : g.arc_out;
            const uint32_t s = off[up], e = off[up + 1];
            bytes += 8 + 4ull * (e - s);
            bool found = false;
            for (uint32_t b = s; b < e; b += 32) {
                const uint32_t j = b + lane;
                bool ok = false;
                if (j < e) {
                    const uint32_t x = __ldg(arc + j);
                    const uint32_t d = x >> g.lbits;
                    ok = lab_ok(x, g.lmask, cs.lab) && d != up && bit_test(cs.Bv, d);
                }
                if (__any_sync(kFull, ok)) {
                    found = true;
                    break;
                }
            }
            alive = found;
        }
        if (!alive) {
            if (lane == 0) atomicAnd(a.Bu + (up >> 5), ~(1u << (up & 31)));
            continue;
        }
        // propagate (Alg. 2 lines 19-22): fitting neighbours become candidates of v
        for (int ci = 0; ci < a.nc; ci++) {
            const Cons cs = a.c[ci];
            if (!cs.X) continue;
            const uint32_t* off = cs.dir ? g.off_in : g.off_out;
            const uint32_t* arc = cs.dir ? g.arc_in : g.arc_out;
            const uint32_t s = off[up], e = off[up + 1];
            for (uint32_t j = s + lane; j < e; j += 32) {
                const uint32_t x = __ldg(arc + j);
                const uint32_t d = x >> g.lbits;
                if (lab_ok(x, g.lmask, cs.lab) && d != up && bit_test(cs.Bv, d))
                    atomicOr(cs.X + (d >> 5), 1u << (d & 31));
            }
        }
    }
    if (bytes_acc) {
        // one lane per warp accounted the bytes; aggregate per block
        unsigned long long v = lane == 0 ? bytes : 0ull;
        v = block_sum(v);
        if (threadIdx.x == 0 && v) atomicAdd(bytes_acc, v);
    }
}

void run_explore(gps_ctx* c, const DevGraph& g, const ExploreArgs& a, uint32_t max_cands) {
    if (max_cands == 0) return;
    uint32_t warps_needed = max_cands;
    uint32_t blocks = std::min<uint32_t>((warps_needed + 7) / 8, (uint32_t)c->nsm * 8);
    launch(c, GPS_K_EXPLORE, dim3(blocks), dim3(256), 0, k_explore, g, a, c->d_bytes + GPS_K_EXPLORE);
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
