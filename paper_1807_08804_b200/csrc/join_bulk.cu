// join_bulk.cu -- write pass of a closing-free join step (a8) with the
// per-row inputs staged by TMA bulk copies (cp.async.bulk, UBLKCP), double-buffered.
//
// Same arithmetic as k_join_fast (join.cu): the output row of pair (row r, segment
// position j) is woff[r] + j - #(row values in the segment before it), valid when the
// new value is not one of the row's values (injectivity, Def. 2).  What
// changes is how the per-row inputs reach the block.  A block owns a contiguous pair
// range, hence a contiguous row range; it walks that range in WINDOWS of kBW rows.
// Every per-row input of a window is a contiguous range of device memory -- the pair
// offsets poff, the segment starts s0, the output offsets woff, the in-segment masks
// imask, and the input rows M (one range per query whose rows the window meets) --
// so one elected thread stages the whole window with a handful of bulk copies
// completing on an mbarrier, and issues window k+1's copies before the block works
// on window k.  The window's pairs then need ONE dependent global access per chunk
// (the new values in the EC segments) instead of the four of the load-as-you-go
// path (row search, offsets, row data, values).
#include <cstdlib>

#include "bulk.cuh"
#include "kernels.cuh"
#include "pairs.cuh"

namespace gps {

constexpr int kBT = 256;                 // threads per block
constexpr int kBI = 4;                   // pairs per thread per chunk
constexpr uint32_t kBCh = kBT * kBI;     // pairs per chunk
constexpr uint32_t kBW = 256;            // rows per window
constexpr uint32_t kBPieces = 8;         // input-row ranges (queries) per window
constexpr uint32_t kNoHole = 0xffu;

struct BHdr {                // window descriptor, written by the producer before the copies
    uint64_t r0;             // first row (global row numbering of the step)
    uint32_t wn;             // rows
    uint32_t np;             // pieces
    uint32_t sh_poff, sh_woff, sh_s0, sh_im;   // byte shifts of the staged arrays in their slots
    uint32_t prow[kBPieces + 1];   // first window row of each piece (prow[np] = wn)
    uint32_t poffs[kBPieces];      // byte offset of each piece's first row inside the M area
    uint32_t pjob[kBPieces];       // job of each piece
};

// Per-buffer layout (bytes): header, poff, woff, s0, imask, M, meta.
template <uint32_t WOUT, bool ST = (WOUT <= 4)>
struct BLay {
    static constexpr uint32_t w = WOUT - 1;
    static __host__ __device__ constexpr size_t a16(size_t x) { return (x + 15) & ~size_t(15); }
    static constexpr size_t HDR = 0;
    static constexpr size_t POFF = a16(sizeof(BHdr));
    static constexpr size_t WOFF = POFF + bulk_slot(8ull * (kBW + 1));
    static constexpr size_t S0 = WOFF + bulk_slot(8ull * kBW);
    static constexpr size_t IM = S0 + bulk_slot(4ull * kBW);
    static constexpr size_t M = IM + bulk_slot(4ull * kBW);
    static constexpr size_t META = M + a16(4ull * w * kBW) + 32ull * kBPieces;
    // meta per row: WOUT template words (new value's column = 0xffffffff), then
    // (hole | in-segment mask of the output columns << 8)
    static constexpr size_t BUF = META + a16(4ull * (WOUT + 1) * kBW);
    // output staging (two buffers, alternating per chunk): a chunk's rows, row-major, placed at the
    // output's address offset mod 16 so the aligned interior goes out as one bulk store
    // (wide rows, WOUT > kStagedMax: no staging -- it would halve the resident blocks -- but one
    // (new value, window row) pair per output row and word-parallel 16-byte stores)
    // (wide rows are staged in ONE buffer -- two would cost resident blocks -- whose previous
    // bulk store must have finished reading before it is rewritten; ST = false: no staging, one
    // (new value, window row) pair per output row and word-parallel 16-byte stores)
    static constexpr bool STAGED = ST;
    static constexpr uint32_t NSTG = (ST && WOUT <= 4) ? 2 : 1;
    static constexpr uint32_t STG = STAGED ? kBCh * WOUT + 4 : 2 * kBCh;   // words
    static constexpr size_t OUT = 2 * BUF;
    static __host__ __device__ size_t jobs_bytes(uint32_t nj) { return a16(8ull * (nj + 1) + 8ull * nj + 4ull * nj + nj); }
    static __host__ __device__ size_t bytes(uint32_t nj) { return jobs_bytes(nj) + OUT + NSTG * a16(4ull * STG) + 16; }
    // STAGED = false: the two staging buffers hold the kBCh uint2 (value, row) entries instead
};

template <uint32_t WOUT>
__device__ __forceinline__ void issue_window(const JoinStep& a, char* buf, uint64_t* bar, uint64_t r0, uint64_t rend,
                                             const uint64_t* s_jr, const uint32_t* const* s_jM, uint32_t nj) {
    using L = BLay<WOUT>;
    constexpr uint32_t w = L::w;
    BHdr* h = reinterpret_cast<BHdr*>(buf + L::HDR);
    uint32_t wn = (uint32_t)((rend - r0) < (uint64_t)kBW ? (rend - r0) : (uint64_t)kBW);
    // pieces: the queries (jobs) whose rows meet [r0, r0 + wn); cut the window at the
    // (kBPieces + 1)-th non-empty job
    uint32_t lo = 0, hi = nj;   // job of row r0: largest j with row0 <= r0
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (s_jr[mid] <= r0) lo = mid; else hi = mid;
    }
    uint32_t np = 0, moff = 0, tx = 0;
    char* marea = buf + L::M;
    for (uint32_t j = lo; j < nj && np < kBPieces; j++) {
        const uint64_t a0 = s_jr[j] > r0 ? s_jr[j] : r0;
        if (a0 >= r0 + wn) break;
        const uint64_t a1 = s_jr[j + 1] < r0 + wn ? s_jr[j + 1] : r0 + wn;
        if (a1 <= a0) continue;   // a query without rows in this step
        h->prow[np] = (uint32_t)(a0 - r0);
        h->pjob[np] = j;
        const uint32_t* src = s_jM[j] + (a0 - s_jr[j]) * w;
        const uint64_t nb = (a1 - a0) * w * 4ull;
        const uint32_t sh = bulk_stage(marea + moff, src, nb, bar, &tx);
        h->poffs[np] = moff + sh;
        moff += (uint32_t)(((reinterpret_cast<uintptr_t>(src) + nb + 15) & ~uintptr_t(15)) -
                           (reinterpret_cast<uintptr_t>(src) & ~uintptr_t(15)));
        np++;
        if (np == kBPieces && a1 < r0 + wn) wn = (uint32_t)(a1 - r0);   // out of piece slots: cut
    }
    h->r0 = r0;
    h->wn = wn;
    h->np = np;
    h->prow[np] = wn;
    h->sh_poff = bulk_stage(buf + L::POFF, a.poff + r0, 8ull * (wn + 1), bar, &tx);
    h->sh_woff = bulk_stage(buf + L::WOFF, a.woff + r0, 8ull * wn, bar, &tx);
    h->sh_s0 = bulk_stage(buf + L::S0, a.s0 + r0, 4ull * wn, bar, &tx);
    h->sh_im = bulk_stage(buf + L::IM, a.imask + r0, 4ull * wn, bar, &tx);
    mbar_arrive_expect_tx(bar, tx);   // the header writes above are released by this arrive
}

template <uint32_t WOUT, bool ST>
__global__ void __launch_bounds__(kBT, (WOUT >= 5 ? 4 : 3)) k_join_bulk(const __grid_constant__ JoinStep a) {
    using L = BLay<WOUT, ST>;
    constexpr uint32_t w = L::w;
    extern __shared__ __align__(16) char s_dyn[];
    uint64_t* s_jr = reinterpret_cast<uint64_t*>(s_dyn);                     // [nj+1] first row of each job
    const uint32_t** s_jM = reinterpret_cast<const uint32_t**>(s_dyn + 8ull * (a.nj + 1));   // [nj] input rows
    uint32_t* s_jperm = reinterpret_cast<uint32_t*>(s_dyn + 16ull * a.nj + 8);   // [nj] perm (nibbles)
    uint8_t* s_jnw = reinterpret_cast<uint8_t*>(s_jperm + a.nj);             // [nj] count only
    char* bufs = s_dyn + L::jobs_bytes(a.nj);
    __shared__ uint64_t s_bar[2];
    __shared__ uint64_t s_rng[2];
    __shared__ uint64_t s_base;
    uint32_t* stage = reinterpret_cast<uint32_t*>(bufs + L::OUT);   // [2][STG] output staging
    uint32_t ob = 0;   // staging buffer of the next chunk with output

    for (uint32_t j = threadIdx.x; j < a.nj; j += blockDim.x) {
        const JoinJob& J = a.jobs[j];
        s_jr[j] = J.row0;
        s_jM[j] = J.M;
        s_jperm[j] = J.perm_packed;
        s_jnw[j] = (uint8_t)(J.nowrite ? 1 : 0);
    }
    if (threadIdx.x == 0) {
        s_jr[a.nj] = a.R;
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        mbar_fence_init();
    }
    const uint64_t P = __ldg(a.poff + a.R);
    uint64_t p0, p1;
    pairs_range(P, blockIdx.x, gridDim.x, p0, p1);
    auto offs = [&](uint64_t i) -> uint64_t { return __ldg(a.poff + i); };
    // the block's rows: [row of p0, row of p1 - 1] (warps 0 and 1 search concurrently)
    if (p0 < p1 && threadIdx.x < 64) {
        const uint64_t r = pairs_find_warp(offs, 0, a.R, threadIdx.x < 32 ? p0 : p1 - 1);
        if (lane_id() == 0) s_rng[threadIdx.x >> 5] = r;
    }
    __syncthreads();
    if (p0 >= p1) return;
    const uint64_t rA = s_rng[0], rEnd = s_rng[1] + 1;

    if (threadIdx.x == 0) issue_window<WOUT>(a, bufs, &s_bar[0], rA, rEnd, s_jr, s_jM, a.nj);
    uint64_t r0 = rA;
    uint32_t phases = 0u;   // bit b: parity of buffer b's next phase
    for (int b = 0; r0 < rEnd; b ^= 1) {
        char* B = bufs + b * L::BUF;
        mbar_wait(&s_bar[b], (phases >> b) & 1u);
        phases ^= 1u << b;
        const BHdr* h = reinterpret_cast<const BHdr*>(B + L::HDR);
        const uint32_t wn = h->wn;
        const uint64_t rnext = r0 + wn;
        // prefetch: the next window's copies go out before this window is worked on (its
        // buffer was released by the barrier that ended the window before this one)
        if (threadIdx.x == 0 && rnext < rEnd) {
            fence_proxy_async_smem();
            issue_window<WOUT>(a, bufs + (b ^ 1) * L::BUF, &s_bar[b ^ 1], rnext, rEnd, s_jr, s_jM, a.nj);
        }
        const uint64_t* wpoff = reinterpret_cast<const uint64_t*>(B + L::POFF + h->sh_poff);
        const uint64_t* wwoff = reinterpret_cast<const uint64_t*>(B + L::WOFF + h->sh_woff);
        const uint32_t* ws0 = reinterpret_cast<const uint32_t*>(B + L::S0 + h->sh_s0);
        const uint32_t* wim = reinterpret_cast<const uint32_t*>(B + L::IM + h->sh_im);
        uint32_t* meta = reinterpret_cast<uint32_t*>(B + L::META);
        // per-row metadata: the output row template (row values in output-column order) and
        // which output columns hold values found in the row's segment
        for (uint32_t i = threadIdx.x; i < wn; i += kBT) {
            uint32_t p = 0;
            while (p + 1 < h->np && h->prow[p + 1] <= i) p++;
            const uint32_t job = h->pjob[p];
            const uint32_t* row = reinterpret_cast<const uint32_t*>(B + L::M + h->poffs[p]) + (i - h->prow[p]) * w;
            const uint32_t perm = s_jperm[job], found = wim[i];
            uint32_t val[w];
#pragma unroll
            for (uint32_t c = 0; c < w; c++) val[c] = row[c];
            uint32_t im = 0;
#pragma unroll
            for (uint32_t oc = 0; oc < WOUT; oc++) {
                uint32_t t = 0xffffffffu, f = 0;
#pragma unroll
                for (uint32_t c = 0; c < w; c++)
                    if (((perm >> (4 * c)) & 15u) == oc) {
                        t = val[c];
                        f = (found >> c) & 1u;
                    }
                meta[i * (WOUT + 1) + oc] = t;
                im |= f << oc;
            }
            const uint32_t hole = s_jnw[job] ? kNoHole : (perm >> (4 * w)) & 15u;
            meta[i * (WOUT + 1) + WOUT] = hole | (im << 8);
        }
        __syncthreads();
        const uint64_t wp0 = wpoff[0] > p0 ? wpoff[0] : p0;
        const uint64_t wp1 = wpoff[wn] < p1 ? wpoff[wn] : p1;
        // the items of the chunk at cp: window row (binary search in the staged offsets for the
        // thread's first pair, a forward walk for the next kBI - 1), segment position, and the
        // candidate value (the one global load, issued here)
        auto items = [&](uint64_t cp, bool (&v)[kBI], uint32_t (&wi)[kBI], uint32_t (&j)[kBI],
                         uint32_t (&cand)[kBI]) {
            const uint64_t q0 = cp + threadIdx.x * kBI;
            uint32_t lo = 0;
            if (q0 < wp1) {
                uint32_t hi = wn;
                while (hi - lo > 1) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (wpoff[mid] <= q0) lo = mid; else hi = mid;
                }
            }
#pragma unroll
            for (int it = 0; it < kBI; it++) {
                const uint64_t q = q0 + it;
                v[it] = q < wp1;
                if (v[it])
                    while (wpoff[lo + 1] <= q) lo++;
                wi[it] = lo;
                j[it] = v[it] ? (uint32_t)(q - wpoff[lo]) : 0u;
                const uint32_t hole = meta[lo * (WOUT + 1) + WOUT] & 0xffu;
                v[it] = v[it] && hole != kNoHole;
                cand[it] = v[it] ? __ldg(a.ec_val + ws0[lo] + j[it]) : 0u;
            }
        };
        bool v[kBI];
        uint32_t wi[kBI], j[kBI], cand[kBI];
        if (wp0 < wp1) items(wp0, v, wi, j, cand);
        for (uint64_t cp = wp0; cp < wp1; cp += kBCh) {
            bool ok[kBI];
            uint32_t mine = 0;
#pragma unroll
            for (int it = 0; it < kBI; it++) {
                const uint32_t* m = meta + wi[it] * (WOUT + 1);
                bool good = v[it];
#pragma unroll
                for (uint32_t c = 0; c < WOUT; c++) good = good && m[c] != cand[it];   // injectivity
                ok[it] = good;
                mine += good ? 1u : 0u;
            }
            // software pipeline: the next chunk's candidate loads go out before this chunk's
            // scan and stores
            bool nv_[kBI];
            uint32_t nwi[kBI], nj_[kBI], ncand[kBI];
            if (cp + kBCh < wp1) items(cp + kBCh, nv_, nwi, nj_, ncand);
            // staging buffer ob was last read by the bulk store of the chunk before the previous one:
            // the issuing thread waits for that read before the scan's barriers release the writers
            if (L::STAGED && threadIdx.x == 0) {
                if (L::NSTG == 2) bulk_wait_read_le1();
                else bulk_wait_read_all();
            }
            uint32_t tot;
            uint32_t lpos = block_excl_scan(mine, &tot);
            auto rotate = [&]() {
#pragma unroll
                for (int it = 0; it < kBI; it++) {
                    v[it] = nv_[it];
                    wi[it] = nwi[it];
                    j[it] = nj_[it];
                    cand[it] = ncand[it];
                }
            };
            if (tot == 0) {   // uniform
                rotate();
                continue;
            }
            if constexpr (!L::STAGED) {
                uint2* s_ri = reinterpret_cast<uint2*>(stage);   // (new value, window row) per output row
                if (mine && lpos == 0) {   // the chunk's first output fixes the chunk's output base
                    uint32_t fc = 0, fw = 0, fj = 0;
#pragma unroll
                    for (int it = kBI - 1; it >= 0; it--)
                        if (ok[it]) {
                            fc = cand[it];
                            fw = wi[it];
                            fj = j[it];
                        }
                    const uint32_t* m = meta + fw * (WOUT + 1);
                    const uint32_t im = m[WOUT] >> 8;
                    uint32_t before = 0;
#pragma unroll
                    for (uint32_t c = 0; c < WOUT; c++) before += ((im >> c) & 1u) && m[c] < fc;
                    s_base = wwoff[fw] + fj - before;
                }
#pragma unroll
                for (int it = 0; it < kBI; it++)
                    if (ok[it]) s_ri[lpos++] = make_uint2(cand[it], wi[it]);
                __syncthreads();
                // word-parallel 16-byte stores of the chunk's consecutive output rows
                uint32_t* g = a.out + s_base * WOUT;
                const uint32_t words = tot * WOUT;
                const uint32_t head = min(words, (uint32_t)((16u - ((uintptr_t)g & 15u)) & 15u) >> 2);
                auto word_at = [&](uint32_t row, uint32_t col) -> uint32_t {
                    const uint2 ri = s_ri[row];
                    const uint32_t* m = meta + ri.y * (WOUT + 1);
                    return col == (m[WOUT] & 0xffu) ? ri.x : m[col];
                };
                if (threadIdx.x < head) g[threadIdx.x] = word_at(threadIdx.x / WOUT, threadIdx.x % WOUT);
                const uint32_t nvec = (words - head) >> 2;
                uint4* g4 = reinterpret_cast<uint4*>(g + head);
                for (uint32_t x = threadIdx.x; x < nvec; x += kBT) {
                    const uint32_t o = head + 4 * x;
                    uint32_t row = o / WOUT, col = o - row * WOUT, wv[4];
                    uint2 ri = s_ri[row];
                    const uint32_t* m = meta + ri.y * (WOUT + 1);
                    uint32_t hole = m[WOUT] & 0xffu;
#pragma unroll
                    for (int k = 0; k < 4; k++) {
                        wv[k] = col == hole ? ri.x : m[col];
                        if (++col == WOUT && k < 3) {
                            col = 0;
                            ri = s_ri[++row];
                            m = meta + ri.y * (WOUT + 1);
                            hole = m[WOUT] & 0xffu;
                        }
                    }
                    g4[x] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
                }
                for (uint32_t o = head + 4 * nvec + threadIdx.x; o < words; o += kBT) g[o] = word_at(o / WOUT, o % WOUT);
                rotate();
                continue;   // s_ri / s_base are rewritten only after the next chunk's scan barriers
            }
            uint32_t* stg = stage + ob * L::STG;
            if (mine) {
                // the global row of this thread's first output fixes the chunk's output base
                uint32_t fc = 0, fw = 0, fj = 0;
#pragma unroll
                for (int it = kBI - 1; it >= 0; it--)
                    if (ok[it]) {
                        fc = cand[it];
                        fw = wi[it];
                        fj = j[it];
                    }
                const uint32_t* m = meta + fw * (WOUT + 1);
                const uint32_t im = m[WOUT] >> 8;
                uint32_t before = 0;
#pragma unroll
                for (uint32_t c = 0; c < WOUT; c++) before += ((im >> c) & 1u) && m[c] < fc;
                const uint64_t base = wwoff[fw] + fj - before - lpos;
                if (lpos == 0) s_base = base;
                const uint32_t shift = (uint32_t)(((uintptr_t)(a.out + base * WOUT) >> 2) & 3u);
                uint32_t* dst = stg + shift + lpos * WOUT;
#pragma unroll
                for (int it = 0; it < kBI; it++) {
                    if (!ok[it]) continue;
                    const uint32_t* mm = meta + wi[it] * (WOUT + 1);
                    const uint32_t hole = mm[WOUT] & 0xffu;
#pragma unroll
                    for (uint32_t c = 0; c < WOUT; c++) dst[c] = c == hole ? cand[it] : mm[c];
                    dst += WOUT;
                }
                fence_proxy_async_smem();   // the staged rows are read by the bulk store (async proxy)
            }
            __syncthreads();
            {
                const uint64_t base = s_base;
                uint32_t* g = a.out + base * WOUT;
                const uint32_t words = tot * WOUT;
                const uint32_t shift = (uint32_t)(((uintptr_t)g >> 2) & 3u);
                const uint32_t head = min(words, (4u - shift) & 3u);         // words before the first 16-byte boundary
                const uint32_t body = ((words - head) >> 2) << 2;            // whole 16-byte vectors
                if (threadIdx.x == 0 && body) {
                    bulk_s2g(g + head, stg + shift + head, body * 4u);
                    bulk_commit();
                }
                const uint32_t rest = words - head - body;                 // tail words after the last vector
                if (threadIdx.x >= 32 && threadIdx.x < 32 + head) g[threadIdx.x - 32] = stg[shift + threadIdx.x - 32];
                if (threadIdx.x >= 64 && threadIdx.x < 64 + rest) {
                    const uint32_t o = head + body + threadIdx.x - 64;
                    g[o] = stg[shift + o];
                }
            }
            if (L::NSTG == 2) ob ^= 1u;
            // s_base is rewritten only after the next chunk's scan barriers
            rotate();
        }
        __syncthreads();   // every thread is done with buffer b: it may be refilled
        r0 = rnext;
    }
    if (threadIdx.x == 0) bulk_wait_all();   // the bulk stores have completed before the block exits
}

template <uint32_t WOUT, bool ST>
static void launch_bulk(gps_ctx* c, const JoinStep& s, uint64_t P) {
    using L = BLay<WOUT, ST>;
    allow_smem((const void*)k_join_bulk<WOUT, ST>, (int)L::bytes(kMaxJobsPerLaunch));
    const uint64_t chunks = (P + kBCh - 1) / kBCh;
    const uint32_t wave = resident_grid(c, (const void*)k_join_bulk<WOUT, ST>, kBT, L::bytes(64));
    const uint32_t G = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)wave, chunks));
    launch(c, GPS_K_JOIN_WRITE, dim3(G), dim3(kBT), L::bytes(s.nj), k_join_bulk<WOUT, ST>, s);
}

template <uint32_t WOUT>
static void launch_bulk_w(gps_ctx* c, const JoinStep& s, uint64_t P) {
    // wide rows: word-parallel stores; GPS_JOIN_WIDE_STAGED=1 stages them in one buffer for bulk
    // stores instead (measured 3 % slower on config 2: the staging costs a resident block)
    const char* e = std::getenv("GPS_JOIN_WIDE_STAGED");
    if (e && *e == '1') launch_bulk<WOUT, true>(c, s, P);
    else launch_bulk<WOUT, false>(c, s, P);
}

bool join_bulk_enabled() { return std::getenv("GPS_JOIN_NO_BULK") == nullptr; }

void run_join_bulk_write(gps_ctx* c, const JoinStep& s, uint64_t P) {
    switch (s.wout) {
        case 2: return launch_bulk<2, true>(c, s, P);
        case 3: return launch_bulk<3, true>(c, s, P);
        case 4: return launch_bulk<4, true>(c, s, P);
        case 5: return launch_bulk_w<5>(c, s, P);
        case 6: return launch_bulk_w<6>(c, s, P);
        case 7: return launch_bulk_w<7>(c, s, P);
        case 8: return launch_bulk_w<8>(c, s, P);
        default: fail(GPS_EINVAL, "internal: bulk join row width out of range");
    }
}

}  // namespace gps
