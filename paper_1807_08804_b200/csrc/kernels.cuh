// kernels.cuh -- job descriptors and host launchers of the batched per-query
// kernels (filter.cu, join.cu, scan.cu).
//
// Batch-synchronous execution: every phase of Alg. 1 runs as ONE launch over all
// queries of a batch.  Per-job arguments live in device memory (uploaded from a
// pinned arena); outputs of a phase are concatenated across jobs in job order,
// so a single global scan / compaction serves the whole batch.  Row numbers
// refer to SURVEY.md §8(a).
#pragma once
#include "internal.cuh"

namespace gps {

// Decoupled look-back scratch owned by a ctx (lookback.cuh).
struct LbScratch {
    uint64_t* status;        // [nslots * max_tiles]
    unsigned int* ctr;       // [nslots] tickets (self-resetting)
    uint32_t max_tiles;      // tiles per slot
};
LbScratch lb_scratch(gps_ctx* c, uint32_t slots, uint32_t tiles_needed);
uint32_t lb_next_epoch(gps_ctx* c);
// Blocks of `func` (block size `threads`, dynamic smem `smem`) resident at once on the
// whole GPU: the grid of a persistent kernel, so no block waits for a second wave.
uint32_t resident_grid(gps_ctx* c, const void* func, int threads, size_t smem);

constexpr uint32_t kMaxJobsPerLaunch = 2048;   // job prefix staged in shared memory
constexpr uint32_t kJoinStageCols = 8;          // join rows of <= 8 columns are staged in shared memory

// ---- a2 kernel_check (Def. 3; Alg. 2 line 7 P:723) -------------------
struct ChkQV {                   // one query vertex of a check launch (all queries flattened)
    int32_t lab;                 // vertex label or -1
    uint32_t qout, qin;          // required out- / in-degree
    uint32_t pad;
    int64_t bound;               // bound data id or -1
    uint32_t* B;                 // its candidate bitmap (nws words)
};
void run_check(gps_ctx* c, const DevGraph& g, const ChkQV* d_qv, uint32_t nf);

// ---- a3 kernel_collect ----------------------------------
// Per job (query, vertex): c_array (sorted candidate ids), rank prefix rp
// (exclusive popcount per bitmap word, rp[nw] = |C|), |C| in *cnt, and the
// exclusive prefix sums of the candidates' out-/in-degrees (seg_out/seg_in,
// C+1 entries) that index the pair spaces of explore and EC.  One single-pass
// launch (decoupled look-back).
// A job may carry the end-of-step bitmap update of its vertex (a folded "post":
// B &= AND of the X scratch bitmaps xs[x0..x1), which are cleared), applied word
// by word before the compaction -- the update needs no grid-wide barrier of its
// own, so it rides on the collect launch that follows it anyway.  post_only jobs
// apply the update and compact nothing.
struct CollectJob {
    uint32_t* B;
    uint32_t* rp;
    uint32_t* carr;
    uint32_t* cnt;
    uint32_t* seg_out;
    uint32_t* seg_in;
    uint32_t* segtot;       // optional [2]: seg_out[C], seg_in[C] (pair-space sizes for the host)
    uint32_t* const* xs = nullptr;
    uint32_t x0 = 0, x1 = 0;
    uint32_t post_only = 0;
};
void run_collect(gps_ctx* c, const DevGraph& g, const CollectJob* d_jobs, uint32_t nj);

// ---- a4/a5 kernel_explore (Alg. 2 lines 14-22) --------------------
// One constraint of the filter: a member a' of set A survives only if it has an
// arc of direction dir (0: a' -> s', 1: s' -> a') with a fitting label to some
// s' != a' of set S.  Prune (lines 14-18) is (A = u, S = v); propagation (lines
// 19-22, reading R15) is (A = v, S = u).  The job writes X = the members of A
// that satisfy it (k_post then ANDs X into B_A).  Both sides hold a (possibly
// stale, i.e. superset) c_array; rows whose key left the current bitmap are
// skipped.  Per job the kernel walks the cheaper side:
//   A-side: pairs (a' in C(A), arc of adj_dir(a')), test s' in B_S, one X bit per a'
//   S-side: pairs (s' in C(S), arc of adj_{1-dir}(s')), test a' in B_A, set X[a']
// (the same set: a' has a fitting arc to S  <=>  a' is a fitting reverse neighbour of S).
struct ExploreJob {
    const uint32_t* candA;  // c_array of A (nullptr: none yet -> S-side; at least one side has one)
    const uint32_t* cntA;   // device |C(A)|
    const uint32_t* segA;   // degree prefix of C(A) in direction dir
    const uint32_t* candS;  // c_array of S (nullptr: none yet -> A-side)
    const uint32_t* cntS;
    const uint32_t* segS;   // degree prefix of C(S) in direction 1 - dir
    const uint32_t* BA;     // current bitmaps
    const uint32_t* BS;
    uint32_t* X;            // [nws] output bits (zero on entry)
    int32_t lab;            // edge label or -1
    uint32_t dir;
    uint8_t freshA, freshS; // the c_array equals the current bitmap (no membership test per row)
};
// cls: GPS_K_EXPLORE (prune jobs) or GPS_K_PROPAGATE (propagation jobs)
void run_explore(gps_ctx* c, const DevGraph& g, const ExploreJob* d_jobs, uint32_t nj, int cls);

// End of an explore launch, one job per bitmap it filters (word-parallel):
// B &= X[x0] & ... & X[x1-1], then that scratch is zeroed.
struct PostJob {
    uint32_t* B;
    uint32_t x0, x1;
};
void run_post(gps_ctx* c, const DevGraph& g, const PostJob* d_jobs, uint32_t* const* d_xs, uint32_t nj);

// ---- a6 collect_edge_candidates, single pass -------------------
// Job = (query, arc, direction).  The job's pair space is cut into tiles of
// kPT*kPI pairs; tile0 = the job's first tile in the launch-wide numbering (job
// order).  Values of all jobs go to one array in global pair order.
struct ECJob {
    const uint32_t* keys;   // c_array of the key endpoint p
    const uint32_t* nkeys;  // device |C(p)|
    const uint32_t* seg;    // degree prefix of the keys in direction dir
    const uint32_t* Bq;     // bitmap of the value endpoint q
    uint32_t* off;          // [|C(p)|+1] written: position of each key's first value, off[C] = end
    unsigned long long* span;  // [2] written: first / one-past-last value position of the job
    uint64_t P;             // pair-space size (host copy of seg[C])
    uint32_t C;             // host copy of |C(p)|
    uint32_t tile0;
    int32_t lab;
    uint32_t dir;           // 0: values are out-neighbours of the key, 1: in-neighbours
};
// values are written at val[base + launch-wide position]; off / span hold absolute positions
void run_ec(gps_ctx* c, const DevGraph& g, const ECJob* d_jobs, uint32_t nj, uint32_t ntiles, uint32_t* val,
            uint64_t base);
constexpr uint32_t kEcPairTile = 4096;   // pairs per tile of the single-pass EC kernel

struct PassCtl {             // two-step bookkeeping of one pair-space launch
    uint64_t* blk;           // [G+1] per-block counts -> exclusive offsets
    unsigned int* done;      // last-block counter
    uint64_t* info;          // [0] = pairs, [1] = written rows
};

// ---- a8 join step: count -> scan -> write ----------------
struct CloseChk {          // fused closing arc p -> q: value(q) must be in EC(p->q)[value(p)]
    uint32_t key_new;      // key endpoint is the vertex added by this step
    uint32_t key_col;      // else its column in the input table
    uint32_t tgt_new;
    uint32_t tgt_col;
    const uint32_t* Bk;    // bitmap + rank prefix of the key endpoint
    const uint32_t* rpk;
    const uint32_t* off;   // EC key offsets of the closing arc (into the shared value array)
};
struct JoinJob {           // one query's share of a join step
    uint64_t row0;         // first input row of this query (global row numbering of the step)
    const uint32_t* M;     // this query's input rows, row-major R_j x w
    const uint32_t* Bx;    // key endpoint bitmap + rank prefix
    const uint32_t* rpx;
    const uint32_t* ec_off;  // EC key offsets of the extension arc
    const uint32_t* Bn;    // candidate bitmap of the new vertex: every extension segment is a subset of it
    unsigned long long* total;  // per-query output count
    uint32_t x_col;
    uint32_t nclose, close0;
    uint32_t final_;       // last step: write in query-vertex order (perm)
    uint32_t nowrite;      // count only (gps_count's last level)
    uint32_t perm_packed;  // perm (identity unless final_) in nibbles, rows of <= kJoinStageCols columns
    uint8_t perm[GPS_MAX_QV + 1];
};
struct JoinStep {
    uint32_t w, wout;
    uint64_t R;
    const JoinJob* jobs;
    uint32_t nj;
    const CloseChk* cl;
    const uint32_t* ec_val;  // values of every EC table of the batch
    uint32_t* s0;          // [R] segment start of each row in ec_val
    uint64_t* poff;        // [R+1] exclusive scan of segment lengths (pair space)
    PassCtl ctl;
    uint32_t* out;         // output rows of the writing jobs, job order
    uint64_t plo = 0, phi = ~0ull;   // pair sub-range to process; phi == ~0: all pairs
    uint64_t cap = ~0ull;            // single pass: output rows the buffer holds (rows past it are not written)
    uint64_t out_base = 0;           // single pass: output row of the first row this launch produces
    // closing-free steps (every job): validity is injectivity only, so a row's outputs are its
    // segment minus the row's own values.  imask[r] = which of row r's values occur in its
    // segment (binary searches in the seg pass); woff = exclusive scan of written
    // outputs per row (R+1).  The count pass disappears and the write pass places each pair
    // at woff[r] + j - #(row values in the segment before it).
    int fast = 0;
    uint32_t* imask = nullptr;
    uint64_t* woff = nullptr;
};
// Row-sharded join: d_out[i] = first row j in [0, R] with poff[j] >= d_t[i] (row cuts).
void run_lower_bound(gps_ctx* c, const uint64_t* poff, uint64_t R, const uint64_t* d_t, uint32_t n, uint64_t* d_out);
void run_join_seg(gps_ctx* c, const JoinStep& s);      // s0 + poff (+ imask / aoff / woff / jobs[].total if fast)
// fast steps: write pass over all P pairs (rows of count-only jobs are skipped)
void run_join_fast_write(gps_ctx* c, const JoinStep& s, uint64_t P);
// the same write pass with the per-row inputs staged by TMA bulk copies (join_bulk.cu);
// GPS_JOIN_NO_BULK selects k_join_fast instead
bool join_bulk_enabled();
void run_join_bulk_write(gps_ctx* c, const JoinStep& s, uint64_t P);
void run_join_count(gps_ctx* c, const JoinStep& s, uint32_t G);
void run_join_write(gps_ctx* c, const JoinStep& s, uint32_t G);
// Single pass (no count pass): P = pairs of the step's range [plo, phi); out holds cap rows
// (rows of the step past cap are produced but not written); per-job totals via
// jobs[].total, info[0] = P, info[1] = rows produced.  Returns the look-back epoch.
uint32_t run_join_tiles(gps_ctx* c, const JoinStep& s, uint64_t P);
// After a capped run_join_tiles of P pairs: d_out[0] = first tile not fully written,
// d_out[1] = its first output row (the tail is rerun from there).
void run_cap_tile(gps_ctx* c, uint64_t P, uint64_t cap, uint64_t* d_out);
constexpr uint32_t kJoinTilePairs = 1024;   // pairs per single-pass tile (join.cu kTile)

}  // namespace gps
