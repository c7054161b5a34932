// kernels.cuh -- argument blocks and host launchers of the per-query kernels
// (filter.cu, join.cu, scan.cu).  Row numbers refer to SURVEY.md §8(a).
#pragma once
#include "internal.cuh"

namespace gps {

// Decoupled look-back scratch owned by a ctx (lookback.cuh).
struct LbScratch {
    uint64_t* status;        // [kLbSlots * max_tiles]
    unsigned int* ctr;       // [kLbSlots] tickets
    uint32_t max_tiles;      // tiles per slot
};
constexpr int kLbSlots = 3 * GPS_MAX_QE;
LbScratch lb_scratch(gps_ctx* c, uint32_t tiles_needed);
uint32_t lb_next_epoch(gps_ctx* c);

// ---- a2 kernel_check (Def. 3; Alg. 2 line 7 P:723) -------------------
struct QDesc {
    int k;
    int32_t lab[GPS_MAX_QV];     // vertex label or -1
    int64_t bound[GPS_MAX_QV];   // bound data id or -1
    uint32_t qout[GPS_MAX_QV];   // required out-degree
    uint32_t qin[GPS_MAX_QV];    // required in-degree
};
void run_check(gps_ctx* c, const DevGraph& g, const QDesc& q, uint32_t* B);

// ---- a3 kernel_collect ----------------------------------
// For each listed query vertex: c_array (sorted candidate ids), rank prefix rp
// (exclusive popcount per bitmap word, rp[nw] = |C|), |C| in *cnt, and the
// exclusive prefix sums of the candidates' out-/in-degrees (seg_out/seg_in,
// C+1 entries) that index the pair spaces of explore and EC.  Optionally
// zeroes mask[0..C).  One single-pass kernel (decoupled look-back).
struct CollectArgs {
    int nu;
    const uint32_t* B[GPS_MAX_QV];
    uint32_t* rp[GPS_MAX_QV];
    uint32_t* carr[GPS_MAX_QV];
    uint32_t* cnt[GPS_MAX_QV];
    uint32_t* seg_out[GPS_MAX_QV];
    uint32_t* seg_in[GPS_MAX_QV];
    unsigned long long* mask[GPS_MAX_QV];
};
void run_collect(gps_ctx* c, const DevGraph& g, CollectArgs a);

// ---- a4/a5 kernel_explore (Alg. 2 lines 14-22) --------------------
// Constraint of a candidate u' of u for one query arc between u and v:
// adj_dir(u') must hold some v' != u' with a fitting label and v' in B[v].
struct Cons {
    const uint32_t* Bv;   // bitmap of the neighbour v
    uint32_t* X;          // propagation scratch for v
    int32_t lab;          // edge label or -1
    int dir;              // 0: arc u -> v (out-adjacency of u'), 1: arc v -> u (in-adjacency)
};
struct ExploreArgs {
    int no, ni;             // constraints c[0..no) are out-arcs, c[no..no+ni) in-arcs
    Cons c[GPS_MAX_QE];
    const uint32_t* cands;  // c_array[u]
    const uint32_t* cnt;    // device |C(u)|
    const uint32_t* seg_out;
    const uint32_t* seg_in;
    unsigned long long* mask;  // [|C(u)|] satisfied-constraint bits (zeroed by collect)
    uint32_t* Bu;           // bitmap of u (pruned bits cleared)
    int propagate;
};
void run_explore(gps_ctx* c, const DevGraph& g, const ExploreArgs& a);

// B[v] &= X_1 & X_2 & ... (each listed scratch), then the scratch is zeroed.
struct AndArgs {
    int nt;
    uint32_t* B[GPS_MAX_QE];
    int xbeg[GPS_MAX_QE + 1];
    uint32_t* X[GPS_MAX_QE];
};
void run_bitand(gps_ctx* c, const DevGraph& g, const AndArgs& a);

// ---- a6 collect_edge_candidates, two-step -----------------------
struct ECArc {
    const uint32_t* keys;   // c_array of the key endpoint p
    uint32_t nkeys;         // |C(p)|
    int dir;                // 0: values are out-neighbours of the key, 1: in-neighbours
    int32_t lab;
    const uint32_t* Bq;     // bitmap of the value endpoint q
    const uint32_t* seg;    // [nkeys+1] degree prefix of the keys in direction dir
    uint32_t* cnt;          // [nkeys] count pass output (zeroed by the host)
    uint32_t* val;          // [total] write pass output
    uint64_t* blk;          // [G+1] per-block counts -> offsets
    unsigned int* done;     // last-block counter
    uint64_t* info;         // [2]: pairs, total
};
struct ECArgs {
    int na;
    ECArc a[GPS_MAX_QE];
};
void run_ec(gps_ctx* c, const DevGraph& g, const ECArgs& a, bool write, uint32_t G);

// ---- a8 join step: count -> scan -> write ----------------
struct CloseChk {          // fused closing arc p -> q: value(q) must be in EC(p->q)[value(p)]
    int key_new;           // key endpoint is the vertex added by this step
    uint32_t key_col;      // else its column in the input table
    int tgt_new;
    uint32_t tgt_col;
    const uint32_t* Bk;    // bitmap + rank prefix of the key endpoint
    const uint32_t* rpk;
    const uint32_t* off;   // EC offsets / values of the closing arc
    const uint32_t* val;
};
struct StepArgs {
    const uint32_t* M;     // input table, row-major R x w
    uint32_t w;
    uint64_t R;
    uint32_t x_col;        // column of the visited endpoint (EC key)
    const uint32_t* Bx;
    const uint32_t* rpx;
    const uint32_t* ec_off;
    const uint32_t* ec_val;
    int nclose;
    CloseChk cl[GPS_MAX_QE];
    uint32_t* s0;          // [R] segment start of each row in ec_val
    uint64_t* poff;        // [R+1] exclusive scan of segment lengths (pair space)
    uint64_t* blk;         // [G+1] per-block valid counts -> exclusive offsets
    uint64_t* info;        // [0] = #pairs P, [1] = #output rows
    unsigned int* done;    // last-block counter (self-resetting)
    uint32_t* out;         // output table
    uint32_t wout;         // output width (w + 1)
    int final_;            // write in query-vertex order via perm
    uint8_t perm[GPS_MAX_QV + 1];
};
void run_join_seg(gps_ctx* c, const StepArgs& s);      // s0 + poff (one look-back pass)
void run_join_count(gps_ctx* c, const StepArgs& s, uint32_t G);
void run_join_write(gps_ctx* c, const StepArgs& s, uint32_t G);

}  // namespace gps
