/*
 * gpsense.h -- C-ABI boundary of the B200-native GpSense subgraph-matching hot path.
 *
 * Problem (PAPER.md §"Subgraph Similarity Search"): "Given a large data
 * graph G and a query graph Q, we find all matches of Q in G"; a match is the
 * injective, edge- and label-preserving map of Def. 2.  The calls
 * below follow Alg. 1 FilteringAndJoining: inputs q and g, output
 * "all matches of q in g", "a set of subgraph isomorphisms".
 * Generalisations (directed labelled arcs, '*' wildcards, bound "concept"
 * vertices P:592, non-induced, injective) are the readings R1-R9 in DESIGN.md.
 *
 * Conventions (all entry points):
 *   - Every function returns gps_status (0 = GPS_OK, < 0 = error) except
 *     gps_last_error / gps_result_free.  On error a thread-local message is
 *     available from gps_last_error(); output arguments are left untouched
 *     unless stated.
 *   - Input arrays are BORROWED for the duration of the call and copied; the
 *     caller keeps ownership.  Pointers are HOST pointers unless a flag says
 *     otherwise.
 *   - A gps_ctx is bound to one CUDA device and one stream; it is not
 *     thread-safe.  A gps_graph is immutable after load and may be used by any
 *     ctx on the same device.
 *   - There is NO CPU fallback: every step of filtering and joining runs in the
 *     library's sm_100a kernels; the only host work is validation, the query
 *     plan ("the only step that runs on the CPU") and the join-order
 *     choice.  Without a usable CUDA device gps_create fails with
 *     GPS_ECUDA.
 */
#ifndef GPSENSE_H
#define GPSENSE_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define GPS_API __attribute__((visibility("default")))
#else
#define GPS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    GPS_OK = 0,
    GPS_EINVAL = -1,         /* malformed argument (see each call) */
    GPS_EDISCONNECTED = -2,  /* query skeleton not connected */
    GPS_ENOMEM = -3,         /* device or host allocation failed */
    GPS_ECUDA = -4,          /* CUDA runtime / launch failure */
    GPS_ENCCL = -5,          /* reserved: collective failure */
    GPS_EOVERFLOW = -6,      /* result does not fit the caller's buffer / 32-bit tables */
    GPS_EUNSUPPORTED = -7    /* graph beyond the packed-arc layout (n << b >= 2^32, m >= 2^32) */
} gps_status;

#define GPS_ANY (-1)         /* wildcard vertex / edge label ('*'; variable edge P:594) */
#define GPS_FREE (-1)        /* unbound query vertex (variable node P:592) */
#define GPS_MAX_QV 32        /* max query vertices */
#define GPS_MAX_QE 64        /* max query arcs */
#define GPS_REFINE_UNTIL_STABLE 0xFFFFFFFFu   /* gps_match_opts.refine_rounds: refine to the fixpoint */
#define GPS_PLAN_RANKING 0                    /* gps_match_opts.plan_mode */
#define GPS_PLAN_COMMONSENSE 1

/* gps_csr_desc.flags */
#define GPS_DIRECTED 0u
#define GPS_UNDIRECTED 1u    /* each listed arc is an unordered edge: the library symmetrises it */

typedef struct gps_ctx gps_ctx;
typedef struct gps_graph gps_graph;
typedef struct gps_result gps_result;

typedef struct {
    int device;              /* CUDA ordinal */
    void* stream;            /* cudaStream_t to run on (e.g. torch.cuda.current_stream().cuda_stream);
                                NULL = the library creates its own non-blocking stream */
    void* nccl_comm;         /* ncclComm_t (e.g. torch ProcessGroupNCCL._comm_ptr()) for the row-sharded
                                join; NULL = single GPU.  world = 1 with a communicator
                                runs the sharded path (and its collectives) on one rank */
    int rank, world;         /* this process's rank and the number of ranks of nccl_comm */
    /* Optional caller allocator for the library's stream-ordered device memory (scratch, join
     * tables, results), e.g. torch's caching allocator: dev_alloc(bytes, stream,
     * user) returns a 16-byte-aligned device pointer usable in stream order on `stream` (NULL =
     * out of memory -> GPS_ENOMEM); dev_free(ptr, stream, user) returns it, in stream order
     * after the work enqueued on `stream` so far.  Both NULL = the library's private memory
     * pool.  Called from the calling thread and from batch worker threads (with the worker's
     * stream), possibly concurrently.  The graph arrays themselves are plain cudaMalloc. */
    void* (*dev_alloc)(size_t bytes, void* stream, void* user);
    void (*dev_free)(void* ptr, void* stream, void* user);
    void* alloc_user;
} gps_ctx_opts;

/* Data graph as CSR ("nodes array ... edges array ... two additional
 * arrays ... labels of nodes and edges").  Rows need not be sorted; duplicate
 * (src, dst, label) arcs are collapsed (set semantics, reading R5).
 *   offsets        [n_vertices+1] u64, offsets[0] = 0, non-decreasing, offsets[n] = n_arcs
 *   targets        [n_arcs] u32 < n_vertices
 *   edge_labels    [n_arcs] u16 or NULL (all 0)
 *   vertex_labels  [n_vertices] u16 or NULL (all 0; commonsense graphs "contain no node labels")
 * Errors: GPS_EINVAL (bad offsets / target >= n / n = 0), GPS_EUNSUPPORTED
 * ((n-1) << b >= 2^32 with b = bits of the largest edge label, or >= 2^32 stored arcs). */
typedef struct {
    uint32_t n_vertices;
    uint64_t n_arcs;
    const uint64_t* offsets;
    const uint32_t* targets;
    const uint16_t* edge_labels;
    const uint16_t* vertex_labels;
    uint32_t flags;
} gps_csr_desc;

/* One query arc src -> dst with an edge label or GPS_ANY.  No self-loops. */
typedef struct { int32_t src, dst, label; } gps_qedge;

/* Query graph (P:580-594 concept / variable nodes, labelled / variable edges).
 *   vertex_labels [n_vertices] label or GPS_ANY (NULL = all GPS_ANY)
 *   bound         [n_vertices] data id or GPS_FREE (NULL = all free)
 *   edges         [n_edges]
 * Errors: GPS_EINVAL (k = 0, k > 32, e > 64, endpoint >= k, self-loop,
 * bound id >= n), GPS_EDISCONNECTED (k > 1 and skeleton not connected). */
typedef struct {
    uint32_t n_vertices, n_edges;
    const int32_t* vertex_labels;
    const int64_t* bound;
    const gps_qedge* edges;
} gps_query;

/* Knobs of the method (NULL = defaults from gps_default_opts). */
typedef struct {
    uint32_t refine_rounds;      /* refinement rounds after initialisation; default 1;
                                    GPS_REFINE_UNTIL_STABLE = rounds until no candidate set shrinks
                                    ("the refinement function until convergence") */
    int32_t reverse_refine;      /* refine in reversed visit order; default 1 */
    uint32_t lowconn_threshold;  /* query degree <= this is "low connectivity"; default 1 */
    int32_t result_on_device;    /* gps_match: 1 = rows stay in device memory (default), 0 = host copy */
    float rebalance_threshold;   /* row-sharded join: exchange rows when max/mean pairs per rank exceeds
                                    this (default 1.10; 0 = always, very large = never) */
    int32_t plan_mode;           /* visit order O: GPS_PLAN_RANKING (default, f(u) = deg/freq) or
                                    GPS_PLAN_COMMONSENSE (concept node of max degree first, then the
                                    neighbour with the most unordered neighbours) */
    uint64_t row_budget_bytes;   /* largest partial-embedding table (bytes) a join step may materialise
                                    at once (reading R27, "intermediate results ... a key
                                    challenge"): a step whose output exceeds it is split into pair
                                    ranges and each piece runs the remaining steps depth-first (the
                                    result set does not depend on it).  0 (default) = a quarter of the
                                    device memory; a table that cannot be allocated below the budget
                                    also goes depth-first.  gps_count never
                                    materialises its last level, so it never fails for lack of
                                    memory on the tables; gps_match returns GPS_ENOMEM only when the
                                    final rows themselves cannot be allocated. */
} gps_match_opts;

GPS_API gps_status gps_default_opts(gps_match_opts* opts);

/* Creates a ctx on opts->device.  The library allocates stream-ordered from a private memory
 * pool per device that keeps up to 3/4 of the device memory cached after frees
 * (GPS_POOL_KEEP_BYTES overrides).  GPS_POOL_RESERVE_BYTES (environment, read when the first
 * ctx of a device is created) maps that many bytes into the pool up front -- workloads with
 * multi-GB join tables then sub-allocate instead of growing the pool mid-query. */
GPS_API gps_status gps_create(const gps_ctx_opts* opts, gps_ctx** out);
/* Frees the ctx and the device memory of any gps_result it still owns. */
GPS_API gps_status gps_destroy(gps_ctx* ctx);

/* a0: copies the CSR to the device, sorts + de-duplicates
 * every row, builds the incoming CSR ("both incoming and outgoing graph
 * representations") and the vertex-label histogram freq(label). */
GPS_API gps_status gps_load_data_graph(gps_ctx* ctx, const gps_csr_desc* desc, gps_graph** out);
GPS_API gps_status gps_free_graph(gps_graph* g);
/* n, stored arcs (after de-duplication / symmetrisation), #vertex labels, edge-label bits. */
GPS_API gps_status gps_graph_info(const gps_graph* g, uint32_t* n, uint64_t* arcs, uint32_t* n_vlabels,
                          uint32_t* elabel_bits);

/* Alg. 1 end to end: plan (host) -> filter (check, collect, explore, refine)
 * -> collect edge candidates -> combine.  *out receives all embeddings as
 * row-major uint32 rows x k, column j = image of query vertex j, rows in an
 * unspecified but deterministic order (reading R25).  Empty result is GPS_OK
 * with rows = 0. */
GPS_API gps_status gps_match(gps_ctx* ctx, const gps_graph* g, const gps_query* q,
                     const gps_match_opts* opts, gps_result** out);
/* Same, writing rows into a caller-owned HOST buffer of cap_rows x k uint32
 * (pinned memory recommended).  *rows = #embeddings; GPS_EOVERFLOW (with *rows
 * set) if it exceeds cap_rows (nothing written then). */
GPS_API gps_status gps_match_host(gps_ctx* ctx, const gps_graph* g, const gps_query* q,
                          const gps_match_opts* opts, uint32_t* host_out, uint64_t cap_rows,
                          uint64_t* rows);
/* #embeddings; the last join level is counted, never written. */
GPS_API gps_status gps_count(gps_ctx* ctx, const gps_graph* g, const gps_query* q,
                     const gps_match_opts* opts, uint64_t* count);

/* Batched execution of nq independent queries (the QA-batch use, BASELINE
 * configs[4]): the library runs them concurrently on a pool of worker host
 * threads, each owning a CUDA stream and scratch (set its size with
 * gps_set_workers; default 2); a batch that fits one slice (gps_set_slice) runs on the
 * ctx's own stream instead.  results[i] / counts[i] / statuses[i] (statuses
 * may be NULL) as for the single-query calls: every entry of statuses is written,
 * a query that failed has results[i] = NULL.  A query whose candidate-edge tables
 * alone exceed the 32-bit table limits fails with GPS_EOVERFLOW without affecting
 * the others.  Results are owned by the caller (gps_result_free) and by the ctx
 * (its stream orders their release).  The ctx stream is ordered before / after the
 * batch.  Returns the first failing status (GPS_OK if all succeeded). */
GPS_API gps_status gps_match_batch(gps_ctx* ctx, const gps_graph* g, const gps_query* queries, uint32_t nq,
                                   const gps_match_opts* opts, gps_result** results, gps_status* statuses);
GPS_API gps_status gps_count_batch(gps_ctx* ctx, const gps_graph* g, const gps_query* queries, uint32_t nq,
                                   const gps_match_opts* opts, uint64_t* counts, gps_status* statuses);
/* Batched execution with every result copied into ONE caller-owned host buffer
 * (pinned memory recommended) of cap_words uint32: query i's rows (row-major,
 * rows[i] x k_i) start at word offset offsets[i] (the order of the segments in
 * the buffer is unspecified).  GPS_EOVERFLOW if the results do not fit (rows[]
 * are still filled). */
GPS_API gps_status gps_match_batch_host(gps_ctx* ctx, const gps_graph* g, const gps_query* queries, uint32_t nq,
                                        const gps_match_opts* opts, uint32_t* host_out, uint64_t cap_words,
                                        uint64_t* offsets, uint64_t* rows, gps_status* statuses);
/* Number of batch workers (1..64; 0 = default 2).  Destroys existing workers (and their results). */
GPS_API gps_status gps_set_workers(gps_ctx* ctx, uint32_t n);
/* Queries per worker hand-out in the batch calls (each hand-out runs batch-synchronously:
 * one launch per phase for all its queries); 0 = default 64. */
GPS_API gps_status gps_set_slice(gps_ctx* ctx, uint32_t queries);

/* ---- multi-GPU (row-sharded join, SPMD) ------------------------------------
 * With a ctx of world > 1 every rank calls gps_match / gps_count with the same
 * graph and query (batches run one query at a time).  Filtering and edge
 * candidates are computed on every rank (replicated); the join's pair space is
 * split across ranks, the per-step counts are all-gathered and partial
 * embeddings are exchanged when the load is unbalanced.  gps_count returns the
 * GLOBAL count on every rank; gps_match returns this rank's shard (shards in rank
 * order = the global result); gps_result_global_rows gives the global size. */
GPS_API gps_status gps_result_global_rows(const gps_result* r, uint64_t* global_rows);

/* Host arithmetic of the row-sharded join (no device work; identical on every rank,
 * exposed so multi-process tests can check it without GPUs).  Rank order is the
 * global row order; rank t's global share of a step's P pairs is
 * [t*P/world, (t+1)*P/world) (remainder to the first ranks).
 *   gps_shard_plan: pairs_all[world] = every rank's local pairs (all-gathered);
 *     local_targets[world+1] = where rank t's share starts in THIS rank's local pair
 *     space, clamped to [0, pairs_all[rank] + 1]: local row i goes to the rank t with
 *     local_targets[t] <= poff[i] < local_targets[t+1] (poff = the rows' exclusive
 *     pair offsets; the last rank also takes rows at the very end); *rebalance = 1 when
 *     max/mean > threshold; *total = global pairs.
 *   gps_shard_recv: send_matrix[src*world + dst] = rows src sends to dst
 *     (all-gathered); at[world] = row offset of src's block in this rank's receive
 *     buffer (blocks in source-rank order); *total = rows received.
 * Errors: GPS_EINVAL (world < 1, rank outside [0, world), NULL input). */
GPS_API gps_status gps_shard_plan(int world, int rank, const uint64_t* pairs_all, float threshold,
                                  uint64_t* local_targets, int* rebalance, uint64_t* total);
GPS_API gps_status gps_shard_recv(int world, int rank, const uint64_t* send_matrix, uint64_t* at, uint64_t* total);

/* In-process ranks on one device (threads sharing a hub): the same sharded path
 * with device-to-device copies instead of NCCL -- used to test sharding and
 * rebalancing with several ranks on one GPU. */
typedef struct gps_local_comm gps_local_comm;
GPS_API gps_status gps_local_comm_create(int world, gps_local_comm** out);
GPS_API gps_status gps_local_comm_destroy(gps_local_comm* comm);
GPS_API gps_status gps_create_local_rank(const gps_ctx_opts* opts, gps_local_comm* comm, int rank, gps_ctx** out);

/* ---- f2: commonsense query semantics -----------------------
 * gps_load_triples: a knowledge base given as (subject, relation, object) triples is the
 *   labelled data graph directly ("direct transformation": concepts -> vertices,
 *   relations -> labelled arcs subject -> object).  subject/object [n_triples] < n_vertices,
 *   relation [n_triples] (NULL = all 0), vertex_labels as for gps_csr_desc (NULL = all 0,
 *   P:528).  flags as gps_csr_desc.flags.  Same errors as gps_load_data_graph.
 * gps_match_project: the matches of the PROJECTION ("a subset of variable
 *   nodes, termed projection"): the set of distinct tuples (f(project[0]), ...,
 *   f(project[n_project-1])) over all embeddings f, in lexicographic order; rows x n_project
 *   in the result.  GPS_EINVAL if n_project is 0 or > 32 or a vertex is out of range;
 *   GPS_EUNSUPPORTED with a row-sharded ctx or more than 2^32 embeddings.
 * gps_count_project: the number of such tuples. */
GPS_API gps_status gps_load_triples(gps_ctx* ctx, uint32_t n_vertices, uint64_t n_triples, const uint32_t* subject,
                                    const uint16_t* relation, const uint32_t* object, const uint16_t* vertex_labels,
                                    uint32_t flags, gps_graph** out);
GPS_API gps_status gps_match_project(gps_ctx* ctx, const gps_graph* g, const gps_query* q, const gps_match_opts* opts,
                                     uint32_t n_project, const int32_t* project, gps_result** out);
GPS_API gps_status gps_count_project(gps_ctx* ctx, const gps_graph* g, const gps_query* q, const gps_match_opts* opts,
                                     uint32_t n_project, const int32_t* project, uint64_t* count);
/* gps_match_named: NAMED variable edges ("query edges are also categorized into variable
 *   and labeled edges", "2 variable edges: ?x, ?y"; "each variable-edge name as a
 *   binding reported in output, with equal names constrained equal"; DESIGN reading R32).
 *   edge_var [q->n_edges] (host): a name id >= 0 for a variable edge (its label must be
 *   GPS_ANY), -1 for an edge without a name.  Let v_0 < v_1 < ... < v_{V-1} be the distinct
 *   ids.  The result is the set of distinct tuples (f(project[0]), ..., f(project[n_project-1]),
 *   beta(v_0), ..., beta(v_{V-1})) over every embedding f (Def. 2) and every assignment beta of
 *   edge labels to the names such that each edge e = (a, b) named v has an arc f(a) -> f(b)
 *   labelled beta(v); lexicographic order, (n_project or k) + V columns (n_project = 0 and
 *   project = NULL: all k query vertices).  Computed on the device by instantiating the query
 *   for every assignment of the labels present in g (one batch) and deduplicating.
 *   Errors: GPS_EINVAL (named edge with a label, projected vertex out of range, more than 32
 *   columns), GPS_EUNSUPPORTED (V > 8, more than 65536 assignments, row-sharded ctx, more than
 *   2^32 rows before deduplication), plus gps_match's.
 * gps_count_named: the number of such tuples. */
GPS_API gps_status gps_match_named(gps_ctx* ctx, const gps_graph* g, const gps_query* q, const gps_match_opts* opts,
                                   const int32_t* edge_var, uint32_t n_project, const int32_t* project,
                                   gps_result** out);
GPS_API gps_status gps_count_named(gps_ctx* ctx, const gps_graph* g, const gps_query* q, const gps_match_opts* opts,
                                   const int32_t* edge_var, uint32_t n_project, const int32_t* project,
                                   uint64_t* count);

/* ---- f3: multi-level graph compression ------------
 * gps_compress: levels 1..n_levels of the compression of g ("a sequence of smaller
 *   graphs G_i ... similar nodes are combined to form a weighted node"; DESIGN readings
 *   R33-R36): level i pairs SIMILAR nodes of level i-1 (same vertex label, identical set of
 *   (direction, edge label, neighbour node) edge ends: R33 at delta = 1), greedily in id
 *   order (R34); node ids of a level follow their smallest member.  Weights (P:846-850,
 *   R35): w_out(U) = max over members x of the arcs x -> M(U) (w_in likewise), edge weights
 *   start at #labelled arcs x -> y and combine as w(U, V) = sum over the parts V' of V of the
 *   max over the parts U' of U of w(U', V').  deltas [n_levels] (host) must each be 1.0 on the
 *   device: GPS_EUNSUPPORTED for delta < 1 (a similarity join, not built), GPS_EINVAL outside
 *   (0, 1] or n_levels outside 1..16; GPS_EUNSUPPORTED when keys need more than 64 bits.
 *   The compression owns device memory until gps_free_compressed (which also detaches it from
 *   g if attached); g must outlive it.
 * gps_compressed_info: nodes and weighted out-/in-edges of level (1..n_levels).
 * gps_compressed_fetch: copies level `level` to HOST arrays (each may be NULL):
 *   group [n] (node of every data vertex: M(U) = {x : group[x] = U}), label / w_out / w_in
 *   [nodes], edge_out [edges_out] (U << 32 | V, ascending) with weight_out, edge_in likewise
 *   (U << 32 | V = in-weight of U from V).
 * gps_compressed_candidates: the weighted candidate test of P:905 (R36: label, bound id in
 *   M(X), distinct query out-/in-degree <= w(X) + sum over Z != X of w(X, Z)) through every
 *   data vertex's node: bitmaps_out (host) k x ceil(n/32) words, bit v of row u = v lies in
 *   the mapping list of a weighted candidate of u (a superset of Def. 3's candidates,
 *   Theorem 1).
 * gps_graph_attach_compressed: subsequent filters on g also apply that test at `level`
 *   (cg = NULL or level 0 detaches); results are unchanged (Theorem 1).  GPS_EINVAL when cg
 *   was built from another graph or level is out of range. */
typedef struct gps_compressed gps_compressed;
GPS_API gps_status gps_compress(gps_ctx* ctx, const gps_graph* g, uint32_t n_levels, const float* deltas,
                                gps_compressed** out);
GPS_API gps_status gps_free_compressed(gps_compressed* cg);
GPS_API gps_status gps_compressed_info(const gps_compressed* cg, uint32_t level, uint32_t* n_nodes,
                                       uint64_t* n_edges_out, uint64_t* n_edges_in);
GPS_API gps_status gps_compressed_fetch(gps_ctx* ctx, const gps_compressed* cg, uint32_t level, uint32_t* group,
                                        uint32_t* label, uint32_t* w_out, uint32_t* w_in, uint64_t* edge_out,
                                        uint32_t* weight_out, uint64_t* edge_in, uint32_t* weight_in);
GPS_API gps_status gps_compressed_candidates(gps_ctx* ctx, const gps_compressed* cg, uint32_t level,
                                             const gps_query* q, uint32_t* bitmaps_out);
GPS_API gps_status gps_graph_attach_compressed(gps_graph* g, const gps_compressed* cg, uint32_t level);

/* ---- f4: gSparql primitives on binary relations --------
 * A relation is a set of (a, b) pairs of u32 terms -- a property table's (subject, object)
 * pairs.  Inputs are HOST column arrays of n pairs (duplicates allowed, any order;
 * NULL columns only with n = 0).  Every result is a DEVICE gps_result of rows x 2 u32
 * (a, b), lexicographically sorted and distinct (sort-based dedup); free with
 * gps_result_free.
 * gps_rel_join: subject/object join rule (sort-merge join): {(x, z) : (x, y) in
 *   R, (y, z) in S}.  GPS_EUNSUPPORTED past 2^32 joined pairs.
 * gps_rel_union / gps_rel_difference: A u B (the merge of a pattern node's rule results,
 *   P:1232) and A \ B.
 * gps_rel_closure: the recursive-rule loop of Algorithm P:1247-1262 (DESIGN R37) for the
 *   transitive rule (x p y), (y p z) -> (x p z): NewT := T; while NewT: InferT := join(NewT, T)
 *   u join(T, NewT); NewT := InferT \ T; T := T u NewT.  *rounds (may be NULL) = loop rounds;
 *   max_rounds > 0 bounds them (GPS_EOVERFLOW past it), 0 = unbounded. */
GPS_API gps_status gps_rel_join(gps_ctx* ctx, const uint32_t* r_src, const uint32_t* r_dst, uint64_t nr,
                                const uint32_t* s_src, const uint32_t* s_dst, uint64_t ns, gps_result** out);
GPS_API gps_status gps_rel_union(gps_ctx* ctx, const uint32_t* a_src, const uint32_t* a_dst, uint64_t na,
                                 const uint32_t* b_src, const uint32_t* b_dst, uint64_t nb, gps_result** out);
GPS_API gps_status gps_rel_difference(gps_ctx* ctx, const uint32_t* a_src, const uint32_t* a_dst, uint64_t na,
                                      const uint32_t* b_src, const uint32_t* b_dst, uint64_t nb, gps_result** out);
GPS_API gps_status gps_rel_closure(gps_ctx* ctx, const uint32_t* src, const uint32_t* dst, uint64_t n,
                                   uint32_t max_rounds, gps_result** out, uint32_t* rounds);

/* rows, cols (= k), data (device or host pointer, owned by the result), on_device. */
GPS_API gps_status gps_result_info(const gps_result* r, uint64_t* rows, uint32_t* cols,
                           const uint32_t** data, int* on_device);
GPS_API void gps_result_free(gps_result* r);
/* Like gps_result_free, but the device memory is released only after the work
 * enqueued so far on `stream` (a cudaStream_t, e.g. the torch stream that read the
 * rows) has completed: the ctx stream waits on an event recorded on `stream`.
 * NULL stream = gps_result_free. */
GPS_API void gps_result_free_after(gps_result* r, void* stream);

GPS_API const char* gps_last_error(void);

/* ---- introspection (tests, bench) ------------------------------------- */

/* Kernel classes for stats / profiling. */
enum {
    GPS_K_CHECK = 0, GPS_K_COLLECT, GPS_K_EXPLORE, GPS_K_BITAND, GPS_K_EC_COUNT, GPS_K_EC_WRITE,
    GPS_K_SCAN, GPS_K_JOIN_LEN, GPS_K_JOIN_COUNT, GPS_K_JOIN_WRITE, GPS_K_LOAD, GPS_K_PROPAGATE, GPS_K_CLEAR,
    GPS_K_NCLASSES
};

typedef struct {
    uint64_t queries;                      /* gps_match / gps_count calls completed */
    uint64_t embeddings;                   /* rows produced / counted */
    uint64_t launches;                     /* kernels launched by this ctx */
    uint64_t host_syncs;                   /* stream synchronisations */
    uint64_t k_launches[GPS_K_NCLASSES];   /* per kernel class */
    double k_bytes[GPS_K_NCLASSES];        /* algorithmic bytes */
    double k_ms[GPS_K_NCLASSES];           /* CUDA-event time, only for profiled classes */
    uint64_t k_timed[GPS_K_NCLASSES];      /* launches that were event-timed */
    uint64_t join_rows_max;                /* largest partial-embedding table (rows, one query) */
    uint64_t join_rows_total;              /* rows of every partial-embedding table materialised */
} gps_stats;

GPS_API gps_status gps_get_stats(gps_ctx* ctx, gps_stats* out);   /* synchronises the ctx stream */
GPS_API gps_status gps_reset_stats(gps_ctx* ctx);
/* Event-time every launch of the classes in class_mask (bit i = class i) on the ctx stream. */
GPS_API gps_status gps_set_profiling(gps_ctx* ctx, uint32_t class_mask);

/* Query plan: visit order O (order_out[k], *n_order entries),
 * ranking f(u) = deg(u) / freq(u.label) as unreduced (deg, freq) pairs
 * (rank_out[2k]). */
GPS_API gps_status gps_debug_plan(gps_ctx* ctx, const gps_graph* g, const gps_query* q,
                          const gps_match_opts* opts, int32_t* order_out, uint32_t* n_order,
                          uint64_t* rank_out);
/* Candidate bitmaps c_set (Alg. 2) after stage 0 = kernel_check, 1 = initialisation
 * (explore over T), 2 = refinement.  bitmaps_out: k x ceil(n/32) uint32 host
 * words, bit v of row u = "v is a candidate of u". */
GPS_API gps_status gps_debug_candidates(gps_ctx* ctx, const gps_graph* g, const gps_query* q,
                                const gps_match_opts* opts, int stage, uint32_t* bitmaps_out);

#ifdef __cplusplus
}
#endif
#endif /* GPSENSE_H */
