/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for subgraph matching.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or helper with the CUDA path
 * (paper_1807_08804_b200/), and the CUDA path never loads it.
 *
 * What it computes (PAPER.md §"Subgraph Similarity Search"):
 *   Def. 1  labelled graph G = (V, E, L, l).
 *   Def. 2  a match is an injective f : V_q -> V_g such that for
 *                       every query edge (u,v): (f(u),f(v)) in E_g and labels
 *                       are preserved.  Generalised per DESIGN.md readings
 *                       R1-R9: directed labelled arcs (data = a SET of
 *                       (src,dst,label) triples), query edge labels may be '*',
 *                       vertex labels may be '*', a vertex may be bound to one
 *                       data id ("concept node"), non-induced.
 *   Problem statement (Alg. 1 output P:656): ALL matches.
 *
 * Algorithm (plain backtracking, the family named at P:364-374 / P:503;
 * SURVEY §8(c) "Algorithm"):
 *   1. pi = BFS order of the query's undirected skeleton from vertex 0
 *      (neighbours in increasing id).  Disconnected -> error.
 *   2. rec(i): u = pi[i]; candidates = {bound(u)} if bound, all V if i == 0,
 *      else the distinct out- (or in-) neighbours of f(p) for the already-mapped
 *      query neighbour p whose image has the shortest adjacency list in the
 *      arc's direction (any mapped neighbour gives the same set once every arc
 *      is checked; the shortest list is the fewest tries).
 *      Keep v iff label(u) in {*, l(v)}, v unused, and EVERY query arc between
 *      u and an already-mapped vertex is present in the data with a matching
 *      label.  Recurse; at i == k emit f.
 *   3. The caller (oracle.py) sorts the emitted rows.
 *   4. Timing variant: OpenMP over the subtrees of the
 *      first BFS depth with enough partial maps; the emitted set is unchanged.
 * Test bookkeeping computed alongside (SURVEY §8(d) "Comparison of results"):
 * an order-independent multiset hash of the rows (sum of splitmix64-chained row
 * hashes mod 2^64), the number of partial maps per BFS depth (= #embeddings of
 * the sub-query induced on the BFS prefix: the intermediate-size measure of the
 * config-3/4 query acceptance), and a first-column range restriction (the
 * partitions of the streaming set comparison).
 * Undirected data: every listed edge is inserted in both directions, so a
 * query arc checked as directed is checked as an unordered edge.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_EINVAL (-1)
#define ORC_EDISCONNECTED (-2)
#define ORC_ELIMIT (-3)
#define ORC_ENOMEM (-4)
#define ORC_MAXK 32

typedef struct { uint32_t a, b; int32_t lab; } triple_t;
typedef struct { uint32_t v; int32_t lab; } oarc_t;

typedef struct {
    uint32_t n;
    uint64_t *out_off, *in_off;   /* [n+1] */
    oarc_t *out_arc, *in_arc;     /* sorted by (v, lab), no duplicates */
    int32_t *vlab;                /* [n] */
} og_graph;

static int cmp_triple(const void *x, const void *y) {
    const triple_t *p = (const triple_t *)x, *q = (const triple_t *)y;
    if (p->a != q->a) return p->a < q->a ? -1 : 1;
    if (p->b != q->b) return p->b < q->b ? -1 : 1;
    if (p->lab != q->lab) return p->lab < q->lab ? -1 : 1;
    return 0;
}

/* Build adjacency rows keyed by t.a, from a triple array (sorted + unique). */
static int build_rows(uint32_t n, triple_t *t, uint64_t m, uint64_t **off_out, oarc_t **arc_out) {
    qsort(t, (size_t)m, sizeof(triple_t), cmp_triple);
    uint64_t w = 0;
    for (uint64_t i = 0; i < m; i++) {
        if (w > 0 && cmp_triple(&t[w - 1], &t[i]) == 0) continue;
        t[w++] = t[i];
    }
    uint64_t *off = (uint64_t *)calloc((size_t)n + 1, sizeof(uint64_t));
    oarc_t *arc = (oarc_t *)malloc(sizeof(oarc_t) * (size_t)(w ? w : 1));
    if (!off || !arc) { free(off); free(arc); return ORC_ENOMEM; }
    for (uint64_t i = 0; i < w; i++) {
        off[t[i].a + 1]++;
        arc[i].v = t[i].b;
        arc[i].lab = t[i].lab;
    }
    for (uint32_t v = 0; v < n; v++) off[v + 1] += off[v];
    *off_out = off;
    *arc_out = arc;
    return 0;
}

void oracle_graph_free(og_graph *g) {
    if (!g) return;
    free(g->out_off); free(g->in_off); free(g->out_arc); free(g->in_arc); free(g->vlab);
    free(g);
}

/* src/dst/elab: the raw edge list (elab may be NULL -> all 0); vlab may be NULL
 * (all 0, "contains no node labels").  Returns NULL on bad input. */
og_graph *oracle_graph_build(uint32_t n, uint64_t m, const uint32_t *src, const uint32_t *dst,
                             const uint16_t *elab, const uint16_t *vlab, int undirected) {
    uint64_t mm = undirected ? 2 * m : m;
    triple_t *t = (triple_t *)malloc(sizeof(triple_t) * (size_t)(mm ? mm : 1));
    og_graph *g = (og_graph *)calloc(1, sizeof(og_graph));
    if (!t || !g) { free(t); free(g); return NULL; }
    g->n = n;
    for (uint64_t i = 0; i < m; i++) {
        if (src[i] >= n || dst[i] >= n) { free(t); free(g); return NULL; }
        int32_t l = elab ? (int32_t)elab[i] : 0;
        t[i].a = src[i]; t[i].b = dst[i]; t[i].lab = l;
        if (undirected) { t[m + i].a = dst[i]; t[m + i].b = src[i]; t[m + i].lab = l; }
    }
    if (build_rows(n, t, mm, &g->out_off, &g->out_arc)) { free(t); oracle_graph_free(g); return NULL; }
    /* incoming rows: swap endpoints of the (already unique) out triples */
    uint64_t w = g->out_off[n];
    uint64_t j = 0;
    for (uint32_t a = 0; a < n; a++)
        for (uint64_t e = g->out_off[a]; e < g->out_off[a + 1]; e++) {
            t[j].a = g->out_arc[e].v; t[j].b = a; t[j].lab = g->out_arc[e].lab; j++;
        }
    if (build_rows(n, t, w, &g->in_off, &g->in_arc)) { free(t); oracle_graph_free(g); return NULL; }
    free(t);
    g->vlab = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
    if (!g->vlab) { oracle_graph_free(g); return NULL; }
    for (uint32_t v = 0; v < n; v++) g->vlab[v] = vlab ? (int32_t)vlab[v] : 0;
    return g;
}

uint64_t oracle_graph_arcs(const og_graph *g) { return g->out_off[g->n]; }

/* Is there an arc a -> b whose label is `lab` (or any label when lab < 0)? */
static int has_arc(const og_graph *g, uint32_t a, uint32_t b, int32_t lab) {
    uint64_t lo = g->out_off[a], hi = g->out_off[a + 1];
    while (lo < hi) {               /* first arc with v >= b */
        uint64_t mid = lo + (hi - lo) / 2;
        if (g->out_arc[mid].v < b) lo = mid + 1; else hi = mid;
    }
    for (; lo < g->out_off[a + 1] && g->out_arc[lo].v == b; lo++)
        if (lab < 0 || g->out_arc[lo].lab == lab) return 1;
    return 0;
}

/* Optional bound on search work (candidate tries), for query-acceptance scripts
 * only: when exceeded the search stops with ORC_ELIMIT.  0 = unlimited (default).
 * It never changes a completed result. */
static uint64_t g_work_limit = 0;
void oracle_set_work_limit(uint64_t tries) { g_work_limit = tries; }

typedef struct { uint32_t other; int out; int32_t lab; } chk_t; /* out: arc u->other, else other->u */

/* The query, prepared once (BFS order, per-position checks); read-only while searching. */
typedef struct {
    const og_graph *g;
    uint32_t k;
    uint32_t pi[ORC_MAXK];
    int32_t qlab[ORC_MAXK];
    int64_t qbound[ORC_MAXK];
    int32_t parent[ORC_MAXK];     /* query vertex whose adjacency generates candidates */
    int parent_out[ORC_MAXK];     /* 1: candidates are out-neighbours of f(parent) */
    chk_t chk[ORC_MAXK][2 * 64];
    int nchk[ORC_MAXK];
    uint32_t lo0, hi0;            /* f(pi[0]) restricted to [lo0, hi0) (first-column partition) */
} orc_plan;

/* Shared between the threads of one search. */
typedef struct {
    uint64_t limit, cap;
    uint32_t *rows;
    volatile int over;
    uint64_t slot;                /* next free row of `rows` (atomic) */
    uint64_t emitted;             /* rows emitted by all searchers, in blocks of 1024 (atomic) */
} orc_shared;

/* One searcher (one per thread). */
typedef struct {
    const orc_plan *p;
    orc_shared *sh;
    uint32_t f[ORC_MAXK];         /* f[u] for query vertex u */
    uint8_t *used;                /* [n] */
    uint64_t count, work, hash;
    uint64_t level[ORC_MAXK];     /* level[i] = #valid partial maps of pi[0..i] found by this searcher */
} orc_state;

/* Order-independent multiset hash of the emitted rows (SURVEY §8(d) "Σ splitmix64(row)
 * mod 2^64"): row_hash chains splitmix64 over the row's k values in query-vertex order,
 * the set hash is the sum of the row hashes mod 2^64.  Test bookkeeping only. */
static uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static uint64_t row_hash(const uint32_t *f, uint32_t k) {
    uint64_t h = 0x243F6A8885A308D3ull ^ (uint64_t)k;
    for (uint32_t j = 0; j < k; j++) h = splitmix64(h ^ (uint64_t)f[j]);
    return h;
}

static int try_vertex(orc_state *s, uint32_t i, uint32_t v) {
    const orc_plan *p = s->p;
    uint32_t u = p->pi[i];
    if (g_work_limit && ++s->work > g_work_limit) { s->sh->over = 1; return 0; }
    if (s->used[v]) return 0;
    if (p->qlab[u] >= 0 && p->g->vlab[v] != p->qlab[u]) return 0;
    if (p->qbound[u] >= 0 && (int64_t)v != p->qbound[u]) return 0;
    for (int c = 0; c < p->nchk[i]; c++) {
        const chk_t *ck = &p->chk[i][c];
        uint32_t w = s->f[ck->other];
        if (ck->out ? !has_arc(p->g, v, w, ck->lab) : !has_arc(p->g, w, v, ck->lab)) return 0;
    }
    return 1;
}

static void emit(orc_state *s) {
    const orc_plan *p = s->p;
    orc_shared *sh = s->sh;
    if (sh->rows) {
        uint64_t at = __atomic_fetch_add(&sh->slot, 1, __ATOMIC_RELAXED);
        if (at < sh->cap) memcpy(sh->rows + at * p->k, s->f, sizeof(uint32_t) * p->k);
    }
    s->hash += row_hash(s->f, p->k);
    s->count++;
    /* the limit is on the total over all searchers: each publishes its count in blocks */
    if (sh->limit && (s->count & 1023) == 0) {
        uint64_t tot = __atomic_add_fetch(&sh->emitted, 1024, __ATOMIC_RELAXED);
        if (tot > sh->limit) sh->over = 1;
    }
    if (sh->limit && s->count > sh->limit) sh->over = 1;
}

/* Depth-first search from position i (positions < i mapped); stop_at: a position at which
 * the partial map is handed to `leaf` instead of being extended (frontier collection), or
 * k + 1 for a full search. */
typedef void (*leaf_fn)(orc_state *s, void *user);

static void rec(orc_state *s, uint32_t i, uint32_t stop_at, leaf_fn leaf, void *user);

static void take(orc_state *s, uint32_t i, uint32_t v, uint32_t stop_at, leaf_fn leaf, void *user) {
    const orc_plan *p = s->p;
    uint32_t u = p->pi[i];
    s->f[u] = v;
    s->used[v] = 1;
    s->level[i]++;
    rec(s, i + 1, stop_at, leaf, user);
    s->used[v] = 0;
}

static void rec(orc_state *s, uint32_t i, uint32_t stop_at, leaf_fn leaf, void *user) {
    const orc_plan *p = s->p;
    if (s->sh->over) return;
    if (i == p->k) { emit(s); return; }
    if (i == stop_at) { leaf(s, user); return; }
    uint32_t u = p->pi[i];
    const og_graph *g = p->g;
    if (p->qbound[u] >= 0) {
        uint32_t v = (uint32_t)p->qbound[u];
        if ((i > 0 || (v >= p->lo0 && v < p->hi0)) && try_vertex(s, i, v)) take(s, i, v, stop_at, leaf, user);
        return;
    }
    if (i == 0) {
        for (uint32_t v = p->lo0; v < p->hi0 && !s->sh->over; v++)
            if (try_vertex(s, i, v)) take(s, i, v, stop_at, leaf, user);
        return;
    }
    /* candidates: the distinct neighbours of the mapped query neighbour whose image has
       the shortest adjacency list in the needed direction (every other arc is checked by
       try_vertex, so any mapped neighbour gives the same set; the shortest list is the
       fewest tries -- a hub image would otherwise be scanned for every partial map) */
    uint32_t w = s->f[p->parent[u]];
    int use_out = p->parent_out[u];
    uint64_t best = (use_out ? g->out_off : g->in_off)[w + 1] - (use_out ? g->out_off : g->in_off)[w];
    for (int c = 0; c < p->nchk[i]; c++) {
        const chk_t *ck = &p->chk[i][c];
        uint32_t x = s->f[ck->other];
        int xo = !ck->out;   /* arc other->u: u is an out-neighbour of f(other) */
        uint64_t len = (xo ? g->out_off : g->in_off)[x + 1] - (xo ? g->out_off : g->in_off)[x];
        if (len < best) { best = len; w = x; use_out = xo; }
    }
    const uint64_t *off = use_out ? g->out_off : g->in_off;
    const oarc_t *arc = use_out ? g->out_arc : g->in_arc;
    for (uint64_t e = off[w]; e < off[w + 1] && !s->sh->over; e++) {
        uint32_t v = arc[e].v;
        if (e > off[w] && arc[e - 1].v == v) continue;   /* distinct neighbours only */
        if (try_vertex(s, i, v)) take(s, i, v, stop_at, leaf, user);
    }
}

/* Frontier of partial maps at one depth (parallel variant only). */
typedef struct { uint32_t *f; uint64_t n, cap; uint32_t k; } frontier_t;
static void collect_leaf(orc_state *s, void *user) {
    frontier_t *fr = (frontier_t *)user;
    if (fr->n == fr->cap) {
        uint64_t nc = fr->cap ? 2 * fr->cap : 4096;
        uint32_t *x = (uint32_t *)realloc(fr->f, sizeof(uint32_t) * fr->k * nc);
        if (!x) { s->sh->over = 2; return; }
        fr->f = x;
        fr->cap = nc;
    }
    memcpy(fr->f + fr->n * fr->k, s->f, sizeof(uint32_t) * fr->k);
    fr->n++;
}

/* Prepare the plan (BFS order + per-position checks).  Returns 0 or an ORC_* code. */
static int make_plan(orc_plan *p, const og_graph *g, uint32_t k, const int32_t *qvlab, const int64_t *qbound,
                     uint32_t eq, const int32_t *qsrc, const int32_t *qdst, const int32_t *qlab) {
    if (k == 0 || k > ORC_MAXK || eq > 64) return ORC_EINVAL;
    memset(p, 0, sizeof(*p));
    p->g = g; p->k = k;
    for (uint32_t u = 0; u < k; u++) {
        p->qlab[u] = qvlab ? qvlab[u] : -1;
        p->qbound[u] = qbound ? qbound[u] : -1;
        if (p->qbound[u] >= (int64_t)g->n) return ORC_EINVAL;
    }
    for (uint32_t e = 0; e < eq; e++) {
        if (qsrc[e] < 0 || qdst[e] < 0 || (uint32_t)qsrc[e] >= k || (uint32_t)qdst[e] >= k ||
            qsrc[e] == qdst[e]) return ORC_EINVAL;
    }
    /* 1. BFS order over the undirected skeleton from vertex 0 */
    int pos[ORC_MAXK];
    for (uint32_t u = 0; u < k; u++) pos[u] = -1;
    uint32_t len = 0, head = 0;
    p->pi[len++] = 0; pos[0] = 0;
    while (head < len) {
        uint32_t x = p->pi[head++];
        for (uint32_t y = 0; y < k; y++) {
            if (pos[y] >= 0) continue;
            int adj = 0;
            for (uint32_t e = 0; e < eq; e++)
                if (((uint32_t)qsrc[e] == x && (uint32_t)qdst[e] == y) ||
                    ((uint32_t)qsrc[e] == y && (uint32_t)qdst[e] == x)) adj = 1;
            if (adj) { pos[y] = (int)len; p->pi[len++] = y; }
        }
    }
    if (len != k) return ORC_EDISCONNECTED;
    /* per position: the generating parent and every arc to an earlier vertex */
    for (uint32_t i = 0; i < k; i++) {
        uint32_t u = p->pi[i];
        p->parent[u] = -1;
        p->nchk[i] = 0;
        for (uint32_t e = 0; e < eq; e++) {
            uint32_t a = (uint32_t)qsrc[e], b = (uint32_t)qdst[e];
            uint32_t other;
            int out;
            if (a == u) { other = b; out = 1; } else if (b == u) { other = a; out = 0; } else continue;
            if (pos[other] >= (int)i) continue;
            chk_t *ck = &p->chk[i][p->nchk[i]++];
            ck->other = other; ck->out = out; ck->lab = qlab ? qlab[e] : -1;
            if (p->parent[u] < 0 || pos[other] < pos[p->parent[u]]) {
                p->parent[u] = (int32_t)other;
                p->parent_out[u] = !out;     /* arc other->u: out-neighbours of f(other) */
            }
        }
    }
    p->lo0 = 0;
    p->hi0 = g->n;
    return 0;
}

static int state_init(orc_state *s, const orc_plan *p, orc_shared *sh) {
    memset(s, 0, sizeof(*s));
    s->p = p;
    s->sh = sh;
    s->used = (uint8_t *)calloc(p->g->n ? p->g->n : 1, 1);
    return s->used ? 0 : ORC_ENOMEM;
}

/* Result of oracle_run. */
typedef struct {
    int64_t count;                /* #embeddings (>= 0) or an ORC_* code */
    uint64_t hash;                /* multiset hash of the embeddings (see row_hash) */
    uint64_t level[ORC_MAXK];     /* level[i]: #partial maps of the BFS prefix pi[0..i] the search
                                     visited = #embeddings of the sub-query induced on pi[0..i]
                                     (restricted by the first-column range); level[k-1] = count */
    uint32_t pi[ORC_MAXK];        /* the BFS order */
    uint32_t threads;             /* threads actually used */
} orc_result;

/* The search of SURVEY §8(c): plain backtracking in BFS order.  threads > 1 is the
 * timing variant of §8(c) step 4: the search tree is expanded serially down to the
 * first depth with >= 64 * threads partial maps, and those subtrees are searched in
 * parallel (OpenMP, dynamic schedule); the emitted set is the same.  [lo0, hi0)
 * restricts the image of query vertex 0 (hi0 = 0: no restriction) -- the
 * first-column partitions of SURVEY §8(d)'s streaming comparison.  Rows (query-vertex
 * order, unsorted) go to `rows` up to `cap`. */
void oracle_run(const og_graph *g, uint32_t k, const int32_t *qvlab, const int64_t *qbound,
                uint32_t eq, const int32_t *qsrc, const int32_t *qdst, const int32_t *qlab,
                uint32_t threads, uint32_t lo0, uint32_t hi0, uint32_t *rows, uint64_t cap, uint64_t limit,
                orc_result *res) {
    memset(res, 0, sizeof(*res));
    orc_plan *p = (orc_plan *)calloc(1, sizeof(orc_plan));
    if (!p) { res->count = ORC_ENOMEM; return; }
    int rc = make_plan(p, g, k, qvlab, qbound, eq, qsrc, qdst, qlab);
    if (rc) { free(p); res->count = rc; return; }
    if (hi0) { p->lo0 = lo0; p->hi0 = hi0 < g->n ? hi0 : g->n; }
    memcpy(res->pi, p->pi, sizeof(p->pi));
    orc_shared sh;
    memset(&sh, 0, sizeof(sh));
    sh.rows = rows; sh.cap = rows ? cap : 0; sh.limit = limit;
    orc_state s0;
    if (state_init(&s0, p, &sh)) { free(p); res->count = ORC_ENOMEM; return; }
    if (threads <= 1) {
        rec(&s0, 0, k + 1, NULL, NULL);
        res->count = s0.count; res->hash = s0.hash;
        memcpy(res->level, s0.level, sizeof(s0.level));
        res->threads = 1;
    } else {
        /* expand serially until the frontier is wide enough (or the search is done) */
        frontier_t fr = {NULL, 0, 0, k};
        uint32_t depth = 0;
        for (depth = 1; depth < k; depth++) {
            frontier_t nx = {NULL, 0, 0, k};
            orc_state t;
            if (state_init(&t, p, &sh)) { res->count = ORC_ENOMEM; break; }
            if (depth == 1) {
                rec(&t, 0, 1, collect_leaf, &nx);
            } else {
                for (uint64_t x = 0; x < fr.n && !sh.over; x++) {
                    memcpy(t.f, fr.f + x * k, sizeof(uint32_t) * k);
                    for (uint32_t i = 0; i + 1 < depth; i++) t.used[t.f[p->pi[i]]] = 1;
                    rec(&t, depth - 1, depth, collect_leaf, &nx);
                    for (uint32_t i = 0; i + 1 < depth; i++) t.used[t.f[p->pi[i]]] = 0;
                }
            }
            free(t.used);
            free(fr.f);
            fr = nx;
            if (sh.over || fr.n >= 64ull * threads || fr.n == 0) break;
        }
        if (depth >= k) depth = k - 1;   /* unreachable for k >= 2 (loop breaks first); k == 1 below */
        if (!res->count) {
            uint64_t cnt = 0, hsum = 0, lev[ORC_MAXK];
            memset(lev, 0, sizeof(lev));
            /* frontier positions 0..depth-1 are mapped; their level counts are the frontier's */
            int bad = 0;
            if (k == 1) {
                rec(&s0, 0, k + 1, NULL, NULL);
                cnt = s0.count; hsum = s0.hash; memcpy(lev, s0.level, sizeof(lev));
            } else {
                /* serial prefix levels: recount by re-running the collection is wasteful; the
                   frontier at depth d has exactly level[d-1] members and the shallower levels are
                   counted by a plain serial pass limited to depth-1 */
                orc_state t;
                if (state_init(&t, p, &sh)) bad = 1;
                else {
                    frontier_t dummy = {NULL, 0, 0, k};
                    if (depth > 1) rec(&t, 0, depth - 1, collect_leaf, &dummy);
                    free(dummy.f);
                    for (uint32_t i = 0; i + 1 < depth; i++) lev[i] = t.level[i];
                    free(t.used);
                }
                lev[depth - 1] = fr.n;
#pragma omp parallel num_threads(threads) reduction(+ : cnt, hsum)
                {
                    orc_state ts;
                    uint64_t tl[ORC_MAXK];
                    memset(tl, 0, sizeof(tl));
                    if (state_init(&ts, p, &sh) == 0) {
#pragma omp for schedule(dynamic, 1)
                        for (uint64_t x = 0; x < fr.n; x++) {
                            if (sh.over) continue;
                            memcpy(ts.f, fr.f + x * k, sizeof(uint32_t) * k);
                            for (uint32_t i = 0; i < depth; i++) ts.used[ts.f[p->pi[i]]] = 1;
                            rec(&ts, depth, k + 1, NULL, NULL);
                            for (uint32_t i = 0; i < depth; i++) ts.used[ts.f[p->pi[i]]] = 0;
                        }
                        cnt += ts.count;
                        hsum += ts.hash;
                        for (uint32_t i = depth; i < k; i++) tl[i] = ts.level[i];
                        free(ts.used);
                    } else {
                        sh.over = 2;
                    }
#pragma omp critical
                    for (uint32_t i = depth; i < k; i++) lev[i] += tl[i];
                }
                if (fr.n == 0) { cnt = 0; }
            }
            if (bad || sh.over == 2) res->count = ORC_ENOMEM;
            else {
                res->count = (int64_t)cnt; res->hash = hsum;
                memcpy(res->level, lev, sizeof(lev));
                if (k > 1 && fr.n == 0) for (uint32_t i = depth; i < k; i++) res->level[i] = 0;
            }
        }
        free(fr.f);
        res->threads = threads;
    }
    if (sh.over == 1 && res->count >= 0) res->count = ORC_ELIMIT;
    if (limit && res->count > (int64_t)limit) res->count = ORC_ELIMIT;
    free(s0.used);
    free(p);
}

/* Returns #embeddings (>= 0) or a negative ORC_* code.  Rows (query-vertex
 * order, k u32 each, unsorted) are written to `rows` up to `cap` rows.  With
 * limit > 0 the search stops once the count exceeds `limit` (ORC_ELIMIT). */
int64_t oracle_match(const og_graph *g, uint32_t k, const int32_t *qvlab, const int64_t *qbound,
                     uint32_t eq, const int32_t *qsrc, const int32_t *qdst, const int32_t *qlab,
                     uint32_t *rows, uint64_t cap, uint64_t limit) {
    orc_result r;
    oracle_run(g, k, qvlab, qbound, eq, qsrc, qdst, qlab, 1, 0, 0, rows, cap, limit, &r);
    return r.count;
}
