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
 *      else the distinct out- (or in-) neighbours of f(p) for the earliest
 *      already-mapped query neighbour p (following the arc's direction).
 *      Keep v iff label(u) in {*, l(v)}, v unused, and EVERY query arc between
 *      u and an already-mapped vertex is present in the data with a matching
 *      label.  Recurse; at i == k emit f.
 *   3. The caller (oracle.py) sorts the emitted rows.
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
    uint32_t f[ORC_MAXK];         /* f[u] for query vertex u */
    uint8_t *used;                /* [n] */
    uint64_t count, limit, cap, work;
    uint32_t *rows;
    int over;
} orc_state;

static int try_vertex(orc_state *s, uint32_t i, uint32_t v) {
    uint32_t u = s->pi[i];
    if (g_work_limit && ++s->work > g_work_limit) { s->over = 1; return 0; }
    if (s->used[v]) return 0;
    if (s->qlab[u] >= 0 && s->g->vlab[v] != s->qlab[u]) return 0;
    if (s->qbound[u] >= 0 && (int64_t)v != s->qbound[u]) return 0;
    for (int c = 0; c < s->nchk[i]; c++) {
        const chk_t *ck = &s->chk[i][c];
        uint32_t w = s->f[ck->other];
        if (ck->out ? !has_arc(s->g, v, w, ck->lab) : !has_arc(s->g, w, v, ck->lab)) return 0;
    }
    return 1;
}

static void rec(orc_state *s, uint32_t i) {
    if (s->over) return;
    if (i == s->k) {
        if (s->rows && s->count < s->cap)
            memcpy(s->rows + s->count * s->k, s->f, sizeof(uint32_t) * s->k);
        s->count++;
        if (s->limit && s->count > s->limit) s->over = 1;
        return;
    }
    uint32_t u = s->pi[i];
    const og_graph *g = s->g;
    if (s->qbound[u] >= 0) {
        uint32_t v = (uint32_t)s->qbound[u];
        if (try_vertex(s, i, v)) { s->f[u] = v; s->used[v] = 1; rec(s, i + 1); s->used[v] = 0; }
        return;
    }
    if (i == 0) {
        for (uint32_t v = 0; v < g->n && !s->over; v++)
            if (try_vertex(s, i, v)) { s->f[u] = v; s->used[v] = 1; rec(s, i + 1); s->used[v] = 0; }
        return;
    }
    uint32_t w = s->f[s->parent[u]];
    const uint64_t *off = s->parent_out[u] ? g->out_off : g->in_off;
    const oarc_t *arc = s->parent_out[u] ? g->out_arc : g->in_arc;
    for (uint64_t e = off[w]; e < off[w + 1] && !s->over; e++) {
        uint32_t v = arc[e].v;
        if (e > off[w] && arc[e - 1].v == v) continue;   /* distinct neighbours only */
        if (try_vertex(s, i, v)) { s->f[u] = v; s->used[v] = 1; rec(s, i + 1); s->used[v] = 0; }
    }
}

/* Returns #embeddings (>= 0) or a negative ORC_* code.  Rows (query-vertex
 * order, k u32 each, unsorted) are written to `rows` up to `cap` rows.  With
 * limit > 0 the search stops once the count exceeds `limit` (ORC_ELIMIT). */
int64_t oracle_match(const og_graph *g, uint32_t k, const int32_t *qvlab, const int64_t *qbound,
                     uint32_t eq, const int32_t *qsrc, const int32_t *qdst, const int32_t *qlab,
                     uint32_t *rows, uint64_t cap, uint64_t limit) {
    if (k == 0 || k > ORC_MAXK || eq > 64) return ORC_EINVAL;
    orc_state *s = (orc_state *)calloc(1, sizeof(orc_state));
    if (!s) return ORC_ENOMEM;
    s->g = g; s->k = k; s->rows = rows; s->cap = rows ? cap : 0; s->limit = limit;
    for (uint32_t u = 0; u < k; u++) {
        s->qlab[u] = qvlab ? qvlab[u] : -1;
        s->qbound[u] = qbound ? qbound[u] : -1;
        if (s->qbound[u] >= (int64_t)g->n) { free(s); return ORC_EINVAL; }
    }
    for (uint32_t e = 0; e < eq; e++) {
        if (qsrc[e] < 0 || qdst[e] < 0 || (uint32_t)qsrc[e] >= k || (uint32_t)qdst[e] >= k ||
            qsrc[e] == qdst[e]) { free(s); return ORC_EINVAL; }
    }
    /* 1. BFS order over the undirected skeleton from vertex 0 */
    int pos[ORC_MAXK];
    for (uint32_t u = 0; u < k; u++) pos[u] = -1;
    uint32_t len = 0, head = 0;
    s->pi[len++] = 0; pos[0] = 0;
    while (head < len) {
        uint32_t x = s->pi[head++];
        for (uint32_t y = 0; y < k; y++) {
            if (pos[y] >= 0) continue;
            int adj = 0;
            for (uint32_t e = 0; e < eq; e++)
                if (((uint32_t)qsrc[e] == x && (uint32_t)qdst[e] == y) ||
                    ((uint32_t)qsrc[e] == y && (uint32_t)qdst[e] == x)) adj = 1;
            if (adj) { pos[y] = (int)len; s->pi[len++] = y; }
        }
    }
    if (len != k) { free(s); return ORC_EDISCONNECTED; }
    /* per position: the generating parent and every arc to an earlier vertex */
    for (uint32_t i = 0; i < k; i++) {
        uint32_t u = s->pi[i];
        s->parent[u] = -1;
        s->nchk[i] = 0;
        for (uint32_t e = 0; e < eq; e++) {
            uint32_t a = (uint32_t)qsrc[e], b = (uint32_t)qdst[e];
            uint32_t other;
            int out;
            if (a == u) { other = b; out = 1; } else if (b == u) { other = a; out = 0; } else continue;
            if (pos[other] >= (int)i) continue;
            chk_t *ck = &s->chk[i][s->nchk[i]++];
            ck->other = other; ck->out = out; ck->lab = qlab ? qlab[e] : -1;
            if (s->parent[u] < 0 || pos[other] < pos[s->parent[u]]) {
                s->parent[u] = (int32_t)other;
                s->parent_out[u] = !out;     /* arc other->u: out-neighbours of f(other) */
            }
        }
    }
    s->used = (uint8_t *)calloc(g->n ? g->n : 1, 1);
    if (!s->used) { free(s); return ORC_ENOMEM; }
    rec(s, 0);
    int64_t r = s->over ? ORC_ELIMIT : (int64_t)s->count;
    free(s->used);
    free(s);
    return r;
}
