/* TEST INFRASTRUCTURE ONLY — see psp_oracle.h for scope and pinning.
 *
 * A restatement of the reference algorithm in plain C (f64 throughout, like
 * the reference: include/psp/graph.hpp:14, include/psp/shortest_paths.hpp:34).
 * Loop orders follow the reference exactly so that results are bitwise equal
 * even for weights whose sums round.
 */
#include "psp_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define INF_D HUGE_VAL

/* ---------------------------------------------------------------- FW ---- */

/* relax_tile (src/shortest_paths.cpp:111-124): kk-outer, i, j-inner; rows
 * whose d(i,kk) is unreachable are skipped (:117). */
static void relax_tile(double* d, uint64_t n, uint64_t k0, uint64_t k1, uint64_t i0,
                       uint64_t i1, uint64_t j0, uint64_t j1) {
    for (uint64_t kk = k0; kk < k1; ++kk) {
        const double* krow = d + kk * n;
        for (uint64_t i = i0; i < i1; ++i) {
            const double dik = d[i * n + kk];
            if (dik == INF_D) continue;
            double* irow = d + i * n;
            for (uint64_t j = j0; j < j1; ++j) {
                const double cand = dik + krow[j];
                if (cand < irow[j]) irow[j] = cand;
            }
        }
    }
}

int pso_apsp_dense(uint64_t n, const uint64_t* off, const uint32_t* to, const double* w,
                   uint64_t block, double* d) {
    if (n == 0) return 0;
    if (block == 0) return -1; /* :131 throws invalid_argument */
    /* init (:133-137): INF, zero diagonal, then edge weights */
    for (uint64_t i = 0; i < n * n; ++i) d[i] = INF_D;
    for (uint64_t v = 0; v < n; ++v) d[v * n + v] = 0.0;
    for (uint64_t u = 0; u < n; ++u)
        for (uint64_t e = off[u]; e < off[u + 1]; ++e) d[u * n + to[e]] = w[e];
    /* three passes per k-block (:139-170) */
    const uint64_t nb = (n + block - 1) / block;
    for (uint64_t kb = 0; kb < nb; ++kb) {
        const uint64_t k0 = kb * block, k1 = (k0 + block < n) ? k0 + block : n;
        relax_tile(d, n, k0, k1, k0, k1, k0, k1);
        for (uint64_t jb = 0; jb < nb; ++jb) {
            if (jb == kb) continue;
            const uint64_t j0 = jb * block, j1 = (j0 + block < n) ? j0 + block : n;
            relax_tile(d, n, k0, k1, k0, k1, j0, j1);
        }
        for (uint64_t ib = 0; ib < nb; ++ib) {
            if (ib == kb) continue;
            const uint64_t i0 = ib * block, i1 = (i0 + block < n) ? i0 + block : n;
            relax_tile(d, n, k0, k1, i0, i1, k0, k1);
        }
        for (uint64_t ib = 0; ib < nb; ++ib) {
            if (ib == kb) continue;
            const uint64_t i0 = ib * block, i1 = (i0 + block < n) ? i0 + block : n;
            for (uint64_t jb = 0; jb < nb; ++jb) {
                if (jb == kb) continue;
                const uint64_t j0 = jb * block, j1 = (j0 + block < n) ? j0 + block : n;
                relax_tile(d, n, k0, k1, i0, i1, j0, j1);
            }
        }
    }
    return 0;
}

/* ---------------------------------------------------------- Dijkstra ---- */

/* DistanceHeap (src/shortest_paths.cpp:13-80): indexed binary min-heap with
 * a position table; sift_up stops on parent <= d, sift_down prefers the
 * right child only when strictly smaller. */
typedef struct {
    uint32_t* heap;
    uint32_t* pos;
    uint32_t size;
} heap_t;

#define ABSENT 0xffffffffu

static void sift_up(heap_t* h, uint32_t i, const double* dist) {
    const uint32_t v = h->heap[i];
    const double d = dist[v];
    while (i > 0) {
        const uint32_t parent = (i - 1) / 2;
        if (dist[h->heap[parent]] <= d) break;
        h->heap[i] = h->heap[parent];
        h->pos[h->heap[i]] = i;
        i = parent;
    }
    h->heap[i] = v;
    h->pos[v] = i;
}

static void sift_down(heap_t* h, uint32_t i, const double* dist) {
    const uint32_t v = h->heap[i];
    const double d = dist[v];
    for (;;) {
        uint32_t child = 2 * i + 1;
        if (child >= h->size) break;
        if (child + 1 < h->size && dist[h->heap[child + 1]] < dist[h->heap[child]]) ++child;
        if (d <= dist[h->heap[child]]) break;
        h->heap[i] = h->heap[child];
        h->pos[h->heap[i]] = i;
        i = child;
    }
    h->heap[i] = v;
    h->pos[v] = i;
}

static void push_or_decrease(heap_t* h, uint32_t v, const double* dist) {
    uint32_t i = h->pos[v];
    if (i == ABSENT) {
        i = h->size++;
        h->heap[i] = v;
        h->pos[v] = i;
    }
    sift_up(h, i, dist);
}

static uint32_t pop_min(heap_t* h, const double* dist) {
    const uint32_t top = h->heap[0];
    h->pos[top] = ABSENT;
    const uint32_t last = h->heap[--h->size];
    if (h->size > 0) {
        h->heap[0] = last;
        h->pos[last] = 0;
        sift_down(h, 0, dist);
    }
    return top;
}

void pso_dijkstra(uint64_t n, const uint64_t* off, const uint32_t* to, const double* w,
                  uint32_t source, double* dist) {
    heap_t h;
    h.heap = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
    h.pos = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
    h.size = 0;
    for (uint64_t v = 0; v < n; ++v) {
        dist[v] = INF_D;
        h.pos[v] = ABSENT;
    }
    dist[source] = 0.0;
    push_or_decrease(&h, source, dist);
    while (h.size) {
        const uint32_t u = pop_min(&h, dist);
        const double du = dist[u];
        for (uint64_t e = off[u]; e < off[u + 1]; ++e) {
            const double nd = du + w[e];
            if (nd < dist[to[e]]) {
                dist[to[e]] = nd;
                push_or_decrease(&h, to[e], dist);
            }
        }
    }
    free(h.heap);
    free(h.pos);
}

double pso_min_plus_combine(uint64_t len, const double* a, const double* b) {
    double best = INF_D;
    for (uint64_t i = 0; i < len; ++i) {
        const double s = a[i] + b[i];
        if (s < best) best = s;
    }
    return best;
}

/* ------------------------------------------------------------ oracle ---- */

struct pso_oracle {
    uint64_t n, b, bg_edges;
    uint32_t k;
    uint32_t* perm;     /* original -> reordered */
    uint32_t* assign;   /* reordered -> component */
    uint64_t* comp_off; /* k+1 */
    uint64_t* bnd_off;  /* k+1 */
    double** ctab;      /* |C| x |C| */
    double** btab;      /* |B(C)| x b */
};

typedef struct {
    uint32_t u, v;
    double w;
} edge_t;

static int cmp_nb(const void* a, const void* b) {
    const uint32_t x = ((const edge_t*)a)->v, y = ((const edge_t*)b)->v;
    return (x > y) - (x < y);
}

/* Graph(n, edges) CSR construction (src/graph.cpp:19-56): both arcs of every
 * edge, each adjacency list sorted by neighbour id. */
static void csr_from_edges(uint64_t n, const edge_t* edges, uint64_t m, uint64_t** off_out,
                           uint32_t** to_out, double** w_out) {
    uint64_t* off = (uint64_t*)calloc(n + 1, sizeof(uint64_t));
    for (uint64_t i = 0; i < m; ++i) {
        ++off[edges[i].u + 1];
        ++off[edges[i].v + 1];
    }
    for (uint64_t v = 0; v < n; ++v) off[v + 1] += off[v];
    edge_t* arcs = (edge_t*)malloc((2 * m + 1) * sizeof(edge_t));
    uint64_t* cur = (uint64_t*)malloc((n + 1) * sizeof(uint64_t));
    memcpy(cur, off, n * sizeof(uint64_t));
    for (uint64_t i = 0; i < m; ++i) {
        arcs[cur[edges[i].u]++] = (edge_t){edges[i].u, edges[i].v, edges[i].w};
        arcs[cur[edges[i].v]++] = (edge_t){edges[i].v, edges[i].u, edges[i].w};
    }
    uint32_t* to = (uint32_t*)malloc((2 * m + 1) * sizeof(uint32_t));
    double* w = (double*)malloc((2 * m + 1) * sizeof(double));
    for (uint64_t v = 0; v < n; ++v) {
        qsort(arcs + off[v], off[v + 1] - off[v], sizeof(edge_t), cmp_nb);
        for (uint64_t e = off[v]; e < off[v + 1]; ++e) {
            to[e] = arcs[e].v;
            w[e] = arcs[e].w;
        }
    }
    free(arcs);
    free(cur);
    *off_out = off;
    *to_out = to;
    *w_out = w;
}

pso_oracle* pso_build(uint64_t n, const uint64_t* off, const uint32_t* to, const double* w,
                      uint32_t k, const uint32_t* perm, const uint32_t* assign,
                      const uint8_t* flags) {
    pso_oracle* o = (pso_oracle*)calloc(1, sizeof(pso_oracle));
    if (!o) return NULL;
    o->n = n;
    o->k = k;
    o->perm = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
    o->assign = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
    memcpy(o->perm, perm, n * sizeof(uint32_t));
    memcpy(o->assign, assign, n * sizeof(uint32_t));
    o->comp_off = (uint64_t*)calloc(k + 1, sizeof(uint64_t));
    o->bnd_off = (uint64_t*)calloc(k + 1, sizeof(uint64_t));
    /* component_ranges (src/oracle.cpp:45-54) and boundary offsets
     * (src/oracle.cpp:80-89) */
    for (uint64_t v = 0; v < n; ++v) {
        ++o->comp_off[assign[v] + 1];
        if (flags[v]) ++o->bnd_off[assign[v] + 1];
    }
    for (uint32_t c = 0; c < k; ++c) {
        o->comp_off[c + 1] += o->comp_off[c];
        o->bnd_off[c + 1] += o->bnd_off[c];
    }
    o->b = o->bnd_off[k];
    o->ctab = (double**)calloc(k, sizeof(double*));
    o->btab = (double**)calloc(k, sizeof(double*));

    /* Phase 2 (src/oracle.cpp:162-169): induced_range_subgraph (:22-43) keeps
     * the parent's (sorted) neighbour order, then apsp_dense with the default
     * block size 64 (include/psp/shortest_paths.hpp:43). */
    for (uint32_t c = 0; c < k; ++c) {
        const uint64_t base = o->comp_off[c], size = o->comp_off[c + 1] - base;
        uint64_t* soff = (uint64_t*)calloc(size + 1, sizeof(uint64_t));
        uint64_t cnt = 0;
        for (uint64_t i = 0; i < size; ++i) {
            for (uint64_t e = off[base + i]; e < off[base + i + 1]; ++e)
                if (to[e] >= base && to[e] < base + size) ++cnt;
            soff[i + 1] = cnt;
        }
        uint32_t* sto = (uint32_t*)malloc((cnt + 1) * sizeof(uint32_t));
        double* sw = (double*)malloc((cnt + 1) * sizeof(double));
        cnt = 0;
        for (uint64_t i = 0; i < size; ++i)
            for (uint64_t e = off[base + i]; e < off[base + i + 1]; ++e)
                if (to[e] >= base && to[e] < base + size) {
                    sto[cnt] = (uint32_t)(to[e] - base);
                    sw[cnt++] = w[e];
                }
        o->ctab[c] = (double*)malloc((size * size + 1) * sizeof(double));
        pso_apsp_dense(size, soff, sto, sw, 64, o->ctab[c]);
        free(soff);
        free(sto);
        free(sw);
    }

    /* Phase 3 (src/oracle.cpp:170-177): build_boundary_graph (:77-125) —
     * cross edges for v < nb.to (:103-109), then per component the clique
     * edges i < j < |B(C)| with finite table entries (:110-122). */
    const uint64_t b = o->b;
    uint64_t cap = 16, m = 0;
    edge_t* edges = (edge_t*)malloc(cap * sizeof(edge_t));
#define PUSH_EDGE(A, B, W)                                           \
    do {                                                             \
        if (m == cap) {                                              \
            cap *= 2;                                                \
            edges = (edge_t*)realloc(edges, cap * sizeof(edge_t));   \
        }                                                            \
        edges[m++] = (edge_t){(uint32_t)(A), (uint32_t)(B), (W)};    \
    } while (0)
    for (uint64_t v = 0; v < n; ++v) {
        if (!flags[v]) continue;
        const uint32_t cv = assign[v];
        for (uint64_t e = off[v]; e < off[v + 1]; ++e) {
            const uint32_t u = to[e], cu = assign[u];
            if (cu != cv && v < u) {
                const uint64_t bv = o->bnd_off[cv] + (v - o->comp_off[cv]);
                const uint64_t bu = o->bnd_off[cu] + (u - o->comp_off[cu]);
                PUSH_EDGE(bv, bu, w[e]);
            }
        }
    }
    for (uint32_t c = 0; c < k; ++c) {
        const uint64_t bc = o->bnd_off[c + 1] - o->bnd_off[c];
        const uint64_t size = o->comp_off[c + 1] - o->comp_off[c];
        for (uint64_t i = 0; i < bc; ++i)
            for (uint64_t j = i + 1; j < bc; ++j) {
                const double d = o->ctab[c][i * size + j];
                if (d < INF_D) PUSH_EDGE(o->bnd_off[c] + i, o->bnd_off[c] + j, d);
            }
    }
#undef PUSH_EDGE
    o->bg_edges = m;
    uint64_t* boff;
    uint32_t* bto;
    double* bw;
    csr_from_edges(b, edges, m, &boff, &bto, &bw);
    free(edges);
    /* boundary_apsp (src/oracle.cpp:127-142): one Dijkstra per boundary id,
     * rows grouped by component. */
    for (uint32_t c = 0; c < k; ++c) {
        const uint64_t lo = o->bnd_off[c], hi = o->bnd_off[c + 1];
        o->btab[c] = (double*)malloc(((hi - lo) * b + 1) * sizeof(double));
        for (uint64_t i = lo; i < hi; ++i)
            pso_dijkstra(b, boff, bto, bw, (uint32_t)i, o->btab[c] + (i - lo) * b);
    }
    free(boff);
    free(bto);
    free(bw);
    return o;
}

void pso_free(pso_oracle* o) {
    if (!o) return;
    for (uint32_t c = 0; c < o->k; ++c) {
        free(o->ctab[c]);
        free(o->btab[c]);
    }
    free(o->ctab);
    free(o->btab);
    free(o->perm);
    free(o->assign);
    free(o->comp_off);
    free(o->bnd_off);
    free(o);
}

void pso_info(const pso_oracle* o, uint64_t* info) {
    info[0] = o->n;
    info[1] = o->k;
    info[2] = o->b;
    info[3] = o->bg_edges;
    uint64_t stored = 0; /* Oracle::stored_entries (src/oracle.cpp:58-65) */
    for (uint32_t c = 0; c < o->k; ++c) {
        const uint64_t s = o->comp_off[c + 1] - o->comp_off[c];
        stored += s * s + (o->bnd_off[c + 1] - o->bnd_off[c]) * o->b;
    }
    info[4] = stored;
}

void pso_offsets(const pso_oracle* o, uint64_t* comp_off, uint64_t* bnd_off) {
    memcpy(comp_off, o->comp_off, (o->k + 1) * sizeof(uint64_t));
    memcpy(bnd_off, o->bnd_off, (o->k + 1) * sizeof(uint64_t));
}

const double* pso_component_table(const pso_oracle* o, uint32_t c) { return o->ctab[c]; }
const double* pso_boundary_rows(const pso_oracle* o, uint32_t c) { return o->btab[c]; }

/* query (src/query.cpp:29-88): make_frame id translation (:29-45),
 * stitch_into (:49-59) with the unreachable-row skip (:53), min_plus_combine
 * with the target column (:61-65), same-component cap (:70-72), and
 * minplus_ops = B1*B2 + B2 (:73). */
int pso_query(const pso_oracle* o, uint32_t v1, uint32_t v2, double* dist, uint64_t* ops) {
    if (v1 >= o->n || v2 >= o->n) return -1;
    const uint32_t r1 = o->perm[v1], r2 = o->perm[v2];
    const uint32_t c1 = o->assign[r1], c2 = o->assign[r2];
    const uint64_t l1 = r1 - o->comp_off[c1], l2 = r2 - o->comp_off[c2];
    const uint64_t s1 = o->comp_off[c1 + 1] - o->comp_off[c1];
    const uint64_t s2 = o->comp_off[c2 + 1] - o->comp_off[c2];
    const uint64_t b1n = o->bnd_off[c1 + 1] - o->bnd_off[c1];
    const uint64_t b2n = o->bnd_off[c2 + 1] - o->bnd_off[c2];
    const double* row1 = o->ctab[c1] + l1 * s1;
    const double* col2 = o->ctab[c2] + l2 * s2;
    const uint64_t bg2 = o->bnd_off[c2];
    double* through = (double*)malloc((b2n + 1) * sizeof(double));
    for (uint64_t j = 0; j < b2n; ++j) through[j] = INF_D;
    for (uint64_t i = 0; i < b1n; ++i) {
        const double d1 = row1[i];
        if (d1 == INF_D) continue;
        const double* bg_row = o->btab[c1] + i * o->b + bg2;
        for (uint64_t j = 0; j < b2n; ++j) {
            const double cand = d1 + bg_row[j];
            /* std::min(a, b) returns a unless b < a */
            if (cand < through[j]) through[j] = cand;
        }
    }
    double d = pso_min_plus_combine(b2n, through, col2);
    free(through);
    if (c1 == c2) {
        const double same = o->ctab[c1][l1 * s1 + l2];
        if (same < d) d = same;
    }
    *dist = d;
    if (ops) *ops = b1n * b2n + b2n;
    return 0;
}

uint64_t pso_batch_query(const pso_oracle* o, uint64_t count, const uint32_t* v1,
                         const uint32_t* v2, double* dist, uint64_t* ops) {
    for (uint64_t i = 0; i < count; ++i)
        if (pso_query(o, v1[i], v2[i], dist + i, ops ? ops + i : NULL) != 0) return i + 1;
    return 0;
}
