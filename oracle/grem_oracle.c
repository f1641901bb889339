/*
 * grem_oracle.c — TEST INFRASTRUCTURE ONLY.  A single-threaded, bit-exact C
 * restatement of the reference GREM partitioner (streamcut, pure Python).
 * It is the checker for the CUDA path at sizes where the Python reference is
 * too slow; it is validated against the Python reference itself
 * (tests/test_oracle.py) on random multigraphs and on committed golden
 * fixtures produced by running streamcut (tests/golden/make_golden.py).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library; the product path never does.
 *
 * Every function cites the reference lines it follows (paths relative to the
 * reference package, pkg/src/streamcut/).  Differences in *method* (not in
 * result): chunk adjacency is built by counting sort instead of
 * np.lexsort (model.py:53-61) — same multiset, same ascending neighbour order;
 * the BFS restart scan (seed.py:69-75) uses a (-degree, index)-sorted list with
 * a skip pointer — the same node is chosen, without the quadratic rescan.
 * Floating point: the running estimates are IEEE binary64 exactly as Python
 * floats ((a + c) * 0.5, grem.py:147-148); build with -ffp-contract=off.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_FORMAT 1
#define OR_CAPACITY 2
#define OR_NOMEM 4

static char g_err[256];
const char* oracle_last_error(void) { return g_err; }

typedef int (*oracle_seed_cb)(int64_t n_chunk_nodes, int8_t* labels_out, void* user);

/* ------------------------------------------------------------------ chunk */

typedef struct {
    int64_t nn;        /* N_c: sorted unique endpoints (model.py:59) */
    int64_t* nodes;    /* global ids ascending */
    int64_t* start;    /* CSR over local ids, len nn+1 */
    int64_t* adj;      /* local ids of neighbours, ascending per row (model.py:56) */
} chunk_t;

typedef struct {
    int64_t n;
    int32_t* stamp;    /* per global node: chunk serial + 1 */
    int64_t* local;    /* per global node: local index when stamped */
    int32_t serial;
} chunk_ws;

static void chunk_free(chunk_t* c) {
    free(c->nodes); free(c->start); free(c->adj);
    memset(c, 0, sizeof(*c));
}

/* EdgeChunk.__init__ (model.py:48-61): nodes = np.unique(edges) incl.
 * self-loop-only nodes; symmetric adjacency without self-loops, duplicates
 * kept, neighbour lists ascending. */
static int chunk_build(chunk_ws* ws, const uint32_t* e, int64_t m, int sorted_adj, chunk_t* c) {
    memset(c, 0, sizeof(*c));
    ws->serial++;
    int32_t tag = ws->serial;
    int64_t nn = 0;
    for (int64_t i = 0; i < 2 * m; ++i) {
        uint32_t v = e[i];
        if (ws->stamp[v] != tag) { ws->stamp[v] = tag; nn++; }
    }
    c->nn = nn;
    c->nodes = (int64_t*)malloc(sizeof(int64_t) * (nn ? nn : 1));
    c->start = (int64_t*)calloc((size_t)nn + 1, sizeof(int64_t));
    if (!c->nodes || !c->start) return OR_NOMEM;
    /* ascending ids: collect then sort (radix by counting would need O(n)) */
    int64_t k = 0;
    ws->serial++;
    int32_t tag2 = ws->serial;
    for (int64_t i = 0; i < 2 * m; ++i) {
        uint32_t v = e[i];
        if (ws->stamp[v] == tag) { ws->stamp[v] = tag2; c->nodes[k++] = v; }
    }
    /* sort ids: LSD radix on 64-bit (values < 2^32) */
    {
        int64_t* tmp = (int64_t*)malloc(sizeof(int64_t) * (nn ? nn : 1));
        if (!tmp) return OR_NOMEM;
        int64_t cnt[65536 + 1];
        for (int pass = 0; pass < 2; ++pass) {
            int sh = pass * 16;
            memset(cnt, 0, sizeof(cnt));
            for (int64_t i = 0; i < nn; ++i) cnt[((c->nodes[i] >> sh) & 0xFFFF) + 1]++;
            for (int b = 0; b < 65536; ++b) cnt[b + 1] += cnt[b];
            for (int64_t i = 0; i < nn; ++i) tmp[cnt[(c->nodes[i] >> sh) & 0xFFFF]++] = c->nodes[i];
            memcpy(c->nodes, tmp, sizeof(int64_t) * nn);
        }
        free(tmp);
    }
    for (int64_t i = 0; i < nn; ++i) ws->local[c->nodes[i]] = i;
    /* degrees (self-loops excluded, model.py:53) */
    int64_t entries = 0;
    for (int64_t i = 0; i < m; ++i) {
        uint32_t u = e[2 * i], v = e[2 * i + 1];
        if (u == v) continue;
        c->start[ws->local[u] + 1]++;
        c->start[ws->local[v] + 1]++;
        entries += 2;
    }
    for (int64_t i = 0; i < nn; ++i) c->start[i + 1] += c->start[i];
    c->adj = (int64_t*)malloc(sizeof(int64_t) * (entries ? entries : 1));
    if (!c->adj) return OR_NOMEM;
    if (!sorted_adj) {
        int64_t* pos = (int64_t*)malloc(sizeof(int64_t) * (nn ? nn : 1));
        if (!pos) return OR_NOMEM;
        memcpy(pos, c->start, sizeof(int64_t) * nn);
        for (int64_t i = 0; i < m; ++i) {
            uint32_t u = e[2 * i], v = e[2 * i + 1];
            if (u == v) continue;
            int64_t lu = ws->local[u], lv = ws->local[v];
            c->adj[pos[lu]++] = lv;
            c->adj[pos[lv]++] = lu;
        }
        free(pos);
        return OR_OK;
    }
    /* sorted rows: counting sort by neighbour, then stable counting sort by
     * owner => rows ascending by neighbour (== np.lexsort((vals, keys))). */
    {
        int64_t* src = (int64_t*)malloc(sizeof(int64_t) * (entries ? entries : 1));
        int64_t* dst = (int64_t*)malloc(sizeof(int64_t) * (entries ? entries : 1));
        int64_t* bucket = (int64_t*)calloc((size_t)nn + 1, sizeof(int64_t));
        if (!src || !dst || !bucket) return OR_NOMEM;
        int64_t q = 0;
        for (int64_t i = 0; i < m; ++i) {
            uint32_t u = e[2 * i], v = e[2 * i + 1];
            if (u == v) continue;
            src[q] = ws->local[u]; dst[q] = ws->local[v]; q++;
            src[q] = ws->local[v]; dst[q] = ws->local[u]; q++;
        }
        for (int64_t i = 0; i < entries; ++i) bucket[dst[i] + 1]++;
        for (int64_t i = 0; i < nn; ++i) bucket[i + 1] += bucket[i];
        int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (entries ? entries : 1));
        if (!order) return OR_NOMEM;
        for (int64_t i = 0; i < entries; ++i) order[bucket[dst[i]]++] = i;
        int64_t* pos = (int64_t*)malloc(sizeof(int64_t) * (nn ? nn : 1));
        if (!pos) return OR_NOMEM;
        memcpy(pos, c->start, sizeof(int64_t) * nn);
        for (int64_t j = 0; j < entries; ++j) {
            int64_t i = order[j];
            c->adj[pos[src[i]]++] = dst[i];
        }
        free(pos); free(order); free(bucket); free(src); free(dst);
    }
    return OR_OK;
}

/* ------------------------------------------------------------------ state */

typedef struct {
    int64_t n;
    int8_t* parts;     /* -1 / 0 / 1 (model.py:91-98) */
    double* nbr0;
    double* nbr1;
    int64_t sizes[2];
    int64_t cap;
} state_t;

/* grem.py:100-116 */
static int assign_side(double c0, double c1, const int64_t* sizes, int64_t cap, int* out) {
    if (c0 < c1 && sizes[1] < cap) { *out = 1; return OR_OK; }
    if (c1 < c0 && sizes[0] < cap) { *out = 0; return OR_OK; }
    if (sizes[0] <= sizes[1]) {
        if (sizes[0] >= cap) { strcpy(g_err, "both partitions at capacity; size accounting is broken"); return OR_CAPACITY; }
        *out = 0; return OR_OK;
    }
    if (sizes[1] >= cap) { strcpy(g_err, "both partitions at capacity; size accounting is broken"); return OR_CAPACITY; }
    *out = 1; return OR_OK;
}

typedef struct {
    int64_t chunks, visits, moves, ties;
} oracle_stats;

/* process_chunk, grem.py:119-155 */
static int process_chunk(state_t* st, const chunk_t* c, const int64_t* gid_of_local, int refine, oracle_stats* stats) {
    int8_t* parts = st->parts;
    for (int64_t i = 0; i < c->nn; ++i) {
        int64_t n = c->nodes[i];
        int old = parts[n];
        if (old != -1 && !refine) continue;
        double c0 = 0.0, c1 = 0.0;
        for (int64_t k = c->start[i]; k < c->start[i + 1]; ++k) {
            int pw = parts[gid_of_local[c->adj[k]]];
            if (pw == 0) c0 += 1.0;
            else if (pw == 1) c1 += 1.0;
        }
        if (old != -1) {
            c0 = (st->nbr0[n] + c0) * 0.5;
            c1 = (st->nbr1[n] + c1) * 0.5;
            st->sizes[old] -= 1;
        }
        int b;
        int rc = assign_side(c0, c1, st->sizes, st->cap, &b);
        if (rc) return rc;
        if (stats) { stats->visits++; if (c0 == c1) stats->ties++; if (old != -1 && b != old) stats->moves++; }
        st->sizes[b] += 1;
        parts[n] = (int8_t)b;
        st->nbr0[n] = c0;
        st->nbr1[n] = c1;
    }
    return OR_OK;
}

/* _bfs_grow, seed.py:56-118.  Restart = highest degree unpicked node, lowest
 * index on ties (seed.py:69-75), taken from a (-degree, index) order with a
 * skip pointer — identical choice without the O(n) rescan. */
static int bfs_grow(const chunk_t* c, int refinement_passes, int64_t capacity, int8_t* labels) {
    int64_t n = c->nn;
    int64_t target = (n + 1) / 2;   /* ceil(n / 2) */
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
    int64_t* queue = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
    uint8_t* picked = (uint8_t*)calloc((size_t)(n ? n : 1), 1);
    if (!order || !queue || !picked) return OR_NOMEM;
    /* stable counting sort by degree descending */
    int64_t maxdeg = 0;
    for (int64_t i = 0; i < n; ++i) {
        int64_t d = c->start[i + 1] - c->start[i];
        if (d > maxdeg) maxdeg = d;
    }
    int64_t* cnt = (int64_t*)calloc((size_t)maxdeg + 2, sizeof(int64_t));
    if (!cnt) return OR_NOMEM;
    for (int64_t i = 0; i < n; ++i) cnt[maxdeg - (c->start[i + 1] - c->start[i]) + 1]++;
    for (int64_t d = 0; d <= maxdeg; ++d) cnt[d + 1] += cnt[d];
    for (int64_t i = 0; i < n; ++i) order[cnt[maxdeg - (c->start[i + 1] - c->start[i])]++] = i;
    free(cnt);
    int64_t rp = 0, qh = 0, qt = 0, count = 0;
    while (count < target) {
        if (qh == qt) {
            while (picked[order[rp]]) rp++;
            int64_t best = order[rp];
            queue[qt++] = best;
            picked[best] = 1;
            count++;
            if (count >= target) break;
        }
        int64_t v = queue[qh++];
        for (int64_t k = c->start[v]; k < c->start[v + 1]; ++k) {
            int64_t w = c->adj[k];
            if (!picked[w]) {
                picked[w] = 1;
                count++;
                queue[qt++] = w;
                if (count >= target) break;
            }
        }
    }
    for (int64_t i = 0; i < n; ++i) labels[i] = picked[i] ? 0 : 1;
    int64_t sizes[2] = {target, n - target};
    for (int pass = 0; pass < refinement_passes; ++pass) {
        int moved = 0;
        for (int64_t i = 0; i < n; ++i) {
            int side = labels[i];
            int64_t same = 0, other = 0;
            for (int64_t k = c->start[i]; k < c->start[i + 1]; ++k) {
                if (labels[c->adj[k]] == side) same++; else other++;
            }
            if (other == 0) continue;
            if (other > same && sizes[1 - side] < capacity) {
                labels[i] = (int8_t)(1 - side);
                sizes[side]--;
                sizes[1 - side]++;
                moved = 1;
            }
        }
        if (!moved) break;
    }
    free(order); free(queue); free(picked);
    return OR_OK;
}

/* _seed_chunk, grem.py:158-174 (+ seed_bisect checks, seed.py:36-53) */
static int seed_chunk(state_t* st, const chunk_t* c, int seed_algo, int refinement_passes,
                      oracle_seed_cb cb, void* user, const int64_t* gid_of_local) {
    int64_t nn = c->nn;
    if (nn == 0) { strcpy(g_err, "cannot seed an empty chunk"); return OR_FORMAT; }
    if (2 * st->cap < nn) { strcpy(g_err, "capacity infeasible for chunk nodes"); return OR_CAPACITY; }
    int8_t* lab = (int8_t*)malloc((size_t)nn);
    if (!lab) return OR_NOMEM;
    int rc;
    if (seed_algo == 0) rc = bfs_grow(c, refinement_passes, st->cap, lab);
    else rc = cb ? cb(nn, lab, user) : OR_FORMAT;
    if (rc) { free(lab); return rc; }
    for (int64_t i = 0; i < nn; ++i) st->parts[c->nodes[i]] = lab[i];
    int64_t s0 = 0, s1 = 0;
    for (int64_t v = 0; v < st->n; ++v) { if (st->parts[v] == 0) s0++; else if (st->parts[v] == 1) s1++; }
    st->sizes[0] = s0; st->sizes[1] = s1;
    for (int64_t i = 0; i < nn; ++i) {
        int64_t a = 0, b = 0;
        for (int64_t k = c->start[i]; k < c->start[i + 1]; ++k) {
            int pw = st->parts[gid_of_local[c->adj[k]]];
            if (pw == 0) a++; else if (pw == 1) b++;
        }
        st->nbr0[c->nodes[i]] = (double)a;
        st->nbr1[c->nodes[i]] = (double)b;
    }
    free(lab);
    return OR_OK;
}

/* _fill_unassigned, grem.py:177-189 */
static int fill_unassigned(state_t* st) {
    for (int64_t v = 0; v < st->n; ++v) {
        if (st->parts[v] != -1) continue;
        int b = st->sizes[0] <= st->sizes[1] ? 0 : 1;
        if (st->sizes[b] >= st->cap) {
            b = 1 - b;
            if (st->sizes[b] >= st->cap) { strcpy(g_err, "no partition has room for unassigned nodes"); return OR_CAPACITY; }
        }
        st->parts[v] = (int8_t)b;
        st->sizes[b]++;
    }
    return OR_OK;
}

typedef void (*oracle_chunk_cb)(const int64_t* sizes, const int8_t* parts, void* user);

/* bisect, grem.py:192-224 (count_cuts is done by the caller) */
int oracle_bisect(const uint32_t* edges, int64_t m, int64_t n, int64_t chunk_edges, int64_t cap,
                  int refine, int passes, int seed_algo, int seed_refinement_passes,
                  oracle_seed_cb seed_cb, void* seed_user,
                  oracle_chunk_cb chunk_cb, void* chunk_user,
                  int8_t* labels_out, int64_t* sizes_out, oracle_stats* stats) {
    g_err[0] = 0;
    if (n < 1) { strcpy(g_err, "num_nodes must be >= 1"); return OR_FORMAT; }
    if (2 * cap < n) { strcpy(g_err, "capacity cannot hold all nodes across two parts"); return OR_CAPACITY; }
    if (chunk_edges < 1) { strcpy(g_err, "chunk_size must be >= 1"); return OR_FORMAT; }
    for (int64_t i = 0; i < 2 * m; ++i)
        if ((int64_t)edges[i] >= n) { strcpy(g_err, "edge endpoint >= num_nodes"); return OR_FORMAT; }
    state_t st;
    st.n = n; st.cap = cap; st.sizes[0] = st.sizes[1] = 0;
    st.parts = labels_out;
    memset(st.parts, 0xFF, (size_t)n);
    st.nbr0 = (double*)calloc((size_t)n, sizeof(double));
    st.nbr1 = (double*)calloc((size_t)n, sizeof(double));
    chunk_ws ws;
    ws.n = n; ws.serial = 0;
    ws.stamp = (int32_t*)calloc((size_t)n, sizeof(int32_t));
    ws.local = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    if (!st.nbr0 || !st.nbr1 || !ws.stamp || !ws.local) return OR_NOMEM;
    int64_t num_chunks = m ? (m + chunk_edges - 1) / chunk_edges : 0;
    int rc = OR_OK;
    for (int pass = 0; pass < passes && rc == OR_OK; ++pass) {
        for (int64_t ci = 0; ci < num_chunks && rc == OR_OK; ++ci) {
            int64_t lo = ci * chunk_edges;
            int64_t cnt = m - lo < chunk_edges ? m - lo : chunk_edges;
            int seeding = (pass == 0 && ci == 0);
            chunk_t c;
            rc = chunk_build(&ws, edges + 2 * lo, cnt, seeding, &c);
            if (rc == OR_OK) {
                if (seeding) rc = seed_chunk(&st, &c, seed_algo, seed_refinement_passes, seed_cb, seed_user, c.nodes);
                else rc = process_chunk(&st, &c, c.nodes, refine, stats);
                if (stats) stats->chunks++;
            }
            chunk_free(&c);
            if (rc == OR_OK && chunk_cb) chunk_cb(st.sizes, st.parts, chunk_user);
        }
    }
    if (rc == OR_OK) rc = fill_unassigned(&st);
    if (sizes_out) { sizes_out[0] = st.sizes[0]; sizes_out[1] = st.sizes[1]; }
    free(st.nbr0); free(st.nbr1); free(ws.stamp); free(ws.local);
    return rc;
}

/* count_cuts, grem.py:227-252: cut count + per-part sizes (num_parts = max+1) */
int oracle_count_cuts(const uint32_t* edges, int64_t m, int64_t n, const int32_t* labels,
                      int64_t* cut_out, int64_t* sizes_out, int64_t max_parts, int64_t* num_parts_out) {
    int64_t cut = 0;
    for (int64_t i = 0; i < m; ++i) {
        int32_t a = labels[edges[2 * i]], b = labels[edges[2 * i + 1]];
        if (a < 0 || b < 0) { strcpy(g_err, "unlabeled endpoint encountered"); return OR_FORMAT; }
        cut += (a != b);
    }
    int32_t mx = -1;
    for (int64_t v = 0; v < n; ++v) if (labels[v] > mx) mx = labels[v];
    int64_t np_ = mx >= 0 ? (int64_t)mx + 1 : 1;
    if (np_ > max_parts) { strcpy(g_err, "too many parts"); return OR_FORMAT; }
    for (int64_t k = 0; k < np_; ++k) sizes_out[k] = 0;
    for (int64_t v = 0; v < n; ++v) if (labels[v] >= 0) sizes_out[labels[v]]++;
    *cut_out = cut;
    *num_parts_out = np_;
    return OR_OK;
}

/* partition, grem.py:277-319 — recursion over in-memory induced subgraphs
 * (_extract_induced, grem.py:255-274: kept edges in file order, dense ids =
 * rank among ascending members). */
typedef struct {
    int64_t total_nodes;
    double slack;
    double frac;          /* < 0 => use chunk_edges */
    int64_t chunk_edges;
    int refine, passes, seed_algo, seed_refinement_passes;
    oracle_seed_cb seed_cb;
    void* seed_user;
    int32_t* final_labels;
    oracle_stats* stats;
} part_ctx;

static int64_t plan_chunk(const part_ctx* pc, int64_t m) {
    if (pc->frac < 0) return pc->chunk_edges;
    double t = pc->frac * (double)m;      /* ceil(chunk_frac * num_edges), edgefile.py:346 */
    int64_t ce = (int64_t)ceil(t);
    return ce < 1 ? 1 : ce;
}

static int recurse(part_ctx* pc, const uint32_t* edges, int64_t m, int64_t n, const int64_t* orig,
                   int64_t p_level, int level, int64_t leaf_base) {
    double capd = ceil((1.0 + pc->slack) * (double)pc->total_nodes / (double)(1LL << (level + 1)));
    int64_t cap = (int64_t)capd;
    int8_t* lab = (int8_t*)malloc((size_t)n);
    if (!lab) return OR_NOMEM;
    int rc = oracle_bisect(edges, m, n, plan_chunk(pc, m), cap, pc->refine, pc->passes, pc->seed_algo,
                           pc->seed_refinement_passes, pc->seed_cb, pc->seed_user, NULL, NULL, lab, NULL, pc->stats);
    if (rc) { free(lab); return rc; }
    if (p_level == 2) {
        for (int64_t v = 0; v < n; ++v) pc->final_labels[orig[v]] = (int32_t)(leaf_base + lab[v]);
        free(lab);
        return OR_OK;
    }
    int64_t* newid = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    if (!newid) { free(lab); return OR_NOMEM; }
    for (int side = 0; side < 2 && rc == OR_OK; ++side) {
        int64_t base = leaf_base + side * (p_level / 2);
        int64_t k = 0;
        for (int64_t v = 0; v < n; ++v) newid[v] = (lab[v] == side) ? k++ : -1;
        if (k == 0) continue;
        int64_t* sub_orig = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
        int64_t ms = 0;
        for (int64_t i = 0; i < m; ++i) if (lab[edges[2 * i]] == side && lab[edges[2 * i + 1]] == side) ms++;
        uint32_t* sub = (uint32_t*)malloc(sizeof(uint32_t) * 2 * (size_t)(ms ? ms : 1));
        if (!sub_orig || !sub) { rc = OR_NOMEM; break; }
        for (int64_t v = 0; v < n; ++v) if (newid[v] >= 0) sub_orig[newid[v]] = orig[v];
        int64_t q = 0;
        for (int64_t i = 0; i < m; ++i) {
            uint32_t a = edges[2 * i], b = edges[2 * i + 1];
            if (lab[a] == side && lab[b] == side) { sub[2 * q] = (uint32_t)newid[a]; sub[2 * q + 1] = (uint32_t)newid[b]; q++; }
        }
        rc = recurse(pc, sub, ms, k, sub_orig, p_level / 2, level + 1, base);
        free(sub); free(sub_orig);
    }
    free(newid); free(lab);
    return rc;
}

int oracle_partition(const uint32_t* edges, int64_t m, int64_t n, int64_t p, double slack, double frac,
                     int64_t chunk_edges, int refine, int passes, int seed_algo, int seed_refinement_passes,
                     oracle_seed_cb seed_cb, void* seed_user, int32_t* labels_out, oracle_stats* stats) {
    g_err[0] = 0;
    if (p < 2 || (p & (p - 1)) != 0) { strcpy(g_err, "number of parts must be a power of two >= 2"); return OR_FORMAT; }
    part_ctx pc;
    pc.total_nodes = n; pc.slack = slack; pc.frac = frac; pc.chunk_edges = chunk_edges;
    pc.refine = refine; pc.passes = passes; pc.seed_algo = seed_algo;
    pc.seed_refinement_passes = seed_refinement_passes; pc.seed_cb = seed_cb; pc.seed_user = seed_user;
    pc.final_labels = labels_out; pc.stats = stats;
    for (int64_t v = 0; v < n; ++v) labels_out[v] = -1;
    int64_t* orig = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    if (!orig) return OR_NOMEM;
    for (int64_t v = 0; v < n; ++v) orig[v] = v;
    int rc = recurse(&pc, edges, m, n, orig, p, 0, 0);
    free(orig);
    return rc;
}
