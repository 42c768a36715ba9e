/*
 * ipgc_oracle.c -- CPU restatement of the reference IPGC hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links, imports or
 * executes this file: it is the checker used by tests/, __graft_entry__.smoke()
 * and the cpu_baseline leg of bench.py.  It is pinned against the reference
 * (`hybridcolor`, /root/reference/pkg) through tests/golden/ fixtures produced
 * by tests/golden/make_golden.py and through oracle/_ref (the reference's own
 * compiled Cython backend) when present.
 *
 * Every routine below restates a reference routine and cites it:
 *   orc_build_csr   <- pkg/src/hybridcolor/graph.py:184-201  (build_csr)
 *   orc_color       <- pkg/src/hybridcolor/driver.py:122-176 (color_graph loop)
 *                      + coloring.py:113-176 (data/topology iterations,
 *                        commits 105-110)
 *                      + _kernels.pyx:29-149 (assign_* / resolve_* kernels)
 *                      + worklist.py:77-91 (swap_and_sort)
 *   orc_verify      <- driver.py:188-204 (verify_coloring)
 *   orc_colors_used <- driver.py:179-185 (colors_used)
 *   orc_gen_*       <- build-owned synthetic generators;
 *                      grid follows pkg/tests/conftest.py:30-41, ER endpoint
 *                      sampling follows conftest.py:53-59 / compare_backends.py:27-31
 *                      with a counter-based hash in place of numpy's PCG64.
 *
 * Semantics are the reference's deterministic synchronous rounds: snapshot
 * reads, lower-id-wins tie break, worklist sorted at swap time.  The loops are
 * written the reference's way (colors_read / colors_write / stamp triple with
 * explicit commits) on purpose, so the oracle does not share the product's
 * single-word state encoding.  OpenMP only parallelises the per-node loops; the
 * result is independent of the thread count exactly as in the reference
 * (test_backends.py:72-91).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------ */
/* counter-based hash shared with the CUDA generators */
/* ------------------------------------------------------------------------ */
static inline uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint64_t orc_hash(uint64_t seed, uint64_t k, uint64_t l) {
    return splitmix64((seed << 40) + (k << 6) + l);
}

/* 2-D grid, ids i*cols+j; edge order exactly as conftest.grid_graph
 * (pkg/tests/conftest.py:30-41): for each (i,j), down edge then right edge. */
int64_t orc_grid_num_edges(int64_t rows, int64_t cols) {
    if (rows <= 0 || cols <= 0) return 0;
    return rows * (cols - 1) + (rows - 1) * cols;
}

void orc_gen_grid(int64_t rows, int64_t cols, int64_t *edges) {
    int64_t k = 0;
    for (int64_t i = 0; i < rows; ++i)
        for (int64_t j = 0; j < cols; ++j) {
            int64_t u = i * cols + j;
            if (i + 1 < rows) { edges[2 * k] = u; edges[2 * k + 1] = u + cols; ++k; }
            if (j + 1 < cols) { edges[2 * k] = u; edges[2 * k + 1] = u + 1; ++k; }
        }
}

/* Erdos-Renyi style: m uniform endpoint pairs; loops/dupes left to build_csr
 * (conftest.py:53-59). endpoint = hash(seed, k, side) mod n. */
void orc_gen_er(int64_t n, int64_t m, uint64_t seed, int64_t *edges) {
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < m; ++k) {
        edges[2 * k] = (int64_t)(orc_hash(seed, (uint64_t)k, 0) % (uint64_t)n);
        edges[2 * k + 1] = (int64_t)(orc_hash(seed, (uint64_t)k, 1) % (uint64_t)n);
    }
}

/* Graph500-shaped R-MAT without noise or vertex permutation.  For edge k and
 * level l, r = hash(seed,k,l) >> 32 picks the quadrant against integer
 * thresholds of a/b/c = .57/.19/.19 (d = .05); the quadrant's (row, col) bits
 * become bit l of (src, dst). */
#define RMAT_TA 2448131359ULL /* round(0.57 * 2^32) */
#define RMAT_TB 3264175145ULL /* + round(0.19 * 2^32) */
#define RMAT_TC 4080218931ULL /* + round(0.19 * 2^32) */
void orc_gen_rmat(int scale, int64_t m, uint64_t seed, int64_t *edges) {
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < m; ++k) {
        int64_t s = 0, d = 0;
        for (int l = 0; l < scale; ++l) {
            uint64_t r = orc_hash(seed, (uint64_t)k, (uint64_t)l) >> 32;
            int64_t sb = r >= RMAT_TB;                       /* c or d quadrant */
            int64_t db = (r >= RMAT_TA && r < RMAT_TB) || r >= RMAT_TC; /* b or d */
            s |= sb << l;
            d |= db << l;
        }
        edges[2 * k] = s;
        edges[2 * k + 1] = d;
    }
}

/* ------------------------------------------------------------------------ */
/* build_csr (graph.py:184-201): symmetric closure, loops dropped, duplicate */
/* pairs collapsed, adjacency sorted ascending.                               */
/* ------------------------------------------------------------------------ */
static int cmp_i64(const void *a, const void *b) {
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

/* ro: int64[n+1]; ci: capacity 2*m.  Returns num_edges (directed). */
int64_t orc_build_csr(int64_t n, int64_t m, const int64_t *edges, int64_t *ro, int64_t *ci) {
    memset(ro, 0, sizeof(int64_t) * (size_t)(n + 1));
    if (n == 0 || m == 0) return 0;  /* graph.py:188-189 */
    int64_t *deg = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    for (int64_t k = 0; k < m; ++k) {  /* both directions, loops dropped (191-192) */
        int64_t u = edges[2 * k], v = edges[2 * k + 1];
        if (u == v) continue;
        deg[u + 1]++; deg[v + 1]++;
    }
    for (int64_t u = 0; u < n; ++u) deg[u + 1] += deg[u];
    int64_t *cur = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    memcpy(cur, deg, sizeof(int64_t) * (size_t)n);
    for (int64_t k = 0; k < m; ++k) {
        int64_t u = edges[2 * k], v = edges[2 * k + 1];
        if (u == v) continue;
        ci[cur[u]++] = v; ci[cur[v]++] = u;
    }
    /* sort + dedupe each row == np.unique on src*n+dst (195-197) */
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t u = 0; u < n; ++u) {
        int64_t b = deg[u], e = deg[u + 1];
        qsort(ci + b, (size_t)(e - b), sizeof(int64_t), cmp_i64);
        int64_t w = b;
        for (int64_t k = b; k < e; ++k)
            if (k == b || ci[k] != ci[k - 1]) ci[w++] = ci[k];
        cur[u] = w - b;  /* unique count */
    }
    /* compact rows (bincount + cumsum, 199-200) */
    int64_t out = 0;
    for (int64_t u = 0; u < n; ++u) {
        int64_t b = deg[u], c = cur[u];
        ro[u] = out;
        memmove(ci + out, ci + b, sizeof(int64_t) * (size_t)c);
        out += c;
    }
    ro[n] = out;
    free(cur); free(deg);
    return out;
}

/* ------------------------------------------------------------------------ */
/* IPGC solve                                                                */
/* ------------------------------------------------------------------------ */
typedef struct {
    int64_t *colors_read, *colors_write, *stamp; /* ColorState, coloring.py:37-52 */
    int64_t *cur; int64_t cur_len;               /* Worklist.current (sorted)     */
    int64_t *next; int64_t cursor;               /* next_storage + cursor          */
    int64_t *scratch; int nthreads; int64_t scratch_w;
    int64_t n;
} orc_state;

/* assign for one node: _kernels.pyx:29-58.  The reference allocates a fresh
 * zeroed tag row per call and tags with u+1; the oracle keeps one row per
 * thread for the whole solve, so the tag also folds in the round number to
 * stay unique: tag = (round_no-1)*(n+1) + u + 1. */
static inline void assign_node(const int64_t *ro, const int64_t *ci, orc_state *s,
                               int64_t u, int64_t round_no, int64_t *row) {
    int64_t tag = (round_no - 1) * (s->n + 1) + u + 1;
    int64_t lim = ro[u + 1] - ro[u] + 1;
    for (int64_t k = ro[u]; k < ro[u + 1]; ++k) {
        int64_t c = s->colors_read[ci[k]];
        if (1 <= c && c <= lim) row[c] = tag;
    }
    int64_t col = 1;
    while (row[col] == tag) ++col;
    s->colors_write[u] = col;
    s->stamp[u] = round_no;
}

/* resolve for one node: _kernels.pyx:94-120; returns the conflict count and
 * reports the loser through *lost. */
static inline int64_t resolve_node(const int64_t *ro, const int64_t *ci, orc_state *s,
                                   int64_t u, int64_t round_no, int *lost) {
    int64_t cu = s->colors_read[u], cnt = 0;
    for (int64_t k = ro[u]; k < ro[u + 1]; ++k) {
        int64_t v = ci[k];
        if (v < u && s->stamp[v] == round_no && s->colors_read[v] == cu) ++cnt;
    }
    *lost = cnt > 0;
    if (cnt > 0) s->colors_write[u] = 0;
    return cnt;
}

static void push_losers(orc_state *s, const int64_t *cand, int64_t ncand, const char *lost) {
    for (int64_t i = 0; i < ncand; ++i)
        if (lost[i]) s->next[s->cursor++] = cand[i];
}

static int64_t swap_and_sort(orc_state *s) {  /* worklist.py:77-91 */
    int64_t m = s->cursor;
    qsort(s->next, (size_t)m, sizeof(int64_t), cmp_i64);
    int64_t *t = s->cur; s->cur = s->next; s->next = t;
    s->cur_len = m;
    s->cursor = 0;
    return m;
}

static int64_t *row_of(orc_state *s) {
#ifdef _OPENMP
    return s->scratch + (int64_t)omp_get_thread_num() * s->scratch_w;
#else
    return s->scratch;
#endif
}

/* data_driven_iteration, coloring.py:113-142 */
static int64_t data_round(int64_t n, const int64_t *ro, const int64_t *ci, orc_state *s,
                          int64_t round_no, char *lost) {
    int64_t m = s->cur_len;
    const int64_t *nodes = s->cur;
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < m; ++i) assign_node(ro, ci, s, nodes[i], round_no, row_of(s));
    for (int64_t i = 0; i < m; ++i) s->colors_read[nodes[i]] = s->colors_write[nodes[i]]; /* _commit_list (132) */
    int64_t conflicts = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : conflicts)
    for (int64_t i = 0; i < m; ++i) {
        int l;
        conflicts += resolve_node(ro, ci, s, nodes[i], round_no, &l);
        lost[i] = (char)l;
    }
    push_losers(s, nodes, m, lost);
    for (int64_t i = 0; i < m; ++i) s->colors_read[nodes[i]] = s->colors_write[nodes[i]]; /* (140) */
    (void)n;
    return conflicts;
}

/* topology_driven_iteration, coloring.py:145-176 */
static int64_t topo_round(int64_t n, const int64_t *ro, const int64_t *ci, orc_state *s,
                          int64_t round_no, char *lost, int64_t *ids) {
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t u = 0; u < n; ++u)  /* assign_sweep: activity colors_read[u]==0 (_kernels.pyx:76-77) */
        if (s->colors_read[u] == 0) assign_node(ro, ci, s, u, round_no, row_of(s));
    for (int64_t u = 0; u < n; ++u)  /* _commit_stamped (coloring.py:109-110) */
        if (s->stamp[u] == round_no) s->colors_read[u] = s->colors_write[u];
    int64_t conflicts = 0;
#pragma omp parallel for schedule(dynamic, 1024) reduction(+ : conflicts)
    for (int64_t u = 0; u < n; ++u) {  /* resolve_sweep: activity stamp==round (135-136) */
        lost[u] = 0;
        if (s->stamp[u] == round_no) {
            int l;
            conflicts += resolve_node(ro, ci, s, u, round_no, &l);
            lost[u] = (char)l;
        }
    }
    for (int64_t u = 0; u < n; ++u) ids[u] = u;
    push_losers(s, ids, n, lost);
    for (int64_t u = 0; u < n; ++u)
        if (s->stamp[u] == round_no) s->colors_read[u] = s->colors_write[u];
    return conflicts;
}

/* color_graph loop, driver.py:122-176.
 *   mode: 0 = data, 1 = topo, 2 = hybrid;  thr_count = ceil(H*n) (driver.py:138)
 *   colors: int64[n] out
 *   rec: int64[4*max_rec] out: (mode_used 0/1 topo flag, wl_in, wl_out, conflicts)
 * Returns the number of rounds (may exceed max_rec; records beyond are dropped). */
int64_t orc_color(int64_t n, const int64_t *ro, const int64_t *ci, int mode, int64_t thr_count,
                  int64_t *colors, int64_t *rec, int64_t max_rec) {
    orc_state s;
    memset(&s, 0, sizeof s);
    s.n = n;
    s.colors_read = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    s.colors_write = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    s.stamp = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    s.cur = (int64_t *)malloc(sizeof(int64_t) * ((size_t)n + 1));
    s.next = (int64_t *)malloc(sizeof(int64_t) * ((size_t)n + 1));
    int64_t maxdeg = 0;
    for (int64_t u = 0; u < n; ++u)
        if (ro[u + 1] - ro[u] > maxdeg) maxdeg = ro[u + 1] - ro[u];
#ifdef _OPENMP
    s.nthreads = omp_get_max_threads();
#else
    s.nthreads = 1;
#endif
    s.scratch_w = maxdeg + 2;
    s.scratch = (int64_t *)calloc((size_t)s.nthreads * (size_t)s.scratch_w, sizeof(int64_t));
    char *lost = (char *)malloc((size_t)n + 1);
    int64_t *ids = (int64_t *)malloc(sizeof(int64_t) * ((size_t)n + 1));
    for (int64_t u = 0; u < n; ++u) s.cur[u] = u;  /* Worklist.init_full (worklist.py:37-39) */
    s.cur_len = n;

    int64_t round_no = 1;
    while (s.cur_len > 0) {
        int64_t size_in = s.cur_len;
        int topo = mode == 1 ? 1 : mode == 0 ? 0 : (size_in > thr_count); /* driver.py:147-152 */
        int64_t conflicts = topo ? topo_round(n, ro, ci, &s, round_no, lost, ids)
                                 : data_round(n, ro, ci, &s, round_no, lost);
        swap_and_sort(&s);
        if (round_no <= max_rec) {
            int64_t *r = rec + 4 * (round_no - 1);
            r[0] = topo; r[1] = size_in; r[2] = s.cur_len; r[3] = conflicts;
        }
        ++round_no;
    }
    memcpy(colors, s.colors_read, sizeof(int64_t) * (size_t)n);
    free(s.colors_read); free(s.colors_write); free(s.stamp); free(s.cur); free(s.next);
    free(s.scratch); free(lost); free(ids);
    return round_no - 1;
}

/* verify_coloring, driver.py:188-204 */
int64_t orc_verify(int64_t n, const int64_t *ro, const int64_t *ci, const int64_t *colors) {
    int64_t bad = 0;
#pragma omp parallel for schedule(dynamic, 1024) reduction(+ : bad)
    for (int64_t u = 0; u < n; ++u)
        for (int64_t k = ro[u]; k < ro[u + 1]; ++k) {
            int64_t v = ci[k];
            if (u < v && (colors[u] == colors[v] || colors[u] == 0)) ++bad;
        }
    return bad;
}

/* colors_used, driver.py:179-185: -1 signals the reference's ValueError. */
int64_t orc_colors_used(int64_t n, const int64_t *colors) {
    if (n == 0) return 0;
    int64_t mx = colors[0];
    for (int64_t u = 0; u < n; ++u) {
        if (colors[u] < 1) return -1;
        if (colors[u] > mx) mx = colors[u];
    }
    return mx;
}

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
