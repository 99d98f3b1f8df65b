/*
 * irls_oracle.c — plain, slow, float64 CPU oracle for the IRLS s-t min-cut
 * hot path of Zhu & Gleich, "A Parallel Min-Cut Algorithm using Iteratively
 * Reweighted Least Squares" (arXiv 1501.03105).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.  It
 * shares no code, header, table or helper with the CUDA path
 * (paper_1501_03105_b200/csrc); the two meet only in the seeded inputs of
 * synthetic/generators.py.
 *
 * Citations: "P:Lnnn" = /root/reference/PAPER.md line nnn (equation numbers
 * as in SURVEY.md §0); "S:Lnnn" = SPEC.md; "A<k>" / "O<k>" / "C<k>" =
 * readings and arithmetic contract recorded in DESIGN.md §2 (taken from
 * SURVEY.md §8(c)).
 *
 * Arithmetic: float64, compiled with -ffp-contract=off (C1: no FMA); sqrt and
 * '/' are IEEE round-to-nearest.  Every sum follows the order stated at the
 * point of use (C2 ascending neighbour id; C3 fixed reduction tree), so the
 * results are a function of the inputs alone.
 *
 * Parity status: every function below is pinned by the
 * `-m "not gpu"` tests in tests/test_oracle_*.py — closed forms, SPEC worked
 * examples, dense numpy solves, brute-force cut enumeration, networkx max
 * flow, invariants.  Functions with no independent pin say so in their
 * comment ("parity unpinned").
 */
#include <math.h>
#include <stdint.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#include <stdlib.h>
#include <string.h>

/* Threads (SURVEY §8(d) "OpenMP over C3 chunks"): every parallel loop below
 * computes elements independently (a node's value from its own inputs in C2
 * order, a chunk's C3 partial from its own 4096 elements), so the results
 * are bitwise independent of the thread count (pinned by
 * tests/test_oracle_threads.py).  Sums across elements happen only in the
 * fixed C3 tree; a block-Jacobi block (A32) is solved by one thread.  Loops
 * run in parallel only above a size where threads pay for themselves. */

int orc_set_num_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
    return omp_get_max_threads();
#else
    (void)n;
    return 1;
#endif
}

/* status codes: numerically equal to irls_status in include/irls_mincut.h by
 * specification; deliberately not shared. */
enum {
    ORC_OK = 0,
    ORC_ERR_INVALID_ARGUMENT = 1,
    ORC_ERR_SOURCE_EQUALS_SINK = 2,
    ORC_ERR_BAD_CAPACITY = 3,
    ORC_ERR_NOT_SYMMETRIC = 4,
    ORC_ERR_SINGULAR = 5,
    ORC_ERR_CG_BREAKDOWN = 6,
    ORC_ERR_BAD_POTENTIAL = 7,
    ORC_ERR_STATE = 8,
    ORC_ERR_OOM = 11,
};

/* ------------------------------------------------------------------------- */
/* Graph: the non-terminal graph G~ in reduced ids, plus the terminal */
/* edges E^T as per-node capacities cs/ct and the direct s-t capacity (A5).  */
/* ------------------------------------------------------------------------- */
typedef struct {
    int64_t n;          /* number of non-terminal nodes (n~) */
    int64_t *adj_ptr;   /* n+1 */
    int64_t *adj_idx;   /* neighbour reduced ids, strictly ascending (C2) */
    double *adj_c;      /* n-link capacities, > 0 (A6: c = 0 is absent) */
    double *cs, *ct;    /* terminal capacities (0 = absent) */
    double c_st;        /* direct s-t capacity (A5) */
    int64_t n_total;    /* ids in outputs: stencil N+2, CSR n */
    int64_t *orig;      /* reduced id -> output id */
    int64_t s_id, t_id; /* output ids of s and t */
} orc_graph;

static int is_bad_cap(double c) { return !(c >= 0.0) || isinf(c); }

void orc_graph_free(orc_graph *g)
{
    if (!g) return;
    free(g->adj_ptr); free(g->adj_idx); free(g->adj_c);
    free(g->cs); free(g->ct); free(g->orig); free(g);
}

static orc_graph *graph_alloc(int64_t n, int64_t nnz)
{
    orc_graph *g = (orc_graph *)calloc(1, sizeof(orc_graph));
    if (!g) return NULL;
    g->n = n;
    g->adj_ptr = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    g->adj_idx = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nnz > 0 ? nnz : 1));
    g->adj_c = (double *)malloc(sizeof(double) * (size_t)(nnz > 0 ? nnz : 1));
    g->cs = (double *)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
    g->ct = (double *)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
    g->orig = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    if (!g->adj_ptr || !g->adj_idx || !g->adj_c || !g->cs || !g->ct || !g->orig) {
        orc_graph_free(g);
        return NULL;
    }
    return g;
}

/* Stencil input: node u = x + nx*(y + ny*z); cx[u] = c(u,u+1),
 * cy[u] = c(u,u+nx), cz[u] = c(u,u+nx*ny); entries past the grid edge are
 * ignored.  s = N, t = N+1 are virtual.  Ascending neighbour order of a grid
 * node is (-z, -y, -x, +x, +y, +z) (C2).  Zero capacities are absent (A6). */
int orc_graph_from_stencil(orc_graph **out, int64_t nx, int64_t ny, int64_t nz,
                           const double *cx, const double *cy, const double *cz,
                           const double *cs, const double *ct)
{
    *out = NULL;
    if (nx < 1 || ny < 1 || nz < 1) return ORC_ERR_INVALID_ARGUMENT;
    int64_t N = nx * ny * nz, pl = nx * ny;
    for (int64_t u = 0; u < N; u++) {
        int64_t x = u % nx, y = (u / nx) % ny, z = u / pl;
        if (x < nx - 1 && is_bad_cap(cx[u])) return ORC_ERR_BAD_CAPACITY;
        if (y < ny - 1 && is_bad_cap(cy[u])) return ORC_ERR_BAD_CAPACITY;
        if (z < nz - 1 && is_bad_cap(cz[u])) return ORC_ERR_BAD_CAPACITY;
        if (is_bad_cap(cs[u]) || is_bad_cap(ct[u])) return ORC_ERR_BAD_CAPACITY;
    }
    orc_graph *g = graph_alloc(N, 6 * N);
    if (!g) return ORC_ERR_OOM;
    int64_t k = 0;
    for (int64_t u = 0; u < N; u++) {
        int64_t x = u % nx, y = (u / nx) % ny, z = u / pl;
        g->adj_ptr[u] = k;
#define PUSH(cond, v, c) do { if ((cond) && (c) > 0.0) { g->adj_idx[k] = (v); g->adj_c[k] = (c); k++; } } while (0)
        PUSH(z > 0, u - pl, (z > 0 ? cz[u - pl] : 0.0));
        PUSH(y > 0, u - nx, (y > 0 ? cy[u - nx] : 0.0));
        PUSH(x > 0, u - 1, (x > 0 ? cx[u - 1] : 0.0));
        PUSH(x < nx - 1, u + 1, cx[u]);
        PUSH(y < ny - 1, u + nx, cy[u]);
        PUSH(z < nz - 1, u + pl, cz[u]);
#undef PUSH
        g->cs[u] = cs[u];
        g->ct[u] = ct[u];
        g->orig[u] = u;
    }
    g->adj_ptr[N] = k;
    g->c_st = 0.0;
    g->n_total = N + 2;
    g->s_id = N;
    g->t_id = N + 1;
    *out = g;
    return ORC_OK;
}

typedef struct { int64_t col; int64_t pos; double w; } csr_ent;

static int ent_cmp(const void *a, const void *b)
{
    const csr_ent *x = (const csr_ent *)a, *y = (const csr_ent *)b;
    if (x->col != y->col) return x->col < y->col ? -1 : 1;
    return x->pos < y->pos ? -1 : (x->pos > y->pos);
}

/* CSR input over all n nodes including s and t.  Duplicate
 * entries of a row are merged by summation in CSR order (A7); self
 * loops are rejected; the merged matrix must be exactly symmetric.  The edge
 * {s,t} becomes the additive constant c_st (A5). */
int orc_graph_from_csr(orc_graph **out, int64_t n, const int64_t *row_ptr,
                       const int32_t *col, const double *w, int64_t s, int64_t t)
{
    *out = NULL;
    if (n < 2 || s < 0 || t < 0 || s >= n || t >= n) return ORC_ERR_INVALID_ARGUMENT;
    if (s == t) return ORC_ERR_SOURCE_EQUALS_SINK;
    if (row_ptr[0] != 0) return ORC_ERR_INVALID_ARGUMENT;
    for (int64_t u = 0; u < n; u++)
        if (row_ptr[u + 1] < row_ptr[u]) return ORC_ERR_INVALID_ARGUMENT;
    int64_t nnz = row_ptr[n];
    for (int64_t e = 0; e < nnz; e++) {
        if (col[e] < 0 || col[e] >= n) return ORC_ERR_INVALID_ARGUMENT;
        if (is_bad_cap(w[e])) return ORC_ERR_BAD_CAPACITY;
    }
    for (int64_t u = 0; u < n; u++)
        for (int64_t e = row_ptr[u]; e < row_ptr[u + 1]; e++)
            if (col[e] == u) return ORC_ERR_INVALID_ARGUMENT;

    /* merged rows: sort each row's entries by (col, position), sum runs */
    int64_t *mptr = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    int64_t *mcol = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nnz > 0 ? nnz : 1));
    double *mw = (double *)malloc(sizeof(double) * (size_t)(nnz > 0 ? nnz : 1));
    csr_ent *tmp = (csr_ent *)malloc(sizeof(csr_ent) * (size_t)(nnz > 0 ? nnz : 1));
    if (!mptr || !mcol || !mw || !tmp) { free(mptr); free(mcol); free(mw); free(tmp); return ORC_ERR_OOM; }
    int64_t m = 0;
    for (int64_t u = 0; u < n; u++) {
        int64_t a = row_ptr[u], b = row_ptr[u + 1];
        for (int64_t e = a; e < b; e++) { tmp[e - a].col = col[e]; tmp[e - a].pos = e; tmp[e - a].w = w[e]; }
        qsort(tmp, (size_t)(b - a), sizeof(csr_ent), ent_cmp);
        mptr[u] = m;
        for (int64_t i = 0; i < b - a; i++) {
            if (i > 0 && tmp[i].col == tmp[i - 1].col) {
                mw[m - 1] = mw[m - 1] + tmp[i].w;
            } else {
                mcol[m] = tmp[i].col; mw[m] = tmp[i].w; m++;
            }
        }
    }
    mptr[n] = m;
    free(tmp);
    /* exact symmetry of the merged matrix */
    int rc = ORC_OK;
    for (int64_t u = 0; u < n && rc == ORC_OK; u++) {
        for (int64_t e = mptr[u]; e < mptr[u + 1]; e++) {
            int64_t v = mcol[e];
            int64_t lo = mptr[v], hi = mptr[v + 1], found = -1;
            while (lo < hi) { int64_t mid = (lo + hi) / 2; if (mcol[mid] < u) lo = mid + 1; else hi = mid; }
            if (lo < mptr[v + 1] && mcol[lo] == u) found = lo;
            if (found < 0 || mw[found] != mw[e]) { rc = ORC_ERR_NOT_SYMMETRIC; break; }
        }
    }
    if (rc != ORC_OK) { free(mptr); free(mcol); free(mw); return rc; }

    int64_t nr = n - 2;
    int64_t nn = 0;
    for (int64_t u = 0; u < n; u++) {
        if (u == s || u == t) continue;
        for (int64_t e = mptr[u]; e < mptr[u + 1]; e++)
            if (mcol[e] != s && mcol[e] != t && mw[e] > 0.0) nn++;
    }
    orc_graph *g = graph_alloc(nr, nn);
    if (!g) { free(mptr); free(mcol); free(mw); return ORC_ERR_OOM; }
    int64_t k = 0, r = 0;
    for (int64_t u = 0; u < n; u++) {
        if (u == s || u == t) continue;
        g->adj_ptr[r] = k;
        g->orig[r] = u;
        for (int64_t e = mptr[u]; e < mptr[u + 1]; e++) {
            int64_t v = mcol[e];
            if (v == s) g->cs[r] = mw[e];
            else if (v == t) g->ct[r] = mw[e];
            else if (mw[e] > 0.0) {
                g->adj_idx[k] = v - (v > s) - (v > t); /* reduced id, monotone in v */
                g->adj_c[k] = mw[e];
                k++;
            }
        }
        r++;
    }
    g->adj_ptr[nr] = k;
    g->c_st = 0.0;
    for (int64_t e = mptr[s]; e < mptr[s + 1]; e++)
        if (mcol[e] == t) g->c_st = mw[e];
    g->n_total = n;
    g->s_id = s;
    g->t_id = t;
    free(mptr); free(mcol); free(mw);
    *out = g;
    return ORC_OK;
}

int64_t orc_graph_n(const orc_graph *g) { return g->n; }
int64_t orc_graph_n_total(const orc_graph *g) { return g->n_total; }
int64_t orc_graph_nnz(const orc_graph *g) { return g->adj_ptr[g->n]; }
double orc_graph_c_st(const orc_graph *g) { return g->c_st; }
void orc_graph_orig_ids(const orc_graph *g, int64_t *out)
{
    for (int64_t u = 0; u < g->n; u++) out[u] = g->orig[u];
}
void orc_graph_terminals(const orc_graph *g, double *cs, double *ct)
{
    for (int64_t u = 0; u < g->n; u++) { cs[u] = g->cs[u]; ct[u] = g->ct[u]; }
}

/* Prop. 1 / A8: L~ is nonsingular iff every connected component
 * of G~ (edges with c > 0) contains a node with a positive terminal edge.
 * Plain BFS.  Returns ORC_OK or ORC_ERR_SINGULAR. */
int orc_check_nonsingular(const orc_graph *g)
{
    int64_t n = g->n;
    if (n == 0) return ORC_OK;
    int64_t *queue = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    char *seen = (char *)calloc((size_t)n, 1);
    if (!queue || !seen) { free(queue); free(seen); return ORC_ERR_OOM; }
    int rc = ORC_OK;
    for (int64_t r = 0; r < n && rc == ORC_OK; r++) {
        if (seen[r]) continue;
        int64_t head = 0, tail = 0; int anchored = 0;
        queue[tail++] = r; seen[r] = 1;
        while (head < tail) {
            int64_t u = queue[head++];
            if (g->cs[u] > 0.0 || g->ct[u] > 0.0) anchored = 1;
            for (int64_t e = g->adj_ptr[u]; e < g->adj_ptr[u + 1]; e++) {
                int64_t v = g->adj_idx[e];
                if (!seen[v]) { seen[v] = 1; queue[tail++] = v; }
            }
        }
        if (!anchored) rc = ORC_ERR_SINGULAR;
    }
    free(queue); free(seen);
    return rc;
}

/* ------------------------------------------------------------------------- */
/* C3: the fixed reduction tree (contract C3).                 */
/* ------------------------------------------------------------------------- */
#define C3_CHUNK 4096
#define C3_THREADS 256
#define C3_GROUPS 8

/* One 4096-element chunk starting at `base` of v[0..n): "thread" t sums
 * sequentially from +0.0 the elements base+2t+512j+v (j=0..7, v=0,1); the 32
 * lanes of each warp combine by offsets 16,8,4,2,1 (lane i += lane i+off);
 * the 8 warp sums by offsets 4,2,1.  Elements past n contribute nothing. */
static double c3_chunk(const double *v, int64_t n, int64_t base)
{
    double th[C3_THREADS];
    for (int t = 0; t < C3_THREADS; t++) {
        double acc = 0.0;
        for (int j = 0; j < 8; j++)
            for (int q = 0; q < 2; q++) {
                int64_t i = base + 2 * t + 512 * j + q;
                if (i < n) acc = acc + v[i];
            }
        th[t] = acc;
    }
    double ws[8];
    for (int w = 0; w < 8; w++) {
        double *lane = th + 32 * w;
        for (int off = 16; off >= 1; off /= 2)
            for (int i = 0; i < off; i++) lane[i] = lane[i] + lane[i + off];
        ws[w] = lane[0];
    }
    for (int off = 4; off >= 1; off /= 2)
        for (int i = 0; i < off; i++) ws[i] = ws[i] + ws[i + off];
    return ws[0];
}

/* A list of m values reduced chunk by chunk, repeated until one remains. */
static double c3_list(double *a, int64_t m)
{
    if (m == 0) return 0.0;
    while (m > 1) {
        int64_t K = (m + C3_CHUNK - 1) / C3_CHUNK;
        for (int64_t k = 0; k < K; k++) a[k] = c3_chunk(a, m, k * C3_CHUNK); /* in place: sequential */
        m = K;
    }
    return a[0];
}

/* Full C3 sum of v[0..n): chunk partials; 8 groups covering chunks
 * [floor(gK/8), floor((g+1)K/8)); each group reduced as a fresh list; the 8
 * group sums combined by offsets 4,2,1. */
double orc_c3_sum(const double *v, int64_t n)
{
    int64_t K = (n + C3_CHUNK - 1) / C3_CHUNK;
    double *part = (double *)malloc(sizeof(double) * (size_t)(K > 0 ? K : 1));
    double gs[C3_GROUPS];
#pragma omp parallel for schedule(static) if((K) > 16)
    for (int64_t k = 0; k < K; k++) part[k] = c3_chunk(v, n, k * C3_CHUNK);
    for (int g = 0; g < C3_GROUPS; g++) {
        int64_t lo = (int64_t)g * K / C3_GROUPS, hi = (int64_t)(g + 1) * K / C3_GROUPS;
        gs[g] = c3_list(part + lo, hi - lo);
    }
    free(part);
    for (int off = 4; off >= 1; off /= 2)
        for (int i = 0; i < off; i++) gs[i] = gs[i] + gs[i + off];
    return gs[0];
}

/* Group sums only (the 8 values before the final tree), for the multi-rank
 * slot-exact allreduce tests. */
void orc_c3_group_sums(const double *v, int64_t n, double *out8)
{
    int64_t K = (n + C3_CHUNK - 1) / C3_CHUNK;
    double *part = (double *)malloc(sizeof(double) * (size_t)(K > 0 ? K : 1));
#pragma omp parallel for schedule(static) if((K) > 16)
    for (int64_t k = 0; k < K; k++) part[k] = c3_chunk(v, n, k * C3_CHUNK);
    for (int g = 0; g < C3_GROUPS; g++) {
        int64_t lo = (int64_t)g * K / C3_GROUPS, hi = (int64_t)(g + 1) * K / C3_GROUPS;
        out8[g] = c3_list(part + lo, hi - lo);
    }
    free(part);
}

/* ------------------------------------------------------------------------- */
/* Assembly: Eq. 4 reweighting, Eq. 8 reweighted Laplacian, Eq. 7 reduction.  */
/* ------------------------------------------------------------------------- */

/* Eq. 4 with A2: w = sqrt((c*d)^2 + eps^2); Eq. 8:
 * the edge's conductance in L^(l) is c^2 / w  (O3). */
static double reweight_g(double c, double d, double eps2)
{
    double a = c * d;
    double w = sqrt(a * a + eps2);
    return (c * c) / w;
}

typedef struct {
    const orc_graph *G;
    double *g;     /* per adjacency entry conductance */
    double *gs, *gt, *D, *Dinv;
    double *x, *r, *z, *p, *q;
    double *w, *sv;  /* CG-CG: w = A z, s = A p */
    double *tmp;
    double eps;
    int32_t T, cg_max_iter, cg_norm, warm_start, cg_variant;
    double cg_rtol;
    int32_t step;  /* number of solves done (0 = none) */
    double *cs, *ct; /* owned copy of terminal capacities (set_terminal_weights) */
    const double *bvec; /* right-hand side override (lambda2); NULL: b = gs (Eq. 7) */
    /* block-Jacobi preconditioner (A32; block_size 0 = point Jacobi) */
    int32_t block_size;
    int64_t nblk;
    int64_t *bptr;      /* nblk+1: block b holds positions bptr[b]..bptr[b+1]-1 */
    int64_t *bnode;     /* n: reduced id at each position (block order) */
    int64_t *bpos;      /* n: position of each reduced id */
    int64_t *bfirst;    /* n: first column f_i of the row at each position (block-local index) */
    int64_t *boff;      /* n+1: start of each row's envelope entries in bL */
    double *bL, *bDd;   /* envelope of the unit lower factor; pivots (block order) */
    double *by;         /* scratch (block order) */
} orc_state;

typedef struct {
    double eps;
    int32_t T;
    double cg_rtol;
    int32_t cg_max_iter;
    int32_t cg_norm;      /* 0 = preconditioned (A9), 1 = unpreconditioned */
    int32_t warm_start;
    int32_t cg_variant;   /* 0 = Hestenes-Stiefel (O5), 1 = Chronopoulos-Gear (O5', A31) */
    int32_t block_size;   /* 0 = point Jacobi M = diag(L~) (A12); B >= 1: block Jacobi (A32) */
} orc_options;

typedef struct {
    int32_t cg_iters, converged;
    double rel_res;       /* recursive residual norm / ref at exit */
    double true_rel_res;  /* ||b - A x|| (same norm) / ref */
    double S_eps;         /* Eq. 9 at x^(l) */
    double flow_value;    /* Prop. 3: x^T L^(l) x */
    double current_s;     /* sum_u gs_u (1 - x_u) */
    double x_min, x_max;
    double ref;
} orc_report;

void orc_state_free(orc_state *S)
{
    if (!S) return;
    free(S->g); free(S->gs); free(S->gt); free(S->D); free(S->Dinv);
    free(S->x); free(S->r); free(S->z); free(S->p); free(S->q); free(S->w); free(S->sv); free(S->tmp);
    free(S->cs); free(S->ct);
    free(S->bptr); free(S->bnode); free(S->bpos); free(S->bfirst); free(S->boff); free(S->bL); free(S->bDd);
    free(S->by); free(S);
}

/* ------------------------------------------------------------------------- */
/* Block-Jacobi preconditioner ("block      */
/* Jacobi" with "LU" blocks).  Reading A32 in DESIGN.md §2.           */
/* ------------------------------------------------------------------------- */

/* A32 partition.  For each C3 group g = 0..7 (ids [4096 floor(gK/8),
 * 4096 floor((g+1)K/8)) clipped to n) and each id u of the group ascending:
 * if u is unassigned it opens a new block; then the earliest node v of the
 * block not yet expanded is expanded — its neighbours w (ascending id, c > 0)
 * inside the group and unassigned are appended in that order — until the
 * block holds B nodes or all its nodes are expanded.  Block order = append
 * order.  Writes bptr[nblk+1], bnode[n]; returns nblk (-1 on OOM). */
int64_t orc_block_partition(const orc_graph *G, int32_t B, int64_t *bptr, int64_t *bnode)
{
    int64_t n = G->n, K = (n + C3_CHUNK - 1) / C3_CHUNK, nb = 0, cnt = 0;
    uint8_t *used = (uint8_t *)calloc((size_t)(n > 0 ? n : 1), 1);
    if (!used) return -1;
    for (int g = 0; g < C3_GROUPS; g++) {
        int64_t lo = (int64_t)g * K / C3_GROUPS * C3_CHUNK, hi = (int64_t)(g + 1) * K / C3_GROUPS * C3_CHUNK;
        if (lo > n) lo = n;
        if (hi > n) hi = n;
        for (int64_t u = lo; u < hi; u++) {
            if (used[u]) continue;
            int64_t start = cnt, head = cnt;
            bptr[nb++] = start;
            bnode[cnt++] = u;
            used[u] = 1;
            while (head < cnt && cnt - start < B) {
                int64_t v = bnode[head++];
                for (int64_t e = G->adj_ptr[v]; e < G->adj_ptr[v + 1] && cnt - start < B; e++) {
                    int64_t w = G->adj_idx[e];
                    if (w < lo || w >= hi || used[w]) continue;
                    used[w] = 1;
                    bnode[cnt++] = w;
                }
            }
        }
    }
    bptr[nb] = cnt;
    free(used);
    return nb;
}

/* Envelope of each block row (A32): f_i = the smallest block position among
 * position i and its in-block neighbours.  Row i of the unit lower factor
 * lives in columns [f_i, i) (LDL^T fills only inside the envelope). */
static int block_setup(orc_state *S)
{
    const orc_graph *G = S->G;
    int64_t n = G->n, N1 = n > 0 ? n : 1;
    S->bptr = (int64_t *)malloc(sizeof(int64_t) * (size_t)(N1 + 1));
    S->bnode = (int64_t *)malloc(sizeof(int64_t) * (size_t)N1);
    S->bpos = (int64_t *)malloc(sizeof(int64_t) * (size_t)N1);
    S->bfirst = (int64_t *)malloc(sizeof(int64_t) * (size_t)N1);
    S->boff = (int64_t *)malloc(sizeof(int64_t) * (size_t)(N1 + 1));
    S->bDd = (double *)malloc(sizeof(double) * (size_t)N1);
    S->by = (double *)malloc(sizeof(double) * (size_t)N1);
    if (!S->bptr || !S->bnode || !S->bpos || !S->bfirst || !S->boff || !S->bDd || !S->by) return ORC_ERR_OOM;
    S->nblk = orc_block_partition(G, S->block_size, S->bptr, S->bnode);
    if (S->nblk < 0) return ORC_ERR_OOM;
    for (int64_t i = 0; i < n; i++) S->bpos[S->bnode[i]] = i;
    S->boff[0] = 0;
    for (int64_t b = 0; b < S->nblk; b++)
        for (int64_t i = S->bptr[b]; i < S->bptr[b + 1]; i++) {
            int64_t u = S->bnode[i], f = i;
            for (int64_t e = G->adj_ptr[u]; e < G->adj_ptr[u + 1]; e++) {
                int64_t j = S->bpos[G->adj_idx[e]];
                if (j >= S->bptr[b] && j < f) f = j;
            }
            S->bfirst[i] = f - S->bptr[b];
            S->boff[i + 1] = S->boff[i] + (i - f);
        }
    S->bL = (double *)malloc(sizeof(double) * (size_t)(S->boff[n] > 0 ? S->boff[n] : 1));
    return S->bL ? ORC_OK : ORC_ERR_OOM;
}

/* A32 factorisation of every block of L~ (after assemble): A_B = L~ restricted
 * to the block in block order (A_ii = D_u, A_ij = -g_uv for an n-link inside
 * the block, +0.0 otherwise); LDL^T by rows (Crout), every sum over k
 * ascending:
 *   L_ij = (A_ij - sum_k (L_ik * L_jk) * d_k) / d_j,  k in [max(f_i, f_j), j)
 *   d_i  =  A_ii - sum_k (L_ik * L_ik) * d_k,         k in [f_i, i)
 * (terms outside the envelope are exact zeros of the dense algorithm, which
 * leave every sum bitwise unchanged — pinned against a dense factorisation). */
static void block_factor(orc_state *S)
{
    const orc_graph *G = S->G;
#pragma omp parallel for schedule(static) if((S->nblk) > 64)
    for (int64_t b = 0; b < S->nblk; b++) {
        int64_t p0 = S->bptr[b], p1 = S->bptr[b + 1];
        for (int64_t i = p0; i < p1; i++) {
            int64_t u = S->bnode[i], fi = S->bfirst[i];
            double *Li = S->bL + S->boff[i] - fi;           /* Li[j], j in [fi, i - p0) */
            for (int64_t j = fi; j < i - p0; j++) Li[j] = 0.0;
            for (int64_t e = G->adj_ptr[u]; e < G->adj_ptr[u + 1]; e++) {
                int64_t j = S->bpos[G->adj_idx[e]] - p0;
                if (j >= fi && j < i - p0) Li[j] = -S->g[e];
            }
            for (int64_t j = fi; j < i - p0; j++) {
                int64_t fj = S->bfirst[p0 + j];
                const double *Lj = S->bL + S->boff[p0 + j] - fj;
                double acc = Li[j];
                for (int64_t k = fi > fj ? fi : fj; k < j; k++) acc = acc - (Li[k] * Lj[k]) * S->bDd[p0 + k];
                Li[j] = acc / S->bDd[p0 + j];
            }
            double acc = S->D[u];
            for (int64_t k = fi; k < i - p0; k++) acc = acc - (Li[k] * Li[k]) * S->bDd[p0 + k];
            S->bDd[i] = acc;
        }
    }
}

/* z = M^-1 r.  Point Jacobi: z_u = r_u * Dinv_u (O5).  Block Jacobi (A32),
 * per block: forward y_i = r_i - sum_{k in [f_i, i), ascending} L_ik * y_k;
 * w_i = y_i / d_i; backward, rows i descending: z_i = w_i after every later
 * row's updates, then z_k = z_k - L_ik * z_i for k in [f_i, i). */
static void precond_apply(orc_state *S, const double *r, double *z)
{
    int64_t n = S->G->n;
    if (S->block_size <= 0) {
#pragma omp parallel for schedule(static) if((n) > 32768)
        for (int64_t u = 0; u < n; u++) z[u] = r[u] * S->Dinv[u];
        return;
    }
    double *y = S->by;
#pragma omp parallel for schedule(static) if((S->nblk) > 64)
    for (int64_t b = 0; b < S->nblk; b++) {
        int64_t p0 = S->bptr[b], p1 = S->bptr[b + 1];
        for (int64_t i = p0; i < p1; i++) {
            int64_t fi = S->bfirst[i];
            const double *Li = S->bL + S->boff[i] - fi;
            double acc = r[S->bnode[i]];
            for (int64_t k = fi; k < i - p0; k++) acc = acc - Li[k] * y[p0 + k];
            y[i] = acc;
        }
        for (int64_t i = p0; i < p1; i++) y[i] = y[i] / S->bDd[i];
        for (int64_t i = p1 - 1; i >= p0; i--) {
            int64_t fi = S->bfirst[i];
            const double *Li = S->bL + S->boff[i] - fi;
            for (int64_t k = fi; k < i - p0; k++) y[p0 + k] = y[p0 + k] - Li[k] * y[i];
        }
        for (int64_t i = p0; i < p1; i++) z[S->bnode[i]] = y[i];
    }
}

orc_state *orc_state_new(const orc_graph *G, const orc_options *o)
{
    orc_state *S = (orc_state *)calloc(1, sizeof(orc_state));
    if (!S) return NULL;
    int64_t n = G->n > 0 ? G->n : 1, m = G->adj_ptr[G->n] > 0 ? G->adj_ptr[G->n] : 1;
    S->G = G;
    S->g = (double *)calloc((size_t)m, sizeof(double));
    double **vecs[] = {&S->gs, &S->gt, &S->D, &S->Dinv, &S->x, &S->r, &S->z, &S->p, &S->q, &S->w, &S->sv,
                       &S->tmp, &S->cs, &S->ct};
    for (size_t i = 0; i < sizeof(vecs) / sizeof(vecs[0]); i++) {
        *vecs[i] = (double *)calloc((size_t)n, sizeof(double));
        if (!*vecs[i]) { orc_state_free(S); return NULL; }
    }
    if (!S->g) { orc_state_free(S); return NULL; }
    for (int64_t u = 0; u < G->n; u++) { S->cs[u] = G->cs[u]; S->ct[u] = G->ct[u]; }
    S->eps = o->eps; S->T = o->T; S->cg_rtol = o->cg_rtol; S->cg_max_iter = o->cg_max_iter;
    S->cg_norm = o->cg_norm; S->warm_start = o->warm_start; S->cg_variant = o->cg_variant;
    S->step = 0;
    S->block_size = o->block_size;
    if (S->block_size < 0 || (S->block_size > 0 && S->cg_variant != 0)) { orc_state_free(S); return NULL; }
    if (S->block_size > 0 && block_setup(S) != ORC_OK) { orc_state_free(S); return NULL; }
    return S;
}

/* O1 + O3/O4: conductances of every edge from x (or g = c when x == NULL,
 * i.e. W^(0) = C), then D_u = ((sum_asc g_uv) + gs_u) + gt_u,
 * Dinv_u = 1/D_u, b_u = gs_u (Eq. 7: b = -Z^T L e_s, x_s = 1, x_t = 0). */
static void assemble(orc_state *S, const double *x)
{
    const orc_graph *G = S->G;
    double eps2 = S->eps * S->eps;
#pragma omp parallel for schedule(static) if((G->n) > 32768)
    for (int64_t u = 0; u < G->n; u++) {
        double acc = 0.0;
        for (int64_t e = G->adj_ptr[u]; e < G->adj_ptr[u + 1]; e++) {
            double c = G->adj_c[e];
            double gv = x ? reweight_g(c, x[u] - x[G->adj_idx[e]], eps2) : c;
            S->g[e] = gv;
            acc = acc + gv;
        }
        double cs = S->cs[u], ct = S->ct[u];
        /* A3: terminal edges are reweighted with x_s = 1, x_t = 0 */
        double gs = x ? reweight_g(cs, 1.0 - x[u], eps2) : cs;
        double gt = x ? reweight_g(ct, x[u], eps2) : ct;
        S->gs[u] = gs; S->gt[u] = gt;
        S->D[u] = (acc + gs) + gt;
        S->Dinv[u] = 1.0 / S->D[u];
    }
}

/* O2: q = L~ p with acc = sum_asc g_uv p_v from +0.0, q_u = D_u p_u - acc. */
static void matvec(const orc_state *S, const double *p, double *q)
{
    const orc_graph *G = S->G;
#pragma omp parallel for schedule(static) if((G->n) > 32768)
    for (int64_t u = 0; u < G->n; u++) {
        double acc = 0.0;
        for (int64_t e = G->adj_ptr[u]; e < G->adj_ptr[u + 1]; e++)
            acc = acc + S->g[e] * p[G->adj_idx[e]];
        q[u] = S->D[u] * p[u] - acc;
    }
}

static double dot_c3(orc_state *S, const double *a, const double *b)
{
#pragma omp parallel for schedule(static) if((S->G->n) > 32768)
    for (int64_t u = 0; u < S->G->n; u++) S->tmp[u] = a[u] * b[u];
    return orc_c3_sum(S->tmp, S->G->n);
}

/* O5: Jacobi-preconditioned CG ("preconditioned conjugate gradient")
 * on L~ v = b with M = diag(L~) (A12) or the block-Jacobi M of A32
 * (z = M^-1 r by precond_apply; ref = ||M^-1 b||), Hestenes-Stiefel form, warm start x0
 * = S->x, stopping test res <= rtol*ref before each iteration (A9,
 * A13). */
static int pcg(orc_state *S, orc_report *rep)
{
    const orc_graph *G = S->G;
    int64_t n = G->n;
    double *x = S->x, *r = S->r, *z = S->z, *p = S->p, *q = S->q;
    /* r = b - A x0 */
    matvec(S, x, q);
    const double *b = S->bvec ? S->bvec : S->gs;
#pragma omp parallel for schedule(static) if((n) > 32768)
    for (int64_t u = 0; u < n; u++) r[u] = b[u] - q[u];
    precond_apply(S, r, z);
#pragma omp parallel for schedule(static) if((n) > 32768)
    for (int64_t u = 0; u < n; u++) p[u] = z[u];
    double rho = dot_c3(S, r, z);
    double ref2;
    if (S->cg_norm == 0) {
        double *mb = S->w;                      /* M^-1 b (w is CG-CG's; free here) */
        precond_apply(S, b, mb);
#pragma omp parallel for schedule(static) if((n) > 32768)
        for (int64_t u = 0; u < n; u++) S->tmp[u] = mb[u] * mb[u];
        ref2 = orc_c3_sum(S->tmp, n);
    } else {
        ref2 = dot_c3(S, b, b);
    }
    double ref = sqrt(ref2);
    rep->ref = ref;
    if (ref == 0.0) { /* b = 0 => v = 0 */
        for (int64_t u = 0; u < n; u++) x[u] = 0.0;
        rep->cg_iters = 0; rep->converged = 1; rep->rel_res = 0.0;
        return ORC_OK;
    }
    double res2 = S->cg_norm == 0 ? dot_c3(S, z, z) : dot_c3(S, r, r);
    double res = sqrt(res2);
    int32_t k = 0;
    for (;;) {
        if (res <= S->cg_rtol * ref || k == S->cg_max_iter) break;
        matvec(S, p, q);
        double pi = dot_c3(S, p, q);
        if (!(pi > 0.0) || isinf(pi)) return ORC_ERR_CG_BREAKDOWN;
        double alpha = rho / pi;
#pragma omp parallel for schedule(static) if((n) > 32768)
        for (int64_t u = 0; u < n; u++) x[u] = x[u] + alpha * p[u];
#pragma omp parallel for schedule(static) if((n) > 32768)
        for (int64_t u = 0; u < n; u++) r[u] = r[u] - alpha * q[u];
        precond_apply(S, r, z);
        double rho1 = dot_c3(S, r, z);
        res2 = S->cg_norm == 0 ? dot_c3(S, z, z) : dot_c3(S, r, r);
        res = sqrt(res2);
        double beta = rho1 / rho;
#pragma omp parallel for schedule(static) if((n) > 32768)
        for (int64_t u = 0; u < n; u++) p[u] = z[u] + beta * p[u];
        rho = rho1;
        k++;
        if (!isfinite(alpha) || !isfinite(beta) || !isfinite(res)) return ORC_ERR_CG_BREAKDOWN;
    }
    rep->cg_iters = k;
    rep->converged = res <= S->cg_rtol * ref;
    rep->rel_res = res / ref;
    return ORC_OK;
}

/* O5' (A31): the same Jacobi-PCG in the Chronopoulos-Gear form (SURVEY
 * §8(f) NEXT #3, single-reduction CG: Chronopoulos & Gear 1989), which
 * carries w = A z and s = A p so that one iteration needs one global
 * reduction instead of two.  In exact arithmetic its iterates equal O5's.
 * Setup, ref, the b = 0 case and the stopping test (res <= rtol*ref before
 * each iteration) are O5's.  Then, if the loop runs at all: w = A z,
 * delta = <z, w> (breakdown if not > 0 or inf), alpha = rho / delta.
 * Iteration k:  p = z (k = 0) | z + beta p;  s = w (k = 0) | w + beta s;
 * x += alpha p;  r -= alpha s;  z = r Dinv;  w = A z (O2);
 * gamma = <r, z>, delta = <z, w>, res = sqrt(<z,z> | <r,r>) (C3 each);
 * k += 1;  beta = gamma / rho;  den = delta - (beta gamma) / alpha;
 * rho = gamma;  breakdown if alpha, beta or res is not finite;  if the loop
 * continues: breakdown unless den > 0 and finite, alpha = gamma / den. */
static int pcg_cgcg(orc_state *S, orc_report *rep)
{
    const orc_graph *G = S->G;
    int64_t n = G->n;
    double *x = S->x, *r = S->r, *z = S->z, *p = S->p, *q = S->q, *w = S->w, *sv = S->sv;
    matvec(S, x, q);
    const double *b = S->bvec ? S->bvec : S->gs;
#pragma omp parallel for schedule(static) if((n) > 32768)
    for (int64_t u = 0; u < n; u++) r[u] = b[u] - q[u];
#pragma omp parallel for schedule(static) if((n) > 32768)
    for (int64_t u = 0; u < n; u++) z[u] = r[u] * S->Dinv[u];
    double rho = dot_c3(S, r, z);
    double ref2;
    if (S->cg_norm == 0) {
#pragma omp parallel for schedule(static) if((n) > 32768)
        for (int64_t u = 0; u < n; u++) { double mb = b[u] * S->Dinv[u]; S->tmp[u] = mb * mb; }
        ref2 = orc_c3_sum(S->tmp, n);
    } else {
        ref2 = dot_c3(S, b, b);
    }
    double ref = sqrt(ref2);
    rep->ref = ref;
    if (ref == 0.0) {
        for (int64_t u = 0; u < n; u++) x[u] = 0.0;
        rep->cg_iters = 0; rep->converged = 1; rep->rel_res = 0.0;
        return ORC_OK;
    }
    double res = sqrt(S->cg_norm == 0 ? dot_c3(S, z, z) : dot_c3(S, r, r));
    int32_t k = 0;
    double alpha = 0.0, beta = 0.0;
    if (!(res <= S->cg_rtol * ref || k == S->cg_max_iter)) {
        matvec(S, z, w);
        double delta = dot_c3(S, z, w);
        if (!(delta > 0.0) || isinf(delta)) return ORC_ERR_CG_BREAKDOWN;
        alpha = rho / delta;
    }
    for (;;) {
        if (res <= S->cg_rtol * ref || k == S->cg_max_iter) break;
#pragma omp parallel for schedule(static) if((n) > 32768)
        for (int64_t u = 0; u < n; u++) p[u] = k == 0 ? z[u] : z[u] + beta * p[u];
#pragma omp parallel for schedule(static) if((n) > 32768)
        for (int64_t u = 0; u < n; u++) sv[u] = k == 0 ? w[u] : w[u] + beta * sv[u];
#pragma omp parallel for schedule(static) if((n) > 32768)
        for (int64_t u = 0; u < n; u++) x[u] = x[u] + alpha * p[u];
#pragma omp parallel for schedule(static) if((n) > 32768)
        for (int64_t u = 0; u < n; u++) r[u] = r[u] - alpha * sv[u];
#pragma omp parallel for schedule(static) if((n) > 32768)
        for (int64_t u = 0; u < n; u++) z[u] = r[u] * S->Dinv[u];
        matvec(S, z, w);
        double gamma = dot_c3(S, r, z);
        double delta = dot_c3(S, z, w);
        res = sqrt(S->cg_norm == 0 ? dot_c3(S, z, z) : dot_c3(S, r, r));
        k++;
        beta = gamma / rho;
        double t = beta * gamma;
        t = t / alpha;
        double den = delta - t;
        rho = gamma;
        if (!isfinite(alpha) || !isfinite(beta) || !isfinite(res)) return ORC_ERR_CG_BREAKDOWN;
        if (!(res <= S->cg_rtol * ref || k == S->cg_max_iter)) {
            if (!(den > 0.0) || isinf(den)) return ORC_ERR_CG_BREAKDOWN;
            alpha = gamma / den;
        }
    }
    rep->cg_iters = k;
    rep->converged = res <= S->cg_rtol * ref;
    rep->rel_res = res / ref;
    return ORC_OK;
}

static int solve(orc_state *S, orc_report *rep)
{
    return S->cg_variant == 1 ? pcg_cgcg(S, rep) : pcg(S, rep);
}

/* O8 diagnostics at x = S->x with the step's conductances. */
static void diagnostics(orc_state *S, orc_report *rep)
{
    const orc_graph *G = S->G;
    int64_t n = G->n;
    const double *x = S->x;
    double eps2 = S->eps * S->eps;
    /* Eq. 9: S_eps = sum over edges with c > 0 of w_e; node u
     * owns its higher-id n-links (ascending) then its s- and t-links. */
#pragma omp parallel for schedule(static) if((n) > 32768)
    for (int64_t u = 0; u < n; u++) {
        double acc = 0.0;
        for (int64_t e = G->adj_ptr[u]; e < G->adj_ptr[u + 1]; e++) {
            int64_t v = G->adj_idx[e];
            if (v < u) continue;
            double a = G->adj_c[e] * (x[u] - x[v]);
            acc = acc + sqrt(a * a + eps2);
        }
        if (S->cs[u] > 0.0) { double a = S->cs[u] * (1.0 - x[u]); acc = acc + sqrt(a * a + eps2); }
        if (S->ct[u] > 0.0) { double a = S->ct[u] * x[u]; acc = acc + sqrt(a * a + eps2); }
        S->tmp[u] = acc;
    }
    rep->S_eps = orc_c3_sum(S->tmp, n);
    /* Prop. 3: flow value x^T L^(l) x = sum_e g_e d_e^2 */
#pragma omp parallel for schedule(static) if((n) > 32768)
    for (int64_t u = 0; u < n; u++) {
        double acc = 0.0;
        for (int64_t e = G->adj_ptr[u]; e < G->adj_ptr[u + 1]; e++) {
            int64_t v = G->adj_idx[e];
            if (v < u) continue;
            double d = x[u] - x[v];
            acc = acc + S->g[e] * (d * d);
        }
        double ds = 1.0 - x[u];
        acc = acc + S->gs[u] * (ds * ds);
        acc = acc + S->gt[u] * (x[u] * x[u]);
        S->tmp[u] = acc;
    }
    rep->flow_value = orc_c3_sum(S->tmp, n);
#pragma omp parallel for schedule(static) if((n) > 32768)
    for (int64_t u = 0; u < n; u++) S->tmp[u] = S->gs[u] * (1.0 - x[u]);
    rep->current_s = orc_c3_sum(S->tmp, n);
    /* true residual in the stopping norm */
    double *q = S->q;
    matvec(S, x, q);
#pragma omp parallel for schedule(static) if((n) > 32768)
    for (int64_t u = 0; u < n; u++) q[u] = S->gs[u] - q[u];
    if (S->cg_norm == 0) precond_apply(S, q, S->w);   /* the stopping norm's M^-1 (b - A x) */
    const double *mv = S->cg_norm == 0 ? S->w : q;
#pragma omp parallel for schedule(static) if((n) > 32768)
    for (int64_t u = 0; u < n; u++) S->tmp[u] = mv[u] * mv[u];
    double tr = sqrt(orc_c3_sum(S->tmp, n));
    rep->true_rel_res = rep->ref > 0.0 ? tr / rep->ref : 0.0;
    double mn = n ? x[0] : 0.0, mx = n ? x[0] : 0.0;
    for (int64_t u = 0; u < n; u++) { if (x[u] < mn) mn = x[u]; if (x[u] > mx) mx = x[u]; }
    rep->x_min = mn; rep->x_max = mx;
}

/* Algorithm 1 step 2 / O4: x^(0) solves Eq. 5 with W^(0) = C, cold. */
int orc_init(orc_state *S, orc_report *rep)
{
    memset(rep, 0, sizeof(*rep));
    assemble(S, NULL);
    if (S->block_size > 0) block_factor(S);
    for (int64_t u = 0; u < S->G->n; u++) S->x[u] = 0.0;
    int rc = solve(S, rep);
    if (rc != ORC_OK) return rc;
    diagnostics(S, rep);
    S->step = 1;
    return ORC_OK;
}

/* Algorithm 1 step 4 / O6: reweight from x^(l-1) (Eq. 4), then
 * solve L~^(l) v = b^(l), warm-started from x^(l-1) or cold. */
int orc_step(orc_state *S, orc_report *rep)
{
    memset(rep, 0, sizeof(*rep));
    if (S->step == 0) return ORC_ERR_STATE;
    assemble(S, S->x);
    if (S->block_size > 0) block_factor(S);
    if (!S->warm_start)
        for (int64_t u = 0; u < S->G->n; u++) S->x[u] = 0.0;
    int rc = solve(S, rep);
    if (rc != ORC_OK) return rc;
    diagnostics(S, rep);
    S->step++;
    return ORC_OK;
}

void orc_get_x(const orc_state *S, double *x)
{
    for (int64_t u = 0; u < S->G->n; u++) x[u] = S->x[u];
}

void orc_set_x(orc_state *S, const double *x)
{
    for (int64_t u = 0; u < S->G->n; u++) S->x[u] = x[u];
    if (S->step == 0) S->step = 1;
}

/* A19 / P:L451: replace the terminal capacities, keep x. */
int orc_set_terminal_weights(orc_state *S, const double *cs, const double *ct)
{
    for (int64_t u = 0; u < S->G->n; u++)
        if (is_bad_cap(cs[u]) || is_bad_cap(ct[u])) return ORC_ERR_BAD_CAPACITY;
    for (int64_t u = 0; u < S->G->n; u++) { S->cs[u] = cs[u]; S->ct[u] = ct[u]; }
    return ORC_OK;
}

/* For unit pins: conductances, D, Dinv, b after assemble(x) (x NULL = init). */
void orc_assemble_export(orc_state *S, const double *x, double *g, double *gs, double *gt,
                         double *D, double *Dinv)
{
    assemble(S, x);
    const orc_graph *G = S->G;
    for (int64_t e = 0; e < G->adj_ptr[G->n]; e++) g[e] = S->g[e];
    for (int64_t u = 0; u < G->n; u++) { gs[u] = S->gs[u]; gt[u] = S->gt[u]; D[u] = S->D[u]; Dinv[u] = S->Dinv[u]; }
}

/* For unit pins of A32: the partition (positions -> ids, block starts, first
 * columns) and, after assemble(x) (x NULL = init) and the factorisation, the
 * factor (boff-indexed envelope, pivots) and z = M^-1 r. */
int64_t orc_block_count(const orc_state *S) { return S->block_size > 0 ? S->nblk : 0; }
int64_t orc_block_env_size(const orc_state *S) { return S->block_size > 0 ? S->boff[S->G->n] : 0; }
void orc_block_export(const orc_state *S, int64_t *bptr, int64_t *bnode, int64_t *bfirst, int64_t *boff)
{
    if (S->block_size <= 0) return;
    int64_t n = S->G->n;
    for (int64_t b = 0; b <= S->nblk; b++) bptr[b] = S->bptr[b];
    for (int64_t i = 0; i < n; i++) { bnode[i] = S->bnode[i]; bfirst[i] = S->bfirst[i]; }
    for (int64_t i = 0; i <= n; i++) boff[i] = S->boff[i];
}
void orc_precond_export(orc_state *S, const double *x, const double *r, double *z, double *L, double *Dd)
{
    assemble(S, x);
    if (S->block_size > 0) block_factor(S);
    precond_apply(S, r, z);
    if (S->block_size > 0) {
        int64_t n = S->G->n;
        for (int64_t e = 0; e < S->boff[n]; e++) L[e] = S->bL[e];
        for (int64_t i = 0; i < n; i++) Dd[i] = S->bDd[i];
    }
}

/* Run a full solve (init + T steps), optionally recording x^(l) for l=0..T
 * (xs has (T+1)*n entries) and the reports (T+1). */
int orc_irls_run(orc_state *S, double *xs, orc_report *reps)
{
    orc_report rep;
    int rc = orc_init(S, &rep);
    if (rc) return rc;
    if (reps) reps[0] = rep;
    int64_t n = S->G->n;
    if (xs) for (int64_t u = 0; u < n; u++) xs[u] = S->x[u];
    for (int32_t l = 1; l <= S->T; l++) {
        rc = orc_step(S, &rep);
        if (rc) return rc;
        if (reps) reps[l] = rep;
        if (xs) for (int64_t u = 0; u < n; u++) xs[(int64_t)l * n + u] = S->x[u];
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* Sweep cut ("sorting the nodes according to x^(T)").    */
/* ------------------------------------------------------------------------- */
typedef __int128 i128;

static const double *sort_x;
static int sweep_cmp(const void *a, const void *b)
{
    int64_t i = *(const int64_t *)a, j = *(const int64_t *)b;
    double xi = sort_x[i], xj = sort_x[j];
    if (xi > xj) return -1;   /* x descending */
    if (xi < xj) return 1;
    return (i > j) - (i < j); /* ties: id ascending (A14) */
}

/* A15: prefix sums of the sweep are exact integer sums of capacities in
 * fixed point with F fractional bits, Q(c) = rint(c * 2^F), F = 124 - e - b
 * where cmax < 2^e (frexp) and b = bit length of the number of positive
 * capacities (n-links + s-links + t-links + direct s-t). */
static int32_t sweep_F(const orc_graph *G, const double *cs, const double *ct)
{
    double cmax = G->c_st;
    int64_t cnt = G->c_st > 0.0;
    for (int64_t u = 0; u < G->n; u++) {
        for (int64_t e = G->adj_ptr[u]; e < G->adj_ptr[u + 1]; e++)
            if (G->adj_idx[e] > u) { cnt++; if (G->adj_c[e] > cmax) cmax = G->adj_c[e]; }
        if (cs[u] > 0.0) { cnt++; if (cs[u] > cmax) cmax = cs[u]; }
        if (ct[u] > 0.0) { cnt++; if (ct[u] > cmax) cmax = ct[u]; }
    }
    if (cmax == 0.0) return 0;
    int e; frexp(cmax, &e);
    int b = 0; while (b < 63 && (((int64_t)1) << b) <= cnt) b++;
    return 124 - e - b;
}

static i128 Qfix(double c, int32_t F) { return (i128)rint(ldexp(c, F)); }

/* O7: order non-terminals by (x desc, id asc); delta_v = sum over neighbours
 * u of (+c if u is later in the order else -c) + ct_v - cs_v; P_0 = sum cs +
 * c_st; P_i = P_{i-1} + delta_{order[i-1]} (exact, fixed point); k = first
 * argmin of P_i over i = 0..n; S = {s} + order[0..k).  The reported cut value
 * is recomputed from S by C3 ("recomputed, not trusted").
 * side: n_total bytes (1 = source side); order: n output ids (or NULL);
 * pk_words: P_k as (lo, hi) 64-bit words (or NULL). */
int orc_sweep(const orc_state *S, const double *x, uint8_t *side, int64_t *order_out,
              int64_t *k_out, double *cut_out, int32_t *F_out, uint64_t *pk_words)
{
    const orc_graph *G = S->G;
    int64_t n = G->n;
    for (int64_t u = 0; u < n; u++) if (isnan(x[u])) return ORC_ERR_BAD_POTENTIAL;
    int64_t *order = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    int64_t *rank = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    i128 *delta = (i128 *)malloc(sizeof(i128) * (size_t)(n > 0 ? n : 1));
    double *cross = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    if (!order || !rank || !delta || !cross) { free(order); free(rank); free(delta); free(cross); return ORC_ERR_OOM; }
    for (int64_t u = 0; u < n; u++) order[u] = u;
    sort_x = x;
    qsort(order, (size_t)n, sizeof(int64_t), sweep_cmp);
    for (int64_t i = 0; i < n; i++) rank[order[i]] = i;
    int32_t F = sweep_F(G, S->cs, S->ct);
    for (int64_t v = 0; v < n; v++) {
        i128 d = 0;
        for (int64_t e = G->adj_ptr[v]; e < G->adj_ptr[v + 1]; e++) {
            int64_t u = G->adj_idx[e];
            i128 qc = Qfix(G->adj_c[e], F);
            d += rank[u] > rank[v] ? qc : -qc;
        }
        d += Qfix(S->ct[v], F);
        d -= Qfix(S->cs[v], F);
        delta[v] = d;
    }
    i128 P = Qfix(G->c_st, F);
    for (int64_t v = 0; v < n; v++) P += Qfix(S->cs[v], F);
    i128 best = P; int64_t k = 0;
    for (int64_t i = 1; i <= n; i++) {
        P += delta[order[i - 1]];
        if (P < best) { best = P; k = i; }
    }
    /* membership and directly recomputed cut value */
    for (int64_t id = 0; id < G->n_total; id++) side[id] = 0;
    side[G->s_id] = 1;
    for (int64_t i = 0; i < k; i++) side[G->orig[order[i]]] = 1;
    for (int64_t v = 0; v < n; v++) {
        if (rank[v] < k) {
            double acc = 0.0;
            for (int64_t e = G->adj_ptr[v]; e < G->adj_ptr[v + 1]; e++)
                if (rank[G->adj_idx[e]] >= k) acc = acc + G->adj_c[e];
            cross[v] = acc + S->ct[v];
        } else {
            cross[v] = S->cs[v];
        }
    }
    double cut = orc_c3_sum(cross, n) + G->c_st;
    if (order_out) for (int64_t i = 0; i < n; i++) order_out[i] = G->orig[order[i]];
    *k_out = k;
    *cut_out = cut;
    if (F_out) *F_out = F;
    if (pk_words) { pk_words[0] = (uint64_t)best; pk_words[1] = (uint64_t)(best >> 64); }
    free(order); free(rank); free(delta); free(cross);
    return ORC_OK;
}

/* cut(S, S-bar) by definition over the graph held by S (with its
 * current terminal capacities); side indexed by output id. */
double orc_cut_value(const orc_state *S, const uint8_t *side)
{
    const orc_graph *G = S->G;
    double cut = 0.0;
    int ss = side[G->s_id], st = side[G->t_id];
    for (int64_t u = 0; u < G->n; u++) {
        int su = side[G->orig[u]];
        for (int64_t e = G->adj_ptr[u]; e < G->adj_ptr[u + 1]; e++) {
            int64_t v = G->adj_idx[e];
            if (v > u && su != side[G->orig[v]]) cut += G->adj_c[e];
        }
        if (su != ss) cut += S->cs[u];
        if (su != st) cut += S->ct[u];
    }
    if (ss != st) cut += G->c_st;
    return cut;
}

/* ------------------------------------------------------------------------- */
/* Exact min cut mu* by Edmonds-Karp (shortest augmenting paths) on the whole */
/* graph, used to evaluate delta (Eq. 13).  Undirected edge {u,v} */
/* = two arcs of capacity c, each the other's residual twin.                  */
/* ------------------------------------------------------------------------- */
int orc_maxflow_ek(const orc_state *S, double *flow_out, uint8_t *side)
{
    const orc_graph *G = S->G;
    int64_t n = G->n, V = n + 2, s = n, t = n + 1;
    int64_t m = G->adj_ptr[n] / 2 + 2 * n + 1; /* undirected edges (upper bound) */
    int64_t *head = (int64_t *)malloc(sizeof(int64_t) * (size_t)V);
    int64_t *nxt = (int64_t *)malloc(sizeof(int64_t) * (size_t)(2 * m));
    int64_t *to = (int64_t *)malloc(sizeof(int64_t) * (size_t)(2 * m));
    double *res = (double *)malloc(sizeof(double) * (size_t)(2 * m));
    int64_t *prev = (int64_t *)malloc(sizeof(int64_t) * (size_t)V);
    int64_t *queue = (int64_t *)malloc(sizeof(int64_t) * (size_t)V);
    if (!head || !nxt || !to || !res || !prev || !queue) {
        free(head); free(nxt); free(to); free(res); free(prev); free(queue); return ORC_ERR_OOM;
    }
    for (int64_t i = 0; i < V; i++) head[i] = -1;
    int64_t A = 0;
    double cmax = G->c_st;
#define ADD_EDGE(a, b, c) do { to[A] = (b); res[A] = (c); nxt[A] = head[a]; head[a] = A; A++; \
                               to[A] = (a); res[A] = (c); nxt[A] = head[b]; head[b] = A; A++; } while (0)
    for (int64_t u = 0; u < n; u++) {
        for (int64_t e = G->adj_ptr[u]; e < G->adj_ptr[u + 1]; e++)
            if (G->adj_idx[e] > u) { ADD_EDGE(u, G->adj_idx[e], G->adj_c[e]); if (G->adj_c[e] > cmax) cmax = G->adj_c[e]; }
        if (S->cs[u] > 0.0) { ADD_EDGE(s, u, S->cs[u]); if (S->cs[u] > cmax) cmax = S->cs[u]; }
        if (S->ct[u] > 0.0) { ADD_EDGE(u, t, S->ct[u]); if (S->ct[u] > cmax) cmax = S->ct[u]; }
    }
    if (G->c_st > 0.0) ADD_EDGE(s, t, G->c_st);
#undef ADD_EDGE
    double tol = 1e-12 * cmax, flow = 0.0;
    for (;;) {
        for (int64_t i = 0; i < V; i++) prev[i] = -2;
        int64_t qh = 0, qt = 0;
        queue[qt++] = s; prev[s] = -1;
        while (qh < qt && prev[t] == -2) {
            int64_t u = queue[qh++];
            for (int64_t a = head[u]; a >= 0; a = nxt[a])
                if (res[a] > tol && prev[to[a]] == -2) { prev[to[a]] = a; queue[qt++] = to[a]; }
        }
        if (prev[t] == -2) break;
        double b = INFINITY;
        for (int64_t v = t; v != s; v = to[prev[v] ^ 1]) if (res[prev[v]] < b) b = res[prev[v]];
        for (int64_t v = t; v != s; v = to[prev[v] ^ 1]) { res[prev[v]] -= b; res[prev[v] ^ 1] += b; }
        flow += b;
    }
    /* reachable set from s in the final residual graph: prev != -2 */
    for (int64_t id = 0; id < G->n_total; id++) side[id] = 0;
    side[G->s_id] = 1;
    for (int64_t u = 0; u < n; u++) if (prev[u] != -2) side[G->orig[u]] = 1;
    *flow_out = flow;
    free(head); free(nxt); free(to); free(res); free(prev); free(queue);
    return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* Two-level rounding ("A two-level rounding procedure";          */
/* SURVEY §8(f) NEXT #1).  Readings A25-A30 in DESIGN.md §2.                  */
/* ------------------------------------------------------------------------- */

/* A25 ("the two centers returned from K-means on x^(T) (with initial
 * guesses 0.1 and 0.9)"): Lloyd's algorithm, k = 2, on the components of
 * x^(T) — the non-terminals plus x_s = 1 and x_t = 0.  Assignment: u goes to
 * cluster 1 iff |x_u - c1| < |x_u - c0| (a tie goes to cluster 0).  Means:
 * sum_j = C3 sum over the non-terminals of (x_u if u is in j, else +0.0),
 * then + x_s if s is in j, then + x_t if t is in j; c_j = sum_j / |j| (an
 * empty cluster keeps its centre).  Stop when both centres are unchanged,
 * or after 100 rounds.  out4 = (c0, c1, gamma0 = c0 + 0.05, gamma1 = c1 - 0.05). */
int orc_kmeans2(const orc_state *S, const double *x, double *out4, int32_t *rounds_out)
{
    const orc_graph *G = S->G;
    int64_t n = G->n;
    double *v0 = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double *v1 = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    if (!v0 || !v1) { free(v0); free(v1); return ORC_ERR_OOM; }
    double c0 = 0.1, c1 = 0.9;
    int32_t r;
    for (r = 1; r <= 100; r++) {
        int64_t n1 = 0;
        for (int64_t u = 0; u < n; u++) {
            int in1 = fabs(x[u] - c1) < fabs(x[u] - c0);
            v0[u] = in1 ? 0.0 : x[u];
            v1[u] = in1 ? x[u] : 0.0;
            n1 += in1;
        }
        double s0 = orc_c3_sum(v0, n), s1 = orc_c3_sum(v1, n);
        const double xt[2] = {1.0, 0.0}; /* x_s, x_t */
        for (int i = 0; i < 2; i++) {
            if (fabs(xt[i] - c1) < fabs(xt[i] - c0)) { s1 = s1 + xt[i]; n1++; }
            else s0 = s0 + xt[i];
        }
        int64_t n0 = n + 2 - n1;
        double d0 = n0 > 0 ? s0 / (double)n0 : c0;
        double d1 = n1 > 0 ? s1 / (double)n1 : c1;
        int same = (d0 == c0) && (d1 == c1);
        c0 = d0; c1 = d1;
        if (same) break;
    }
    if (r > 100) r = 100;
    out4[0] = c0; out4[1] = c1; out4[2] = c0 + 0.05; out4[3] = c1 - 0.05;
    /* A26': crossing thresholds (centres less than 0.1 apart) fall back to
     * gamma = (c0, c1) (the degenerate-threshold reading of SPEC S:L404). */
    if (!(out4[2] < out4[3])) { out4[2] = c0; out4[3] = c1; }
    *rounds_out = r;
    free(v0); free(v1);
    return ORC_OK;
}

static void put_q(uint64_t *w, i128 v) { w[0] = (uint64_t)v; w[1] = (uint64_t)(v >> 64); }
static i128 get_q(const uint64_t *w) { return (i128)(((unsigned __int128)w[1] << 64) | w[0]); }

/* The partition and the coarsened graph G_c, in the fixed point
 * of A15 (Q(c) = rint(c 2^F), the sweep's F), so every coarse capacity is an
 * exact integer sum (A27).  cls[u] = 0 if x_u <= gamma0 (S0), else 1 if
 * x_u >= gamma1 (S1), else 2 (Sc); s is in S1 and t in S0 by definition
 * (they are what S1 and S0 contract into).  Coarse ids: Sc in ascending
 * reduced id.  The four bullets of P:L278-281:
 *   {u,v} in Sc x Sc:  Q(c_uv)                          (ccol / ccap, ascending)
 *   {s_c,u}:           sum_{v in S1} Q(c_uv) + Q(cs_u)  (the s-link: s in S1)
 *   {t_c,u}:           sum_{v in S0} Q(c_uv) + Q(ct_u)  (the t-link: t in S0)
 *   {s_c,t_c}:         Q(c_st) + sum_{u in S1}(sum_{v in S0} Q(c_uv) + Q(ct_u))
 *                      + sum_{u in S0} Q(cs_u)
 * Caller buffers: cls, cid [n]; cptr [n+1]; ccol, ccap(2 words) [nnz];
 * cqs, cqt (2 words) [n]; cqst [2].  Returns nc and the coarse entry count. */
int orc_coarsen(const orc_state *S, const double *x, double g0, double g1, int8_t *cls, int64_t *cid,
                int64_t *nc_out, int64_t *cptr, int64_t *ccol, uint64_t *ccap, uint64_t *cqs, uint64_t *cqt,
                uint64_t *cqst, int32_t *F_out)
{
    const orc_graph *G = S->G;
    int64_t n = G->n;
    int32_t F = sweep_F(G, S->cs, S->ct);
    int64_t nc = 0;
    for (int64_t u = 0; u < n; u++) {
        cls[u] = x[u] <= g0 ? 0 : (x[u] >= g1 ? 1 : 2);
        cid[u] = cls[u] == 2 ? nc++ : -1;
    }
    i128 qst = Qfix(G->c_st, F);
    int64_t m = 0;
    cptr[0] = 0;
    for (int64_t u = 0; u < n; u++) {
        if (cls[u] == 2) {
            i128 qs = 0, qt = 0;
            for (int64_t e = G->adj_ptr[u]; e < G->adj_ptr[u + 1]; e++) {
                int64_t v = G->adj_idx[e];
                i128 q = Qfix(G->adj_c[e], F);
                if (cls[v] == 2) { ccol[m] = cid[v]; put_q(ccap + 2 * m, q); m++; }
                else if (cls[v] == 1) qs += q;
                else qt += q;
            }
            put_q(cqs + 2 * cid[u], qs + Qfix(S->cs[u], F));
            put_q(cqt + 2 * cid[u], qt + Qfix(S->ct[u], F));
            cptr[cid[u] + 1] = m;
        } else if (cls[u] == 1) {
            for (int64_t e = G->adj_ptr[u]; e < G->adj_ptr[u + 1]; e++)
                if (cls[G->adj_idx[e]] == 0) qst += Qfix(G->adj_c[e], F);
            qst += Qfix(S->ct[u], F);
        } else {
            qst += Qfix(S->cs[u], F);
        }
    }
    put_q(cqst, qst);
    *nc_out = nc;
    if (F_out) *F_out = F;
    return ORC_OK;
}

/* Exact max-flow / min-cut on G_c (the paper's "combinatorial max-flow/
 * min-cut solver") by Edmonds-Karp (shortest augmenting paths) in
 * 128-bit integers.  Coarse nodes 0..nc-1, s_c = nc, t_c = nc+1; the direct
 * s_c-t_c edge is in every cut and is added to the flow value.  src[u] = 1 iff
 * u is reachable from s_c in the final residual graph: the source side of
 * the minimal minimum cut, which is the same for every maximum flow (A28). */
int orc_maxflow_coarse(int64_t nc, const int64_t *cptr, const int64_t *ccol, const uint64_t *ccap,
                       const uint64_t *cqs, const uint64_t *cqt, const uint64_t *cqst, uint8_t *src,
                       uint64_t *flow_out)
{
    int64_t V = nc + 2, s = nc, t = nc + 1;
    int64_t m = cptr[nc] / 2 + 2 * nc + 1;
    int64_t *head = (int64_t *)malloc(sizeof(int64_t) * (size_t)V);
    int64_t *nxt = (int64_t *)malloc(sizeof(int64_t) * (size_t)(2 * m));
    int64_t *to = (int64_t *)malloc(sizeof(int64_t) * (size_t)(2 * m));
    i128 *res = (i128 *)malloc(sizeof(i128) * (size_t)(2 * m));
    int64_t *prev = (int64_t *)malloc(sizeof(int64_t) * (size_t)V);
    int64_t *queue = (int64_t *)malloc(sizeof(int64_t) * (size_t)V);
    if (!head || !nxt || !to || !res || !prev || !queue) {
        free(head); free(nxt); free(to); free(res); free(prev); free(queue); return ORC_ERR_OOM;
    }
    for (int64_t i = 0; i < V; i++) head[i] = -1;
    int64_t A = 0;
#define ADD_EDGE(a, b, c) do { to[A] = (b); res[A] = (c); nxt[A] = head[a]; head[a] = A; A++; \
                               to[A] = (a); res[A] = (c); nxt[A] = head[b]; head[b] = A; A++; } while (0)
    for (int64_t u = 0; u < nc; u++) {
        for (int64_t e = cptr[u]; e < cptr[u + 1]; e++)
            if (ccol[e] > u) ADD_EDGE(u, ccol[e], get_q(ccap + 2 * e));
        i128 qs = get_q(cqs + 2 * u), qt = get_q(cqt + 2 * u);
        if (qs > 0) ADD_EDGE(s, u, qs);
        if (qt > 0) ADD_EDGE(u, t, qt);
    }
#undef ADD_EDGE
    i128 flow = get_q(cqst);
    for (;;) {
        for (int64_t i = 0; i < V; i++) prev[i] = -2;
        int64_t qh = 0, qt = 0;
        queue[qt++] = s; prev[s] = -1;
        while (qh < qt && prev[t] == -2) {
            int64_t u = queue[qh++];
            for (int64_t a = head[u]; a >= 0; a = nxt[a])
                if (res[a] > 0 && prev[to[a]] == -2) { prev[to[a]] = a; queue[qt++] = to[a]; }
        }
        if (prev[t] == -2) break;
        i128 b = -1;
        for (int64_t v = t; v != s; v = to[prev[v] ^ 1]) if (b < 0 || res[prev[v]] < b) b = res[prev[v]];
        for (int64_t v = t; v != s; v = to[prev[v] ^ 1]) { res[prev[v]] -= b; res[prev[v] ^ 1] += b; }
        flow += b;
    }
    for (int64_t u = 0; u < nc; u++) src[u] = prev[u] != -2;
    put_q(flow_out, flow);
    free(head); free(nxt); free(to); free(res); free(prev); free(queue);
    return ORC_OK;
}

/* The cut value of a node set by C3 (O7 step 7): cross_v = (v in S) ?
 * (sum_asc over neighbours u not in S of c_uv) + ct_v : cs_v, plus c_st. */
static double cut_c3(const orc_state *S, const uint8_t *in)
{
    const orc_graph *G = S->G;
    int64_t n = G->n;
    double *cross = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    if (!cross) return NAN;
    for (int64_t v = 0; v < n; v++) {
        if (in[v]) {
            double acc = 0.0;
            for (int64_t e = G->adj_ptr[v]; e < G->adj_ptr[v + 1]; e++)
                if (!in[G->adj_idx[e]]) acc = acc + G->adj_c[e];
            cross[v] = acc + S->ct[v];
        } else {
            cross[v] = S->cs[v];
        }
    }
    double cut = orc_c3_sum(cross, n) + G->c_st;
    free(cross);
    return cut;
}

/* Two-level rounding of x: K-means thresholds (A25) -> S0/S1/Sc
 * -> G_c (A27) -> exact min cut on G_c (A28) -> the induced cut on G
 * ("An s-t cut on G_c induces an s-t cut on G"): S = {s} + S1 + the
 * source side of G_c.  The cut value is recomputed on G by C3 (A29).
 * dinfo = (c0, c1, gamma0, gamma1); iinfo = (rounds, |S0|, |S1|, |Sc|, coarse
 * entries); flow = max-flow value on G_c in fixed point (2 words). */
int orc_two_level(const orc_state *S, const double *x, uint8_t *side, double *cut_out, double *dinfo,
                  int64_t *iinfo, uint64_t *flow, int32_t *F_out)
{
    const orc_graph *G = S->G;
    int64_t n = G->n, nnz = G->adj_ptr[n];
    for (int64_t u = 0; u < n; u++) if (isnan(x[u])) return ORC_ERR_BAD_POTENTIAL;
    int32_t rounds;
    int rc = orc_kmeans2(S, x, dinfo, &rounds);
    if (rc) return rc;
    size_t N1 = (size_t)(n > 0 ? n : 1), M1 = (size_t)(nnz > 0 ? nnz : 1);
    int8_t *cls = (int8_t *)malloc(N1);
    int64_t *cid = (int64_t *)malloc(sizeof(int64_t) * N1);
    int64_t *cptr = (int64_t *)malloc(sizeof(int64_t) * (N1 + 1));
    int64_t *ccol = (int64_t *)malloc(sizeof(int64_t) * M1);
    uint64_t *ccap = (uint64_t *)malloc(16 * M1), *cqs = (uint64_t *)malloc(16 * N1),
             *cqt = (uint64_t *)malloc(16 * N1), cqst[2];
    uint8_t *src = (uint8_t *)malloc(N1), *in = (uint8_t *)malloc(N1);
    if (!cls || !cid || !cptr || !ccol || !ccap || !cqs || !cqt || !src || !in) { rc = ORC_ERR_OOM; goto out; }
    int64_t nc;
    if (!(dinfo[2] < dinfo[3])) {
        /* A26': still degenerate (c0 >= c1; Lloyd from (0.1, 0.9) keeps
         * c0 < c1, so only a NaN-free rounding tie reaches this): the sweep
         * cut of x. */
        int64_t k;
        uint64_t pk[2];
        rc = orc_sweep(S, x, side, NULL, &k, cut_out, F_out, pk);
        iinfo[0] = rounds; iinfo[1] = iinfo[2] = iinfo[3] = iinfo[4] = 0;
        flow[0] = flow[1] = 0;
        goto out;
    }
    orc_coarsen(S, x, dinfo[2], dinfo[3], cls, cid, &nc, cptr, ccol, ccap, cqs, cqt, cqst, F_out);
    rc = orc_maxflow_coarse(nc, cptr, ccol, ccap, cqs, cqt, cqst, src, flow);
    if (rc) goto out;
    int64_t n0 = 0, n1 = 0;
    for (int64_t u = 0; u < n; u++) {
        in[u] = cls[u] == 1 || (cls[u] == 2 && src[cid[u]]);
        n0 += cls[u] == 0; n1 += cls[u] == 1;
    }
    for (int64_t id = 0; id < G->n_total; id++) side[id] = 0;
    side[G->s_id] = 1;
    for (int64_t u = 0; u < n; u++) if (in[u]) side[G->orig[u]] = 1;
    *cut_out = cut_c3(S, in);
    iinfo[0] = rounds; iinfo[1] = n0; iinfo[2] = n1; iinfo[3] = nc; iinfo[4] = cptr[nc];
out:
    free(cls); free(cid); free(cptr); free(ccol); free(ccap); free(cqs); free(cqt); free(src); free(in);
    return rc;
}

/* ------------------------------------------------------------------------- */
/* Cheeger-type diagnostic lambda_2 (Theorem 4; characterised by  */
/* the constrained WLS of P:L543-551; reading A30).     */
/* ------------------------------------------------------------------------- */

/* lambda_2 = min (1/2C) x^T L x s.t. x_s = 1, x_t = -1 (Eq. lambda2-
 * constrained-wls), L the Laplacian of G with the capacities c
 * (W = C) and C = 2 sum_e c_e.  Reduced system as Eq. 7 with
 * f = (1, -1): L~ v = b, b_u = cs_u - ct_u, solved by the same Jacobi-PCG
 * (O5) from x0 = 0 with the given rtol / cap / norm.  Then
 *   x^T L x = C3 over u of own_u, plus 4 c_st, where own_u = sum over the
 *     higher-id neighbours v (ascending) of c_uv * (d * d), d = x_u - x_v,
 *     then + cs_u * (ds * ds), ds = 1 - x_u, then + ct_u * (dt * dt),
 *     dt = x_u + 1;
 *   C = 2 * (C3 over u of (sum_{v > u, asc} c_uv + cs_u + ct_u) + c_st);
 *   lambda_2 = x^T L x / (2 C).
 * out3 = (lambda_2, x^T L x, C); x_out (may be NULL) = v.  The IRLS state
 * (x) is restored. */
int orc_lambda2(orc_state *S, double rtol, int32_t max_iter, int32_t norm, double *out3, int32_t *iters,
                double *x_out)
{
    const orc_graph *G = S->G;
    int64_t n = G->n;
    size_t N1 = (size_t)(n > 0 ? n : 1);
    double *xs = (double *)malloc(sizeof(double) * N1), *b = (double *)malloc(sizeof(double) * N1);
    double *own = (double *)malloc(sizeof(double) * N1), *cap = (double *)malloc(sizeof(double) * N1);
    if (!xs || !b || !own || !cap) { free(xs); free(b); free(own); free(cap); return ORC_ERR_OOM; }
    memcpy(xs, S->x, sizeof(double) * (size_t)n);
    double r0 = S->cg_rtol; int32_t m0 = S->cg_max_iter, n0 = S->cg_norm;
    S->cg_rtol = rtol; S->cg_max_iter = max_iter; S->cg_norm = norm;
    int32_t bs0 = S->block_size;
    S->block_size = 0;                 /* lambda_2's solve: point Jacobi (A30) */
    assemble(S, NULL);
    for (int64_t u = 0; u < n; u++) { b[u] = S->gs[u] - S->gt[u]; S->x[u] = 0.0; }
    S->bvec = b;
    orc_report rep;
    memset(&rep, 0, sizeof(rep));
    int rc = solve(S, &rep);
    S->bvec = NULL;
    S->block_size = bs0;
    S->cg_rtol = r0; S->cg_max_iter = m0; S->cg_norm = n0;
    if (rc == ORC_OK) {
        const double *x = S->x;
        for (int64_t u = 0; u < n; u++) {
            double q = 0.0, c = 0.0;
            for (int64_t e = G->adj_ptr[u]; e < G->adj_ptr[u + 1]; e++) {
                int64_t v = G->adj_idx[e];
                if (v < u) continue;
                double d = x[u] - x[v];
                q = q + G->adj_c[e] * (d * d);
                c = c + G->adj_c[e];
            }
            double ds = 1.0 - x[u], dt = x[u] + 1.0;
            q = q + S->cs[u] * (ds * ds);
            q = q + S->ct[u] * (dt * dt);
            own[u] = q;
            cap[u] = (c + S->cs[u]) + S->ct[u];
        }
        double xLx = orc_c3_sum(own, n) + 4.0 * G->c_st;
        double C = 2.0 * (orc_c3_sum(cap, n) + G->c_st);
        out3[0] = xLx / (2.0 * C); out3[1] = xLx; out3[2] = C;
        *iters = rep.cg_iters;
        if (x_out) memcpy(x_out, S->x, sizeof(double) * (size_t)n);
    }
    memcpy(S->x, xs, sizeof(double) * (size_t)n);
    free(xs); free(b); free(own); free(cap);
    return rc;
}
