/*
 * irls_mincut.h — C ABI of the B200-native IRLS s-t min-cut hot path.
 *
 * Method: Zhu & Gleich, "A Parallel Min-Cut Algorithm using Iteratively
 * Reweighted Least Squares", arXiv 1501.03105.  Citations "P:Lnnn"
 * are PAPER.md lines; readings A<k>, the oracle steps O<k> and the arithmetic
 * contract C1-C3 are listed in DESIGN.md §2.
 *
 * What the library computes (Algorithm 1, without the partition
 * step):
 *   x^(0)  = solution of the constrained WLS Eq. 5 with W^(0) = C,
 *   for l = 1..T:
 *     w^(l) = sqrt((C B x^(l-1))^2 + eps^2)                 (Eq. 4)
 *     L^(l) = B^T C (W^(l))^-1 C B                           (Eq. 8)
 *     solve the reduced system L~^(l) v = b^(l)               (Eq. 7)
 *       by Jacobi-preconditioned CG warm-started from v^(l-1)
 *   sweep cut of x^(T): sort by potential, prefix-sum the per-node cut
 *   deltas, take the first argmin
 *
 * Conventions shared by every entry point
 *   - All floating point is IEEE float64 without FMA contraction (C1); all
 *     sums follow C2/C3, so results are bitwise identical to the CPU oracle
 *     and independent of the number of GPUs.
 *   - Input arrays are HOST memory, copied at create; the caller keeps
 *     ownership.  Output arrays are caller-owned HOST memory unless a
 *     function says otherwise.  Device memory is owned by the context.
 *   - Multi-GPU: one process per GPU; every call is collective (all ranks,
 *     same order).  Only rank 0 fills sweep / potential outputs; other ranks
 *     may pass NULL.
 *   - Every call is stream-ordered on the context's stream and returns after
 *     its results are final.
 *   - Argument errors (IRLS_ERR_INVALID_ARGUMENT and the validation codes
 *     BAD_CAPACITY / SINGULAR, at create or irls_set_terminal_weights) are
 *     detected on the host before device work and leave the context usable.
 *     After any other error the context is poisoned: later calls return
 *     IRLS_ERR_STATE until irls_mincut_destroy.  A non-converged CG is NOT an error: the
 *     report says converged = 0.
 *   - No C++ exception crosses this boundary.
 */
#ifndef IRLS_MINCUT_H
#define IRLS_MINCUT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct irls_ctx irls_ctx; /* opaque; one per rank; not thread-safe */

typedef enum {
    IRLS_OK = 0,
    IRLS_ERR_INVALID_ARGUMENT = 1,   /* bad sizes, NULL pointers, self loop, eps <= 0, ... */
    IRLS_ERR_SOURCE_EQUALS_SINK = 2, /* s == t */
    IRLS_ERR_BAD_CAPACITY = 3,       /* c < 0, NaN or Inf (P:L42 requires c >= 0; A6) */
    IRLS_ERR_NOT_SYMMETRIC = 4,      /* CSR after duplicate merging is not symmetric */
    IRLS_ERR_SINGULAR = 5,           /* a component of G~ has no positive terminal edge (Prop. 1; A8) */
    IRLS_ERR_CG_BREAKDOWN = 6,       /* p'Ap <= 0 or a non-finite CG scalar */
    IRLS_ERR_BAD_POTENTIAL = 7,      /* NaN in x at the sweep */
    IRLS_ERR_STATE = 8,              /* wrong call order, or poisoned context */
    IRLS_ERR_CUDA = 9,
    IRLS_ERR_NCCL = 10,              /* an NCCL call or a peer-memory collective (p2p wait timeout) failed */
    IRLS_ERR_OOM = 11
} irls_status;

typedef enum { IRLS_NORM_PRECONDITIONED = 0, IRLS_NORM_UNPRECONDITIONED = 1 } irls_cg_norm;
/* GRAPH (default): CUDA graphs with device-side WHILE loops — on a
 * communicator the NCCL collectives are captured inside the loop bodies
 * (with p2p only the per-solve ones: the per-iteration exchanges are peer
 * stores), so there is no host round trip per CG iteration; GRAPH_NCCL: the
 * same (kept for compatibility); HOST: a host loop with one 4-byte readback
 * of the device stopping flag per CG iteration (every kernel a plain launch,
 * visible to profilers). */
typedef enum { IRLS_LOOP_GRAPH = 0, IRLS_LOOP_HOST = 1, IRLS_LOOP_GRAPH_NCCL = 2 } irls_loop_mode;
/* PCG form (A31): Hestenes-Stiefel (O5, two reductions per iteration) or
 * Chronopoulos-Gear (O5': one reduction per iteration,
 * one kernel per iteration on one GPU; iterates equal O5's in exact
 * arithmetic, bitwise equal to the oracle's O5'). */
typedef enum { IRLS_CG_HS = 0, IRLS_CG_CG = 1 } irls_cg_variant;

/* Solver options (A9-A13). */
typedef struct {
    double eps;          /* smoothing eps of Eq. 4, > 0; default 1e-6 */
    int32_t T;           /* IRLS steps after x^(0) (A1); default 50 */
    double cg_rtol;      /* stop when ||res|| <= cg_rtol * ||ref|| (A9); default 1e-3 */
    int32_t cg_max_iter; /* PCG iteration cap per solve; default 50 */
    int32_t cg_norm;     /* irls_cg_norm: PRECONDITIONED ||M^-1 r|| vs ||M^-1 b|| (default), or ||r|| vs ||b|| */
    int32_t warm_start;  /* 1: CG starts from v^(l-1); 0: cold start from 0 */
    int32_t record_trace;/* 1: fill S_eps / flow / true residual / x range in reports (extra passes) */
    int32_t loop_mode;   /* irls_loop_mode: CUDA graph with device-side WHILE loop (default) or host loop */
    int32_t fixed_point_exit; /* 1: within one irls_solve, once a warm reweight step stops before its first
                                 CG iteration (x unchanged), the remaining steps repeat it bit for bit and are
                                 skipped on the device (their reports are copies).  x^(T) and the reports are
                                 identical to running every step; default 0 (every step executed). */
    int32_t p2p;         /* multi-rank contexts (world > 1, or world 1 with an NCCL id): 1 = the per-iteration
                            collectives go over peer memory, fused into the kernels that produce their data
                            (DESIGN.md §6): each group owner stores its C3 slot sums straight into every
                            rank's slot buffer and bumps an arrival counter that the finalize kernel waits
                            on (no slot allreduce), and on z-slabs K5 (CG-CG: the iteration kernel) also
                            stores z's (w's) boundary planes into the neighbours' ghost planes; on CSR
                            id strips a store kernel writes the send lists' z values into the peers'
                            ghost blocks before K5's sums are pushed (no per-iteration halo exchange).  Peer buffers
                            are exchanged at create with CUDA IPC handles over NCCL (allocated with
                            cudaMalloc, outside device_alloc); virtual groups use the other ranks' buffers
                            directly.  Results are bit-identical to p2p = 0.  A wait longer than 120 s
                            ends the solve with IRLS_ERR_NCCL.  Ignored on a single-rank context.
                            Default 0 (NCCL). */
    int32_t cg_variant;  /* irls_cg_variant; default IRLS_CG_HS */
    int32_t block_size;  /* preconditioner (A12 / A32): 0 = point Jacobi M = diag(L~) (default); B in [1, 256]
                            = block Jacobi with exact block solves (the paper's "block Jacobi" with "LU"
                            blocks): BFS blocks of at most B nodes
                            inside one C3 group (so identical for every world size), each factored per IRLS
                            step as A_B = L D L^T (envelope, by rows, sums ascending) and applied per CG
                            iteration by forward / backward substitution, bitwise equal to the oracle's
                            definition (A32).  The partition is built at create.  Not combinable
                            with cg_variant IRLS_CG_CG, p2p or record_trace (IRLS_ERR_INVALID_ARGUMENT).
                            irls_lambda2's solve stays point Jacobi (A30). */
} irls_options;

void irls_options_default(irls_options *opt);

/* Process / device description.  world_size 1: nccl_unique_id may be NULL;
 * a stencil context given world_size 1 AND an id runs the multi-rank code
 * path over a 1-rank NCCL communicator (host loop, slot allreduce, finalize
 * kernels, gather / broadcast) — a self-test of the NCCL plumbing on one GPU.
 * cuda_stream: a cudaStream_t to run on, or NULL for a library-owned one.
 * device_alloc / device_free: the caller's device memory (e.g. torch
 * tensors from its caching allocator) for every array the context owns —
 * called at create, on the first sweep / two-level rounding and when the
 * coarse graph grows, with the context's stream; freed at destroy.  NULL:
 * the library's stream-ordered pool.  alloc_user is passed through. */
typedef void *(*irls_device_alloc_fn)(size_t bytes, void *stream, void *user);
typedef void (*irls_device_free_fn)(void *ptr, void *stream, void *user);
typedef struct {
    int32_t world_size, rank, device;
    const uint8_t *nccl_unique_id; /* 128 bytes from irls_nccl_unique_id on rank 0, broadcast by the caller */
    void *cuda_stream;
    irls_device_alloc_fn device_alloc;
    irls_device_free_fn device_free;
    void *alloc_user;
} irls_comm_desc;

/* Fill a fresh NCCL unique id (128 bytes) on rank 0. */
irls_status irls_nccl_unique_id(uint8_t out[128]);

/* Structured 2-D/3-D grid (the GraphCut / MRI configs).  N = nx*ny*nz
 * non-terminal nodes, u = x + nx*(y + ny*z); s = N and t = N+1 are virtual.
 * cx[u] = c(u, u+1) (ignored at x = nx-1), cy[u] = c(u, u+nx) (ignored at
 * y = ny-1), cz[u] = c(u, u+nx*ny) (ignored at z = nz-1); cs[u] = c(s,u),
 * ct[u] = c(u,t).  All arrays length N, host, float64, >= 0 (0 = absent edge,
 * A6).  Multi-GPU: z-slab partition aligned to the C3 groups (every rank owns
 * whole groups); world_size must divide 8 and the partition must be
 * group-aligned, else IRLS_ERR_INVALID_ARGUMENT.  Every rank passes the full
 * arrays. */
irls_status irls_mincut_create_stencil(irls_ctx **ctx, const irls_comm_desc *comm,
                                       int32_t nx, int32_t ny, int32_t nz,
                                       const double *cx, const double *cy, const double *cz,
                                       const double *cs, const double *ct,
                                       const irls_options *opt);

/* General undirected graph as CSR over all n nodes including s and t:
 * row_ptr[n+1] (int64), col[row_ptr[n]] (int32), w (float64 >= 0).  Entries of
 * a row with the same column are merged by summation in CSR order (A7); self
 * loops are rejected; the merged matrix must be exactly symmetric.  The edge
 * {s,t}, if present, is the additive constant c_st (A5).  Multi-GPU: id
 * strips — rank r owns the reduced ids of C3 groups [8r/W, 8(r+1)/W) (chunk
 * boundaries; W must divide 8 and the graph must have >= 8 chunks of 4096
 * non-terminals); its rows keep their neighbours' values in a ghost block
 * refreshed by one grouped NCCL exchange per halo (send lists follow from the
 * symmetry of G~); every rank passes the full CSR. */
irls_status irls_mincut_create_csr(irls_ctx **ctx, const irls_comm_desc *comm, int64_t n,
                                   const int64_t *row_ptr, const int32_t *col, const double *w,
                                   int64_t s, int64_t t, const irls_options *opt);

/* Per-solve diagnostics. */
typedef struct {
    int32_t cg_iters, converged, status, reserved;
    double rel_res;      /* recursive residual / ref at exit */
    double true_rel_res; /* record_trace: ||b - A x|| / ref (same norm) */
    double S_eps;        /* record_trace: Eq. 9 at x^(l) */
    double flow_value;   /* record_trace: Prop. 3, x^T L^(l) x */
    double current_s;    /* record_trace: sum_u g_su (1 - x_u) */
    double x_min, x_max; /* record_trace */
    double ref;          /* ||M^-1 b|| or ||b|| */
    float ms;            /* device time of this solve */
    float ms_assemble;   /* irls_solve's one-graph mode: device time from the previous solve's end to the
                            end of this solve's assembly (K1 incl. its START reduction); else 0 */
} irls_step_report;

/* x^(0): W = C, cold CG (Alg. 1 step 2).  report may be NULL. */
irls_status irls_init(irls_ctx *ctx, irls_step_report *report);
/* One IRLS step: reweight from the current x (Eq. 4), assemble (Eq. 7-8),
 * PCG warm or cold per options.  Requires irls_init (or set_potentials). */
irls_status irls_step(irls_ctx *ctx, irls_step_report *report);

typedef enum { IRLS_FROM_SCRATCH = 0, IRLS_CONTINUE = 1 } irls_solve_mode;
/* FROM_SCRATCH: irls_init then T steps (T+1 solves).  CONTINUE: T steps from
 * the current x (a warm-started sequence of related problems).
 * per_step: T+1 (FROM_SCRATCH) or T (CONTINUE) reports, or NULL. */
irls_status irls_solve(irls_ctx *ctx, int32_t mode, irls_step_report *per_step,
                       int64_t *total_cg_iters);

/* Sweep cut of the current x (O7): order non-terminals by (x desc, id
 * asc), prefix sums of per-node cut deltas in exact fixed point (A15), first
 * argmin.  side: host bytes, one per output id (stencil N+2, CSR n), 1 =
 * source side; order: host, n~ output ids in sweep order, or NULL; k: number
 * of non-terminals on the source side; cut_value: recomputed from the set
 * (C3).  side may be NULL: the result stays on the device (irls_get_side).
 * Only rank 0 writes outputs. */
irls_status irls_sweep_cut(irls_ctx *ctx, uint8_t *side, int32_t *order, int64_t *k,
                           double *cut_value);
irls_status irls_get_side(irls_ctx *ctx, uint8_t *side);

/* ---- two-level rounding --------------
 * Rounds the current x^(T) (gathered to rank 0) instead of the sweep:
 *   1. K-means (Lloyd, k = 2) on the components of x^(T) — the non-terminals
 *      plus x_s = 1, x_t = 0 — from centres 0.1 / 0.9 (A25): u joins
 *      cluster 1 iff |x_u - c1| < |x_u - c0|; centres are C3 sums / counts;
 *      stop when both centres repeat (<= 100 rounds).
 *   2. gamma0 = c0 + 0.05, gamma1 = c1 - 0.05; S0 = {x <= gamma0},
 *      S1 = {x >= gamma1} \ S0, Sc = the rest; s in S1, t in S0.
 *   3. G_c: Sc + {s_c, t_c}, capacities per the four bullets of P:L278-281
 *      in the sweep's 128-bit fixed point Q(c) = rint(c 2^F) (A27), built on
 *      the GPU.
 *   4. Exact max-flow on G_c on the HOST (Boykov-Kolmogorov, timed
 *      separately, A28); source side = the set reachable from s_c in the
 *      final residual graph (minimal min cut, unique).
 *   5. S = {s} + S1 + that set ("an s-t cut on G_c induces an s-t cut on G",
 *      P:L283); the cut value is recomputed on G by C3 (A29).
 * side: n_total bytes on the host (as irls_sweep_cut) or NULL; rep: may be
 * NULL.  Collective in multi-GPU mode; rank 0 computes, every rank returns
 * the report.  Requires a solve (IRLS_ERR_STATE); NaN in x ->
 * IRLS_ERR_BAD_POTENTIAL; a max-flow whose value differs from the cut value
 * of its set (strong duality fails: an internal error) -> IRLS_ERR_CUDA. */
typedef struct {
    double c0, c1, gamma0, gamma1;   /* K-means centres and thresholds */
    int32_t kmeans_rounds;
    int32_t certified;               /* 1: max-flow value == cut value of the returned set on G_c */
    int64_t n0, n1, nc;              /* |S0|, |S1|, |Sc| over the non-terminals */
    int64_t coarse_nlinks;           /* n-links of G_c (undirected) */
    int64_t augmentations;           /* max-flow augmenting paths */
    int32_t F, pad;                  /* fixed-point fraction bits */
    double coarse_flow;              /* max-flow value on G_c including the s_c-t_c edge (Q / 2^F) */
    double cut_value;                /* cut of the returned set on G (C3) */
    float ms_gpu;                    /* K-means + coarsening + lift + cut on the device */
    float ms_copy;                   /* coarse graph to the host and source side back */
    float ms_maxflow;                /* host max-flow (the paper's sequential second level) */
    float ms_total;                  /* wall time of the call on rank 0 */
} irls_two_level_report;
irls_status irls_two_level_cut(irls_ctx *ctx, uint8_t *side, irls_two_level_report *rep);

/* mu*, the exact minimum cut of G, by the same pipeline with no contraction
 * (gamma0 = -inf, gamma1 = +inf: G_c = G, the no-coarsening limit of S:L384)
 * — the denominator of delta = (mu - mu*) / mu* (Eq. 13).  Needs
 * no solve; host memory ~60 B per n-link.  Multi-rank contexts: collective,
 * computed on rank 0 (which holds the whole graph), report broadcast. */
irls_status irls_exact_min_cut(irls_ctx *ctx, uint8_t *side, irls_two_level_report *rep);

/* ---- Cheeger-type diagnostic (Theorem 4) ----
 * lambda_2, the non-zero finite generalized eigenvalue of the pencil (L, D)
 * (Eq. spectral; D = diag(d), d_s = d_t = C = 2 sum_e c_e),
 * by its constrained-WLS characterisation: minimise
 * (1/2C) x^T L x subject to x_s = 1, x_t = -1 on the capacities c (W = C).
 * One cold Jacobi-PCG solve of the reduced system (Eq. 7 with f = (1,-1):
 * b_u = cs_u - ct_u) with the given rtol / cap / norm (irls_cg_norm), then
 * x^T L x and C by C3 (A30).  phi^2/2 <= lambda_2 <= 2 phi with phi =
 * mu_star / C (Theorem 4).  The IRLS state (x, options) is restored afterwards.
 * x_out: the solution v (n~ doubles, host; rank 0) or NULL.  Multi-rank
 * contexts: collective; the solve runs distributed, the quadratic form on
 * rank 0 over the gathered v (like the sweep), every rank returns its
 * values. */
typedef struct {
    double lambda2, xLx, C, rel_res;
    int32_t cg_iters, converged;
    float ms;            /* device time of the solve */
    int32_t launches;    /* kernels launched */
} irls_lambda2_report;
irls_status irls_lambda2(irls_ctx *ctx, double cg_rtol, int32_t cg_max_iter, int32_t cg_norm, double *x_out,
                         irls_lambda2_report *rep);

/* The coarse graph of the last irls_two_level_cut (rank 0, host copies), for
 * parity tests: cls [n~] per reduced node (0 = S0, 1 = S1, 2 = Sc); ptr
 * [nc+1], col [entries] (coarse ids, ascending; both directions stored), cap
 * [entries] (capacity, float64); qs, qt [2*nc] and qst [2]: the s_c / t_c /
 * s_c-t_c links as 128-bit fixed point (lo, hi) words.  Any pointer may be
 * NULL; sizes from the report (entries = 2 * coarse_nlinks). */
irls_status irls_two_level_get_coarse(irls_ctx *ctx, int8_t *cls, int32_t *ptr, int32_t *col, double *cap,
                                      uint64_t *qs, uint64_t *qt, uint64_t *qst);

/* Host-only: the library's exact max-flow on a coarse graph in fixed point
 * (the one irls_two_level_cut runs), for CPU tests.  ptr [nc+1] / col:
 * symmetric CSR with ascending columns; cap, qs, qt, flow: 128-bit (lo, hi)
 * words; flow excludes any direct s_c-t_c edge.  src [nc]: 1 = reachable
 * from s_c.  certified = 1 when the flow equals the cut of src.  Returns
 * IRLS_ERR_INVALID_ARGUMENT for a non-symmetric graph. */
irls_status irls_coarse_maxflow(int32_t nc, const int32_t *ptr, const int32_t *col, const uint64_t *cap,
                                const uint64_t *qs, const uint64_t *qt, uint8_t *src, uint64_t *flow,
                                int32_t *certified);

/* Replace the terminal capacities (full arrays, length n~ in reduced order:
 * stencil u, CSR ascending original id without s and t); keeps x. */
irls_status irls_set_terminal_weights(irls_ctx *ctx, const double *cs, const double *ct);

/* Potentials of the n~ non-terminals in reduced order (host). */
irls_status irls_get_potentials(irls_ctx *ctx, double *x);
irls_status irls_set_potentials(irls_ctx *ctx, const double *x);

/* Counters of the last solve: kernel launches of this library and device
 * time of the dominant kernels, for the roofline. */
typedef struct {
    int64_t launches;        /* kernels launched by the library in the last irls_solve / sweep */
    int64_t cg_iters;        /* CG iterations in the last irls_solve */
    int64_t n_nonterminal;   /* n~ (global) */
    int64_t n_links;         /* |E~| with c > 0 (global) */
    int64_t n_local;         /* non-terminals owned by this rank */
    int64_t sweep_sorted;    /* nodes the last rank-0 sweep radix-sorted: n~ (full sort), or the
                                candidate buckets' nodes of the branch-and-bound sweep */
} irls_stats;
irls_status irls_get_stats(irls_ctx *ctx, irls_stats *stats);

/* Kernel timing with CUDA events on the context's stream, on the current
 * state: runs `reps` launches of kernel `which` (0 = CG SpMV+p-update K3,
 * 1 = CG axpy+Jacobi K5, 2 = reweight+assemble K1) and returns the mean ms.
 * The CG state is saved and restored, so the solve state is unchanged.
 * which = 3 (multi-rank NCCL contexts only; COLLECTIVE: every rank calls it
 * with the same reps): the per-CG-iteration z halo exchange (one plane / the
 * packed send lists to each neighbour over NCCL), timed on this rank; it only
 * rewrites z's ghost entries with the values they already hold.
 * which = 4 (cg_variant = IRLS_CG_CG only): the Chronopoulos-Gear iteration
 * kernel (one iteration at k = 1; state saved and restored as above). */
irls_status irls_time_kernel(irls_ctx *ctx, int32_t which, int32_t reps, float *mean_ms);

void irls_mincut_destroy(irls_ctx *ctx);
const char *irls_status_string(irls_status st);
const char *irls_last_error(const irls_ctx *ctx);

/* ---- virtual groups: the multi-GPU data path on ONE device --------------- */
/* All `world` ranks of the z-slab partition of one grid, driven by one host
 * thread on one device and one stream, phase by phase (every rank's kernel,
 * then the collective, ...); halo exchange, slot allreduce and gather are
 * device copies instead of NCCL.  Everything else — slabs, ghost planes,
 * per-rank reductions, ghost p updates, finalize kernels, rank-0 sweep — is
 * the multi-GPU code.  Used to test that path without several GPUs; results
 * are bitwise those of world 1.  world must divide 8 and the slabs must be
 * group-aligned (see irls_plan_stencil). */
typedef struct irls_vgroup irls_vgroup;
irls_status irls_vgroup_create_stencil(irls_vgroup **g, int32_t world, int32_t device, int32_t nx, int32_t ny,
                                       int32_t nz, const double *cx, const double *cy, const double *cz,
                                       const double *cs, const double *ct, const irls_options *opt);
/* The CSR graph's id strips (rank r owns C3 groups [8r/W, 8(r+1)/W): reduced
 * ids on chunk boundaries; W > 1 needs >= 8 chunks), ghost blocks and halo
 * lists, as irls_mincut_create_csr builds them on each of W processes. */
irls_status irls_vgroup_create_csr(irls_vgroup **g, int32_t world, int32_t device, int64_t n, const int64_t *row_ptr,
                                   const int32_t *col, const double *w, int64_t s, int64_t t,
                                   const irls_options *opt);
irls_status irls_vgroup_solve(irls_vgroup *g, int32_t mode, irls_step_report *per_step, int64_t *total_cg_iters);
irls_status irls_vgroup_sweep_cut(irls_vgroup *g, uint8_t *side, int32_t *order, int64_t *k, double *cut_value);
irls_status irls_vgroup_two_level_cut(irls_vgroup *g, uint8_t *side, irls_two_level_report *rep);
irls_status irls_vgroup_get_potentials(irls_vgroup *g, double *x);
irls_status irls_vgroup_set_terminal_weights(irls_vgroup *g, const double *cs, const double *ct);
const char *irls_vgroup_last_error(const irls_vgroup *g);  /* first rank's error detail */
void irls_vgroup_destroy(irls_vgroup *g);

/* ---- host-only helpers of the multi-GPU plan (no device work) ----------- */
/* C3 groups of a length-n index space: chunk count K = ceil(n/4096); group g
 * covers chunks [floor(gK/8), floor((g+1)K/8)). */
irls_status irls_plan_stencil(int32_t nx, int32_t ny, int32_t nz, int32_t world, int32_t rank,
                              int32_t *z0, int32_t *z1, int32_t *g0, int32_t *g1);
/* Id strip of rank `rank` of a CSR graph with nr non-terminals: reduced ids
 * [lo, hi) = the chunks of C3 groups [g0, g1) = [8r/W, 8(r+1)/W); W > 1 needs
 * every rank to own >= 1 chunk (else IRLS_ERR_INVALID_ARGUMENT). */
irls_status irls_plan_csr(int64_t nr, int32_t world, int32_t rank, int64_t *lo, int64_t *hi, int32_t *g0, int32_t *g1);
/* Host-only: the halo of id strip `rank` over
 * the REDUCED adjacency (nr non-terminals, aptr[nr+1], aidx ascending per row,
 * terminals removed), as irls_mincut_create_csr builds it: lo_hi[2] = the
 * strip [lo, hi); ghosts (ascending global ids, grouped by owner) with
 * recv_off[world+1] the per-owner ranges; send_idx (local ids, ascending per
 * peer) with send_off[world+1] the per-peer ranges.  ghosts / send_idx are
 * filled only when non-NULL and large enough (ghosts_cap, send_cap entries;
 * call once with NULL to learn recv_off[world] / send_off[world]).  Entry i of
 * rank q's send list to rank r lands at ghost slot recv_off_r[q] + i of r. */
irls_status irls_csr_halo_plan(int64_t nr, const int64_t *aptr, const int32_t *aidx, int32_t world, int32_t rank,
                               int64_t *lo_hi, int64_t *recv_off, int64_t *send_off, int32_t *ghosts,
                               int64_t ghosts_cap, int32_t *send_idx, int64_t send_cap);
/* Halo plan of rank `rank`'s z-slab: element offsets relative to its first
 * owned node (send_lo/send_hi: boundary planes sent to peer_lo/peer_hi;
 * recv_lo/recv_hi: ghost planes received from them), count = nx*ny values
 * per message; peers are -1 when absent. */
typedef struct {
    int64_t count, n_own, send_lo, recv_lo, send_hi, recv_hi;
    int32_t peer_lo, peer_hi, first_plane, reserved;
} irls_halo;
irls_status irls_halo_plan(int32_t nx, int32_t ny, int32_t nz, int32_t world, int32_t rank, irls_halo *h);
/* The fixed 8-leaf tree of C3 step 6: ((s0+s4)+(s2+s6))+((s1+s5)+(s3+s7)). */
double irls_combine_slots(const double slots[8]);

#ifdef __cplusplus
}
#endif
#endif /* IRLS_MINCUT_H */
