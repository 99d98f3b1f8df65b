// kernels.h — argument blocks and launchers of the IRLS kernels (internal).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace irls {

// Which assembly to run (Algorithm 1: step 2 vs step 4).
// ASM_LAMBDA2: W = C with the boundary x_s = 1, x_t = -1 (b = gs - gt), the
// Cheeger diagnostic's constrained WLS.
enum AssembleMode { ASM_INIT = 0, ASM_REWEIGHT_WARM = 1, ASM_REWEIGHT_COLD = 2, ASM_LAMBDA2 = 3 };

// Per-node CG vectors (local indexing; owned nodes are [0, n_own); arrays
// marked "ghost" also hold one plane below (negative indices) and above).
struct VecArgs {
    int64_t n_own;
    int32_t chunk0;      // global chunk index of local chunk 0
    double *x;           // ghost
    double *D, *Dinv, *r, *q;
    double *z;           // ghost
    double *p0, *p1;     // ghost (ping-pong: iteration k reads p[k&1], writes p[(k+1)&1])
    const int32_t *frozen;  // DevCtrl::frozen: assembly kernels skip a step that repeats a fixed point
    // K5 only, z-slabs with irls_options.p2p: the boundary planes of z are also
    // stored into the neighbours' ghost planes over peer memory (the halo
    // exchange fused into the kernel that produces z)
    double *zpeer_lo = nullptr;  // lower neighbour's upper ghost plane <- my first owned plane
    double *zpeer_hi = nullptr;  // upper neighbour's lower ghost plane <- my last owned plane
    int64_t plane = 0;           // nx * ny
};

// Chronopoulos-Gear PCG (irls_options.cg_variant = IRLS_CG_CG): iteration k
// reads r[k&1], w[k&1], s[(k+1)&1] (also at neighbours, incl. ghosts) and
// writes r[(k+1)&1], w[(k+1)&1], s[k&1]; p and x are updated in place.
struct CgArgs {
    double *r[2], *w[2], *s[2];  // ghosted like x
    double *p;
    // z-slabs with irls_options.p2p: the new w of the first / last owned plane
    // is also stored into the lower / upper neighbour's ghost plane of w[b]
    double *wpeer_lo[2] = {nullptr, nullptr}, *wpeer_hi[2] = {nullptr, nullptr};
    int64_t plane = 0;
};

struct StencilArgs {
    int32_t nx, ny, nz;
    int64_t P;           // nx*ny
    int64_t lo;          // global id of local node 0
    FastDiv fd_nx, fd_ny;
    int32_t lo_ghost;    // a rank below owns plane z0-1 (ghost planes valid)
    const double *cx, *cy, *cz;  // cz: ghost below
    const double *cs, *ct;
    double *gx, *gy, *gz;        // gz: ghost below
};

struct SellArgs {
    int64_t n;                   // rows
    const int64_t *slice_ptr;    // [nslices+1] entry offsets (multiples of kSell)
    const int32_t *col;          // -1 = padding (always after the real entries)
    const double *c;             // capacities
    double *g;                   // conductances
    const double *cs, *ct;
    int32_t wmax;                // widest slice (max degree)
    int64_t gbase, glow;         // strips: columns >= gbase are ghosts; the first glow ghosts have lower ids
};

// Block-Jacobi preconditioner (A32, block_jacobi.cu).  Blocks are stored in
// the order of decreasing size (independent blocks: the order changes no
// bit); block b occupies positions [bptr[b], bptr[b+1]); position i holds
// local node bnode[i]; its in-block lower neighbours are (ecol[e], *eg[e])
// for e in [eptr[i], eptr[i+1]).  One thread per block; the 32 blocks of a
// lane group G = b / 32 share a row table (rows gR[G] .. gR[G+1]): row i spans
// block-local columns [rowF, i) — the union of the 32 blocks' envelopes,
// zero-padded (exact no-ops of the dense algorithm) — and starts rowOff band
// elements into G's band.  Band element t of row i of lane l lives at
// L[32 (gL[G] + rowOff + t) + l], the pivot of row i at Dd[32 (gR[G] + i) + l]:
// a warp reads 256 contiguous bytes per element.
struct BlockArgs {
    int64_t nblk = 0;
    int32_t m_max = 0;           // largest block
    const int32_t *bptr = nullptr, *bnode = nullptr, *eptr = nullptr, *ecol = nullptr;
    const double *const *eg = nullptr;  // the conductance of each in-block edge (device pointers)
    const int64_t *gL = nullptr, *gR = nullptr;  // per lane group: band start, row-table start
    const int32_t *rowF = nullptr, *rowOff = nullptr;
    double *L = nullptr, *Dd = nullptr;  // factor: unit lower L (band), pivots
    double *mb = nullptr;        // M^-1 b (START)
};

struct CondArgs {
    cudaGraphConditionalHandle handle;
    int32_t use;                 // 1: set the WHILE condition from device code
    int32_t finalize;            // 1: world == 1, the last block finalizes the scalars
};

// assembly (K1 / K2): fills g*, D, Dinv, r, z and START reduction
void launch_stencil_assemble(const StencilArgs &s, const VecArgs &v, const RedArgs &ra, const CondArgs &cd,
                             int mode, double eps, cudaStream_t st);
void launch_sell_assemble(const SellArgs &s, const VecArgs &v, const RedArgs &ra, const CondArgs &cd,
                          int mode, double eps, cudaStream_t st);
// _ex: also store the terminal conductances gs/gt (record_trace diagnostics)
int launch_stencil_assemble_ex(const StencilArgs &s, const VecArgs &v, const RedArgs &ra, const CondArgs &cd,
                                int mode, double eps, double *gs_out, double *gt_out, cudaStream_t st);
int launch_sell_assemble_ex(const SellArgs &s, const VecArgs &v, const RedArgs &ra, const CondArgs &cd,
                             int mode, double eps, double *gs_out, double *gt_out, cudaStream_t st);
// K3: p = z + beta p_old (fused), lazy x += alpha p_old, q = L~ p, PQ reduction
void launch_stencil_pspmv(const StencilArgs &s, const VecArgs &v, const RedArgs &ra, const CondArgs &cd,
                          cudaStream_t st, bool w0 = false);
void launch_sell_pspmv(const SellArgs &s, const VecArgs &v, const RedArgs &ra, const CondArgs &cd,
                       cudaStream_t st, bool w0 = false);
// small.cu: the whole CG loop of a <= one-chunk graph in one block (kind 0
// stencil, 1 SELL); runs after the assembly, before finish / report
void small_cg_prepare();  // once per process, outside stream capture (128 KB dynamic shared memory)
void launch_small_cg(int kind, const StencilArgs &s, const SellArgs &sl, const VecArgs &v, DevCtrl *ctrl,
                     double *slots, cudaStream_t st);
// ghost planes of p for the next iteration (multi-GPU stencil)
void launch_ghost_pupdate(const VecArgs &v, int64_t ghost_lo, int64_t ghost_hi, int64_t plane, DevCtrl *ctrl,
                          cudaStream_t st);
// CSR multi-rank: ghost block of p updated from the exchanged z; halo packing
void launch_ghost_range_pupdate(const VecArgs &v, int64_t start, int64_t count, DevCtrl *ctrl, cudaStream_t st);
void launch_halo_pack(const double *arr, const int32_t *idx, int64_t n, double *out, cudaStream_t st);
// block Jacobi (A32): KF factor per IRLS step; START: z0 = M^-1 r0, mb = M^-1 b
// + the 5 START reductions; iteration: r -= alpha q, z = M^-1 r + the 3 RZ
// reductions.  Return the number of kernels launched.
int launch_block_factor(const BlockArgs &b, const double *D, const int32_t *frozen, cudaStream_t st);
int launch_block_start(const BlockArgs &b, const VecArgs &v, const double *gs, const RedArgs &ra,
                       const CondArgs &cd, cudaStream_t st);
int launch_block_iter(const BlockArgs &b, const VecArgs &v, const RedArgs &ra, const CondArgs &cd, cudaStream_t st);
// K5: r -= alpha q, z = Dinv r, RZ reduction
void launch_axpy_jacobi(const VecArgs &v, const RedArgs &ra, const CondArgs &cd, cudaStream_t st);
// after the loop: x += alpha p_last (or x = 0 if b = 0)
void launch_finish(const VecArgs &v, DevCtrl *ctrl, cudaStream_t st);
// scalar finalizers for the multi-GPU path (after the slot allreduce)
// Chronopoulos-Gear iteration (one kernel; C3 quantities [<r,z>, <z,w>,
// <z,z>, <r,r>]; world 1: the last block finalizes and sets the condition)
void launch_stencil_cgcg(const StencilArgs &s, const VecArgs &v, const CgArgs &g, const RedArgs &ra,
                         const CondArgs &cd, cudaStream_t st);
void launch_sell_cgcg(const SellArgs &s, const VecArgs &v, const CgArgs &g, const RedArgs &ra, const CondArgs &cd,
                      cudaStream_t st);
// ghost entries [lo, lo + n): s = w + beta s_old, r = r - alpha s (the owner's formulas)
void launch_cgcg_ghost(const CgArgs &g, int64_t lo, int64_t n, const DevCtrl *ctrl, cudaStream_t st);
void launch_cgcg_finish(const VecArgs &v, const DevCtrl *ctrl, cudaStream_t st);
// CSR strips with p2p: the z halo as peer stores, then this rank's group sums
// (nq quantities of groups [g0, g1)) and arrivals pushed to every rank
void launch_p2p_halo_push(const double *z, const int32_t *send_idx, const int32_t *peer, const int64_t *pos,
                          int64_t n, double *const *zpeers, const double *slots, int nq, int g0, int g1, int32_t K,
                          int n_fin, double *const *pslots, unsigned long long *const *pcnt, int world,
                          const DevCtrl *ctrl, cudaStream_t st);
void launch_finalize(int phase, DevCtrl *ctrl, const double *slots, const CondArgs &cd, const P2PWait &pw,
                     cudaStream_t st);
// write the step report from the control block
struct DevReport {
    int32_t cg_iters, converged, status, pad;
    double rel_res, true_rel_res, S_eps, flow_value, current_s, x_min, x_max, ref;
    unsigned long long t_end;  // %globaltimer (ns) when the solve's report was written
    unsigned long long t_asm;  // %globaltimer (ns) when the solve's START reduction was finalized
};
// freeze: set DevCtrl::frozen when this (warm reweight) solve ended with 0 CG
// iterations and x unchanged (fixed_point_exit)
void launch_report(DevCtrl *ctrl, DevReport *reports, int freeze, cudaStream_t st);
// fixed_point_exit graph gate: IF condition = !frozen
void launch_gate(const DevCtrl *ctrl, cudaGraphConditionalHandle h, cudaStream_t st);
// multi-step graph: time mark; outer WHILE over `count` IRLS steps (stops
// early at a fixed point when freeze_exit); copies of the frozen report
void launch_mark(DevCtrl *ctrl, cudaStream_t st);
void launch_outer_init(DevCtrl *ctrl, cudaGraphConditionalHandle h, int count, cudaStream_t st);
void launch_outer_next(DevCtrl *ctrl, cudaGraphConditionalHandle h, int freeze_exit, cudaStream_t st);
void launch_fill_reports(DevCtrl *ctrl, DevReport *reports, cudaStream_t st);
// record_trace diagnostics: [S_eps, flow, current_s, true_res^2] + x range
void launch_stencil_diag_ex(const StencilArgs &s, const VecArgs &v, const RedArgs &ra, double eps, int norm,
                            const double *gsv, const double *gtv, cudaStream_t st);
void launch_sell_diag_ex(const SellArgs &s, const VecArgs &v, const RedArgs &ra, double eps, int norm,
                         const double *gsv, const double *gtv, cudaStream_t st);
void launch_diag_finalize(DevCtrl *ctrl, const double *slots, DevReport *reports, int norm, const P2PWait &pw,
                          cudaStream_t st);

enum { PH_START = 0, PH_PQ = 1, PH_RZ = 2, PH_W0 = 3, PH_CG = 4 };
// virtual-group slot sum: dst[i] = sum_r src[r][i]
void launch_vsum(double *const *src, int W, int n, double *dst, cudaStream_t st);
void launch_vminmax(DevCtrl *const *ctrl, int W, cudaStream_t st);

// stencil_pair.cu (nx even): K1a+K1b, K3, K5, finish with 128-bit pair access
int launch_pair_assemble(const StencilArgs &s, const VecArgs &v, const RedArgs &ra, const CondArgs &cd, int mode,
                          double eps, double *gs_out, double *gt_out, cudaStream_t st);
void launch_pair_pspmv(const StencilArgs &s, const VecArgs &v, const RedArgs &ra, const CondArgs &cd,
                       cudaStream_t st, bool w0 = false);
void launch_pair_axpy(const VecArgs &v, const RedArgs &ra, const CondArgs &cd, cudaStream_t st);
void launch_pair_cgcg(const StencilArgs &s, const VecArgs &v, const CgArgs &g, const RedArgs &ra, const CondArgs &cd,
                      cudaStream_t st);
void launch_pair_finish(const VecArgs &v, DevCtrl *ctrl, cudaStream_t st);
// sell_pair.cu (widest slice <= 8): false when the generic SELL kernel must run
bool launch_sellp_assemble(const SellArgs &s, const VecArgs &v, const RedArgs &ra, const CondArgs &cd, int mode,
                           double eps, double *gs_out, double *gt_out, cudaStream_t st);
bool launch_sellp_pspmv(const SellArgs &s, const VecArgs &v, const RedArgs &ra, const CondArgs &cd, cudaStream_t st,
                        bool w0 = false);

// ---------------------------------------------------------------------------
// Sweep cut (K8-K12)
// ---------------------------------------------------------------------------
struct SweepBuffers {
    int64_t n;
    unsigned long long *keys, *keys_alt;
    int32_t *vals, *vals_alt;
    int32_t *rank;
    int32_t *tile_hist;      // [256][ntiles]: the radix passes' look-back words
    int32_t *tile_off;       // [256][ntiles]
    int32_t *scan_tmp;       // scan block totals
    unsigned long long *digit_hist;  // [8][256] global histograms
    __int128 *delta;         // [n+2] delta_v in id order (+ P0, P_k)
    __int128 *tile_sum;      // [ntiles] scan look-back: tile aggregates
    __int128 *tile_incl;     // [ntiles] scan look-back: inclusive prefixes
    __int128 *qcs_tile;      // [ntiles] per-tile sums of Q(cs) (P_0)
    __int128 *tile_min;      // [ntiles]
    int64_t *tile_argmin;    // [ntiles]
    int32_t *flags;          // [0] NaN seen, [1] radix tile ticket
    int64_t *k_out;
    int32_t *lastv;          // the k-th node of the order when ord is not materialised (sweep_bb.cu)
    double *cross;
    uint8_t *side;           // n_total
};
int64_t sweep_ntiles(int64_t n);
// prep: keys (x desc), ids, delta_v in id order (exact fixed point), global
// digit histograms, per-tile Q(cs) sums, NaN flag (digit_hist and flags zeroed
// by the caller)
void sweep_prep_stencil(const StencilArgs &s, int64_t N, int32_t F, const double *x, SweepBuffers &b,
                        cudaStream_t st);
void sweep_prep_sell(const SellArgs &s, int32_t F, const double *x, SweepBuffers &b, cudaStream_t st);
// returns pointer to the sorted ids buffer (vals or vals_alt); *nan: a NaN key
// (nothing sorted)
int32_t *sweep_sort(SweepBuffers &b, cudaStream_t st, int *launches, bool *nan);
void sweep_scan_argmin(SweepBuffers &b, const int32_t *ord, __int128 P0, cudaStream_t st);
// branch-and-bound sweep (sweep_bb.cu): buckets from a sorted sample of x;
// one pass for the per-bucket counts / exact delta sums / negative bounds;
// only the buckets that can hold the first minimum are extracted, sorted and
// scanned.  Partials: [4][bb_num_ctas()][nb] u64, [bb_num_ctas()] i128.
typedef unsigned long long u64_t;
int bb_num_ctas();
size_t bb_table_bytes();  // splitter cell table + meta (one buffer)
void bb_sample_sort(const double *x, int64_t n, int32_t ns, int32_t nb, u64_t *skey, int32_t *sid, u64_t *spk,
                    int32_t *spi, void *table, cudaStream_t st);
void bb_pass_stencil(const StencilArgs &s, int64_t N, int32_t F, const double *x, const u64_t *spk,
                     const int32_t *spi, const void *table, int32_t nb, u64_t *part, __int128 *pqcs, int32_t *flags,
                     uint16_t *bkt, cudaStream_t st);
void bb_pass_sell(const SellArgs &s, int32_t F, const double *x, const u64_t *spk, const int32_t *spi,
                  const void *table, int32_t nb, u64_t *part, __int128 *pqcs, int32_t *flags, uint16_t *bkt,
                  cudaStream_t st);
void bb_reduce(const u64_t *part, const __int128 *pqcs, int32_t nb, __int128 qcst, unsigned *cnt, __int128 *bsum,
               __int128 *bneg, __int128 *p0, cudaStream_t st);
void bb_extract(int64_t N, const double *x, const uint16_t *bkt, int32_t nb, const int16_t *slot_of, u64_t *cursor,
                u64_t *ck, int32_t *cid, u64_t *ida, int32_t *posa, u64_t *digit_hist, cudaStream_t st);
void bb_cdelta_stencil(const StencilArgs &s, int32_t F, const double *x, const int32_t *cid, const int32_t *perm,
                       int64_t C, __int128 *cdel, cudaStream_t st);
void bb_cdelta_sell(const SellArgs &s, int32_t F, const double *x, const int32_t *cid, const int32_t *perm, int64_t C,
                    __int128 *cdel, cudaStream_t st);
void bb_gather(const u64_t *ck, const int32_t *perm, int64_t C, u64_t *kb, int32_t *jb, u64_t *digit_hist,
               cudaStream_t st);
void bb_cand_scan(const __int128 *cdel, const int32_t *sorted, const int64_t *cdst, const int64_t *cpos,
                  const __int128 *cP, int32_t ncand, __int128 *cmin, int64_t *carg, cudaStream_t st);
void bb_finish(const __int128 *cmin, const int64_t *carg, int32_t nc, __int128 bP, int64_t bpos, const int64_t *cdst,
               const int64_t *cpos, const int32_t *sorted, const int32_t *cid, int64_t *k_out, int32_t *lastv,
               int32_t *flags, cudaStream_t st);
// side + cut of the first k of the order, membership from x (the sweep)
void sweep_side_cross_x_stencil(const StencilArgs &s, int64_t N, const double *x, const int32_t *ord, SweepBuffers &b,
                                const RedArgs &ra, cudaStream_t st);
void sweep_side_cross_x_sell(const SellArgs &s, const double *x, const int32_t *ord, const int64_t *orig,
                             SweepBuffers &b, const RedArgs &ra, cudaStream_t st);
// side + cut of {v : rank[v] < k} (two-level lift)
void sweep_side_cross_stencil(const StencilArgs &s, int64_t N, SweepBuffers &b, const RedArgs &ra,
                              cudaStream_t st);
void sweep_side_cross_sell(const SellArgs &s, const int64_t *orig, int64_t n_total, SweepBuffers &b,
                           const RedArgs &ra, cudaStream_t st);
void sweep_order_out(const int32_t *order, const int64_t *orig, int32_t *out, int64_t n, cudaStream_t st);
__int128 qfix_host(double c, int32_t F);
// create-time CSR preparation on the GPU (csr_prep.cu)
void csrp_check(const int64_t *rp, const int32_t *col, const double *w, int64_t n, unsigned long long *first_bad,
                int32_t *selfloop, cudaStream_t st);
void csrp_merge(const int64_t *rp, const int32_t *col, const double *w, int64_t n, int32_t *scol, double *sw,
                int32_t *mcnt, cudaStream_t st);
void csrp_compact(const int64_t *rp, const int32_t *scol, const double *sw, const int32_t *mptr, int64_t n,
                  int32_t *mcol, double *mw, cudaStream_t st);
void csrp_symmetry(const int32_t *mptr, const int32_t *mcol, const double *mw, int64_t n, int32_t *asym,
                   cudaStream_t st);
void csrp_reduce(const int32_t *mptr, const int32_t *mcol, const double *mw, int64_t nr, int64_t s, int64_t t,
                 double *cs, double *ct, int64_t *orig, int32_t *acnt, unsigned long long *cnt,
                 unsigned long long *cmax_bits, double *cst, cudaStream_t st);
void csrp_fill(const int32_t *mptr, const int32_t *mcol, const double *mw, const int64_t *orig, const int32_t *aptr,
               int64_t nr, int64_t s, int64_t t, int32_t *aidx, double *ac, cudaStream_t st);
void csrp_components(const int32_t *aptr, const int32_t *aidx, const double *cs, const double *ct, int64_t nr,
                     int32_t *par, int32_t *root, uint8_t *anchored, int32_t *lonely, cudaStream_t st);
void csrp_sell_width(const int32_t *aptr, int64_t nr, int32_t *sw, unsigned long long *wmax, cudaStream_t st);
void csrp_i32_to_i64(const int32_t *in, int64_t n, int64_t *out, cudaStream_t st);
void csrp_sell_fill(const int32_t *aptr, const int32_t *aidx, const double *ac, const int64_t *sptr, int64_t nr,
                    int32_t *scol, double *scap, cudaStream_t st);
void exclusive_scan_i32(const int32_t *in, int64_t m, int32_t *out, int64_t *tmp, cudaStream_t st, int *launches);

// ---------------------------------------------------------------------------
// Two-level rounding (twolevel.cu, maxflow.cu)
// ---------------------------------------------------------------------------
struct TLState {
    double c0, c1;
    int32_t done, rounds;
};
struct TLBuffers {
    int64_t n;               // non-terminals
    TLState *st;
    double *part, *slots;    // private C3 scratch: [3][K], [3][8]
    DevCtrl *ctrl;           // private group counters
    int8_t *cls;             // [n] 0 = S0, 1 = S1, 2 = Sc
    int32_t *flag, *cid;     // [n] Sc indicator, coarse id (exclusive scan)
    int32_t *deg, *eoff;     // [n] coarse degree, coarse row offset (exclusive scan)
    int64_t *scan_tmp;
    __int128 *tile_a;        // [ntiles] s_c-t_c partials
    int32_t *tile_n1;        // [ntiles] |S1| partials
    int32_t *cp;             // [n+1] coarse row pointer
    __int128 *cqs, *cqt;     // [n] coarse terminal links (by coarse id)
    int32_t *ccol;           // [cap_entries]
    double *ccap;
    int64_t cap_entries;
    uint8_t *src;            // [n] coarse source side (by coarse id)
    int32_t *prank;          // [n] 0 = source side
    int64_t *one;            // device constant 1 (the "k" of the side/cut kernel)
    uint8_t *side;           // [n_total]
};
int64_t tl_ntiles(int64_t n);
// lambda2.cu: [x^T L x owned terms, owned capacities] -> slots (2 quantities)
void launch_l2_quad_stencil(const StencilArgs &s, int64_t N, const double *x, const RedArgs &ra, cudaStream_t st);
void launch_l2_quad_sell(const SellArgs &s, const double *x, const RedArgs &ra, cudaStream_t st);
void tl_kmeans_round(const double *x, int64_t n, TLState *st, const RedArgs &ra, cudaStream_t stream);
void tl_classify_stencil(const StencilArgs &s, int64_t N, const double *x, double g0, double g1, int32_t F,
                         TLBuffers &b, cudaStream_t st);
void tl_classify_sell(const SellArgs &s, const double *x, double g0, double g1, int32_t F, TLBuffers &b,
                      cudaStream_t st);
void tl_fill_stencil(const StencilArgs &s, int64_t N, int32_t F, TLBuffers &b, cudaStream_t st);
void tl_fill_sell(const SellArgs &s, int32_t F, TLBuffers &b, cudaStream_t st);
void tl_lift(TLBuffers &b, cudaStream_t st);

// Exact max-flow on the coarse graph (host; maxflow.cu).  Undirected coarse
// CSR (nc nodes, symmetric, fixed-point capacities), terminal links qs/qt.
// Returns the flow value (without the direct s_c-t_c edge) and src[u] = 1 iff
// u is reachable from s_c in the final residual graph.
__int128 maxflow_bk(int32_t nc, const int32_t *ptr, const int32_t *col, const __int128 *cap, const __int128 *qs,
                    const __int128 *qt, uint8_t *src, int64_t *stats);

}  // namespace irls

namespace irls {
// validate.cu: out[0..5] = bad, zero interior n-links, nodes with a positive
// terminal edge, positive capacities, bits of the max capacity, positive n-links
int validate_stencil(int32_t nx, int32_t ny, int32_t nz, const double *cx, const double *cy, const double *cz,
                     const double *cs, const double *ct, unsigned long long *out_host, cudaStream_t st);
}  // namespace irls
