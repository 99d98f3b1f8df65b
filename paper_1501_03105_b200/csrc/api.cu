// api.cu — the C ABI (include/irls_mincut.h): options and status, the
// multi-GPU plans and collectives, the per-solve CUDA graphs (device-side
// WHILE loops, the multi-step graph, the one-block path), the solve entry
// points, potentials / terminal weights, stats and kernel timing, destroy and
// the virtual groups.  Context creation: api_create.cu; rounding (sweep,
// two-level, exact min cut) and lambda_2: api_round.cu.
#include "api_internal.h"

// ---------------------------------------------------------------------------
// error plumbing
// ---------------------------------------------------------------------------
irls_status fail(irls_ctx *c, irls_status st, const std::string &msg)
{
    if (c) {
        c->err = msg;
        // host-side validation errors leave the context usable
        if (st != IRLS_ERR_INVALID_ARGUMENT && st != IRLS_ERR_BAD_POTENTIAL && st != IRLS_ERR_STATE &&
            st != IRLS_ERR_SINGULAR && st != IRLS_ERR_BAD_CAPACITY)
            c->poisoned = true;
    }
    return st;
}


extern "C" void irls_options_default(irls_options *o)
{
    if (!o) return;
    o->eps = 1e-6;
    o->T = 50;
    o->cg_rtol = 1e-3;
    o->cg_max_iter = 50;
    o->cg_norm = IRLS_NORM_PRECONDITIONED;
    o->warm_start = 1;
    o->record_trace = 0;
    o->loop_mode = IRLS_LOOP_GRAPH;
    o->fixed_point_exit = 0;
    o->p2p = 0;
    o->cg_variant = IRLS_CG_HS;
    o->block_size = 0;
}

extern "C" const char *irls_status_string(irls_status st)
{
    switch (st) {
    case IRLS_OK: return "IRLS_OK";
    case IRLS_ERR_INVALID_ARGUMENT: return "IRLS_ERR_INVALID_ARGUMENT";
    case IRLS_ERR_SOURCE_EQUALS_SINK: return "IRLS_ERR_SOURCE_EQUALS_SINK";
    case IRLS_ERR_BAD_CAPACITY: return "IRLS_ERR_BAD_CAPACITY";
    case IRLS_ERR_NOT_SYMMETRIC: return "IRLS_ERR_NOT_SYMMETRIC";
    case IRLS_ERR_SINGULAR: return "IRLS_ERR_SINGULAR";
    case IRLS_ERR_CG_BREAKDOWN: return "IRLS_ERR_CG_BREAKDOWN";
    case IRLS_ERR_BAD_POTENTIAL: return "IRLS_ERR_BAD_POTENTIAL";
    case IRLS_ERR_STATE: return "IRLS_ERR_STATE";
    case IRLS_ERR_CUDA: return "IRLS_ERR_CUDA";
    case IRLS_ERR_NCCL: return "IRLS_ERR_NCCL";
    case IRLS_ERR_OOM: return "IRLS_ERR_OOM";
    }
    return "IRLS_ERR_UNKNOWN";
}

extern "C" const char *irls_last_error(const irls_ctx *c) { return c ? c->err.c_str() : "null context"; }

extern "C" irls_status irls_nccl_unique_id(uint8_t out[128])
{
    if (!out) return IRLS_ERR_INVALID_ARGUMENT;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return IRLS_ERR_NCCL;
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    memcpy(out, &id, 128);
    return IRLS_OK;
}

// C3 step 6 on the host (slots after the slot-exact allreduce).
extern "C" double irls_combine_slots(const double s[8])
{
    return ((s[0] + s[4]) + (s[2] + s[6])) + ((s[1] + s[5]) + (s[3] + s[7]));
}

// z-slab plan: rank r owns C3 groups [8r/W, 8(r+1)/W); the slab must start
// and end on z-plane boundaries.
extern "C" irls_status irls_plan_stencil(int32_t nx, int32_t ny, int32_t nz, int32_t world, int32_t rank,
                                         int32_t *z0, int32_t *z1, int32_t *g0, int32_t *g1)
{
    if (nx < 1 || ny < 1 || nz < 1 || world < 1 || rank < 0 || rank >= world) return IRLS_ERR_INVALID_ARGUMENT;
    if (8 % world != 0) return IRLS_ERR_INVALID_ARGUMENT;
    const int64_t N = (int64_t)nx * ny * nz, P = (int64_t)nx * ny;
    const int32_t K = (int32_t)((N + kChunk - 1) / kChunk);
    const int a = rank * 8 / world, b = (rank + 1) * 8 / world;
    const int64_t lo = std::min<int64_t>((int64_t)group_lo(a, K) * kChunk, N);
    const int64_t hi = std::min<int64_t>((int64_t)group_lo(b, K) * kChunk, N);
    if (lo % P != 0 || (hi % P != 0 && hi != N)) return IRLS_ERR_INVALID_ARGUMENT;
    if (world > 1 && hi <= lo) return IRLS_ERR_INVALID_ARGUMENT;
    if (z0) *z0 = (int32_t)(lo / P);
    if (z1) *z1 = (int32_t)((hi + P - 1) / P);
    if (g0) *g0 = a;
    if (g1) *g1 = b;
    return IRLS_OK;
}

// ---------------------------------------------------------------------------
// multi-GPU collectives (NCCL over NVLink): halo planes, slot allreduce
// ---------------------------------------------------------------------------
// Halo plan of a z-slab (offsets relative to the first owned node): the
// boundary planes go to the neighbour ranks and their planes land in the
// ghost planes just outside [0, n_own).  Peers are -1 when absent.
extern "C" irls_status irls_halo_plan(int32_t nx, int32_t ny, int32_t nz, int32_t world, int32_t rank,
                                      irls_halo *h)
{
    if (!h) return IRLS_ERR_INVALID_ARGUMENT;
    int32_t z0, z1;
    irls_status s = irls_plan_stencil(nx, ny, nz, world, rank, &z0, &z1, nullptr, nullptr);
    if (s) return s;
    const int64_t P = (int64_t)nx * ny;
    const int64_t n_own = (int64_t)(z1 - z0) * P;
    h->count = P;
    h->n_own = n_own;
    h->first_plane = z0;
    h->peer_lo = rank > 0 ? rank - 1 : -1;
    h->peer_hi = rank < world - 1 ? rank + 1 : -1;
    h->send_lo = 0;
    h->recv_lo = -P;
    h->send_hi = n_own - P;
    h->recv_hi = n_own;
    return IRLS_OK;
}

// CSR: pack the owned values the peers need, then one grouped exchange; the
// peers' values land in the ghost block (contiguous per peer, ascending ids).
static irls_status halo_csr(irls_ctx *c, double *arr, cudaStream_t st)
{
    const int64_t ns = c->send_off[c->world];
    if (ns > 0) launch_halo_pack(arr, c->send_idx, ns, c->sendbuf, st);
    NK(ncclGroupStart());
    for (int q = 0; q < c->world; q++) {
        const int64_t sc = c->send_off[q + 1] - c->send_off[q], rc = c->recv_off[q + 1] - c->recv_off[q];
        if (sc > 0) NK(ncclSend(c->sendbuf + c->send_off[q], (size_t)sc, ncclDouble, q, c->nccl, st));
        if (rc > 0) NK(ncclRecv(arr + c->npad_own + c->recv_off[q], (size_t)rc, ncclDouble, q, c->nccl, st));
    }
    NK(ncclGroupEnd());
    return IRLS_OK;
}

static irls_status halo(irls_ctx *c, double *arr, cudaStream_t st)
{
    if (!c->multi) return IRLS_OK;
    if (c->kind == 1) return halo_csr(c, arr, st);
    const irls_halo &h = c->hplan;
    NK(ncclGroupStart());
    if (h.peer_lo >= 0) {
        NK(ncclSend(arr + h.send_lo, (size_t)h.count, ncclDouble, h.peer_lo, c->nccl, st));
        NK(ncclRecv(arr + h.recv_lo, (size_t)h.count, ncclDouble, h.peer_lo, c->nccl, st));
    }
    if (h.peer_hi >= 0) {
        NK(ncclSend(arr + h.send_hi, (size_t)h.count, ncclDouble, h.peer_hi, c->nccl, st));
        NK(ncclRecv(arr + h.recv_hi, (size_t)h.count, ncclDouble, h.peer_hi, c->nccl, st));
    }
    NK(ncclGroupEnd());
    return IRLS_OK;
}

// Virtual group: rank 0's x_full <- every rank's slab (device copies).
irls_status vgather_x(irls_vgroup *g, double **full)
{
    irls_ctx *c = g->ranks[0];
    if (!c->x_full) {
        c->x_full = dalloc<double>(c, c->n_glob);
        if (!c->x_full) return fail(c, IRLS_ERR_OOM, "x_full");
    }
    for (irls_ctx *d : g->ranks)
        CK(cudaMemcpyAsync(c->x_full + d->lo, d->x, sizeof(double) * d->n_own, cudaMemcpyDeviceToDevice, g->stream));
    *full = c->x_full;
    return IRLS_OK;
}

// Rank 0 receives every slab of x (Algorithm 1 step 5: "Gather the
// voltage vector to the root process"); returns the full vector's pointer on
// rank 0 (the local x when world == 1).
irls_status gather_x(irls_ctx *c, double **full)
{
    *full = c->x;
    if (!c->multi) return IRLS_OK;
    cudaStream_t st = c->stream;
    if (c->rank == 0 && !c->x_full) {
        c->x_full = dalloc<double>(c, c->n_glob);
        if (!c->x_full) return fail(c, IRLS_ERR_OOM, "x_full");
    }
    NK(ncclGroupStart());
    if (c->rank == 0) {
        for (int r = 1; r < c->world; r++) {
            const int64_t lo = c->rank_lo[r], n = c->rank_lo[r + 1] - lo;
            if (n > 0) NK(ncclRecv(c->x_full + lo, (size_t)n, ncclDouble, r, c->nccl, st));
        }
    } else if (c->n_own > 0) {
        NK(ncclSend(c->x, (size_t)c->n_own, ncclDouble, 0, c->nccl, st));
    }
    NK(ncclGroupEnd());
    if (c->rank == 0) CK(cudaMemcpyAsync(c->x_full, c->x, sizeof(double) * c->n_own, cudaMemcpyDeviceToDevice, st));
    *full = c->x_full;
    return IRLS_OK;
}

static irls_status allreduce_slots(irls_ctx *c, int nq, cudaStream_t st)
{
    if (!c->multi) return IRLS_OK;
    NK(ncclAllReduce(c->slots_local, c->slots_glob, (size_t)nq * kGroups, ncclDouble, ncclSum, c->nccl, st));
    return IRLS_OK;
}

// ---------------------------------------------------------------------------
// Collectives over the ranks a host thread drives: one rank with NCCL (one
// process per GPU), or every rank of a virtual group (one process, one device,
// one stream; the same data movement done with device copies).
// ---------------------------------------------------------------------------

// The array of a ghosted vector on one rank (halo exchanges name it this way).
typedef double *(*ArrSel)(irls_ctx *);
static double *sel_x(irls_ctx *c) { return c->x; }
static double *sel_z(irls_ctx *c) { return c->z; }
static double *sel_r(irls_ctx *c) { return c->r; }
static double *sel_dinv(irls_ctx *c) { return c->Dinv; }
static double *sel_w0(irls_ctx *c) { return c->cg_w[0]; }
static double *sel_w1(irls_ctx *c) { return c->cg_w[1]; }

static irls_status coll_halo_sel(Ranks &R, ArrSel sel, cudaStream_t st)
{
    irls_ctx *c = R[0];
    if (!c->multi) return IRLS_OK;
    if (!c->vg) return halo(c, sel(c), st);
    if (c->kind == 1) {  // pack on every rank, then the same copies NCCL would make
        for (irls_ctx *d : R) {
            const int64_t ns = d->send_off[d->world];
            if (ns > 0) launch_halo_pack(sel(d), d->send_idx, ns, d->sendbuf, st);
        }
        for (irls_ctx *d : R)
            for (int q = 0; q < d->world; q++) {
                const int64_t rc = d->recv_off[q + 1] - d->recv_off[q];
                if (rc == 0) continue;
                irls_ctx *o = R[q];
                CK(cudaMemcpyAsync(sel(d) + d->npad_own + d->recv_off[q], o->sendbuf + o->send_off[d->rank],
                                   sizeof(double) * rc, cudaMemcpyDeviceToDevice, st));
            }
        return IRLS_OK;
    }
    for (irls_ctx *d : R) {
        const irls_halo &h = d->hplan;
        double *arr = sel(d);
        const size_t bytes = sizeof(double) * (size_t)h.count;
        if (h.peer_lo >= 0) {
            irls_ctx *o = R[h.peer_lo];
            CK(cudaMemcpyAsync(arr + h.recv_lo, sel(o) + o->hplan.send_hi, bytes, cudaMemcpyDeviceToDevice, st));
        }
        if (h.peer_hi >= 0) {
            irls_ctx *o = R[h.peer_hi];
            CK(cudaMemcpyAsync(arr + h.recv_hi, sel(o) + o->hplan.send_lo, bytes, cudaMemcpyDeviceToDevice, st));
        }
    }
    return IRLS_OK;
}

static irls_status coll_halo(Ranks &R, bool z_not_x, cudaStream_t st)
{
    return coll_halo_sel(R, z_not_x ? sel_z : sel_x, st);
}

static irls_status coll_allreduce(Ranks &R, int nq, cudaStream_t st)
{
    irls_ctx *c = R[0];
    if (!c->multi || c->p2p) return IRLS_OK;  // p2p: the producers already stored every slot
    if (!c->vg) return allreduce_slots(c, nq, st);
    // sum of every rank's slots in rank order (each slot has one non-zero
    // contributor, so this is the same exact value NCCL's sum produces)
    launch_vsum(c->vg->src_slots, (int)R.size(), nq * kGroups, R[0]->slots_glob, st);
    for (size_t r = 1; r < R.size(); r++)
        CK(cudaMemcpyAsync(R[r]->slots_glob, R[0]->slots_glob, sizeof(double) * nq * kGroups,
                           cudaMemcpyDeviceToDevice, st));
    return IRLS_OK;
}

// x range of the diagnostics: min / max of the order-preserving keys.
static irls_status coll_minmax(Ranks &R, cudaStream_t st)
{
    irls_ctx *c = R[0];
    if (!c->multi) return IRLS_OK;
    if (!c->vg) {
        NK(ncclGroupStart());
        NK(ncclAllReduce(&c->ctrl->xmin_key, &c->ctrl->xmin_key, 1, ncclUint64, ncclMin, c->nccl, st));
        NK(ncclAllReduce(&c->ctrl->xmax_key, &c->ctrl->xmax_key, 1, ncclUint64, ncclMax, c->nccl, st));
        NK(ncclGroupEnd());
        return IRLS_OK;
    }
    launch_vminmax(c->vg->src_ctrl, (int)R.size(), st);
    return IRLS_OK;
}

// ---------------------------------------------------------------------------
// enqueue pieces of one solve (over the ranks this thread drives)
// ---------------------------------------------------------------------------
// The p2p consumer side of one rank (an inactive wait when p2p is off).
static P2PWait p2p_wait_args(const irls_ctx *c)
{
    P2PWait pw;
    pw.buf = c->p2p ? c->p2p_buf : nullptr;
    pw.cnt = c->p2p ? (const unsigned long long *)(c->p2p_buf + 2 * kMaxQ * kGroups) : nullptr;
    pw.n_groups = c->n_groups_all;
    return pw;
}

// RedArgs of the solve's reductions: with p2p the owner blocks push to peers.
static RedArgs red_args_solve(const irls_ctx *c)
{
    RedArgs ra = red_args(c);
    if (c->p2p) {
        ra.pslots = c->d_pslots;
        ra.pcnt = c->d_pcnt;
        ra.world = c->world;
    }
    return ra;
}

static irls_status enq_assemble(Ranks &R, int mode, const CondArgs &cd, cudaStream_t st)
{
    irls_status s;
    if (mode != ASM_INIT && mode != ASM_LAMBDA2 && (s = coll_halo(R, false, st))) return s;
    for (irls_ctx *c : R) {
        const VecArgs v = vec_args(c);
        const RedArgs ra = red_args_solve(c);
        // block Jacobi (A32): K1 assembles (its Jacobi z0 and START sums are
        // superseded), then factor, z0 = M^-1 r0, mb = M^-1 b, START sums
        CondArgs cdk = cd;
        if (c->blk_on) cdk.finalize = 0;
        if (c->kind == 0)
            c->launches += launch_stencil_assemble_ex(stencil_args(c, false), v, ra, cdk, mode, c->opt.eps,
                                                      c->gs_diag, c->gt_diag, st);
        else
            c->launches += launch_sell_assemble_ex(sell_args(c), v, ra, cdk, mode, c->opt.eps, c->gs_diag,
                                                   c->gt_diag, st);
        if (c->blk_on) {
            c->launches += launch_block_factor(c->blk, c->D, v.frozen, st);
            c->launches += launch_block_start(c->blk, v, c->gs_diag, ra, cd, st);
        }
    }
    if (R[0]->multi) {
        if ((s = coll_allreduce(R, 5, st))) return s;
        for (irls_ctx *c : R) {
            launch_finalize(PH_START, c->ctrl, c->slots_glob, cd, p2p_wait_args(c), st);
            c->launches++;
        }
        if ((s = coll_halo(R, true, st))) return s;
    }
    if (R[0]->cgcg) {  // CG-CG: w0 = A z0 and alpha_0 = rho / <z0, w0> (a K3 pass at k = 0 into w[0])
        if (R[0]->multi && ((s = coll_halo_sel(R, sel_r, st)) || (s = coll_halo_sel(R, sel_dinv, st)))) return s;
        for (irls_ctx *c : R) {
            VecArgs v = vec_args(c);
            v.q = c->cg_w[0];
            if (c->kind == 0) launch_stencil_pspmv(stencil_args(c, false), v, red_args_solve(c), cd, st, true);
            else launch_sell_pspmv(sell_args(c), v, red_args_solve(c), cd, st, true);
            c->launches++;
        }
        if (R[0]->multi) {
            if ((s = coll_allreduce(R, 1, st))) return s;
            for (irls_ctx *c : R) {
                launch_finalize(PH_W0, c->ctrl, c->slots_glob, cd, p2p_wait_args(c), st);
                c->launches++;
            }
            if ((s = coll_halo_sel(R, sel_w0, st))) return s;
        }
    }
    return last_launch(R[0], "assemble");
}

// Chronopoulos-Gear body: TWO iterations (k even, then k odd) so that the
// ping-pong buffer each halo moves is fixed at capture time; the second one
// is skipped on the device when the first one stopped.
static irls_status enq_body_cgcg(Ranks &R, const CondArgs &cd, cudaStream_t st)
{
    irls_status s;
    for (int half = 0; half < 2; half++) {
        for (irls_ctx *c : R) {
            const VecArgs v = vec_args(c);
            CgArgs g = cg_args(c);
            // ghost s, r first (they only read this iteration's ghost values,
            // which peers may overwrite once this rank's sums are published)
            if (c->multi && c->kind == 0) {
                if (c->lo_ghost) launch_cgcg_ghost(g, -c->P, c->P, c->ctrl, st);
                if (c->hi_ghost) launch_cgcg_ghost(g, c->n_own, c->P, c->ctrl, st);
                c->launches += (c->lo_ghost ? 1 : 0) + (c->hi_ghost ? 1 : 0);
            } else if (c->multi && c->n_ghost > 0) {
                launch_cgcg_ghost(g, c->npad_own, c->n_ghost, c->ctrl, st);
                c->launches++;
            }
            if (c->p2p && c->kind == 0) {  // the w halo fused into the iteration kernel (peer stores)
                for (int b = 0; b < 2; b++) {
                    g.wpeer_lo[b] = c->wpeer_lo[b];
                    g.wpeer_hi[b] = c->wpeer_hi[b];
                }
                g.plane = c->P;
            }
            if (c->kind == 0) launch_stencil_cgcg(stencil_args(c, false), v, g, red_args_solve(c), cd, st);
            else launch_sell_cgcg(sell_args(c), v, g, red_args_solve(c), cd, st);
            c->launches++;
        }
        if (R[0]->multi) {
            if ((s = coll_allreduce(R, 4, st))) return s;
            for (irls_ctx *c : R) {
                launch_finalize(PH_CG, c->ctrl, c->slots_glob, cd, p2p_wait_args(c), st);
                c->launches++;
            }
            if (!(R[0]->p2p && R[0]->kind == 0) && (s = coll_halo_sel(R, half == 0 ? sel_w1 : sel_w0, st)))
                return s;
        }
    }
    return last_launch(R[0], "cg-cg body");
}

static irls_status enq_body(Ranks &R, const CondArgs &cd, cudaStream_t st)
{
    if (R[0]->cgcg) return enq_body_cgcg(R, cd, st);
    irls_status s;
    for (irls_ctx *c : R) {
        const VecArgs v = vec_args(c);
        const RedArgs ra = red_args_solve(c);
        // ghost p first: it reads the ghost z of this iteration, which a
        // neighbour's K5 may overwrite over peer memory (p2p) as soon as this
        // rank's K3 has published its group sums
        if (c->multi && c->kind == 0) {
            launch_ghost_pupdate(v, c->lo_ghost, c->hi_ghost, c->P, c->ctrl, st);
            c->launches++;
        } else if (c->multi && c->n_ghost > 0) {
            launch_ghost_range_pupdate(v, c->npad_own, c->n_ghost, c->ctrl, st);
            c->launches++;
        }
        if (c->kind == 0) launch_stencil_pspmv(stencil_args(c, false), v, ra, cd, st);
        else launch_sell_pspmv(sell_args(c), v, ra, cd, st);
        c->launches++;
    }
    if (R[0]->multi) {
        if ((s = coll_allreduce(R, 1, st))) return s;
        for (irls_ctx *c : R) {
            launch_finalize(PH_PQ, c->ctrl, c->slots_glob, cd, p2p_wait_args(c), st);
            c->launches++;
        }
    }
    for (irls_ctx *c : R) {
        VecArgs v = vec_args(c);
        if (c->p2p && c->kind == 0) {  // the z halo fused into K5 (peer stores)
            v.zpeer_lo = c->zpeer_lo;
            v.zpeer_hi = c->zpeer_hi;
            v.plane = c->P;
        }
        const bool csr_p2p = c->p2p && c->kind == 1;
        if (c->blk_on) {  // block Jacobi (A32): r -= alpha q, z = M^-1 r, RZ sums
            c->launches += launch_block_iter(c->blk, v, red_args_solve(c), cd, st);
            continue;
        }
        launch_axpy_jacobi(v, csr_p2p ? red_args(c) : red_args_solve(c), cd, st);
        c->launches++;
        if (csr_p2p) {  // z halo as peer stores, then the group sums' push (after the stores)
            launch_p2p_halo_push(c->z, c->send_idx, c->halo_peer_dev, c->halo_pos_dev, c->send_off[c->world],
                                 c->d_zpeers, c->slots_local, 3, c->g0, c->g1, c->K, c->n_fin, c->d_pslots,
                                 c->d_pcnt, c->world, c->ctrl, st);
            c->launches += 2;
        }
    }
    if (R[0]->multi) {
        if ((s = coll_allreduce(R, 3, st))) return s;
        for (irls_ctx *c : R) {
            launch_finalize(PH_RZ, c->ctrl, c->slots_glob, cd, p2p_wait_args(c), st);
            c->launches++;
        }
        if (!R[0]->p2p && (s = coll_halo(R, true, st))) return s;
    }
    return last_launch(R[0], "cg body");
}

static void enq_finish(Ranks &R, cudaStream_t st)
{
    for (irls_ctx *c : R) {
        if (c->cgcg) launch_cgcg_finish(vec_args(c), c->ctrl, st);
        else launch_finish(vec_args(c), c->ctrl, st);
        c->launches += 1;
    }
}

// report (+ record_trace diagnostics); `finish` = also enqueue the x update
static irls_status enq_tail(Ranks &R, int mode, cudaStream_t st, bool finish = true)
{
    irls_status s;
    if (finish) enq_finish(R, st);
    for (irls_ctx *c : R) {
        launch_report(c->ctrl, c->reports, mode == ASM_REWEIGHT_WARM && c->opt.fixed_point_exit ? 1 : 0, st);
        c->launches += 1;
    }
    if (R[0]->opt.record_trace) {
        if (R[0]->multi && (s = coll_halo(R, false, st))) return s;
        for (irls_ctx *c : R) {
            const VecArgs v = vec_args(c);
            const RedArgs ra = red_args_solve(c);
            if (c->kind == 0)
                launch_stencil_diag_ex(stencil_args(c, false), v, ra, c->opt.eps, c->opt.cg_norm, c->gs_diag,
                                       c->gt_diag, st);
            else
                launch_sell_diag_ex(sell_args(c), v, ra, c->opt.eps, c->opt.cg_norm, c->gs_diag, c->gt_diag, st);
        }
        if (R[0]->multi && (s = coll_allreduce(R, 4, st))) return s;
        if ((s = coll_minmax(R, st))) return s;
        for (irls_ctx *c : R) {
            launch_diag_finalize(c->ctrl, c->slots_glob, c->reports, c->opt.cg_norm, p2p_wait_args(c), st);
            c->launches += 2;
        }
    }
    return last_launch(R[0], "tail");
}

// Per-solve CUDA graph (one rank, world 1): [x = 0] -> K1 (sets the WHILE
// condition) -> [x = 0] -> WHILE { K3 ; K5 (sets the condition) } -> finish
// -> report [-> diag].  With fixed_point_exit, a warm reweight solve is
// wrapped as  gate -> IF (not frozen) { K1 -> WHILE {...} -> finish } ->
// report: a frozen solve costs one graph launch and two one-thread kernels.
// One-block CG loop (small.cu) for a single rank whose graph is one C3 chunk.
static bool small_path(const irls_ctx *c)
{
    return !c->multi && !c->cgcg && !c->blk_on && c->n_own > 0 && c->n_own <= kChunk;
}

// Block Jacobi (A32) serves every IRLS solve; lambda_2's stays point Jacobi (A30).
static void set_blk_mode(Ranks &R, int mode)
{
    for (irls_ctx *c : R) c->blk_on = c->opt.block_size > 0 && mode != ASM_LAMBDA2;
}

static void enq_small(irls_ctx *c, cudaStream_t st)
{
    SellArgs sl{};
    StencilArgs sa{};
    if (c->kind == 0) sa = stencil_args(c, false);
    else sl = sell_args(c);
    launch_small_cg(c->kind, sa, sl, vec_args(c), c->ctrl, c->slots_local, st);
    c->launches++;
}

static irls_status capture_solve_body(irls_ctx *c, Ranks &R, int mode, cudaStream_t st)
{
    cudaStreamCaptureStatus cs;
    cudaGraph_t graph;
    const cudaGraphNode_t *deps = nullptr;
    size_t nd = 0;
    CK(cudaStreamGetCaptureInfo(st, &cs, nullptr, &graph, &deps, &nd));
    set_blk_mode(R, mode);
    const bool small = small_path(c);
    cudaGraphConditionalHandle h{};
    // default 0 at every launch: the assembly's last block turns the loop on
    if (!small) CK(cudaGraphConditionalHandleCreate(&h, graph, 0, cudaGraphCondAssignDefault));
    CondArgs cd;
    cd.handle = h;
    cd.use = small ? 0 : 1;
    cd.finalize = c->multi ? 0 : 1;  // multi-rank: the finalize kernels after the slot allreduce
    if (mode == ASM_INIT || mode == ASM_LAMBDA2) CK(cudaMemsetAsync(c->x, 0, sizeof(double) * c->n_own, st));
    irls_status s = enq_assemble(R, mode, cd, st);
    if (s) return s;
    if (mode == ASM_REWEIGHT_COLD) CK(cudaMemsetAsync(c->x, 0, sizeof(double) * c->n_own, st));
    if (small) {  // no WHILE node: the block loops itself
        enq_small(c, st);
        c->gl_body = 0;
        return last_launch(c, "small cg");
    }
    CK(cudaStreamGetCaptureInfo(st, &cs, nullptr, &graph, &deps, &nd));
    cudaGraphNodeParams p{};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t cnode;
    CK(cudaGraphAddNode(&cnode, graph, deps, nd, &p));
    cudaGraph_t body = p.conditional.phGraph_out[0];
    CK(cudaStreamUpdateCaptureDependencies(st, &cnode, 1, cudaStreamSetCaptureDependencies));
    CK(cudaStreamBeginCaptureToGraph(c->side_stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    const int64_t pre = c->launches;
    s = enq_body(R, cd, c->side_stream);
    c->gl_body = (c->launches - pre) / (c->cgcg ? 2 : 1);  // CG-CG bodies hold two iterations
    c->launches = pre;
    cudaGraph_t bodyg;
    CK(cudaStreamEndCapture(c->side_stream, &bodyg));
    return s;
}

// One solve, captured on `st` (which must be capturing): K1 -> WHILE {body}
// -> finish -> report, wrapped as gate -> IF (not frozen) {K1 -> WHILE ->
// finish} -> report when the fixed-point exit is on for this mode.
static irls_status capture_step(irls_ctx *c, Ranks &R, int mode, cudaStream_t st)
{
    const bool gated = c->opt.fixed_point_exit && mode == ASM_REWEIGHT_WARM;
    if (!gated) {
        irls_status s = capture_solve_body(c, R, mode, st);
        if (!s) s = enq_tail(R, mode, st);
        return s;
    }
    irls_status s = IRLS_OK;
    cudaStreamCaptureStatus cs;
    cudaGraph_t graph;
    const cudaGraphNode_t *deps = nullptr;
    size_t nd = 0;
    cudaGraphConditionalHandle hif;
    cudaError_t e = cudaStreamGetCaptureInfo(st, &cs, nullptr, &graph, &deps, &nd);
    if (e == cudaSuccess) e = cudaGraphConditionalHandleCreate(&hif, graph, 0, cudaGraphCondAssignDefault);
    if (e == cudaSuccess) {
        launch_gate(c->ctrl, hif, st);
        c->launches++;
        e = cudaStreamGetCaptureInfo(st, &cs, nullptr, &graph, &deps, &nd);
    }
    cudaGraphNodeParams p{};
    cudaGraphNode_t ifnode;
    if (e == cudaSuccess) {
        p.type = cudaGraphNodeTypeConditional;
        p.conditional.handle = hif;
        p.conditional.type = cudaGraphCondTypeIf;
        p.conditional.size = 1;
        e = cudaGraphAddNode(&ifnode, graph, deps, nd, &p);
    }
    if (e == cudaSuccess) e = cudaStreamUpdateCaptureDependencies(st, &ifnode, 1, cudaStreamSetCaptureDependencies);
    if (e == cudaSuccess)
        e = cudaStreamBeginCaptureToGraph(c->side_stream2, p.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                          cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) return fail(c, IRLS_ERR_CUDA, std::string("gated graph: ") + cudaGetErrorString(e));
    s = capture_solve_body(c, R, mode, c->side_stream2);
    if (!s) enq_finish(R, c->side_stream2);
    cudaGraph_t ifg;
    e = cudaStreamEndCapture(c->side_stream2, &ifg);
    if (!s && e != cudaSuccess) s = fail(c, IRLS_ERR_CUDA, std::string("gated graph: ") + cudaGetErrorString(e));
    if (!s) s = enq_tail(R, mode, st, false);
    return s;
}

static irls_status build_graph(irls_ctx *c, int mode)
{
    cudaStream_t st = c->stream;
    Ranks R{c};
    const int64_t lsave = c->launches;
    c->launches = 0;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    irls_status s = capture_step(c, R, mode, st);
    cudaGraph_t full = nullptr;
    cudaError_t e = cudaStreamEndCapture(st, &full);
    if (s) { if (full) cudaGraphDestroy(full); c->launches = lsave; return s; }
    CK(e);
    CK(cudaGraphInstantiate(&c->gexec[mode], full, 0));
    cudaGraphDestroy(full);
    c->gl_fixed[mode] = c->launches;
    c->launches = lsave;
    return IRLS_OK;
}

// T reweight steps of one irls_solve in ONE graph (world 1): mark ->
// WHILE_outer (T times, or until a fixed point with fixed_point_exit) {
// K1 -> WHILE_cg {K3; K5} -> finish -> report -> next } -> fill reports.
// One graph launch per irls_solve instead of one per IRLS step.
static irls_status build_graph_multi(irls_ctx *c, int mode)
{
    cudaStream_t st = c->stream;
    Ranks R{c};
    const int count = c->opt.T;
    const int fpx = c->opt.fixed_point_exit && mode == ASM_REWEIGHT_WARM ? 1 : 0;
    const int64_t lsave = c->launches;
    c->launches = 0;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    irls_status s = IRLS_OK;
    cudaStreamCaptureStatus cs;
    cudaGraph_t graph;
    const cudaGraphNode_t *deps = nullptr;
    size_t nd = 0;
    cudaGraphConditionalHandle hout;
    cudaError_t e = cudaStreamGetCaptureInfo(st, &cs, nullptr, &graph, &deps, &nd);
    if (e == cudaSuccess) e = cudaGraphConditionalHandleCreate(&hout, graph, 0, cudaGraphCondAssignDefault);
    if (e == cudaSuccess) {
        launch_outer_init(c->ctrl, hout, count, st);
        e = cudaStreamGetCaptureInfo(st, &cs, nullptr, &graph, &deps, &nd);
    }
    cudaGraphNodeParams p{};
    cudaGraphNode_t wnode;
    if (e == cudaSuccess) {
        p.type = cudaGraphNodeTypeConditional;
        p.conditional.handle = hout;
        p.conditional.type = cudaGraphCondTypeWhile;
        p.conditional.size = 1;
        e = cudaGraphAddNode(&wnode, graph, deps, nd, &p);
    }
    if (e == cudaSuccess) e = cudaStreamUpdateCaptureDependencies(st, &wnode, 1, cudaStreamSetCaptureDependencies);
    if (e == cudaSuccess)
        e = cudaStreamBeginCaptureToGraph(c->side_stream2, p.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                          cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) {
        s = fail(c, IRLS_ERR_CUDA, std::string("multi-step graph: ") + cudaGetErrorString(e));
    } else {
        s = capture_solve_body(c, R, mode, c->side_stream2);
        if (!s) s = enq_tail(R, mode, c->side_stream2);
        if (!s) {
            launch_outer_next(c->ctrl, hout, fpx, c->side_stream2);
            c->launches++;
        }
        cudaGraph_t bg;
        e = cudaStreamEndCapture(c->side_stream2, &bg);
        if (!s && e != cudaSuccess)
            s = fail(c, IRLS_ERR_CUDA, std::string("multi-step graph: ") + cudaGetErrorString(e));
    }
    const int64_t per_step = c->launches;
    if (!s && fpx) launch_fill_reports(c->ctrl, c->reports, st);
    cudaGraph_t full = nullptr;
    e = cudaStreamEndCapture(st, &full);
    if (s) { if (full) cudaGraphDestroy(full); c->launches = lsave; return s; }
    CK(e);
    CK(cudaGraphInstantiate(&c->gmulti[mode], full, 0));
    cudaGraphDestroy(full);
    c->gm_fixed[mode] = per_step;
    c->launches = lsave;
    return IRLS_OK;
}

// CUDA-graph loops: one rank without collectives, or (IRLS_LOOP_GRAPH_NCCL)
// a rank of a communicator, whose NCCL calls are captured into the graphs.
static bool graph_mode(const irls_ctx *c)
{
    if (c->vg) return false;
    // a communicator: the NCCL calls (or, with p2p, the per-solve ones only)
    // are captured into the graphs — no host round trip per CG iteration
    return c->opt.loop_mode == IRLS_LOOP_GRAPH || c->opt.loop_mode == IRLS_LOOP_GRAPH_NCCL;
}

static irls_status enqueue_solve(Ranks &R, int mode)
{
    irls_ctx *c = R[0];
    cudaStream_t st = c->stream;
    if (graph_mode(c) && R.size() == 1) {
        if (!c->gexec[mode]) {
            irls_status s = build_graph(c, mode);
            if (s) return s;
        }
        CK(cudaGraphLaunch(c->gexec[mode], st));
        c->launches += c->gl_fixed[mode];
        c->graph_iters_pending = true;
        return IRLS_OK;
    }
    // host loop: one 4-byte readback of the device "done" flag per iteration
    // (every rank computes the identical flag: the slot allreduce is exact)
    CondArgs cd;
    memset(&cd, 0, sizeof(cd));
    cd.use = 0;
    cd.finalize = c->multi ? 0 : 1;
    set_blk_mode(R, mode);
    if (mode == ASM_INIT || mode == ASM_LAMBDA2)
        for (irls_ctx *d : R) CK(cudaMemsetAsync(d->x, 0, sizeof(double) * d->n_own, st));
    irls_status s = enq_assemble(R, mode, cd, st);
    if (s) return s;
    if (mode == ASM_REWEIGHT_COLD)
        for (irls_ctx *d : R) CK(cudaMemsetAsync(d->x, 0, sizeof(double) * d->n_own, st));
    if (R.size() == 1 && small_path(c)) enq_small(c, st);
    for (;;) {
        CK(cudaMemcpyAsync(c->h_done, &c->ctrl->done, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (*c->h_done) break;
        s = enq_body(R, cd, st);
        if (s) return s;
    }
    return enq_tail(R, mode, st);
}

static void copy_report(const DevReport &d, irls_step_report *o, float ms, float ms_asm)
{
    o->cg_iters = d.cg_iters;
    o->converged = d.converged;
    o->status = d.status;
    o->reserved = 0;
    o->rel_res = d.rel_res;
    o->true_rel_res = d.true_rel_res;
    o->S_eps = d.S_eps;
    o->flow_value = d.flow_value;
    o->current_s = d.current_s;
    o->x_min = d.x_min;
    o->x_max = d.x_max;
    o->ref = d.ref;
    o->ms = ms;
    o->ms_assemble = ms_asm;
}

// Run `count` solves (first one with mode0, the rest with mode_rest); fill
// reports from rank 0 and check that every driven rank reports the same.
irls_status run_solves(Ranks &R, int mode0, int mode_rest, int count, irls_step_report *reps, int64_t *total)
{
    irls_ctx *c = R[0];
    cudaStream_t st = c->stream;
    for (irls_ctx *d : R) {
        d->launches = 0;
        CK(cudaMemsetAsync(&d->ctrl->step, 0, 2 * sizeof(int32_t), st));  // step, frozen
    }
    std::vector<cudaEvent_t> ev(count + 1);
    for (auto &e : ev) CK(cudaEventCreate(&e));
    CK(cudaEventRecord(ev[0], st));
    irls_status s = IRLS_OK;
    // graph mode, one rank: the T reweight steps run as ONE graph (outer WHILE);
    // per-step times then come from device timestamps in the reports
    const int nrest = mode0 == mode_rest ? count : count - 1;
    const bool multi_graph = graph_mode(c) && R.size() == 1 && nrest == c->opt.T &&
                             nrest >= 2 && (mode_rest == ASM_REWEIGHT_WARM || mode_rest == ASM_REWEIGHT_COLD);
    if (multi_graph) {
        launch_mark(c->ctrl, st);
        if (mode0 != mode_rest) s = enqueue_solve(R, mode0);
        if (!s && !c->gmulti[mode_rest]) s = build_graph_multi(c, mode_rest);
        if (!s) {
            CK(cudaGraphLaunch(c->gmulti[mode_rest], st));
            c->graph_iters_pending = true;
        }
    } else {
        for (int i = 0; i < count && !s; i++) {
            s = enqueue_solve(R, i == 0 ? mode0 : mode_rest);
            if (!s) {
                cudaError_t e = cudaEventRecord(ev[i + 1], st);
                if (e != cudaSuccess) s = fail(c, IRLS_ERR_CUDA, cudaGetErrorString(e));
            }
        }
    }
    cudaError_t e = cudaStreamSynchronize(st);
    if (!s && e != cudaSuccess) s = fail(c, IRLS_ERR_CUDA, std::string("solve: ") + cudaGetErrorString(e));
    std::vector<DevReport> h(count), h2(count);
    if (!s) {
        e = memcpy_sync(c, h.data(), c->reports, sizeof(DevReport) * count, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) s = fail(c, IRLS_ERR_CUDA, cudaGetErrorString(e));
        for (size_t r = 1; r < R.size() && !s; r++) {
            e = memcpy_sync(R[r], h2.data(), R[r]->reports, sizeof(DevReport) * count, cudaMemcpyDeviceToHost);
            if (e != cudaSuccess) s = fail(c, IRLS_ERR_CUDA, cudaGetErrorString(e));
            for (int i = 0; i < count && !s; i++)
                if (h2[i].cg_iters != h[i].cg_iters || h2[i].status != h[i].status || h2[i].rel_res != h[i].rel_res)
                    s = fail(c, IRLS_ERR_STATE, "ranks disagree on the CG scalars");
        }
    }
    int64_t tot = 0;
    unsigned long long t0 = 0;
    if (!s && multi_graph) {
        DevCtrl hc;
        e = memcpy_sync(c, &hc, c->ctrl, sizeof(hc), cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) s = fail(c, IRLS_ERR_CUDA, cudaGetErrorString(e));
        t0 = hc.t_mark;
        // kernels: the first (init) graph's fixed part, then per executed step
        int executed = 0;
        for (int i = (mode0 != mode_rest ? 1 : 0); i < count; i++)
            if (i == 0 || h[i].t_end != h[i - 1].t_end) executed++;
        c->launches += (int64_t)executed * c->gm_fixed[mode_rest] + 2;
    }
    if (!s) {
        for (int i = 0; i < count; i++) {
            float ms = 0.f, ms_asm = 0.f;
            if (multi_graph) {
                const unsigned long long prev = i == 0 ? t0 : h[i - 1].t_end;
                ms = h[i].t_end > prev ? (float)((double)(h[i].t_end - prev) * 1e-6) : 0.f;
                ms_asm = h[i].t_asm > prev && h[i].t_asm <= h[i].t_end ? (float)((double)(h[i].t_asm - prev) * 1e-6)
                                                                       : 0.f;
            } else {
                cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
            }
            tot += h[i].cg_iters;
            if (reps) copy_report(h[i], reps + i, ms, ms_asm);
            if (h[i].status != 0 && !s)
                s = fail(c, (irls_status)h[i].status,
                         h[i].status == ST_P2P_TIMEOUT ? "peer-memory collective: wait timed out (120 s)"
                                                       : "CG breakdown (p'Ap <= 0 or non-finite scalar)");
        }
        if (c->graph_iters_pending) c->launches += c->gl_body * tot;
        c->graph_iters_pending = false;
    }
    for (auto &ee : ev) cudaEventDestroy(ee);
    for (irls_ctx *d : R) {
        d->last_cg_iters = tot;
        if (!s) d->state = 1;
    }
    if (total) *total = tot;
    return s;
}

// ---------------------------------------------------------------------------
// solves
// ---------------------------------------------------------------------------
extern "C" irls_status irls_init(irls_ctx *c, irls_step_report *rep)
{
    NvtxRange nvtx_("irls_init");
    GUARD(c);
    if (c->n_glob == 0) { c->state = 1; return IRLS_OK; }
    irls_step_report tmp;
    Ranks R{c};
    return run_solves(R, ASM_INIT, ASM_INIT, 1, rep ? rep : &tmp, nullptr);
}

extern "C" irls_status irls_step(irls_ctx *c, irls_step_report *rep)
{
    NvtxRange nvtx_("irls_step");
    GUARD(c);
    if (c->state == 0) return fail(c, IRLS_ERR_STATE, "irls_step before irls_init / irls_set_potentials");
    if (c->n_glob == 0) return IRLS_OK;
    const int mode = c->opt.warm_start ? ASM_REWEIGHT_WARM : ASM_REWEIGHT_COLD;
    irls_step_report tmp;
    Ranks R{c};
    return run_solves(R, mode, mode, 1, rep ? rep : &tmp, nullptr);
}

extern "C" irls_status irls_solve(irls_ctx *c, int32_t mode, irls_step_report *per_step, int64_t *total)
{
    NvtxRange nvtx_("irls_solve");
    GUARD(c);
    if (mode != IRLS_FROM_SCRATCH && mode != IRLS_CONTINUE) return IRLS_ERR_INVALID_ARGUMENT;
    if (mode == IRLS_CONTINUE && c->state == 0) return fail(c, IRLS_ERR_STATE, "IRLS_CONTINUE without potentials");
    if (c->n_glob == 0) {  // no unknowns: every solve is trivially converged (b = 0, v = [])
        c->state = 1;
        if (total) *total = 0;
        const int count = mode == IRLS_FROM_SCRATCH ? c->opt.T + 1 : c->opt.T;
        for (int i = 0; per_step && i < count; i++) {
            memset(per_step + i, 0, sizeof(irls_step_report));
            per_step[i].converged = 1;
        }
        return IRLS_OK;
    }
    const int step_mode = c->opt.warm_start ? ASM_REWEIGHT_WARM : ASM_REWEIGHT_COLD;
    Ranks R{c};
    if (mode == IRLS_FROM_SCRATCH) return run_solves(R, ASM_INIT, step_mode, c->opt.T + 1, per_step, total);
    if (c->opt.T == 0) { if (total) *total = 0; return IRLS_OK; }
    return run_solves(R, step_mode, step_mode, c->opt.T, per_step, total);
}

// ---------------------------------------------------------------------------
// potentials / terminal weights
// ---------------------------------------------------------------------------
extern "C" irls_status irls_get_potentials(irls_ctx *c, double *x)
{
    GUARD(c);
    if (c->state == 0) return fail(c, IRLS_ERR_STATE, "no potentials yet");
    if (c->rank == 0 && !x) return IRLS_ERR_INVALID_ARGUMENT;
    double *full = nullptr;
    irls_status s = gather_x(c, &full);
    if (s) return s;
    if (c->rank == 0) CK(cudaMemcpyAsync(x, full, sizeof(double) * c->n_glob, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return IRLS_OK;
}

extern "C" irls_status irls_set_potentials(irls_ctx *c, const double *x)
{
    GUARD(c);
    if (!x) return IRLS_ERR_INVALID_ARGUMENT;
    CK(cudaMemcpyAsync(c->x, x + c->lo, sizeof(double) * c->n_own, cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->state = 1;
    c->sweep_valid = false;
    return IRLS_OK;
}

extern "C" irls_status irls_set_terminal_weights(irls_ctx *c, const double *cs, const double *ct)
{
    GUARD(c);
    if (!cs || !ct) return IRLS_ERR_INVALID_ARGUMENT;
    const int64_t n = c->n_glob;
    double cmax = c->c_st;
    int64_t cnt = c->c_st > 0;
    for (int64_t u = 0; u < n; u++) {
        if (!(cs[u] >= 0.0) || isinf(cs[u]) || !(ct[u] >= 0.0) || isinf(ct[u])) return IRLS_ERR_BAD_CAPACITY;
        if (cs[u] > 0) { cnt++; cmax = std::max(cmax, cs[u]); }
        if (ct[u] > 0) { cnt++; cmax = std::max(cmax, ct[u]); }
    }
    // n-link part of F: recomputed from the device copies
    if (c->kind == 0) {
        // Validate the new weights in scratch buffers: the context's cs/ct
        // (and F) change only once the weights are accepted, so a rejected
        // call (SINGULAR is not poisoning) leaves the previous problem intact.
        unsigned long long vo[6];
        double *scs = nullptr, *sct = nullptr;
        CK(cudaMallocAsync((void **)&scs, sizeof(double) * std::max<int64_t>(n, 1), c->stream));
        CK(cudaMallocAsync((void **)&sct, sizeof(double) * std::max<int64_t>(n, 1), c->stream));
        auto release = [&]() { cudaFreeAsync(scs, c->stream); cudaFreeAsync(sct, c->stream); };
        CK(cudaMemcpyAsync(scs, cs, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(sct, ct, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
        if (validate_stencil(c->nx, c->ny, c->nz, c->cx, c->cy, c->cz, scs, sct, vo, c->stream)) {
            release();
            return fail(c, IRLS_ERR_CUDA, "validate");
        }
        if (vo[1] != 0 || vo[2] == 0) {
            // zero n-links present: full check on the host copy
            std::vector<double> hx(n), hy(n), hz(n);
            memcpy_sync(c, hx.data(), c->cx, sizeof(double) * n, cudaMemcpyDeviceToHost);
            memcpy_sync(c, hy.data(), c->cy, sizeof(double) * n, cudaMemcpyDeviceToHost);
            memcpy_sync(c, hz.data(), c->cz, sizeof(double) * n, cudaMemcpyDeviceToHost);
            if (!grid_nonsingular(c->nx, c->ny, c->nz, hx.data(), hy.data(), hz.data(), cs, ct)) {
                release();
                CK(cudaStreamSynchronize(c->stream));
                return fail(c, IRLS_ERR_SINGULAR, "terminal weights make L~ singular");
            }
        }
        CK(cudaMemcpyAsync(c->cs, scs, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
        CK(cudaMemcpyAsync(c->ct, sct, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
        release();
        CK(cudaStreamSynchronize(c->stream));
        double m;
        memcpy(&m, &vo[4], sizeof(double));
        c->F = compute_F(m, (int64_t)vo[3]);
    } else {
        std::vector<double> cp(c->n_entries);
        std::vector<int32_t> cl(c->n_entries);
        memcpy_sync(c, cp.data(), c->cap, sizeof(double) * c->n_entries, cudaMemcpyDeviceToHost);
        memcpy_sync(c, cl.data(), c->col, sizeof(int32_t) * c->n_entries, cudaMemcpyDeviceToHost);
        // each n-link appears twice (both rows): count once via v > u
        std::vector<int64_t> sp((c->n_glob + kSell - 1) / kSell + 1);
        memcpy_sync(c, sp.data(), c->slice_ptr, sizeof(int64_t) * sp.size(), cudaMemcpyDeviceToHost);
        for (int64_t sl = 0; sl + 1 < (int64_t)sp.size(); sl++)
            for (int64_t e = sp[sl]; e < sp[sl + 1]; e++) {
                const int64_t u = sl * kSell + ((e - sp[sl]) % kSell);
                if (cl[e] > u) { cnt++; cmax = std::max(cmax, cp[e]); }
            }
        // Prop. 1 / A8 with the new terminals: every component keeps an anchor
        if (!c->comp_root.empty() && n > 0) {
            std::vector<uint8_t> anch(n, 0);
            for (int64_t u = 0; u < n; u++)
                if (cs[u] > 0.0 || ct[u] > 0.0) anch[c->comp_root[u]] = 1;
            for (int64_t u = 0; u < n; u++)
                if (!anch[c->comp_root[u]]) return fail(c, IRLS_ERR_SINGULAR, "terminal weights make L~ singular");
        }
        c->F = compute_F(cmax, cnt);
        CK(cudaMemcpyAsync(c->cs, cs, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(c->ct, ct, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
        if (c->lcs != c->cs && c->n_own > 0) {  // the strip's own copy
            CK(cudaMemcpyAsync(c->lcs, cs + c->lo, sizeof(double) * c->n_own, cudaMemcpyHostToDevice, c->stream));
            CK(cudaMemcpyAsync(c->lct, ct + c->lo, sizeof(double) * c->n_own, cudaMemcpyHostToDevice, c->stream));
        }
        CK(cudaStreamSynchronize(c->stream));
    }
    c->sweep_valid = false;
    return IRLS_OK;
}

// ---------------------------------------------------------------------------
// stats / kernel timing / destroy
// ---------------------------------------------------------------------------
extern "C" irls_status irls_get_stats(irls_ctx *c, irls_stats *o)
{
    if (!c || !o) return IRLS_ERR_INVALID_ARGUMENT;
    o->launches = c->launches;
    o->cg_iters = c->last_cg_iters;
    o->n_nonterminal = c->n_glob;
    o->n_links = c->n_links;
    o->n_local = c->n_own;
    o->sweep_sorted = c->sweep_sorted;
    return IRLS_OK;
}

extern "C" irls_status irls_time_kernel(irls_ctx *c, int32_t which, int32_t reps, float *mean_ms)
{
    GUARD(c);
    if (!mean_ms || reps < 1 || which < 0 || which > 4) return IRLS_ERR_INVALID_ARGUMENT;
    if (which == 4 && !c->cgcg) return fail(c, IRLS_ERR_INVALID_ARGUMENT, "CG-CG kernel timing needs cg_variant 1");
    if (c->state == 0) return fail(c, IRLS_ERR_STATE, "time_kernel needs a solved state");
    cudaStream_t st = c->stream;
    if (which == 3) {  // the z halo (NCCL), collective
        if (!c->multi || c->vg) return fail(c, IRLS_ERR_INVALID_ARGUMENT, "halo timing needs an NCCL context");
        Ranks R{c};
        irls_status s = coll_halo(R, true, st);  // warm-up
        if (s) return s;
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0, st));
        for (int i = 0; i < reps && !s; i++) s = coll_halo(R, true, st);
        CK(cudaEventRecord(e1, st));
        CK(cudaEventSynchronize(e1));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        *mean_ms = ms / reps;
        return s;
    }
    const int64_t npad = (int64_t)c->nchunks * kChunk;
    // snapshot everything the kernels write
    std::vector<double *> arrs = {c->x, c->q, c->r, c->z, c->p0, c->p1, c->D, c->Dinv};
    if (c->cgcg)
        for (double *a : {c->cg_r2, c->cg_w[0], c->cg_w[1], c->cg_s[0], c->cg_s[1]}) arrs.push_back(a);
    std::vector<double *> save;
    for (double *a : arrs) {
        double *b = nullptr;
        if (cudaMalloc(&b, sizeof(double) * npad) != cudaSuccess) {
            for (double *s2 : save) cudaFree(s2);
            return fail(c, IRLS_ERR_OOM, "time_kernel snapshot");
        }
        cudaMemcpyAsync(b, a, sizeof(double) * npad, cudaMemcpyDeviceToDevice, st);
        save.push_back(b);
    }
    double *gsave = nullptr;
    const int64_t gbytes = c->kind == 0 ? 3 * npad : c->ln_entries;
    CK(cudaMalloc(&gsave, sizeof(double) * std::max<int64_t>(gbytes, 1)));
    if (c->kind == 0) {
        cudaMemcpyAsync(gsave, c->gx, sizeof(double) * npad, cudaMemcpyDeviceToDevice, st);
        cudaMemcpyAsync(gsave + npad, c->gy, sizeof(double) * npad, cudaMemcpyDeviceToDevice, st);
        cudaMemcpyAsync(gsave + 2 * npad, c->gz, sizeof(double) * npad, cudaMemcpyDeviceToDevice, st);
    } else {
        cudaMemcpyAsync(gsave, c->lg, sizeof(double) * c->ln_entries, cudaMemcpyDeviceToDevice, st);
    }
    DevCtrl hc;
    CK(cudaMemcpyAsync(&hc, c->ctrl, sizeof(hc), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    DevCtrl tc = hc;
    tc.k = 1;  // a steady-state iteration (p-update and lazy x update active)
    if (!(tc.alpha == tc.alpha) || tc.alpha == 0.0) tc.alpha = 0.5;
    if (!(tc.beta == tc.beta)) tc.beta = 0.5;
    tc.done = 0;
    tc.frozen = 0;  // time the real kernels even after a fixed-point exit
    CK(cudaMemcpyAsync(c->ctrl, &tc, sizeof(tc), cudaMemcpyHostToDevice, st));
    CondArgs cd;
    memset(&cd, 0, sizeof(cd));
    const VecArgs v = vec_args(c);
    const RedArgs ra = red_args(c);
    const int mode = c->opt.warm_start ? ASM_REWEIGHT_WARM : ASM_REWEIGHT_COLD;
    auto launch = [&]() {
        if (which == 0) {
            if (c->kind == 0) launch_stencil_pspmv(stencil_args(c, false), v, ra, cd, st);
            else launch_sell_pspmv(sell_args(c), v, ra, cd, st);
        } else if (which == 1) {
            launch_axpy_jacobi(v, ra, cd, st);
        } else if (which == 4) {
            if (c->kind == 0) launch_stencil_cgcg(stencil_args(c, false), v, cg_args(c), ra, cd, st);
            else launch_sell_cgcg(sell_args(c), v, cg_args(c), ra, cd, st);
        } else {
            if (c->kind == 0) launch_stencil_assemble(stencil_args(c, false), v, ra, cd, mode, c->opt.eps, st);
            else launch_sell_assemble(sell_args(c), v, ra, cd, mode, c->opt.eps, st);
        }
    };
    launch();  // warm-up
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, st));
    for (int i = 0; i < reps; i++) launch();
    CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *mean_ms = ms / reps;
    // restore
    for (size_t i = 0; i < save.size(); i++)
        cudaMemcpyAsync(arrs[i], save[i], sizeof(double) * npad, cudaMemcpyDeviceToDevice, st);
    if (c->kind == 0) {
        cudaMemcpyAsync(c->gx, gsave, sizeof(double) * npad, cudaMemcpyDeviceToDevice, st);
        cudaMemcpyAsync(c->gy, gsave + npad, sizeof(double) * npad, cudaMemcpyDeviceToDevice, st);
        cudaMemcpyAsync(c->gz, gsave + 2 * npad, sizeof(double) * npad, cudaMemcpyDeviceToDevice, st);
    } else {
        cudaMemcpyAsync(c->lg, gsave, sizeof(double) * c->ln_entries, cudaMemcpyDeviceToDevice, st);
    }
    cudaMemcpyAsync(c->ctrl, &hc, sizeof(hc), cudaMemcpyHostToDevice, st);
    CK(cudaStreamSynchronize(st));
    for (double *s2 : save) cudaFree(s2);
    cudaFree(gsave);
    return last_launch(c, "time_kernel");
}

extern "C" void irls_mincut_destroy(irls_ctx *c)
{
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    for (auto &g : c->gexec)
        if (g) cudaGraphExecDestroy(g);
    for (auto &g : c->gmulti)
        if (g) cudaGraphExecDestroy(g);
    for (void *p : std::vector<void *>(c->allocs)) dfree(c, p);
    if (c->stream) cudaStreamSynchronize(c->stream);
    for (void *p : c->ipc_open) cudaIpcCloseMemHandle(p);
    for (void *p : c->raw_allocs) cudaFree(p);
    pinned_flag_put(c->h_done);
    if (c->nccl) ncclCommDestroy(c->nccl);
    if (c->side_stream) cudaStreamDestroy(c->side_stream);
    if (c->side_stream2) cudaStreamDestroy(c->side_stream2);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

// ---------------------------------------------------------------------------
// Virtual groups: every rank of the z-slab path in one process on one device.
// ---------------------------------------------------------------------------
extern "C" void irls_vgroup_destroy(irls_vgroup *g)
{
    if (!g) return;
    for (irls_ctx *c : g->ranks) irls_mincut_destroy(c);
    if (g->src_slots) cudaFree(g->src_slots);
    if (g->src_ctrl) cudaFree(g->src_ctrl);
    if (g->stream) cudaStreamDestroy(g->stream);
    delete g;
}

// W contexts of one graph on one device and one stream (every rank's strip
// or slab), plus the device arrays the virtual collectives read.
template <class MakeRank>
static irls_status vgroup_create(irls_vgroup **out, int32_t world, int32_t device, MakeRank make)
{
    if (!out || world < 1 || 8 % world != 0) return IRLS_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    if (cudaSetDevice(device) != cudaSuccess) return IRLS_ERR_CUDA;
    irls_vgroup *g = new irls_vgroup();
    if (cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete g;
        return IRLS_ERR_CUDA;
    }
    for (int r = 0; r < world; r++) {
        irls_comm_desc comm;
        comm.world_size = world;
        comm.rank = r;
        comm.device = device;
        comm.nccl_unique_id = nullptr;
        comm.cuda_stream = g->stream;
        comm.device_alloc = nullptr;
        comm.device_free = nullptr;
        comm.alloc_user = nullptr;
        irls_ctx *c = nullptr;
        irls_status s = make(&c, &comm, g);
        if (s) {
            irls_vgroup_destroy(g);
            return s;
        }
        g->ranks.push_back(c);
    }
    std::vector<double *> src(world);
    std::vector<DevCtrl *> ctl(world);
    for (int r = 0; r < world; r++) {
        src[r] = g->ranks[r]->slots_local;
        ctl[r] = g->ranks[r]->ctrl;
    }
    if (cudaMalloc(&g->src_slots, sizeof(double *) * world) != cudaSuccess ||
        cudaMemcpy(g->src_slots, src.data(), sizeof(double *) * world, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMalloc(&g->src_ctrl, sizeof(DevCtrl *) * world) != cudaSuccess ||
        cudaMemcpy(g->src_ctrl, ctl.data(), sizeof(DevCtrl *) * world, cudaMemcpyHostToDevice) != cudaSuccess) {
        irls_vgroup_destroy(g);
        return IRLS_ERR_CUDA;
    }
    if (g->ranks[0]->p2p) {  // peer memory = the other ranks' buffers on this device
        std::vector<double *> bufs(world);
        for (int r = 0; r < world; r++) bufs[r] = g->ranks[r]->p2p_buf;
        for (int r = 0; r < world; r++) {
            irls_ctx *c = g->ranks[r];
            irls_status s = p2p_set_peers(c, bufs);
            if (s) {
                irls_vgroup_destroy(g);
                return s;
            }
            if (c->kind == 0 && c->hplan.peer_lo >= 0) {
                irls_ctx *o = g->ranks[c->hplan.peer_lo];
                c->zpeer_lo = o->z + o->hplan.recv_hi;
            }
            if (c->kind == 0 && c->hplan.peer_hi >= 0) {
                irls_ctx *o = g->ranks[c->hplan.peer_hi];
                c->zpeer_hi = o->z + o->hplan.recv_lo;
            }
            if (c->kind == 1) {  // CSR strips: every rank's z and ghost-block layout
                std::vector<double *> zp(world);
                std::vector<int64_t> npad(world);
                std::vector<std::vector<int64_t>> roff(world);
                for (int q = 0; q < world; q++) {
                    zp[q] = g->ranks[q]->z;
                    npad[q] = g->ranks[q]->npad_own;
                    roff[q] = g->ranks[q]->recv_off;
                }
                s = p2p_set_halo(c, zp, npad, roff);
                if (s) {
                    irls_vgroup_destroy(g);
                    return s;
                }
            }
            for (int b = 0; b < 2 && c->cgcg && c->kind == 0; b++) {
                if (c->hplan.peer_lo >= 0) {
                    irls_ctx *o = g->ranks[c->hplan.peer_lo];
                    c->wpeer_lo[b] = o->cg_w[b] + o->hplan.recv_hi;
                }
                if (c->hplan.peer_hi >= 0) {
                    irls_ctx *o = g->ranks[c->hplan.peer_hi];
                    c->wpeer_hi[b] = o->cg_w[b] + o->hplan.recv_lo;
                }
            }
        }
    }
    *out = g;
    return IRLS_OK;
}

extern "C" irls_status irls_vgroup_create_stencil(irls_vgroup **out, int32_t world, int32_t device, int32_t nx,
                                                  int32_t ny, int32_t nz, const double *cx, const double *cy,
                                                  const double *cz, const double *cs, const double *ct,
                                                  const irls_options *opt)
{
    return vgroup_create(out, world, device, [&](irls_ctx **c, const irls_comm_desc *comm, irls_vgroup *g) {
        return create_stencil_impl(c, comm, nx, ny, nz, cx, cy, cz, cs, ct, opt, g);
    });
}

extern "C" const char *irls_vgroup_last_error(const irls_vgroup *g)
{
    if (!g || g->ranks.empty()) return "null group";
    for (const irls_ctx *c : g->ranks)
        if (!c->err.empty()) return c->err.c_str();
    return "";
}

extern "C" irls_status irls_vgroup_create_csr(irls_vgroup **out, int32_t world, int32_t device, int64_t n,
                                              const int64_t *row_ptr, const int32_t *col, const double *w, int64_t s,
                                              int64_t t, const irls_options *opt)
{
    return vgroup_create(out, world, device, [&](irls_ctx **c, const irls_comm_desc *comm, irls_vgroup *g) {
        return create_csr_impl(c, comm, n, row_ptr, col, w, s, t, opt, g);
    });
}

extern "C" irls_status irls_vgroup_solve(irls_vgroup *g, int32_t mode, irls_step_report *per_step, int64_t *total)
{
    if (!g) return IRLS_ERR_INVALID_ARGUMENT;
    irls_ctx *c = g->ranks[0];
    GUARD(c);
    if (mode != IRLS_FROM_SCRATCH && mode != IRLS_CONTINUE) return IRLS_ERR_INVALID_ARGUMENT;
    if (mode == IRLS_CONTINUE && c->state == 0) return fail(c, IRLS_ERR_STATE, "IRLS_CONTINUE without potentials");
    const int step_mode = c->opt.warm_start ? ASM_REWEIGHT_WARM : ASM_REWEIGHT_COLD;
    Ranks &R = g->ranks;
    if (mode == IRLS_FROM_SCRATCH) return run_solves(R, ASM_INIT, step_mode, c->opt.T + 1, per_step, total);
    if (c->opt.T == 0) { if (total) *total = 0; return IRLS_OK; }
    return run_solves(R, step_mode, step_mode, c->opt.T, per_step, total);
}

extern "C" irls_status irls_vgroup_sweep_cut(irls_vgroup *g, uint8_t *side, int32_t *order, int64_t *k,
                                             double *cut_value)
{
    if (!g) return IRLS_ERR_INVALID_ARGUMENT;
    irls_ctx *c = g->ranks[0];
    GUARD(c);
    if (c->state == 0) return fail(c, IRLS_ERR_STATE, "sweep before solve");
    double *full = nullptr;
    irls_status s = vgather_x(g, &full);
    if (s) return s;
    return sweep_rank0(c, full, side, order, k, cut_value);
}

extern "C" irls_status irls_vgroup_get_potentials(irls_vgroup *g, double *x)
{
    if (!g || !x) return IRLS_ERR_INVALID_ARGUMENT;
    irls_ctx *c = g->ranks[0];
    GUARD(c);
    if (c->state == 0) return fail(c, IRLS_ERR_STATE, "no potentials yet");
    double *full = nullptr;
    irls_status s = vgather_x(g, &full);
    if (s) return s;
    CK(cudaMemcpyAsync(x, full, sizeof(double) * c->n_glob, cudaMemcpyDeviceToHost, g->stream));
    CK(cudaStreamSynchronize(g->stream));
    return IRLS_OK;
}

extern "C" irls_status irls_vgroup_set_terminal_weights(irls_vgroup *g, const double *cs, const double *ct)
{
    if (!g) return IRLS_ERR_INVALID_ARGUMENT;
    for (irls_ctx *c : g->ranks) {
        irls_status s = irls_set_terminal_weights(c, cs, ct);
        if (s) return s;
    }
    return IRLS_OK;
}

