// api.cu — the C ABI (include/irls_mincut.h): validation, device memory,
// the per-solve CUDA graph with a device-side WHILE loop, the host-loop and
// multi-GPU paths, and the sweep orchestration.
#include <math.h>
#include <atomic>
#include <memory>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <string.h>

#include <algorithm>
#include <queue>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "ctx.h"

using namespace irls;

// NVTX ranges around every entry point and phase (header-only NVTX 3: a
// profiler that injects itself sees them; otherwise they cost a branch).
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

// ---------------------------------------------------------------------------
// error plumbing
// ---------------------------------------------------------------------------
static irls_status fail(irls_ctx *c, irls_status st, const std::string &msg)
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

#define CK(call)                                                                                      \
    do {                                                                                              \
        cudaError_t e__ = (call);                                                                     \
        if (e__ != cudaSuccess)                                                                       \
            return fail(c, e__ == cudaErrorMemoryAllocation ? IRLS_ERR_OOM : IRLS_ERR_CUDA,           \
                        std::string(#call) + ": " + cudaGetErrorString(e__));                         \
    } while (0)

#define NK(call)                                                                                      \
    do {                                                                                              \
        ncclResult_t r__ = (call);                                                                    \
        if (r__ != ncclSuccess) return fail(c, IRLS_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(r__)); \
    } while (0)

#define GUARD(c)                                                                  \
    do {                                                                          \
        if (!(c)) return IRLS_ERR_INVALID_ARGUMENT;                               \
        if ((c)->poisoned) return IRLS_ERR_STATE;                                 \
        if (cudaSetDevice((c)->device) != cudaSuccess) return IRLS_ERR_CUDA;      \
    } while (0)

// Blocking copy ordered on the context stream (its allocations are stream-ordered).
static cudaError_t memcpy_sync(irls_ctx *c, void *dst, const void *src, size_t n, cudaMemcpyKind k)
{
    cudaError_t e = cudaMemcpyAsync(dst, src, n, k, c->stream);
    if (e != cudaSuccess) return e;
    return cudaStreamSynchronize(c->stream);
}

static irls_status last_launch(irls_ctx *c, const char *what)
{
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(c, IRLS_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return IRLS_OK;
}

// Device memory comes from the device's stream-ordered pool with an unbounded
// release threshold: a create / destroy cycle maps HBM once and then reuses
// it (sizes here are GBs; cudaMalloc / cudaFree would remap every time).
static void setup_pool(int device)
{
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
}

template <class T>
static T *dalloc(irls_ctx *c, int64_t count)
{
    void *p = nullptr;
    const size_t bytes = ((size_t)std::max<int64_t>(count, 1) * sizeof(T) + 255) & ~(size_t)255;
    if (c->dev_alloc) {
        p = c->dev_alloc(bytes, (void *)c->stream, c->alloc_user);
        if (!p) return nullptr;
    } else if (cudaMallocAsync(&p, bytes, c->stream) != cudaSuccess) {
        return nullptr;
    }
    cudaMemsetAsync(p, 0, bytes, c->stream);
    c->allocs.push_back(p);
    return (T *)p;
}

// Release one of the context's arrays (stream-ordered for the pool).
static cudaError_t dfree(irls_ctx *c, void *p)
{
    c->allocs.erase(std::remove(c->allocs.begin(), c->allocs.end(), p), c->allocs.end());
    if (c->dev_free) {
        c->dev_free(p, (void *)c->stream, c->alloc_user);
        return cudaSuccess;
    }
    return cudaFreeAsync(p, c->stream);
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
    o->reserved = 0;
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

static int count_nonempty(int32_t K, int g0, int g1)
{
    int n = 0;
    for (int g = g0; g < g1; g++)
        if (group_lo(g + 1, K) > group_lo(g, K)) n++;
    return n;
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

static irls_status check_opts(const irls_options *o)
{
    if (!o) return IRLS_ERR_INVALID_ARGUMENT;
    if (!(o->eps > 0.0) || isinf(o->eps) || o->T < 0 || !(o->cg_rtol >= 0.0) || o->cg_max_iter < 0 ||
        (o->cg_norm != 0 && o->cg_norm != 1) || (o->loop_mode < 0 || o->loop_mode > 2) ||
        (o->fixed_point_exit != 0 && o->fixed_point_exit != 1))
        return IRLS_ERR_INVALID_ARGUMENT;
    return IRLS_OK;
}

static int32_t compute_F(double cmax, int64_t cnt)
{
    if (cmax == 0.0) return 0;
    int e;
    frexp(cmax, &e);
    int b = 0;
    while (b < 63 && (((int64_t)1) << b) <= cnt) b++;
    return 124 - e - b;
}

// ---------------------------------------------------------------------------
// argument blocks
// ---------------------------------------------------------------------------
static VecArgs vec_args(const irls_ctx *c)
{
    VecArgs v;
    v.n_own = c->n_own;
    v.chunk0 = c->chunk0;
    v.x = c->x;
    v.D = c->D;
    v.Dinv = c->Dinv;
    v.r = c->r;
    v.q = c->q;
    v.z = c->z;
    v.p0 = c->p0;
    v.p1 = c->p1;
    v.frozen = &c->ctrl->frozen;
    return v;
}

static StencilArgs stencil_args(const irls_ctx *c, bool full)
{
    StencilArgs s;
    s.nx = c->nx;
    s.ny = c->ny;
    s.nz = c->nz;
    s.P = c->P;
    s.lo = full ? 0 : c->lo;
    s.fd_nx = make_fastdiv((uint32_t)c->nx);
    s.fd_ny = make_fastdiv((uint32_t)c->ny);
    s.lo_ghost = full ? 0 : (c->lo_ghost ? 1 : 0);
    const int64_t off = full ? 0 : c->lo;  // capacity arrays are full-size on every rank
    s.cx = c->cx + off;
    s.cy = c->cy + off;
    s.cz = c->cz + off;
    s.cs = c->cs + off;
    s.ct = c->ct + off;
    s.gx = c->gx;
    s.gy = c->gy;
    s.gz = c->gz;
    return s;
}

// The solve's rows (local strip with ghost columns; the whole graph on one rank).
static SellArgs sell_args(const irls_ctx *c)
{
    SellArgs s;
    s.n = c->n_own;
    s.slice_ptr = c->lslice_ptr;
    s.col = c->lcol;
    s.c = c->lcap;
    s.g = c->lg;
    s.cs = c->lcs;
    s.ct = c->lct;
    s.wmax = c->lwmax;
    s.gbase = c->multi ? c->npad_own : INT64_MAX;
    s.glow = c->multi ? c->recv_off[c->rank] : 0;
    return s;
}

// The whole graph in reduced ids (rank 0's sweep, two-level rounding, lambda_2).
static SellArgs sell_args_full(const irls_ctx *c)
{
    SellArgs s;
    s.n = c->n_glob;
    s.slice_ptr = c->slice_ptr;
    s.col = c->col;
    s.c = c->cap;
    s.g = c->gsell;
    s.cs = c->cs;
    s.ct = c->ct;
    s.wmax = c->sell_wmax;
    s.gbase = INT64_MAX;
    s.glow = 0;
    return s;
}

static RedArgs red_args(const irls_ctx *c)
{
    RedArgs r;
    r.part = c->part;
    r.slots = c->slots_local;
    r.ctrl = c->ctrl;
    r.K = c->K;
    r.g0 = c->g0;
    r.g1 = c->g1;
    r.n_fin = c->n_fin;
    return r;
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
static irls_status vgather_x(irls_vgroup *g, double **full)
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
static irls_status gather_x(irls_ctx *c, double **full)
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
typedef std::vector<irls_ctx *> Ranks;

static irls_status coll_halo(Ranks &R, bool z_not_x, cudaStream_t st)
{
    irls_ctx *c = R[0];
    if (!c->multi) return IRLS_OK;
    if (!c->vg) return halo(c, z_not_x ? c->z : c->x, st);
    if (c->kind == 1) {  // pack on every rank, then the same copies NCCL would make
        for (irls_ctx *d : R) {
            const int64_t ns = d->send_off[d->world];
            if (ns > 0) launch_halo_pack(z_not_x ? d->z : d->x, d->send_idx, ns, d->sendbuf, st);
        }
        for (irls_ctx *d : R)
            for (int q = 0; q < d->world; q++) {
                const int64_t rc = d->recv_off[q + 1] - d->recv_off[q];
                if (rc == 0) continue;
                irls_ctx *o = R[q];
                CK(cudaMemcpyAsync((z_not_x ? d->z : d->x) + d->npad_own + d->recv_off[q], o->sendbuf + o->send_off[d->rank],
                                   sizeof(double) * rc, cudaMemcpyDeviceToDevice, st));
            }
        return IRLS_OK;
    }
    for (irls_ctx *d : R) {
        const irls_halo &h = d->hplan;
        double *arr = z_not_x ? d->z : d->x;
        const size_t bytes = sizeof(double) * (size_t)h.count;
        if (h.peer_lo >= 0) {
            irls_ctx *o = R[h.peer_lo];
            CK(cudaMemcpyAsync(arr + h.recv_lo, (z_not_x ? o->z : o->x) + o->hplan.send_hi, bytes,
                               cudaMemcpyDeviceToDevice, st));
        }
        if (h.peer_hi >= 0) {
            irls_ctx *o = R[h.peer_hi];
            CK(cudaMemcpyAsync(arr + h.recv_hi, (z_not_x ? o->z : o->x) + o->hplan.send_lo, bytes,
                               cudaMemcpyDeviceToDevice, st));
        }
    }
    return IRLS_OK;
}

static irls_status coll_allreduce(Ranks &R, int nq, cudaStream_t st)
{
    irls_ctx *c = R[0];
    if (!c->multi) return IRLS_OK;
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
static irls_status enq_assemble(Ranks &R, int mode, const CondArgs &cd, cudaStream_t st)
{
    irls_status s;
    if (mode != ASM_INIT && mode != ASM_LAMBDA2 && (s = coll_halo(R, false, st))) return s;
    for (irls_ctx *c : R) {
        const VecArgs v = vec_args(c);
        const RedArgs ra = red_args(c);
        if (c->kind == 0)
            c->launches += launch_stencil_assemble_ex(stencil_args(c, false), v, ra, cd, mode, c->opt.eps, c->gs_diag,
                                                      c->gt_diag, st);
        else
            c->launches += launch_sell_assemble_ex(sell_args(c), v, ra, cd, mode, c->opt.eps, c->gs_diag, c->gt_diag, st);
    }
    if (R[0]->multi) {
        if ((s = coll_allreduce(R, 5, st))) return s;
        for (irls_ctx *c : R) {
            launch_finalize(PH_START, c->ctrl, c->slots_glob, cd, st);
            c->launches++;
        }
        if ((s = coll_halo(R, true, st))) return s;
    }
    return last_launch(R[0], "assemble");
}

static irls_status enq_body(Ranks &R, const CondArgs &cd, cudaStream_t st)
{
    irls_status s;
    for (irls_ctx *c : R) {
        const VecArgs v = vec_args(c);
        const RedArgs ra = red_args(c);
        if (c->kind == 0) launch_stencil_pspmv(stencil_args(c, false), v, ra, cd, st);
        else launch_sell_pspmv(sell_args(c), v, ra, cd, st);
        c->launches++;
        if (c->multi && c->kind == 0) {
            launch_ghost_pupdate(v, c->lo_ghost, c->hi_ghost, c->P, c->ctrl, st);
            c->launches++;
        } else if (c->multi && c->n_ghost > 0) {
            launch_ghost_range_pupdate(v, c->npad_own, c->n_ghost, c->ctrl, st);
            c->launches++;
        }
    }
    if (R[0]->multi) {
        if ((s = coll_allreduce(R, 1, st))) return s;
        for (irls_ctx *c : R) {
            launch_finalize(PH_PQ, c->ctrl, c->slots_glob, cd, st);
            c->launches++;
        }
    }
    for (irls_ctx *c : R) {
        launch_axpy_jacobi(vec_args(c), red_args(c), cd, st);
        c->launches++;
    }
    if (R[0]->multi) {
        if ((s = coll_allreduce(R, 3, st))) return s;
        for (irls_ctx *c : R) {
            launch_finalize(PH_RZ, c->ctrl, c->slots_glob, cd, st);
            c->launches++;
        }
        if ((s = coll_halo(R, true, st))) return s;
    }
    return last_launch(R[0], "cg body");
}

static void enq_finish(Ranks &R, cudaStream_t st)
{
    for (irls_ctx *c : R) {
        launch_finish(vec_args(c), c->ctrl, st);
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
            const RedArgs ra = red_args(c);
            if (c->kind == 0)
                launch_stencil_diag_ex(stencil_args(c, false), v, ra, c->opt.eps, c->opt.cg_norm, c->gs_diag,
                                       c->gt_diag, st);
            else
                launch_sell_diag_ex(sell_args(c), v, ra, c->opt.eps, c->opt.cg_norm, c->gs_diag, c->gt_diag, st);
        }
        if (R[0]->multi && (s = coll_allreduce(R, 4, st))) return s;
        if ((s = coll_minmax(R, st))) return s;
        for (irls_ctx *c : R) {
            launch_diag_finalize(c->ctrl, c->slots_glob, c->reports, c->opt.cg_norm, st);
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
static bool small_path(const irls_ctx *c) { return !c->multi && c->n_own > 0 && c->n_own <= kChunk; }

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
    c->gl_body = c->launches - pre;
    c->launches = pre;
    cudaGraph_t bodyg;
    CK(cudaStreamEndCapture(c->side_stream, &bodyg));
    return s;
}

static irls_status build_graph(irls_ctx *c, int mode)
{
    cudaStream_t st = c->stream;
    Ranks R{c};
    const bool gated = c->opt.fixed_point_exit && mode == ASM_REWEIGHT_WARM;
    const int64_t lsave = c->launches;
    c->launches = 0;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    irls_status s = IRLS_OK;
    if (!gated) {
        s = capture_solve_body(c, R, mode, st);
        if (!s) s = enq_tail(R, mode, st);
    } else {
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
        if (e != cudaSuccess) {
            s = fail(c, IRLS_ERR_CUDA, std::string("gated graph: ") + cudaGetErrorString(e));
        } else {
            s = capture_solve_body(c, R, mode, c->side_stream2);
            if (!s) enq_finish(R, c->side_stream2);
            cudaGraph_t ifg;
            e = cudaStreamEndCapture(c->side_stream2, &ifg);
            if (!s && e != cudaSuccess) s = fail(c, IRLS_ERR_CUDA, std::string("gated graph: ") + cudaGetErrorString(e));
            if (!s) s = enq_tail(R, mode, st, false);
        }
    }
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
        if (!s && e != cudaSuccess) s = fail(c, IRLS_ERR_CUDA, std::string("multi-step graph: ") + cudaGetErrorString(e));
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
    if (!c->multi) return c->opt.loop_mode == IRLS_LOOP_GRAPH || c->opt.loop_mode == IRLS_LOOP_GRAPH_NCCL;
    return c->opt.loop_mode == IRLS_LOOP_GRAPH_NCCL;
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

static void copy_report(const DevReport &d, irls_step_report *o, float ms)
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
    o->reserved2 = 0.f;
}

// Run `count` solves (first one with mode0, the rest with mode_rest); fill
// reports from rank 0 and check that every driven rank reports the same.
static irls_status run_solves(Ranks &R, int mode0, int mode_rest, int count, irls_step_report *reps, int64_t *total)
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
            float ms = 0.f;
            if (multi_graph) {
                const unsigned long long prev = i == 0 ? t0 : h[i - 1].t_end;
                ms = h[i].t_end > prev ? (float)((double)(h[i].t_end - prev) * 1e-6) : 0.f;
            } else {
                cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
            }
            tot += h[i].cg_iters;
            if (reps) copy_report(h[i], reps + i, ms);
            if (h[i].status != 0 && !s) s = fail(c, (irls_status)h[i].status, "CG breakdown (p'Ap <= 0 or non-finite scalar)");
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
// create
// ---------------------------------------------------------------------------
static irls_status common_setup(irls_ctx *c, const irls_comm_desc *comm, const irls_options *opt)
{
    c->opt = *opt;
    c->world = comm ? comm->world_size : 1;
    c->rank = comm ? comm->rank : 0;
    c->device = comm ? comm->device : 0;
    if (comm && (!comm->device_alloc) != (!comm->device_free)) return IRLS_ERR_INVALID_ARGUMENT;
    c->dev_alloc = comm ? comm->device_alloc : nullptr;
    c->dev_free = comm ? comm->device_free : nullptr;
    c->alloc_user = comm ? comm->alloc_user : nullptr;
    if (c->world < 1 || c->rank < 0 || c->rank >= c->world) return IRLS_ERR_INVALID_ARGUMENT;
    if (c->world > 1 && ((!comm->nccl_unique_id && !c->vg) || 8 % c->world != 0)) return IRLS_ERR_INVALID_ARGUMENT;
    // world 1 with an NCCL id: the multi-rank code path over a 1-rank
    // communicator (host loop, slot allreduce, finalize kernels, broadcasts)
    c->multi = c->world > 1 || c->vg != nullptr || (comm && comm->nccl_unique_id != nullptr);
    CK(cudaSetDevice(c->device));
    if (comm && comm->cuda_stream) {
        c->stream = (cudaStream_t)comm->cuda_stream;
    } else {
        CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
    }
    CK(cudaStreamCreateWithFlags(&c->side_stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->side_stream2, cudaStreamNonBlocking));
    CK(cudaMallocHost(&c->h_done, sizeof(int)));
    setup_pool(c->device);
    small_cg_prepare();
    return IRLS_OK;
}

static irls_status alloc_solver(irls_ctx *c, int64_t ghost)
{
    const int64_t npad = (int64_t)c->nchunks * kChunk;
    const int64_t gpad = (ghost + 1) & ~(int64_t)1;  // keep the owned start 16-byte aligned
    auto ghosted = [&](double *&ptr) -> bool {
        double *b = dalloc<double>(c, npad + 2 * gpad);
        if (!b) return false;
        ptr = b + gpad;
        return true;
    };
    if (!ghosted(c->x) || !ghosted(c->z) || !ghosted(c->p0) || !ghosted(c->p1)) return IRLS_ERR_OOM;
    c->D = dalloc<double>(c, npad);
    c->Dinv = dalloc<double>(c, npad);
    c->r = dalloc<double>(c, npad);
    c->q = dalloc<double>(c, npad);
    c->ctrl = dalloc<DevCtrl>(c, 1);
    c->part = dalloc<double>(c, (int64_t)kMaxQ * std::max<int32_t>(c->K, 1));
    c->slots_local = dalloc<double>(c, kMaxQ * kGroups);
    c->slots_glob = c->multi ? dalloc<double>(c, kMaxQ * kGroups) : c->slots_local;
    c->max_reports = std::max(c->opt.T + 1, 1);
    c->reports = dalloc<DevReport>(c, c->max_reports);
    if (!c->D || !c->Dinv || !c->r || !c->q || !c->ctrl || !c->part || !c->slots_local || !c->slots_glob || !c->reports)
        return IRLS_ERR_OOM;
    if (c->opt.record_trace) {
        c->gs_diag = dalloc<double>(c, npad);
        c->gt_diag = dalloc<double>(c, npad);
        if (!c->gs_diag || !c->gt_diag) return IRLS_ERR_OOM;
    }
    DevCtrl h;
    memset(&h, 0, sizeof(h));
    h.rtol = c->opt.cg_rtol;
    h.max_iter = c->opt.cg_max_iter;
    h.norm = c->opt.cg_norm;
    h.done = 1;
    CK(memcpy_sync(c, c->ctrl, &h, sizeof(h), cudaMemcpyHostToDevice));
    return IRLS_OK;
}

static irls_status init_nccl(irls_ctx *c, const irls_comm_desc *comm)
{
    if (!c->multi || c->vg) return IRLS_OK;
    ncclUniqueId id;
    memcpy(&id, comm->nccl_unique_id, sizeof(id));
    NK(ncclCommInitRank(&c->nccl, c->world, id, c->rank));
    return IRLS_OK;
}

// Host BFS for Prop. 1 / A8 on a grid (used only when some n-link is zero).
static bool grid_nonsingular(int32_t nx, int32_t ny, int32_t nz, const double *cx, const double *cy, const double *cz,
                             const double *cs, const double *ct)
{
    const int64_t N = (int64_t)nx * ny * nz, P = (int64_t)nx * ny;
    std::vector<uint8_t> seen(N, 0);
    std::vector<int64_t> q;
    q.reserve(1024);
    for (int64_t r0 = 0; r0 < N; r0++) {
        if (seen[r0]) continue;
        bool anchored = false;
        q.clear();
        q.push_back(r0);
        seen[r0] = 1;
        for (size_t h = 0; h < q.size(); h++) {
            const int64_t u = q[h];
            if (cs[u] > 0.0 || ct[u] > 0.0) anchored = true;
            const int64_t x = u % nx, y = (u / nx) % ny, z = u / P;
            const int64_t nb[6] = {z > 0 && cz[u - P] > 0 ? u - P : -1, y > 0 && cy[u - nx] > 0 ? u - nx : -1,
                                   x > 0 && cx[u - 1] > 0 ? u - 1 : -1, x < nx - 1 && cx[u] > 0 ? u + 1 : -1,
                                   y < ny - 1 && cy[u] > 0 ? u + nx : -1, z < nz - 1 && cz[u] > 0 ? u + P : -1};
            for (int k = 0; k < 6; k++)
                if (nb[k] >= 0 && !seen[nb[k]]) { seen[nb[k]] = 1; q.push_back(nb[k]); }
        }
        if (!anchored) return false;
    }
    return true;
}

static irls_status create_stencil_impl(irls_ctx **out, const irls_comm_desc *comm, int32_t nx, int32_t ny, int32_t nz,
                                       const double *cx, const double *cy, const double *cz, const double *cs,
                                       const double *ct, const irls_options *opt, irls_vgroup *vg);

extern "C" irls_status irls_mincut_create_stencil(irls_ctx **out, const irls_comm_desc *comm, int32_t nx, int32_t ny,
                                                  int32_t nz, const double *cx, const double *cy, const double *cz,
                                                  const double *cs, const double *ct, const irls_options *opt)
{
    return create_stencil_impl(out, comm, nx, ny, nz, cx, cy, cz, cs, ct, opt, nullptr);
}

static irls_status create_stencil_impl(irls_ctx **out, const irls_comm_desc *comm, int32_t nx, int32_t ny, int32_t nz,
                                       const double *cx, const double *cy, const double *cz, const double *cs,
                                       const double *ct, const irls_options *opt, irls_vgroup *vg)
{
    NvtxRange nvtx_("irls_mincut_create_stencil");
    if (!out) return IRLS_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    if (check_opts(opt) || nx < 1 || ny < 1 || nz < 1 || !cx || !cy || !cz || !cs || !ct)
        return IRLS_ERR_INVALID_ARGUMENT;
    const int64_t N = (int64_t)nx * ny * nz;
    if (N >= ((int64_t)1 << 31) - 2 * ((int64_t)nx * ny) - kChunk) return IRLS_ERR_INVALID_ARGUMENT;
    irls_ctx *c = new irls_ctx();
    c->vg = vg;
    irls_status s = common_setup(c, comm, opt);
    if (!s) {
        c->kind = 0;
        c->nx = nx; c->ny = ny; c->nz = nz;
        c->P = (int64_t)nx * ny;
        c->n_glob = N;
        c->n_total = N + 2;
        c->s_id = N;
        c->t_id = N + 1;
        c->K = (int32_t)((N + kChunk - 1) / kChunk);
        int32_t g0, g1, z0, z1;
        s = irls_plan_stencil(nx, ny, nz, c->world, c->rank, &z0, &z1, &g0, &g1);
        if (!s) {
            c->g0 = g0; c->g1 = g1; c->z0 = z0; c->z1 = z1;
            c->lo = (int64_t)z0 * c->P;
            c->n_own = std::min<int64_t>((int64_t)z1 * c->P, N) - c->lo;
            c->chunk0 = (int32_t)(c->lo / kChunk);
            c->nchunks = (int32_t)((c->n_own + kChunk - 1) / kChunk);
            c->n_fin = count_nonempty(c->K, g0, g1);
            c->lo_ghost = c->world > 1 && c->rank > 0;
            c->hi_ghost = c->world > 1 && c->rank < c->world - 1;
            c->rank_lo.assign(c->world + 1, N);
            for (int r = 0; r < c->world; r++) {
                int32_t a0, a1;
                irls_plan_stencil(nx, ny, nz, c->world, r, &a0, &a1, nullptr, nullptr);
                c->rank_lo[r] = std::min<int64_t>((int64_t)a0 * c->P, N);
            }
            if (c->multi) s = irls_halo_plan(nx, ny, nz, c->world, c->rank, &c->hplan);
        }
        if (!s) {
            s = alloc_solver(c, c->world > 1 ? c->P : 0);
        }
        if (!s) {
            // static capacities: full arrays on every rank (rank 0 sweeps the whole graph)
            c->cx = dalloc<double>(c, N); c->cy = dalloc<double>(c, N); c->cz = dalloc<double>(c, N);
            c->cs = dalloc<double>(c, N); c->ct = dalloc<double>(c, N);
            c->gx = dalloc<double>(c, (int64_t)c->nchunks * kChunk);
            c->gy = dalloc<double>(c, (int64_t)c->nchunks * kChunk);
            const int64_t gp = c->lo_ghost ? ((c->P + 1) & ~(int64_t)1) : 0;
            double *gzb = dalloc<double>(c, (int64_t)c->nchunks * kChunk + gp);
            if (!c->cx || !c->cy || !c->cz || !c->cs || !c->ct || !c->gx || !c->gy || !gzb) s = IRLS_ERR_OOM;
            else c->gz = gzb + gp;
        }
        if (!s) {
            const size_t b = sizeof(double) * N;
            cudaMemcpyAsync(c->cx, cx, b, cudaMemcpyHostToDevice, c->stream);
            cudaMemcpyAsync(c->cy, cy, b, cudaMemcpyHostToDevice, c->stream);
            cudaMemcpyAsync(c->cz, cz, b, cudaMemcpyHostToDevice, c->stream);
            cudaMemcpyAsync(c->cs, cs, b, cudaMemcpyHostToDevice, c->stream);
            cudaMemcpyAsync(c->ct, ct, b, cudaMemcpyHostToDevice, c->stream);
            unsigned long long vo[6];
            if (validate_stencil(nx, ny, nz, c->cx, c->cy, c->cz, c->cs, c->ct, vo, c->stream))
                s = fail(c, IRLS_ERR_CUDA, "validate_stencil");
            else if (vo[0]) s = IRLS_ERR_BAD_CAPACITY;
            else {
                bool ok = vo[1] == 0 ? (vo[2] > 0) : grid_nonsingular(nx, ny, nz, cx, cy, cz, cs, ct);
                if (!ok) s = IRLS_ERR_SINGULAR;
                double cmax;
                memcpy(&cmax, &vo[4], sizeof(double));
                c->F = compute_F(cmax, (int64_t)vo[3]);
                c->n_links = (int64_t)vo[5];  // |E~| with c > 0
            }
        }
        if (!s) s = init_nccl(c, comm);
    }
    if (s) {
        irls_mincut_destroy(c);
        return s;
    }
    *out = c;
    return IRLS_OK;
}

// Uninitialised host array (filled in parallel; avoids serial zeroing).
template <class T>
struct HostBuf {
    std::unique_ptr<T[]> p;
    explicit HostBuf(int64_t n) : p(new T[(size_t)std::max<int64_t>(n, 1)]) {}
    T &operator[](int64_t i) { return p[i]; }
    const T &operator[](int64_t i) const { return p[i]; }
    T *data() { return p.get(); }
    const T *data() const { return p.get(); }
};

// Host thread pool for create-time preparation (row blocks).
static int host_threads(int64_t n)
{
    if (n < 200000) return 1;
    const unsigned hc = std::thread::hardware_concurrency();
    return (int)std::min<unsigned>(std::max(1u, hc), 32u);
}

template <class F>
static void parallel_for(int64_t n, F f)
{
    const int nt = host_threads(n);
    if (nt == 1) {
        f(0, (int64_t)0, n);
        return;
    }
    std::vector<std::thread> th;
    for (int i = 0; i < nt; i++)
        th.emplace_back([&, i]() { f(i, n * i / nt, n * (i + 1) / nt); });
    for (auto &t : th) t.join();
}

struct Ent {
    int32_t col;
    int64_t pos;
    double w;
};

static irls_status create_csr_impl(irls_ctx **out, const irls_comm_desc *comm, int64_t n, const int64_t *row_ptr,
                                   const int32_t *col, const double *w, int64_t s_, int64_t t_, const irls_options *opt,
                                   irls_vgroup *vg);

extern "C" irls_status irls_mincut_create_csr(irls_ctx **out, const irls_comm_desc *comm, int64_t n,
                                              const int64_t *row_ptr, const int32_t *col, const double *w, int64_t s_,
                                              int64_t t_, const irls_options *opt)
{
    return create_csr_impl(out, comm, n, row_ptr, col, w, s_, t_, opt, nullptr);
}

// Id-strip plan of a CSR graph with nr non-terminals over `world` ranks:
// rank r owns C3 groups [8r/W, 8(r+1)/W), i.e. reduced ids [lo, hi) on chunk
// boundaries; every rank needs at least one chunk.
static bool csr_strips(int64_t nr, int world, std::vector<int64_t> &lo)
{
    const int32_t K = (int32_t)((nr + kChunk - 1) / kChunk);
    lo.assign(world + 1, nr);
    for (int r = 0; r < world; r++) {
        const int64_t c0 = group_lo(kGroups * r / world, K), c1 = group_lo(kGroups * (r + 1) / world, K);
        if (world > 1 && c1 <= c0) return false;
        lo[r] = std::min<int64_t>(c0 * kChunk, nr);
    }
    return true;
}

extern "C" irls_status irls_plan_csr(int64_t nr, int32_t world, int32_t rank, int64_t *lo, int64_t *hi, int32_t *g0,
                                     int32_t *g1)
{
    if (nr < 0 || world < 1 || 8 % world != 0 || rank < 0 || rank >= world) return IRLS_ERR_INVALID_ARGUMENT;
    std::vector<int64_t> v;
    if (!csr_strips(nr, world, v)) return IRLS_ERR_INVALID_ARGUMENT;
    if (lo) *lo = v[rank];
    if (hi) *hi = v[rank + 1];
    if (g0) *g0 = kGroups * rank / world;
    if (g1) *g1 = kGroups * (rank + 1) / world;
    return IRLS_OK;
}

static irls_status create_csr_impl(irls_ctx **out, const irls_comm_desc *comm, int64_t n, const int64_t *row_ptr,
                                   const int32_t *col, const double *w, int64_t s_, int64_t t_, const irls_options *opt,
                                   irls_vgroup *vg)
{
    NvtxRange nvtx_("irls_mincut_create_csr");
    if (!out) return IRLS_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    if (check_opts(opt) || n < 2 || !row_ptr || !col || !w || s_ < 0 || t_ < 0 || s_ >= n || t_ >= n)
        return IRLS_ERR_INVALID_ARGUMENT;
    if (s_ == t_) return IRLS_ERR_SOURCE_EQUALS_SINK;
    if (n >= ((int64_t)1 << 31)) return IRLS_ERR_INVALID_ARGUMENT;
    if (row_ptr[0] != 0) return IRLS_ERR_INVALID_ARGUMENT;
    for (int64_t u = 0; u < n; u++)
        if (row_ptr[u + 1] < row_ptr[u]) return IRLS_ERR_INVALID_ARGUMENT;
    const int64_t nnz = row_ptr[n];
    // Host preparation runs on the host threads (row blocks); every result is
    // independent of the thread count (first offending entry wins, integer
    // counts, per-row sums in CSR order).
    {
        std::vector<int64_t> bad(host_threads(nnz), INT64_MAX);
        std::vector<int> code(bad.size(), 0);
        parallel_for(nnz, [&](int i, int64_t a, int64_t b) {
            for (int64_t e = a; e < b; e++) {
                if (col[e] < 0 || col[e] >= n) { bad[i] = e; code[i] = IRLS_ERR_INVALID_ARGUMENT; return; }
                if (!(w[e] >= 0.0) || isinf(w[e])) { bad[i] = e; code[i] = IRLS_ERR_BAD_CAPACITY; return; }
            }
        });
        for (size_t i = 0; i < bad.size(); i++)
            if (bad[i] != INT64_MAX) return (irls_status)code[i];
        std::vector<uint8_t> loop(host_threads(n), 0);
        parallel_for(n, [&](int i, int64_t a, int64_t b) {
            for (int64_t u = a; u < b && !loop[i]; u++)
                for (int64_t e = row_ptr[u]; e < row_ptr[u + 1]; e++)
                    if (col[e] == u) { loop[i] = 1; break; }
        });
        for (uint8_t l : loop)
            if (l) return IRLS_ERR_INVALID_ARGUMENT;
    }
    // merge duplicates in CSR order (A7): count per row, then fill
    std::vector<int64_t> mptr(n + 1, 0);
    std::vector<int32_t> comp_root;
    auto merge_row = [&](int64_t u, std::vector<Ent> &tmp, int32_t *oc, double *ow) -> int64_t {
        const int64_t a = row_ptr[u], b = row_ptr[u + 1];
        bool sorted = true;
        for (int64_t e = a + 1; e < b; e++)
            if (col[e] <= col[e - 1]) { sorted = false; break; }
        if (sorted) {
            if (oc)
                for (int64_t e = a; e < b; e++) { oc[e - a] = col[e]; ow[e - a] = w[e]; }
            return b - a;
        }
        tmp.clear();
        for (int64_t e = a; e < b; e++) tmp.push_back({col[e], e, w[e]});
        std::stable_sort(tmp.begin(), tmp.end(), [](const Ent &x, const Ent &y) { return x.col < y.col; });
        int64_t m = 0;
        double last = 0.0;
        for (size_t i = 0; i < tmp.size(); i++) {
            if (i > 0 && tmp[i].col == tmp[i - 1].col) {
                last = last + tmp[i].w;
                if (ow) ow[m - 1] = last;
            } else {
                last = tmp[i].w;
                if (oc) { oc[m] = tmp[i].col; ow[m] = last; }
                m++;
            }
        }
        return m;
    };
    parallel_for(n, [&](int, int64_t a, int64_t b) {
        std::vector<Ent> tmp;
        for (int64_t u = a; u < b; u++) mptr[u + 1] = merge_row(u, tmp, nullptr, nullptr);
    });
    for (int64_t u = 0; u < n; u++) mptr[u + 1] += mptr[u];
    HostBuf<int32_t> mcol(mptr[n]);
    HostBuf<double> mw(mptr[n]);
    parallel_for(n, [&](int, int64_t a, int64_t b) {
        std::vector<Ent> tmp;
        for (int64_t u = a; u < b; u++) merge_row(u, tmp, mcol.data() + mptr[u], mw.data() + mptr[u]);
    });
    // exact symmetry
    {
        std::vector<uint8_t> asym(host_threads(n), 0);
        parallel_for(n, [&](int i, int64_t a, int64_t b) {
            for (int64_t u = a; u < b && !asym[i]; u++)
                for (int64_t e = mptr[u]; e < mptr[u + 1]; e++) {
                    const int32_t v = mcol[e];
                    const int32_t *beg = mcol.data() + mptr[v], *end = mcol.data() + mptr[v + 1];
                    const int32_t *it = std::lower_bound(beg, end, (int32_t)u);
                    if (it == end || *it != u || mw[it - mcol.data()] != mw[e]) { asym[i] = 1; break; }
                }
        });
        for (uint8_t a : asym)
            if (a) return IRLS_ERR_NOT_SYMMETRIC;
    }
    const int64_t nr = n - 2;
    auto red = [&](int64_t v) { return v - (v > s_) - (v > t_); };
    auto orig_of = [&](int64_t r) {  // reduced id -> original id
        int64_t u = r;
        const int64_t lo2 = std::min(s_, t_), hi2 = std::max(s_, t_);
        if (u >= lo2) u++;
        if (u >= hi2) u++;
        return u;
    };
    std::vector<double> hcs(std::max<int64_t>(nr, 1), 0.0), hct(std::max<int64_t>(nr, 1), 0.0);
    std::vector<int64_t> orig(std::max<int64_t>(nr, 1), 0);
    std::vector<int64_t> aptr(nr + 1, 0);
    double cst = 0.0;
    for (int64_t e = mptr[s_]; e < mptr[s_ + 1]; e++)
        if (mcol[e] == t_) cst = mw[e];
    parallel_for(nr, [&](int, int64_t a, int64_t b) {
        for (int64_t r = a; r < b; r++) {
            const int64_t u = orig_of(r);
            orig[r] = u;
            int64_t k = 0;
            for (int64_t e = mptr[u]; e < mptr[u + 1]; e++) {
                const int64_t v = mcol[e];
                if (v == s_) hcs[r] = mw[e];
                else if (v == t_) hct[r] = mw[e];
                else if (mw[e] > 0.0) k++;
            }
            aptr[r + 1] = k;
        }
    });
    for (int64_t r = 0; r < nr; r++) aptr[r + 1] += aptr[r];
    HostBuf<int32_t> aidx(aptr[nr]);
    HostBuf<double> ac(aptr[nr]);
    std::vector<int64_t> tcnt(host_threads(nr), 0);
    std::vector<double> tmax(tcnt.size(), 0.0);
    parallel_for(nr, [&](int i, int64_t a, int64_t b) {
        int64_t cn = 0;
        double cm = 0.0;
        for (int64_t r = a; r < b; r++) {
            const int64_t u = orig[r];
            int64_t k = aptr[r];
            for (int64_t e = mptr[u]; e < mptr[u + 1]; e++) {
                const int64_t v = mcol[e];
                if (v == s_ || v == t_ || !(mw[e] > 0.0)) continue;
                aidx[k] = (int32_t)red(v);
                ac[k] = mw[e];
                k++;
                if (v > u) { cn++; cm = std::max(cm, mw[e]); }
            }
            if (hcs[r] > 0) { cn++; cm = std::max(cm, hcs[r]); }
            if (hct[r] > 0) { cn++; cm = std::max(cm, hct[r]); }
        }
        tcnt[i] = cn;
        tmax[i] = cm;
    });
    double cmax = cst;
    int64_t cnt = cst > 0.0;
    for (size_t i = 0; i < tcnt.size(); i++) { cnt += tcnt[i]; cmax = std::max(cmax, tmax[i]); }
    // Prop. 1 / A8: every component of G~ touches a positive terminal edge.
    // Lock-free union-find over the edges (the components do not depend on
    // the union order), then every component's root must be anchored.
    {
        std::unique_ptr<std::atomic<int32_t>[]> par(new std::atomic<int32_t>[(size_t)std::max<int64_t>(nr, 1)]);
        std::unique_ptr<std::atomic<uint8_t>[]> anc(new std::atomic<uint8_t>[(size_t)std::max<int64_t>(nr, 1)]);
        parallel_for(nr, [&](int, int64_t a, int64_t b) {
            for (int64_t r = a; r < b; r++) {
                par[r].store((int32_t)r, std::memory_order_relaxed);
                anc[r].store(0, std::memory_order_relaxed);
            }
        });
        auto find = [&](int32_t x) {
            for (;;) {
                int32_t p = par[x].load(std::memory_order_relaxed);
                if (p == x) return x;
                const int32_t gp = par[p].load(std::memory_order_relaxed);
                if (gp != p) par[x].compare_exchange_weak(p, gp, std::memory_order_relaxed);
                x = gp;
            }
        };
        parallel_for(nr, [&](int, int64_t a, int64_t b) {
            for (int64_t r = a; r < b; r++)
                for (int64_t e = aptr[r]; e < aptr[r + 1]; e++) {
                    if (aidx[e] < r) continue;
                    int32_t x = (int32_t)r, y = aidx[e];
                    for (;;) {
                        x = find(x);
                        y = find(y);
                        if (x == y) break;
                        if (x < y) std::swap(x, y);  // link the larger root below the smaller
                        int32_t expect = x;
                        if (par[x].compare_exchange_strong(expect, y, std::memory_order_relaxed)) break;
                    }
                }
        });
        parallel_for(nr, [&](int, int64_t a, int64_t b) {
            for (int64_t r = a; r < b; r++)
                if (hcs[r] > 0.0 || hct[r] > 0.0) anc[find((int32_t)r)].store(1, std::memory_order_relaxed);
        });
        std::vector<uint8_t> lonely(host_threads(nr), 0);
        comp_root.resize(std::max<int64_t>(nr, 1));
        parallel_for(nr, [&](int i, int64_t a, int64_t b) {
            for (int64_t r = a; r < b; r++) {
                const int32_t root = find((int32_t)r);
                comp_root[r] = root;  // kept: the components of G~ never change (A8 at set_terminal_weights)
                if (!anc[root].load(std::memory_order_relaxed)) lonely[i] = 1;
            }
        });
        for (uint8_t l : lonely)
            if (l) return IRLS_ERR_SINGULAR;
    }
    // SELL-64 (slices of 64 consecutive rows, column-major inside a slice: the
    // k-th neighbour of rows 2t and 2t+1 are adjacent, one 128-bit load)
    const int64_t nsl = (nr + kSell - 1) / kSell;
    std::vector<int64_t> sptr(nsl + 1, 0);
    int64_t sell_wmax = 0;
    for (int64_t sl = 0; sl < nsl; sl++) {
        int64_t wmax = 0;
        for (int64_t r = sl * kSell; r < std::min<int64_t>(nr, sl * kSell + kSell); r++)
            wmax = std::max(wmax, aptr[r + 1] - aptr[r]);
        sptr[sl + 1] = sptr[sl] + kSell * wmax;
        sell_wmax = std::max(sell_wmax, wmax);
    }
    const int64_t nent = sptr[nsl];
    HostBuf<int32_t> scol(nent);
    HostBuf<double> scap(nent);
    parallel_for(nsl, [&](int, int64_t a, int64_t b) {  // padding slots: col -1, c 0
        for (int64_t e = sptr[a]; e < sptr[b]; e++) { scol[e] = -1; scap[e] = 0.0; }
    });
    parallel_for(nr, [&](int, int64_t a, int64_t b) {
        for (int64_t r = a; r < b; r++) {
            const int64_t sl = r / kSell, ln = r % kSell;
            for (int64_t k = 0; k < aptr[r + 1] - aptr[r]; k++) {
                scol[sptr[sl] + kSell * k + ln] = aidx[aptr[r] + k];
                scap[sptr[sl] + kSell * k + ln] = ac[aptr[r] + k];
            }
        }
    });
    irls_ctx *c = new irls_ctx();
    c->vg = vg;
    irls_status st = common_setup(c, comm, opt);
    if (!st && c->multi && !csr_strips(nr, c->world, c->rank_lo)) st = IRLS_ERR_INVALID_ARGUMENT;
    if (!st && !c->multi) c->rank_lo = {0, nr};
    if (!st) {
        c->kind = 1;
        c->n_glob = nr;
        c->n_total = n;
        c->s_id = s_;
        c->t_id = t_;
        c->c_st = cst;
        c->K = (int32_t)((nr + kChunk - 1) / kChunk);
        c->g0 = kGroups * c->rank / c->world;
        c->g1 = kGroups * (c->rank + 1) / c->world;
        c->lo = c->rank_lo[c->rank];
        c->n_own = c->rank_lo[c->rank + 1] - c->lo;
        c->chunk0 = (int32_t)(c->lo / kChunk);
        c->nchunks = (int32_t)((c->n_own + kChunk - 1) / kChunk);
        c->n_fin = count_nonempty(c->K, c->g0, c->g1);
        c->n_links = aptr[nr] / 2;
        c->F = compute_F(cmax, cnt);
        c->n_entries = nent;
        c->sell_wmax = (int32_t)sell_wmax;
        c->npad_own = (int64_t)c->nchunks * kChunk;
        c->comp_root = std::move(comp_root);
    }
    // the strip's local SELL: owned neighbours -> v - lo, others -> ghost block
    // (ascending global id, hence grouped by owner rank); send lists by the
    // symmetry of G~: u goes to peer q iff u has a neighbour owned by q
    std::vector<int64_t> lsptr;
    std::vector<int32_t> lscol, lsend;
    std::vector<double> lscap;
    int64_t lwmax = 0;
    if (!st && c->multi) {
        const int64_t lo = c->lo, hi = c->lo + c->n_own, W = c->world;
        auto owner = [&](int64_t v) {
            return (int)(std::upper_bound(c->rank_lo.begin(), c->rank_lo.end() - 1, v) - c->rank_lo.begin()) - 1;
        };
        std::vector<int32_t> ghosts;
        for (int64_t r = lo; r < hi; r++)
            for (int64_t e = aptr[r]; e < aptr[r + 1]; e++)
                if (aidx[e] < lo || aidx[e] >= hi) ghosts.push_back(aidx[e]);
        std::sort(ghosts.begin(), ghosts.end());
        ghosts.erase(std::unique(ghosts.begin(), ghosts.end()), ghosts.end());
        c->n_ghost = (int64_t)ghosts.size();
        c->recv_off.assign(W + 1, 0);
        for (int32_t v : ghosts) c->recv_off[owner(v) + 1]++;
        for (int q = 0; q < W; q++) c->recv_off[q + 1] += c->recv_off[q];
        std::vector<std::vector<int32_t>> sendq(W);
        for (int64_t r = lo; r < hi; r++) {
            int peers[16], np = 0;
            for (int64_t e = aptr[r]; e < aptr[r + 1]; e++) {
                const int64_t v = aidx[e];
                if (v >= lo && v < hi) continue;
                const int q = owner(v);
                bool seen = false;
                for (int i = 0; i < np; i++) seen |= peers[i] == q;
                if (!seen && np < 16) peers[np++] = q;
            }
            for (int i = 0; i < np; i++) sendq[peers[i]].push_back((int32_t)(r - lo));
        }
        c->send_off.assign(W + 1, 0);
        for (int q = 0; q < W; q++) {
            c->send_off[q + 1] = c->send_off[q] + (int64_t)sendq[q].size();
            lsend.insert(lsend.end(), sendq[q].begin(), sendq[q].end());
        }
        const int64_t nl = c->n_own, lnsl = (nl + kSell - 1) / kSell;
        lsptr.assign(lnsl + 1, 0);
        for (int64_t sl = 0; sl < lnsl; sl++) {
            int64_t wm = 0;
            for (int64_t r = sl * kSell; r < std::min<int64_t>(nl, sl * kSell + kSell); r++)
                wm = std::max(wm, aptr[lo + r + 1] - aptr[lo + r]);
            lsptr[sl + 1] = lsptr[sl] + kSell * wm;
            lwmax = std::max(lwmax, wm);
        }
        lscol.assign(std::max<int64_t>(lsptr[lnsl], 1), -1);
        lscap.assign(std::max<int64_t>(lsptr[lnsl], 1), 0.0);
        for (int64_t r = 0; r < nl; r++) {
            const int64_t sl = r / kSell, ln = r % kSell, gr = lo + r;
            for (int64_t k = 0; k < aptr[gr + 1] - aptr[gr]; k++) {
                const int64_t v = aidx[aptr[gr] + k];
                const int64_t lv = (v >= lo && v < hi)
                                       ? v - lo
                                       : c->npad_own + (std::lower_bound(ghosts.begin(), ghosts.end(), (int32_t)v) - ghosts.begin());
                lscol[lsptr[sl] + kSell * k + ln] = (int32_t)lv;
                lscap[lsptr[sl] + kSell * k + ln] = ac[aptr[gr] + k];
            }
        }
        c->ln_entries = lsptr[lnsl];
        c->lwmax = (int32_t)lwmax;
        if (c->npad_own + c->n_ghost >= ((int64_t)1 << 31)) st = IRLS_ERR_INVALID_ARGUMENT;
    }
    if (!st) st = alloc_solver(c, c->multi ? c->n_ghost : 0);
    if (!st) {
        const int64_t gpad = (int64_t)c->K * kChunk;  // the whole graph (rank 0 sweeps it)
        c->cs = dalloc<double>(c, gpad);
        c->ct = dalloc<double>(c, gpad);
        c->slice_ptr = dalloc<int64_t>(c, nsl + 1);
        c->col = dalloc<int32_t>(c, nent);
        c->cap = dalloc<double>(c, nent);
        c->gsell = dalloc<double>(c, nent);
        c->orig_dev = dalloc<int64_t>(c, std::max<int64_t>(nr, 1));
        if (!c->cs || !c->ct || !c->slice_ptr || !c->col || !c->cap || !c->gsell || !c->orig_dev) st = IRLS_ERR_OOM;
    }
    if (!st && !c->multi) {  // one rank: the solve runs on the global structure
        c->lslice_ptr = c->slice_ptr;
        c->lcol = c->col;
        c->lcap = c->cap;
        c->lg = c->gsell;
        c->lcs = c->cs;
        c->lct = c->ct;
        c->lwmax = c->sell_wmax;
        c->ln_entries = c->n_entries;
    } else if (!st) {
        const int64_t npad = c->npad_own, le = std::max<int64_t>(c->ln_entries, 1);
        c->lslice_ptr = dalloc<int64_t>(c, (int64_t)lsptr.size());
        c->lcol = dalloc<int32_t>(c, le);
        c->lcap = dalloc<double>(c, le);
        c->lg = dalloc<double>(c, le);
        c->lcs = dalloc<double>(c, npad);
        c->lct = dalloc<double>(c, npad);
        c->send_idx = dalloc<int32_t>(c, std::max<int64_t>((int64_t)lsend.size(), 1));
        c->sendbuf = dalloc<double>(c, std::max<int64_t>((int64_t)lsend.size(), 1));
        if (!c->lslice_ptr || !c->lcol || !c->lcap || !c->lg || !c->lcs || !c->lct || !c->send_idx || !c->sendbuf)
            st = IRLS_ERR_OOM;
        cudaError_t e = cudaSuccess;
        auto up = [&](void *dst, const void *src, size_t bytes) {
            if (e == cudaSuccess && bytes > 0) e = memcpy_sync(c, dst, src, bytes, cudaMemcpyHostToDevice);
        };
        if (!st) {
            up(c->lslice_ptr, lsptr.data(), sizeof(int64_t) * lsptr.size());
            up(c->lcol, lscol.data(), sizeof(int32_t) * lscol.size());
            up(c->lcap, lscap.data(), sizeof(double) * lscap.size());
            if (c->n_own > 0) {
                up(c->lcs, hcs.data() + c->lo, sizeof(double) * c->n_own);
                up(c->lct, hct.data() + c->lo, sizeof(double) * c->n_own);
            }
            up(c->send_idx, lsend.data(), sizeof(int32_t) * lsend.size());
            if (e != cudaSuccess) st = fail(c, IRLS_ERR_CUDA, std::string("csr strip upload: ") + cudaGetErrorString(e));
        }
    }
    if (!st) st = init_nccl(c, comm);
    if (!st && nr > 0) {
        cudaError_t e = cudaSuccess;
        auto up = [&](void *dst, const void *src, size_t bytes) {
            if (e == cudaSuccess && bytes > 0) e = memcpy_sync(c, dst, src, bytes, cudaMemcpyHostToDevice);
        };
        up(c->cs, hcs.data(), sizeof(double) * nr);
        up(c->ct, hct.data(), sizeof(double) * nr);
        up(c->slice_ptr, sptr.data(), sizeof(int64_t) * (nsl + 1));
        up(c->col, scol.data(), sizeof(int32_t) * nent);
        up(c->cap, scap.data(), sizeof(double) * nent);
        up(c->orig_dev, orig.data(), sizeof(int64_t) * nr);
        if (e != cudaSuccess) st = fail(c, IRLS_ERR_CUDA, std::string("csr upload: ") + cudaGetErrorString(e));
    }
    if (st) {
        irls_mincut_destroy(c);
        return st;
    }
    *out = c;
    return IRLS_OK;
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
        unsigned long long vo[6];
        CK(cudaMemcpyAsync(c->cs, cs, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(c->ct, ct, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
        if (validate_stencil(c->nx, c->ny, c->nz, c->cx, c->cy, c->cz, c->cs, c->ct, vo, c->stream))
            return fail(c, IRLS_ERR_CUDA, "validate");
        if (vo[1] != 0 || vo[2] == 0) {
            // zero n-links present: full check on the host copy
            std::vector<double> hx(n), hy(n), hz(n);
            memcpy_sync(c, hx.data(), c->cx, sizeof(double) * n, cudaMemcpyDeviceToHost);
            memcpy_sync(c, hy.data(), c->cy, sizeof(double) * n, cudaMemcpyDeviceToHost);
            memcpy_sync(c, hz.data(), c->cz, sizeof(double) * n, cudaMemcpyDeviceToHost);
            if (!grid_nonsingular(c->nx, c->ny, c->nz, hx.data(), hy.data(), hz.data(), cs, ct))
                return fail(c, IRLS_ERR_SINGULAR, "terminal weights make L~ singular");
        }
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
// sweep cut
// ---------------------------------------------------------------------------
static irls_status alloc_sweep(irls_ctx *c)
{
    if (c->sb.keys) return IRLS_OK;
    SweepBuffers &b = c->sb;
    const int64_t n = c->n_glob, nt = sweep_ntiles(n);
    b.n = n;
    b.keys = dalloc<unsigned long long>(c, n);
    b.keys_alt = dalloc<unsigned long long>(c, n);
    b.vals = dalloc<int32_t>(c, n);
    b.vals_alt = dalloc<int32_t>(c, n);
    b.rank = dalloc<int32_t>(c, n);
    b.tile_hist = dalloc<int32_t>(c, 256 * nt);
    b.tile_off = dalloc<int32_t>(c, 256 * nt);
    b.scan_tmp = (int32_t *)dalloc<int64_t>(c, (256 * nt + 4095) / 4096 + 1);
    b.digit_hist = dalloc<unsigned long long>(c, 8 * 256);
    b.delta = dalloc<__int128>(c, n + 2);
    b.delta_id = dalloc<__int128>(c, n);
    b.tile_sum = dalloc<__int128>(c, nt);
    b.tile_min = dalloc<__int128>(c, nt);
    b.tile_argmin = dalloc<int64_t>(c, nt);
    b.flags = dalloc<int32_t>(c, 4);
    b.k_out = dalloc<int64_t>(c, 1);
    b.side = dalloc<uint8_t>(c, c->n_total);
    c->order_out = dalloc<int32_t>(c, n);
    if (!b.keys || !b.keys_alt || !b.vals || !b.vals_alt || !b.rank || !b.tile_hist || !b.tile_off || !b.scan_tmp ||
        !b.digit_hist || !b.delta || !b.delta_id || !b.tile_sum || !b.tile_min || !b.tile_argmin || !b.flags || !b.k_out || !b.side ||
        !c->order_out)
        return fail(c, IRLS_ERR_OOM, "sweep buffers");
    return IRLS_OK;
}

// Rank 0 result of the sweep, broadcast so every rank returns the same values.
struct SweepResultMsg {
    int64_t status, k;
    double cut;
};

static irls_status sweep_rank0(irls_ctx *c, const double *xfull, uint8_t *side, int32_t *order, int64_t *k,
                               double *cut_value);

extern "C" irls_status irls_sweep_cut(irls_ctx *c, uint8_t *side, int32_t *order, int64_t *k, double *cut_value)
{
    NvtxRange nvtx_("irls_sweep_cut");
    GUARD(c);
    if (c->state == 0) return fail(c, IRLS_ERR_STATE, "sweep before solve");
    double *xfull = nullptr;
    irls_status s = gather_x(c, &xfull);
    if (s) return s;
    SweepResultMsg msg{0, 0, 0.0};
    if (c->rank == 0) {
        s = sweep_rank0(c, xfull, side, order, &msg.k, &msg.cut);
        msg.status = s;
        if (s && s != IRLS_ERR_BAD_POTENTIAL && !c->multi) return s;
    }
    if (c->multi) {
        if (!c->msg_dev) {
            c->msg_dev = dalloc<SweepResultMsg>(c, 1);
            if (!c->msg_dev) return fail(c, IRLS_ERR_OOM, "sweep msg");
        }
        if (c->rank == 0)
            CK(cudaMemcpyAsync(c->msg_dev, &msg, sizeof(msg), cudaMemcpyHostToDevice, c->stream));
        NK(ncclBroadcast(c->msg_dev, c->msg_dev, sizeof(msg), ncclUint8, 0, c->nccl, c->stream));
        CK(cudaMemcpyAsync(&msg, c->msg_dev, sizeof(msg), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    }
    if (msg.status) return fail(c, (irls_status)msg.status, c->rank == 0 ? c->err : "sweep failed on rank 0");
    if (k) *k = msg.k;
    if (cut_value) *cut_value = msg.cut;
    return IRLS_OK;
}

static irls_status sweep_rank0(irls_ctx *c, const double *xfull, uint8_t *side, int32_t *order, int64_t *k,
                               double *cut_value)
{
    cudaStream_t st = c->stream;
    const int64_t n = c->n_glob;
    irls_status s = alloc_sweep(c);
    if (s) return s;
    int launches = 0;
    c->launches = 0;
    SweepBuffers &b = c->sb;
    CK(cudaMemsetAsync(b.flags, 0, sizeof(int32_t) * 4, st));
    sweep_keys(xfull, b, st);
    launches++;
    int32_t *ord = sweep_sort(b, st, &launches);
    int32_t hflag = 0;
    CK(cudaMemcpyAsync(&hflag, b.flags, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (hflag) return fail(c, IRLS_ERR_BAD_POTENTIAL, "NaN in potentials");
    sweep_rank(ord, b, st);
    launches++;
    if (c->kind == 0) sweep_delta_stencil(stencil_args(c, true), n, c->F, b, st);
    else sweep_delta_sell(sell_args_full(c), c->F, b, st);
    sweep_delta_order(ord, b, st);
    launches += 2;
    sweep_scan_argmin(b, qfix_host(c->c_st, c->F), st);
    launches += 4;
    RedArgs ra;
    ra.part = c->part;
    ra.slots = c->slots_local;
    ra.ctrl = c->ctrl;
    ra.K = (int32_t)((n + kChunk - 1) / kChunk);
    ra.g0 = 0;
    ra.g1 = 8;
    ra.n_fin = count_nonempty(ra.K, 0, 8);
    if (c->kind == 0) {
        sweep_side_cross_stencil(stencil_args(c, true), n, b, ra, st);
    } else {
        CK(cudaMemsetAsync(b.side, 0, c->n_total, st));
        sweep_side_cross_sell(sell_args_full(c), c->orig_dev, c->n_total, b, ra, st);
        const uint8_t one = 1;
        CK(cudaMemcpyAsync(b.side + c->s_id, &one, 1, cudaMemcpyHostToDevice, st));
    }
    launches++;
    irls_status ls = last_launch(c, "sweep");
    if (ls) return ls;
    double slots[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int64_t hk = 0;
    if (n > 0) CK(cudaMemcpyAsync(slots, c->slots_local, sizeof(slots), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&hk, b.k_out, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    if (order && n > 0) {
        sweep_order_out(ord, c->kind == 1 ? c->orig_dev : nullptr, c->order_out, n, st);
        launches++;
        CK(cudaMemcpyAsync(order, c->order_out, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
    }
    if (side) CK(cudaMemcpyAsync(side, b.side, c->n_total, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (n == 0) hk = 0;
    c->sweep_k = hk;
    c->sweep_cut = irls_combine_slots(slots) + c->c_st;
    c->sweep_valid = true;
    c->order_dev = ord;
    c->launches += launches;
    if (k) *k = hk;
    if (cut_value) *cut_value = c->sweep_cut;
    return IRLS_OK;
}

extern "C" irls_status irls_get_side(irls_ctx *c, uint8_t *side)
{
    GUARD(c);
    if (!c->sweep_valid) return fail(c, IRLS_ERR_STATE, "no sweep result");
    if (!side) return IRLS_ERR_INVALID_ARGUMENT;
    CK(memcpy_sync(c, side, c->sb.side, c->n_total, cudaMemcpyDeviceToHost));
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
    return IRLS_OK;
}

extern "C" irls_status irls_time_kernel(irls_ctx *c, int32_t which, int32_t reps, float *mean_ms)
{
    GUARD(c);
    if (!mean_ms || reps < 1 || which < 0 || which > 2) return IRLS_ERR_INVALID_ARGUMENT;
    if (c->state == 0) return fail(c, IRLS_ERR_STATE, "time_kernel needs a solved state");
    cudaStream_t st = c->stream;
    const int64_t npad = (int64_t)c->nchunks * kChunk;
    // snapshot everything the kernels write
    double *arrs[] = {c->x, c->q, c->r, c->z, c->p0, c->p1, c->D, c->Dinv};
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
    if (c->h_done) cudaFreeHost(c->h_done);
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

// ---------------------------------------------------------------------------
// Two-level rounding (include/irls_mincut.h, DESIGN.md §2 A25-A29)
// ---------------------------------------------------------------------------
#include <chrono>

static irls_status alloc_tl(irls_ctx *c)
{
    TLBuffers &b = c->tl;
    if (b.st) return IRLS_OK;
    const int64_t n = c->n_glob, K = (n + kChunk - 1) / kChunk, nt = tl_ntiles(n);
    b.n = n;
    b.st = dalloc<TLState>(c, 1);
    b.part = dalloc<double>(c, 3 * K);
    b.slots = dalloc<double>(c, 3 * kGroups);
    b.ctrl = dalloc<DevCtrl>(c, 1);
    b.cls = dalloc<int8_t>(c, n);
    b.flag = dalloc<int32_t>(c, n);
    b.cid = dalloc<int32_t>(c, n);
    b.deg = dalloc<int32_t>(c, n);
    b.eoff = dalloc<int32_t>(c, n);
    b.scan_tmp = dalloc<int64_t>(c, nt + 1);
    b.tile_a = dalloc<__int128>(c, nt);
    b.tile_n1 = dalloc<int32_t>(c, nt);
    b.cp = dalloc<int32_t>(c, n + 1);
    b.cqs = dalloc<__int128>(c, n);
    b.cqt = dalloc<__int128>(c, n);
    b.src = dalloc<uint8_t>(c, n);
    b.prank = dalloc<int32_t>(c, n);
    b.one = dalloc<int64_t>(c, 1);
    b.side = dalloc<uint8_t>(c, c->n_total);
    b.ccol = nullptr;
    b.ccap = nullptr;
    b.cap_entries = 0;
    if (!b.st || !b.part || !b.slots || !b.ctrl || !b.cls || !b.flag || !b.cid || !b.deg || !b.eoff || !b.scan_tmp ||
        !b.tile_a || !b.tile_n1 || !b.cp || !b.cqs || !b.cqt || !b.src || !b.prank || !b.one || !b.side)
        return fail(c, IRLS_ERR_OOM, "two-level buffers");
    const int64_t one = 1;
    CK(cudaMemcpyAsync(b.one, &one, sizeof(one), cudaMemcpyHostToDevice, c->stream));
    return IRLS_OK;
}

// Coarse entry buffers grow to the largest coarse graph seen.
static irls_status tl_reserve(irls_ctx *c, int64_t entries)
{
    TLBuffers &b = c->tl;
    if (entries <= b.cap_entries && b.ccol) return IRLS_OK;
    for (void *p : {(void *)b.ccol, (void *)b.ccap}) {
        if (!p) continue;
        CK(dfree(c, p));
    }
    b.ccol = dalloc<int32_t>(c, entries);
    b.ccap = dalloc<double>(c, entries);
    if (!b.ccol || !b.ccap) return fail(c, IRLS_ERR_OOM, "coarse graph");
    b.cap_entries = std::max<int64_t>(entries, 1);
    return IRLS_OK;
}

static double q_to_double(__int128 q, int32_t F) { return ldexp((double)q, -F); }

// exact: no contraction (gamma0 = -inf, gamma1 = +inf, every node in Sc): the
// exact min cut mu* of G by the same pipeline (for delta, Eq. 13).
static irls_status two_level_rank0(irls_ctx *c, const double *xfull, uint8_t *side, irls_two_level_report *r,
                                   bool exact = false)
{
    auto t_start = std::chrono::steady_clock::now();
    cudaStream_t st = c->stream;
    const int64_t n = c->n_glob;
    irls_status s = alloc_tl(c);
    if (s) return s;
    TLBuffers &b = c->tl;
    memset(r, 0, sizeof(*r));
    r->F = c->F;
    cudaEvent_t ev[4];
    for (auto &e : ev) CK(cudaEventCreate(&e));
    struct EvGuard {
        cudaEvent_t *e;
        ~EvGuard() { for (int i = 0; i < 4; i++) cudaEventDestroy(e[i]); }
    } guard{ev};
    int launches = 0;
    CK(cudaEventRecord(ev[0], st));
    // A NaN in x lands in cluster 0 (the comparison is false) and makes c0 NaN.
    // 1. K-means (A25): batches of rounds, the device stops itself
    TLState h{0.1, 0.9, 0, 0};
    CK(cudaMemcpyAsync(b.st, &h, sizeof(h), cudaMemcpyHostToDevice, st));
    if (exact) {
        h.done = 1;
    } else if (n > 0) {
        RedArgs ra;
        ra.part = b.part;
        ra.slots = b.slots;
        ra.ctrl = b.ctrl;
        ra.K = (int32_t)((n + kChunk - 1) / kChunk);
        ra.g0 = 0;
        ra.g1 = kGroups;
        ra.n_fin = count_nonempty(ra.K, 0, kGroups);
        for (int batch = 0; batch < 13 && !h.done; batch++) {
            for (int i = 0; i < 8; i++) tl_kmeans_round(xfull, n, b.st, ra, st);
            launches += 8;
            CK(cudaMemcpyAsync(&h, b.st, sizeof(h), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
        }
    } else if (!exact) {  // only the terminals' values {1, 0}
        for (h.rounds = 1; h.rounds <= 100; h.rounds++) {
            double s0 = 0.0, s1 = 0.0;
            int64_t n1 = 0;
            const double xt[2] = {1.0, 0.0};
            for (double v : xt) {
                if (fabs(v - h.c1) < fabs(v - h.c0)) { s1 = s1 + v; n1++; } else { s0 = s0 + v; }
            }
            const double d0 = (2 - n1) > 0 ? s0 / (double)(2 - n1) : h.c0, d1 = n1 > 0 ? s1 / (double)n1 : h.c1;
            const bool same = d0 == h.c0 && d1 == h.c1;
            h.c0 = d0;
            h.c1 = d1;
            if (same) break;
        }
        if (h.rounds > 100) h.rounds = 100;
    }
    if (exact) h.rounds = 0;
    if (isnan(h.c0) || isnan(h.c1)) return fail(c, IRLS_ERR_BAD_POTENTIAL, "NaN in potentials");
    r->c0 = h.c0;
    r->c1 = h.c1;
    r->gamma0 = exact ? -INFINITY : h.c0 + 0.05;
    r->gamma1 = exact ? INFINITY : h.c1 - 0.05;
    r->kmeans_rounds = h.rounds;
    // 2-3. classify, coarse ids / offsets, G_c
    const int64_t nt = tl_ntiles(n);
    int32_t last[4] = {0, 0, 0, 0};
    std::vector<__int128> tiles((size_t)std::max<int64_t>(nt, 1));
    std::vector<int32_t> tiles_n1((size_t)std::max<int64_t>(nt, 1), 0);
    if (n > 0) {
        if (c->kind == 0) tl_classify_stencil(stencil_args(c, true), n, xfull, r->gamma0, r->gamma1, c->F, b, st);
        else tl_classify_sell(sell_args_full(c), xfull, r->gamma0, r->gamma1, c->F, b, st);
        exclusive_scan_i32(b.flag, n, b.cid, b.scan_tmp, st, &launches);
        exclusive_scan_i32(b.deg, n, b.eoff, b.scan_tmp, st, &launches);
        launches += 1;
        CK(cudaMemcpyAsync(&last[0], b.cid + n - 1, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&last[1], b.flag + n - 1, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&last[2], b.eoff + n - 1, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&last[3], b.deg + n - 1, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(tiles.data(), b.tile_a, sizeof(__int128) * nt, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(tiles_n1.data(), b.tile_n1, sizeof(int32_t) * nt, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }
    const int64_t nc = (int64_t)last[0] + last[1], E = (int64_t)last[2] + last[3];
    if (E > INT32_MAX - 1) return fail(c, IRLS_ERR_INVALID_ARGUMENT, "coarse graph too large");
    s = tl_reserve(c, E);
    if (s) return s;
    __int128 qst = qfix_host(c->c_st, c->F);
    for (int64_t i = 0; i < nt && n > 0; i++) qst += tiles[i];
    if (nc > 0) {
        if (c->kind == 0) tl_fill_stencil(stencil_args(c, true), n, c->F, b, st);
        else tl_fill_sell(sell_args_full(c), c->F, b, st);
        launches++;
    }
    irls_status ls = last_launch(c, "two-level coarsening");
    if (ls) return ls;
    CK(cudaEventRecord(ev[1], st));
    if (!c->h_cp.resize(nc + 1) || !c->h_ccol.resize(E) || !c->h_ccap.resize(E) || !c->h_cqs.resize(nc) ||
        !c->h_cqt.resize(nc))
        return fail(c, IRLS_ERR_OOM, "pinned coarse-graph buffers");
    if (nc > 0) {
        CK(cudaMemcpyAsync(c->h_cp.data(), b.cp, sizeof(int32_t) * nc, cudaMemcpyDeviceToHost, st));
        if (E > 0) {
            CK(cudaMemcpyAsync(c->h_ccol.data(), b.ccol, sizeof(int32_t) * E, cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(c->h_ccap.data(), b.ccap, sizeof(double) * E, cudaMemcpyDeviceToHost, st));
        }
        CK(cudaMemcpyAsync(c->h_cqs.data(), b.cqs, sizeof(__int128) * nc, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(c->h_cqt.data(), b.cqt, sizeof(__int128) * nc, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaEventRecord(ev[2], st));
    CK(cudaStreamSynchronize(st));
    c->h_cp[nc] = (int32_t)E;
    c->h_qst = qst;
    // 4. exact max-flow on G_c (host)
    auto t0 = std::chrono::steady_clock::now();
    HostBuf<__int128> qcap(E);
    parallel_for(E, [&](int, int64_t a, int64_t b2) {
        for (int64_t e = a; e < b2; e++) qcap[e] = qfix_host(c->h_ccap[e], c->F);
    });
    std::vector<uint8_t> src((size_t)std::max<int64_t>(nc, 1), 0);
    int64_t stats[3] = {0, 0, 0};
    __int128 flow = 0;
    if (nc > 0) {
        NvtxRange nvtx_mf("two_level: host max-flow");
        flow = maxflow_bk((int32_t)nc, c->h_cp.data(), c->h_ccol.data(), qcap.data(), c->h_cqs.data(),
                          c->h_cqt.data(), src.data(), stats);
        if (stats[0] != 1) return fail(c, IRLS_ERR_CUDA, "coarse max-flow not certified (flow != cut)");
    } else {
        stats[0] = 1;
    }
    auto t1 = std::chrono::steady_clock::now();
    r->ms_maxflow = (float)std::chrono::duration<double, std::milli>(t1 - t0).count();
    r->certified = (int32_t)stats[0];
    r->augmentations = stats[1];
    r->coarse_flow = q_to_double(flow + qst, c->F);
    // 5. lift + cut on G (C3)
    CK(cudaEventRecord(ev[3], st));
    if (nc > 0) CK(cudaMemcpyAsync(b.src, src.data(), nc, cudaMemcpyHostToDevice, st));
    float ms_copy_back = 0.0f;
    cudaEvent_t e4, e5;
    CK(cudaEventCreate(&e4));
    CK(cudaEventCreate(&e5));
    CK(cudaEventRecord(e4, st));
    tl_lift(b, st);
    RedArgs ra;
    ra.part = c->part;
    ra.slots = c->slots_local;
    ra.ctrl = c->ctrl;
    ra.K = (int32_t)((n + kChunk - 1) / kChunk);
    ra.g0 = 0;
    ra.g1 = 8;
    ra.n_fin = count_nonempty(ra.K, 0, 8);
    SweepBuffers sb = c->sb;
    sb.rank = b.prank;
    sb.k_out = b.one;
    sb.side = b.side;
    if (n > 0) {
        if (c->kind == 0) {
            sweep_side_cross_stencil(stencil_args(c, true), n, sb, ra, st);
        } else {
            CK(cudaMemsetAsync(b.side, 0, c->n_total, st));
            sweep_side_cross_sell(sell_args_full(c), c->orig_dev, c->n_total, sb, ra, st);
            const uint8_t one = 1;
            CK(cudaMemcpyAsync(b.side + c->s_id, &one, 1, cudaMemcpyHostToDevice, st));
        }
        launches += 2;
    } else {
        CK(cudaMemsetAsync(b.side, 0, c->n_total, st));
        const uint8_t one = 1;
        CK(cudaMemcpyAsync(b.side + (c->kind == 0 ? 0 : c->s_id), &one, 1, cudaMemcpyHostToDevice, st));
    }
    ls = last_launch(c, "two-level lift");
    if (ls) return ls;
    double slots[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (n > 0) CK(cudaMemcpyAsync(slots, c->slots_local, sizeof(slots), cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(e5, st));
    if (side) CK(cudaMemcpyAsync(side, b.side, c->n_total, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    float ms_a = 0, ms_b = 0, ms_c = 0;
    cudaEventElapsedTime(&ms_a, ev[0], ev[1]);
    cudaEventElapsedTime(&ms_b, ev[1], ev[2]);
    cudaEventElapsedTime(&ms_c, e4, e5);
    cudaEventElapsedTime(&ms_copy_back, ev[3], e4);
    cudaEventDestroy(e4);
    cudaEventDestroy(e5);
    r->ms_gpu = ms_a + ms_c;
    r->ms_copy = ms_b + ms_copy_back;
    int64_t n1 = 0;
    for (int64_t i = 0; i < nt && n > 0; i++) n1 += tiles_n1[i];
    const int64_t n0 = n - n1 - nc;
    r->n0 = n0;
    r->n1 = n1;
    r->nc = nc;
    r->coarse_nlinks = E / 2;
    r->cut_value = (n > 0 ? irls_combine_slots(slots) : 0.0) + c->c_st;
    c->tl_valid = true;
    c->launches = launches;
    r->ms_total = (float)std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
    return IRLS_OK;
}

struct TwoLevelMsg {
    int64_t status;
    irls_two_level_report rep;
};

extern "C" irls_status irls_two_level_cut(irls_ctx *c, uint8_t *side, irls_two_level_report *rep)
{
    NvtxRange nvtx_("irls_two_level_cut");
    GUARD(c);
    if (c->state == 0) return fail(c, IRLS_ERR_STATE, "two-level rounding before solve");
    double *xfull = nullptr;
    irls_status s = gather_x(c, &xfull);
    if (s) return s;
    TwoLevelMsg msg;
    memset(&msg, 0, sizeof(msg));
    if (c->rank == 0) {
        s = two_level_rank0(c, xfull, side, &msg.rep);
        msg.status = s;
        if (s && !c->multi) return s;
    }
    if (c->multi) {
        void *dmsg = nullptr;
        CK(cudaMallocAsync(&dmsg, sizeof(msg), c->stream));
        if (c->rank == 0) CK(cudaMemcpyAsync(dmsg, &msg, sizeof(msg), cudaMemcpyHostToDevice, c->stream));
        NK(ncclBroadcast(dmsg, dmsg, sizeof(msg), ncclUint8, 0, c->nccl, c->stream));
        CK(cudaMemcpyAsync(&msg, dmsg, sizeof(msg), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaFreeAsync(dmsg, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    }
    if (msg.status) return fail(c, (irls_status)msg.status, c->rank == 0 ? c->err : "two-level failed on rank 0");
    if (rep) *rep = msg.rep;
    return IRLS_OK;
}

extern "C" irls_status irls_exact_min_cut(irls_ctx *c, uint8_t *side, irls_two_level_report *rep)
{
    NvtxRange nvtx_("irls_exact_min_cut");
    GUARD(c);
    if (c->world > 1) return fail(c, IRLS_ERR_INVALID_ARGUMENT, "irls_exact_min_cut is single-process");
    irls_two_level_report r;
    irls_status s = two_level_rank0(c, c->x, side, &r, true);
    if (s) return s;
    if (rep) *rep = r;
    return IRLS_OK;
}

extern "C" irls_status irls_vgroup_two_level_cut(irls_vgroup *g, uint8_t *side, irls_two_level_report *rep)
{
    if (!g) return IRLS_ERR_INVALID_ARGUMENT;
    irls_ctx *c = g->ranks[0];
    GUARD(c);
    if (c->state == 0) return fail(c, IRLS_ERR_STATE, "two-level rounding before solve");
    double *full = nullptr;
    irls_status s = vgather_x(g, &full);
    if (s) return s;
    irls_two_level_report r;
    s = two_level_rank0(c, full, side, &r);
    if (s) return s;
    if (rep) *rep = r;
    return IRLS_OK;
}

static void put_words(uint64_t *w, __int128 v)
{
    w[0] = (uint64_t)v;
    w[1] = (uint64_t)((unsigned __int128)v >> 64);
}
static __int128 get_words(const uint64_t *w) { return (__int128)(((unsigned __int128)w[1] << 64) | w[0]); }

extern "C" irls_status irls_two_level_get_coarse(irls_ctx *c, int8_t *cls, int32_t *ptr, int32_t *col, double *cap,
                                                 uint64_t *qs, uint64_t *qt, uint64_t *qst)
{
    GUARD(c);
    if (!c->tl_valid) return fail(c, IRLS_ERR_STATE, "no two-level result");
    const int64_t nc = (int64_t)c->h_cp.size() - 1, E = c->h_cp[nc];
    if (cls && c->n_glob > 0) CK(memcpy_sync(c, cls, c->tl.cls, c->n_glob, cudaMemcpyDeviceToHost));
    if (ptr) memcpy(ptr, c->h_cp.data(), sizeof(int32_t) * (nc + 1));
    if (col && E) memcpy(col, c->h_ccol.data(), sizeof(int32_t) * E);
    if (cap && E) memcpy(cap, c->h_ccap.data(), sizeof(double) * E);
    for (int64_t i = 0; i < nc; i++) {
        if (qs) put_words(qs + 2 * i, c->h_cqs[i]);
        if (qt) put_words(qt + 2 * i, c->h_cqt[i]);
    }
    if (qst) put_words(qst, c->h_qst);
    return IRLS_OK;
}

extern "C" irls_status irls_coarse_maxflow(int32_t nc, const int32_t *ptr, const int32_t *col, const uint64_t *cap,
                                           const uint64_t *qs, const uint64_t *qt, uint8_t *src, uint64_t *flow,
                                           int32_t *certified)
{
    if (nc < 0 || (nc > 0 && (!ptr || !qs || !qt || !src)) || !flow) return IRLS_ERR_INVALID_ARGUMENT;
    if (nc == 0) {
        put_words(flow, 0);
        if (certified) *certified = 1;
        return IRLS_OK;
    }
    const int32_t E = ptr[nc];
    std::vector<__int128> qc(E), a(nc), b(nc);
    for (int32_t e = 0; e < E; e++) qc[e] = get_words(cap + 2 * e);
    for (int32_t u = 0; u < nc; u++) {
        a[u] = get_words(qs + 2 * u);
        b[u] = get_words(qt + 2 * u);
    }
    int64_t stats[3] = {0, 0, 0};
    __int128 f = maxflow_bk(nc, ptr, col, qc.data(), a.data(), b.data(), src, stats);
    if (stats[0] < 0) return IRLS_ERR_INVALID_ARGUMENT;
    put_words(flow, f);
    if (certified) *certified = (int32_t)stats[0];
    return IRLS_OK;
}

// ---------------------------------------------------------------------------
// Cheeger-type diagnostic lambda_2 (A30)
// ---------------------------------------------------------------------------
extern "C" irls_status irls_lambda2(irls_ctx *c, double cg_rtol, int32_t cg_max_iter, int32_t cg_norm, double *x_out,
                                    irls_lambda2_report *rep)
{
    NvtxRange nvtx_("irls_lambda2");
    GUARD(c);
    if (c->world > 1) return fail(c, IRLS_ERR_INVALID_ARGUMENT, "irls_lambda2 is single-process");
    if (!(cg_rtol >= 0.0) || cg_max_iter < 0 || (cg_norm != 0 && cg_norm != 1))
        return fail(c, IRLS_ERR_INVALID_ARGUMENT, "lambda2 CG options");
    cudaStream_t st = c->stream;
    const int64_t n = c->n_own;
    if (n == 0) {  // only s and t: x = (1, -1), x^T L x = 4 c_st, C = 2 c_st
        if (rep) {
            memset(rep, 0, sizeof(*rep));
            rep->xLx = 4.0 * c->c_st;
            rep->C = 2.0 * c->c_st;
            rep->lambda2 = rep->xLx / (2.0 * rep->C);
            rep->converged = 1;
        }
        return IRLS_OK;
    }
    double *xs = dalloc<double>(c, n);
    if (!xs) return fail(c, IRLS_ERR_OOM, "lambda2 x save");
    CK(cudaMemcpyAsync(xs, c->x, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    const int state0 = c->state;
    const int64_t iters0 = c->last_cg_iters;
    // the CG options live in the control block: set, solve, restore
    DevCtrl *d = c->ctrl;
    auto set_opts = [&](double rt, int32_t mi, int32_t nm) -> cudaError_t {
        cudaError_t e = cudaMemcpyAsync(&d->rtol, &rt, sizeof(double), cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(&d->max_iter, &mi, sizeof(int32_t), cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(&d->norm, &nm, sizeof(int32_t), cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        return e;
    };
    CK(set_opts(cg_rtol, cg_max_iter, cg_norm));
    irls_step_report sr;
    int64_t total = 0;
    Ranks R{c};
    irls_status s = run_solves(R, ASM_LAMBDA2, ASM_LAMBDA2, 1, &sr, &total);
    const int64_t launches = c->launches;
    if (!s) {
        RedArgs ra;
        ra.part = c->part;
        ra.slots = c->slots_local;
        ra.ctrl = c->ctrl;
        ra.K = c->K;
        ra.g0 = 0;
        ra.g1 = 8;
        ra.n_fin = count_nonempty(ra.K, 0, 8);
        if (c->kind == 0) launch_l2_quad_stencil(stencil_args(c, true), n, c->x, ra, st);
        else launch_l2_quad_sell(sell_args_full(c), c->x, ra, st);
        s = last_launch(c, "lambda2 quadratic form");
    }
    double slots[2 * kGroups];
    memset(slots, 0, sizeof(slots));
    if (!s && n > 0) CK(memcpy_sync(c, slots, c->slots_local, sizeof(slots), cudaMemcpyDeviceToHost));
    if (!s && x_out && n > 0) CK(memcpy_sync(c, x_out, c->x, sizeof(double) * n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpyAsync(c->x, xs, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    CK(set_opts(c->opt.cg_rtol, c->opt.cg_max_iter, c->opt.cg_norm));
    CK(dfree(c, xs));
    CK(cudaStreamSynchronize(st));
    c->state = state0;
    c->last_cg_iters = iters0;
    if (s) return s;
    const double xLx = irls_combine_slots(slots) + 4.0 * c->c_st;
    const double C = 2.0 * (irls_combine_slots(slots + kGroups) + c->c_st);
    if (rep) {
        rep->lambda2 = xLx / (2.0 * C);
        rep->xLx = xLx;
        rep->C = C;
        rep->rel_res = sr.rel_res;
        rep->cg_iters = sr.cg_iters;
        rep->converged = sr.converged;
        rep->ms = sr.ms;
        rep->launches = (int32_t)(launches + 1);
    }
    return IRLS_OK;
}
