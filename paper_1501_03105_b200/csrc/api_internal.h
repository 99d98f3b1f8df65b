// api_internal.h — shared internals of the C ABI implementation (api.cu,
// api_create.cu, api_round.cu): error plumbing, device memory, argument
// blocks, host thread helpers and the functions the three files share.
#pragma once

#include <math.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <string>
#include <thread>
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

// Records the error on the context (poisoning it unless it is a host-side
// validation error) and returns st.
irls_status fail(irls_ctx *c, irls_status st, const std::string &msg);

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
static inline cudaError_t memcpy_sync(irls_ctx *c, void *dst, const void *src, size_t n, cudaMemcpyKind k)
{
    cudaError_t e = cudaMemcpyAsync(dst, src, n, k, c->stream);
    if (e != cudaSuccess) return e;
    return cudaStreamSynchronize(c->stream);
}

static inline irls_status last_launch(irls_ctx *c, const char *what)
{
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(c, IRLS_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return IRLS_OK;
}


template <class T>
static inline T *dalloc(irls_ctx *c, int64_t count)
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
static inline cudaError_t dfree(irls_ctx *c, void *p)
{
    c->allocs.erase(std::remove(c->allocs.begin(), c->allocs.end(), p), c->allocs.end());
    if (c->dev_free) {
        c->dev_free(p, (void *)c->stream, c->alloc_user);
        return cudaSuccess;
    }
    return cudaFreeAsync(p, c->stream);
}

static inline int count_nonempty(int32_t K, int g0, int g1)
{
    int n = 0;
    for (int g = g0; g < g1; g++)
        if (group_lo(g + 1, K) > group_lo(g, K)) n++;
    return n;
}

static inline irls_status check_opts(const irls_options *o)
{
    if (!o) return IRLS_ERR_INVALID_ARGUMENT;
    if (!(o->eps > 0.0) || isinf(o->eps) || o->T < 0 || !(o->cg_rtol >= 0.0) || o->cg_max_iter < 0 ||
        (o->cg_norm != 0 && o->cg_norm != 1) || (o->loop_mode < 0 || o->loop_mode > 2) ||
        (o->fixed_point_exit != 0 && o->fixed_point_exit != 1) || (o->p2p != 0 && o->p2p != 1) ||
        (o->cg_variant != IRLS_CG_HS && o->cg_variant != IRLS_CG_CG) || o->block_size < 0 ||
        o->block_size > 256 ||
        (o->block_size > 0 && (o->cg_variant != IRLS_CG_HS || o->p2p || o->record_trace)))
        return IRLS_ERR_INVALID_ARGUMENT;
    return IRLS_OK;
}

// block-Jacobi preconditioner setup at create (api_block.cu; no-op unless
// opt.block_size > 0): host capacities of the grid / the reduced CSR
irls_status block_setup_stencil(irls_ctx *c, const double *cx, const double *cy, const double *cz);
irls_status block_setup_csr(irls_ctx *c, const int64_t *aptr, const int32_t *aidx, const int64_t *lsptr);

static inline int32_t compute_F(double cmax, int64_t cnt)
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
static inline VecArgs vec_args(const irls_ctx *c)
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

static inline StencilArgs stencil_args(const irls_ctx *c, bool full)
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
static inline SellArgs sell_args(const irls_ctx *c)
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
static inline SellArgs sell_args_full(const irls_ctx *c)
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

static inline RedArgs red_args(const irls_ctx *c)
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

static inline CgArgs cg_args(const irls_ctx *c)
{
    CgArgs g;
    g.r[0] = c->r;
    g.r[1] = c->cg_r2;
    g.w[0] = c->cg_w[0];
    g.w[1] = c->cg_w[1];
    g.s[0] = c->cg_s[0];
    g.s[1] = c->cg_s[1];
    g.p = c->p0;
    return g;
}

typedef std::vector<irls_ctx *> Ranks;

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
static inline int host_threads(int64_t n)
{
    if (n < 200000) return 1;
    const unsigned hc = std::thread::hardware_concurrency();
    return (int)std::min<unsigned>(std::max(1u, hc), 32u);
}

template <class F>
static inline void parallel_for(int64_t n, F f)
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

// p[i + 1] += p[i] for i = 0 .. n - 1 (counts in p[1..n] -> offsets), on the
// host threads: block sums, their serial scan, then each block adds its
// offset.  Integer sums: the result does not depend on the thread count.
static inline void parallel_prefix(int64_t *p, int64_t n)
{
    const int nt = host_threads(n);
    if (nt == 1) {
        for (int64_t i = 0; i < n; i++) p[i + 1] += p[i];
        return;
    }
    std::vector<int64_t> tot(nt, 0);
    parallel_for(n, [&](int t, int64_t a, int64_t b) {
        int64_t acc = 0;
        for (int64_t i = a; i < b; i++) acc += p[i + 1];
        tot[t] = acc;
    });
    std::vector<int64_t> off(nt, p[0]);
    for (int t = 1; t < nt; t++) off[t] = off[t - 1] + tot[t - 1];
    parallel_for(n, [&](int t, int64_t a, int64_t b) {
        int64_t run = off[t];
        for (int64_t i = a; i < b; i++) {
            run += p[i + 1];
            p[i + 1] = run;
        }
    });
}

// ---- shared between the files
// api.cu
irls_status gather_x(irls_ctx *c, double **full);
irls_status vgather_x(irls_vgroup *g, double **full);
irls_status run_solves(Ranks &R, int mode0, int mode_rest, int count, irls_step_report *reps, int64_t *total);
// api_create.cu
irls_status create_stencil_impl(irls_ctx **out, const irls_comm_desc *comm, int32_t nx, int32_t ny, int32_t nz,
                                const double *cx, const double *cy, const double *cz, const double *cs,
                                const double *ct, const irls_options *opt, irls_vgroup *vg);
irls_status create_csr_impl(irls_ctx **out, const irls_comm_desc *comm, int64_t n, const int64_t *row_ptr,
                            const int32_t *col, const double *w, int64_t s_, int64_t t_, const irls_options *opt,
                            irls_vgroup *vg);
bool grid_nonsingular(int32_t nx, int32_t ny, int32_t nz, const double *cx, const double *cy, const double *cz,
                      const double *cs, const double *ct);
// api_round.cu
irls_status sweep_rank0(irls_ctx *c, const double *xfull, uint8_t *side, int32_t *order, int64_t *k,
                        double *cut_value);
irls_status p2p_set_peers(irls_ctx *c, const std::vector<double *> &bufs);
int *pinned_flag_get();
void pinned_flag_put(int *p);
irls_status p2p_set_halo(irls_ctx *c, const std::vector<double *> &zpeers, const std::vector<int64_t> &peer_npad,
                         const std::vector<std::vector<int64_t>> &peer_recv_off);
irls_status two_level_rank0(irls_ctx *c, const double *xfull, uint8_t *side, irls_two_level_report *r,
                            bool exact = false);
