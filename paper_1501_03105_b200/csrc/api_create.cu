// api_create.cu — context creation: validation of the
// inputs (A6-A8), the stencil slab plan, the CSR preparation (duplicate
// merging, symmetry, terminal split, Prop. 1, SELL-64, id strips with ghost
// blocks and send lists) on host threads, device allocation and upload.
#include <mutex>
#include "api_internal.h"

// Device memory comes from the device's stream-ordered pool with an unbounded
// release threshold: a create / destroy cycle maps HBM once and then reuses
// it (sizes here are GBs; cudaMalloc / cudaFree would remap every time).
// One pinned int per context for the host loop's "done" readback, from a
// process-wide pinned page (a cudaMallocHost / cudaFreeHost pair per context
// costs milliseconds and cudaFreeHost synchronises the device).
static std::mutex g_pin_mu;
static int *g_pin_page = nullptr;
static std::vector<int> g_pin_free;
int *pinned_flag_get()
{
    std::lock_guard<std::mutex> lk(g_pin_mu);
    if (!g_pin_page) {
        constexpr int kSlots = 4096;
        if (cudaMallocHost(&g_pin_page, sizeof(int) * kSlots) != cudaSuccess) {
            g_pin_page = nullptr;
            return nullptr;
        }
        for (int i = kSlots - 1; i >= 0; i--) g_pin_free.push_back(i);
    }
    if (g_pin_free.empty()) {  // more live contexts than slots: a private pinned int
        int *p = nullptr;
        return cudaMallocHost(&p, sizeof(int)) == cudaSuccess ? p : nullptr;
    }
    const int i = g_pin_free.back();
    g_pin_free.pop_back();
    return g_pin_page + i;
}
void pinned_flag_put(int *p)
{
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_pin_mu);
    if (g_pin_page && p >= g_pin_page && p < g_pin_page + 4096) g_pin_free.push_back((int)(p - g_pin_page));
    else cudaFreeHost(p);
}

static void setup_pool(int device)
{
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
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
    c->p2p = c->multi && opt->p2p != 0;
    CK(cudaSetDevice(c->device));
    if (comm && comm->cuda_stream) {
        c->stream = (cudaStream_t)comm->cuda_stream;
    } else {
        CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
    }
    CK(cudaStreamCreateWithFlags(&c->side_stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->side_stream2, cudaStreamNonBlocking));
    c->h_done = pinned_flag_get();
    if (!c->h_done) return IRLS_ERR_OOM;
    setup_pool(c->device);
    small_cg_prepare();
    return IRLS_OK;
}

static irls_status alloc_solver(irls_ctx *c, int64_t ghost)
{
    const int64_t npad = (int64_t)c->nchunks * kChunk;
    const int64_t gpad = (ghost + 1) & ~(int64_t)1;  // keep the owned start 16-byte aligned
    // multi-process p2p: buffers that peers open through CUDA IPC come from
    // cudaMalloc (pool and caller-allocator memory cannot be exported)
    const bool ipc = c->p2p && !c->vg;
    auto raw = [&](int64_t count) -> double * {
        void *p = nullptr;
        if (cudaMalloc(&p, sizeof(double) * (size_t)std::max<int64_t>(count, 1)) != cudaSuccess) return nullptr;
        c->raw_allocs.push_back(p);
        return (double *)p;
    };
    double *last_base = nullptr;
    auto ghosted = [&](double *&ptr, bool export_) -> bool {
        double *b = export_ ? raw(npad + 2 * gpad) : dalloc<double>(c, npad + 2 * gpad);
        if (!b) return false;
        ptr = b + gpad;
        last_base = b;
        return true;
    };
    const bool ipc_z = ipc;  // z (and CG-CG's w on slabs) are stored into by the neighbours
    if (!ghosted(c->z, ipc_z)) return IRLS_ERR_OOM;
    if (ipc_z) c->z_base = last_base;
    if (!ghosted(c->x, false) || !ghosted(c->p0, false) || !ghosted(c->p1, false) || !ghosted(c->r, false) ||
        !ghosted(c->Dinv, false))
        return IRLS_ERR_OOM;
    c->cgcg = c->opt.cg_variant == IRLS_CG_CG;
    if (c->cgcg) {
        for (int b = 0; b < 2; b++) {
            if (!ghosted(c->cg_w[b], ipc_z && c->kind == 0)) return IRLS_ERR_OOM;
            if (ipc_z && c->kind == 0) c->w_base[b] = last_base;
        }
        if (!ghosted(c->cg_r2, false) || !ghosted(c->cg_s[0], false) || !ghosted(c->cg_s[1], false))
            return IRLS_ERR_OOM;
    }
    if (c->p2p) {
        const int64_t nb = 2 * kMaxQ * kGroups + 1;  // slots by parity + the arrival counter
        c->p2p_buf = ipc ? raw(nb) : dalloc<double>(c, nb);
        c->d_pslots = (double **)dalloc<double *>(c, c->world);
        c->d_pcnt = (unsigned long long **)dalloc<unsigned long long *>(c, c->world);
        if (!c->p2p_buf || !c->d_pslots || !c->d_pcnt) return IRLS_ERR_OOM;
        CK(cudaMemsetAsync(c->p2p_buf, 0, sizeof(double) * nb, c->stream));
        c->n_groups_all = count_nonempty(c->K, 0, kGroups);
    }
    c->D = dalloc<double>(c, npad);
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

// Every rank's p2p slot buffer / counter (and, on z-slabs, the neighbours'
// z ghost planes) as device pointers usable by this rank's kernels.
irls_status p2p_set_peers(irls_ctx *c, const std::vector<double *> &bufs)
{
    std::vector<unsigned long long *> cnt(bufs.size());
    for (size_t w = 0; w < bufs.size(); w++) cnt[w] = (unsigned long long *)(bufs[w] + 2 * kMaxQ * kGroups);
    CK(memcpy_sync(c, c->d_pslots, bufs.data(), sizeof(double *) * bufs.size(), cudaMemcpyHostToDevice));
    CK(memcpy_sync(c, c->d_pcnt, cnt.data(), sizeof(unsigned long long *) * cnt.size(), cudaMemcpyHostToDevice));
    return IRLS_OK;
}

// CSR strips with p2p: where entry i of this rank's send lists lands — rank q
// (the list's peer) at offset npad_own_q + recv_off_q[me] + (i - send_off[q])
// of q's z (its ghost block keeps each sender's values contiguous, in the
// order of the sender's list).
irls_status p2p_set_halo(irls_ctx *c, const std::vector<double *> &zpeers, const std::vector<int64_t> &peer_npad,
                         const std::vector<std::vector<int64_t>> &peer_recv_off)
{
    const int W = c->world;
    const int64_t ns = c->send_off[W];
    std::vector<int32_t> hp(std::max<int64_t>(ns, 1), 0);
    std::vector<int64_t> pos(std::max<int64_t>(ns, 1), 0);
    for (int q = 0; q < W; q++)
        for (int64_t i = c->send_off[q]; i < c->send_off[q + 1]; i++) {
            hp[i] = q;
            pos[i] = peer_npad[q] + peer_recv_off[q][c->rank] + (i - c->send_off[q]);
        }
    c->halo_peer_dev = dalloc<int32_t>(c, std::max<int64_t>(ns, 1));
    c->halo_pos_dev = dalloc<int64_t>(c, std::max<int64_t>(ns, 1));
    c->d_zpeers = (double **)dalloc<double *>(c, W);
    if (!c->halo_peer_dev || !c->halo_pos_dev || !c->d_zpeers) return fail(c, IRLS_ERR_OOM, "p2p halo");
    CK(memcpy_sync(c, c->halo_peer_dev, hp.data(), sizeof(int32_t) * hp.size(), cudaMemcpyHostToDevice));
    CK(memcpy_sync(c, c->halo_pos_dev, pos.data(), sizeof(int64_t) * pos.size(), cudaMemcpyHostToDevice));
    CK(memcpy_sync(c, c->d_zpeers, zpeers.data(), sizeof(double *) * W, cudaMemcpyHostToDevice));
    return IRLS_OK;
}

// One rank's exported buffers, exchanged with an NCCL all-gather at create.
struct PeerRec {
    cudaIpcMemHandle_t hbuf, hz, hw[2];
    int64_t zoff_recv_lo, zoff_recv_hi;  // ghost planes, in doubles from the allocation start (z and w alike)
    int64_t zoff_own, npad_own, recv_off[9];  // CSR strips: z's owned start and the ghost block layout
};

static irls_status p2p_exchange(irls_ctx *c)
{
    const int W = c->world;
    PeerRec mine;
    memset(&mine, 0, sizeof(mine));
    CK(cudaIpcGetMemHandle(&mine.hbuf, c->p2p_buf));
    CK(cudaIpcGetMemHandle(&mine.hz, c->z_base));
    mine.zoff_own = c->z - c->z_base;
    if (c->kind == 0) {
        mine.zoff_recv_lo = (c->z - c->z_base) + c->hplan.recv_lo;
        mine.zoff_recv_hi = (c->z - c->z_base) + c->hplan.recv_hi;
        if (c->cgcg)
            for (int b = 0; b < 2; b++) CK(cudaIpcGetMemHandle(&mine.hw[b], c->w_base[b]));
    } else {
        mine.npad_own = c->npad_own;
        for (int q = 0; q <= W && q < 9; q++) mine.recv_off[q] = c->recv_off[q];
    }
    std::vector<PeerRec> all(W);
    void *dev = nullptr;
    CK(cudaMalloc(&dev, sizeof(PeerRec) * W));
    char *slot = (char *)dev + sizeof(PeerRec) * c->rank;
    cudaError_t e = cudaMemcpyAsync(slot, &mine, sizeof(mine), cudaMemcpyHostToDevice, c->stream);
    ncclResult_t nr = e == cudaSuccess ? ncclAllGather(slot, dev, sizeof(PeerRec), ncclUint8, c->nccl, c->stream)
                                       : ncclSuccess;
    if (e == cudaSuccess && nr == ncclSuccess)
        e = cudaMemcpyAsync(all.data(), dev, sizeof(PeerRec) * W, cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    cudaFree(dev);
    if (nr != ncclSuccess) return fail(c, IRLS_ERR_NCCL, std::string("p2p exchange: ") + ncclGetErrorString(nr));
    CK(e);
    auto open = [&](const cudaIpcMemHandle_t &h, double **out) -> irls_status {
        void *p = nullptr;
        cudaError_t oe = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
        if (oe != cudaSuccess) return fail(c, IRLS_ERR_CUDA, std::string("p2p: cudaIpcOpenMemHandle: ") +
                                                                 cudaGetErrorString(oe));
        c->ipc_open.push_back(p);
        *out = (double *)p;
        return IRLS_OK;
    };
    std::vector<double *> bufs(W);
    irls_status s;
    for (int w = 0; w < W; w++) {
        if (w == c->rank) bufs[w] = c->p2p_buf;
        else if ((s = open(all[w].hbuf, &bufs[w]))) return s;
    }
    if (c->kind == 1) {  // every peer's z (its ghost block receives this rank's send lists)
        std::vector<double *> zp(W);
        std::vector<int64_t> npad(W);
        std::vector<std::vector<int64_t>> roff(W);
        for (int w = 0; w < W; w++) {
            double *b = c->z_base;
            if (w != c->rank && (s = open(all[w].hz, &b))) return s;
            zp[w] = b + all[w].zoff_own;
            npad[w] = all[w].npad_own;
            roff[w].assign(all[w].recv_off, all[w].recv_off + W + 1);
        }
        if ((s = p2p_set_halo(c, zp, npad, roff))) return s;
    }
    if (c->kind == 0) {
        double *b;
        if (c->hplan.peer_lo >= 0) {
            if ((s = open(all[c->hplan.peer_lo].hz, &b))) return s;
            c->zpeer_lo = b + all[c->hplan.peer_lo].zoff_recv_hi;
        }
        if (c->hplan.peer_hi >= 0) {
            if ((s = open(all[c->hplan.peer_hi].hz, &b))) return s;
            c->zpeer_hi = b + all[c->hplan.peer_hi].zoff_recv_lo;
        }
        for (int w = 0; w < 2 && c->cgcg; w++) {  // same ghosted layout as z
            if (c->hplan.peer_lo >= 0) {
                if ((s = open(all[c->hplan.peer_lo].hw[w], &b))) return s;
                c->wpeer_lo[w] = b + all[c->hplan.peer_lo].zoff_recv_hi;
            }
            if (c->hplan.peer_hi >= 0) {
                if ((s = open(all[c->hplan.peer_hi].hw[w], &b))) return s;
                c->wpeer_hi[w] = b + all[c->hplan.peer_hi].zoff_recv_lo;
            }
        }
    }
    return p2p_set_peers(c, bufs);
}

static irls_status init_nccl(irls_ctx *c, const irls_comm_desc *comm)
{
    if (!c->multi || c->vg) return IRLS_OK;
    ncclUniqueId id;
    memcpy(&id, comm->nccl_unique_id, sizeof(id));
    NK(ncclCommInitRank(&c->nccl, c->world, id, c->rank));
    if (c->p2p) return p2p_exchange(c);
    return IRLS_OK;
}

// Host BFS for Prop. 1 / A8 on a grid (used only when some n-link is zero).
bool grid_nonsingular(int32_t nx, int32_t ny, int32_t nz, const double *cx, const double *cy, const double *cz,
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

irls_status create_stencil_impl(irls_ctx **out, const irls_comm_desc *comm, int32_t nx, int32_t ny, int32_t nz,
                                       const double *cx, const double *cy, const double *cz, const double *cs,
                                       const double *ct, const irls_options *opt, irls_vgroup *vg);

extern "C" irls_status irls_mincut_create_stencil(irls_ctx **out, const irls_comm_desc *comm, int32_t nx, int32_t ny,
                                                  int32_t nz, const double *cx, const double *cy, const double *cz,
                                                  const double *cs, const double *ct, const irls_options *opt)
{
    return create_stencil_impl(out, comm, nx, ny, nz, cx, cy, cz, cs, ct, opt, nullptr);
}

irls_status create_stencil_impl(irls_ctx **out, const irls_comm_desc *comm, int32_t nx, int32_t ny, int32_t nz,
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
        if (!s) s = block_setup_stencil(c, cx, cy, cz);
        if (!s) s = init_nccl(c, comm);
    }
    if (s) {
        irls_mincut_destroy(c);
        return s;
    }
    *out = c;
    return IRLS_OK;
}

struct Ent {
    int32_t col;
    int64_t pos;
    double w;
};

static bool csr_strips(int64_t nr, int world, std::vector<int64_t> &lo);

// The halo of one id strip: the ghosts are the neighbours
// owned by other ranks, in ascending global id (hence grouped by owner);
// by the symmetry of G~ owned row u goes to rank q iff u has a neighbour
// owned by q, in ascending u — exactly the order of q's ghost block, so the
// lists need no communication.  aptr/aidx: the reduced adjacency (ascending).
static void csr_strip_halo(const int64_t *aptr, const int32_t *aidx, const std::vector<int64_t> &rank_lo, int rank,
                           std::vector<int32_t> &ghosts, std::vector<int64_t> &recv_off, std::vector<int64_t> &send_off,
                           std::vector<int32_t> &lsend)
{
    const int W = (int)rank_lo.size() - 1;
    const int64_t lo = rank_lo[rank], hi = rank_lo[rank + 1];
    auto owner = [&](int64_t v) {
        return (int)(std::upper_bound(rank_lo.begin(), rank_lo.end() - 1, v) - rank_lo.begin()) - 1;
    };
    ghosts.clear();
    for (int64_t r = lo; r < hi; r++)
        for (int64_t e = aptr[r]; e < aptr[r + 1]; e++)
            if (aidx[e] < lo || aidx[e] >= hi) ghosts.push_back(aidx[e]);
    std::sort(ghosts.begin(), ghosts.end());
    ghosts.erase(std::unique(ghosts.begin(), ghosts.end()), ghosts.end());
    recv_off.assign(W + 1, 0);
    for (int32_t v : ghosts) recv_off[owner(v) + 1]++;
    for (int q = 0; q < W; q++) recv_off[q + 1] += recv_off[q];
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
    send_off.assign(W + 1, 0);
    lsend.clear();
    for (int q = 0; q < W; q++) {
        send_off[q + 1] = send_off[q] + (int64_t)sendq[q].size();
        lsend.insert(lsend.end(), sendq[q].begin(), sendq[q].end());
    }
}

extern "C" irls_status irls_csr_halo_plan(int64_t nr, const int64_t *aptr, const int32_t *aidx, int32_t world,
                                          int32_t rank, int64_t *lo_hi, int64_t *recv_off, int64_t *send_off,
                                          int32_t *ghosts, int64_t ghosts_cap, int32_t *send_idx, int64_t send_cap)
{
    if (nr < 0 || !aptr || (!aidx && nr > 0 && aptr[nr] > 0) || world < 1 || rank < 0 || rank >= world || !lo_hi ||
        !recv_off || !send_off)
        return IRLS_ERR_INVALID_ARGUMENT;
    std::vector<int64_t> rank_lo;
    if (!csr_strips(nr, world, rank_lo)) return IRLS_ERR_INVALID_ARGUMENT;
    std::vector<int32_t> g, ls;
    std::vector<int64_t> ro, so;
    csr_strip_halo(aptr, aidx, rank_lo, rank, g, ro, so, ls);
    lo_hi[0] = rank_lo[rank];
    lo_hi[1] = rank_lo[rank + 1];
    for (int q = 0; q <= world; q++) {
        recv_off[q] = ro[q];
        send_off[q] = so[q];
    }
    if (ghosts && (int64_t)g.size() <= ghosts_cap) std::copy(g.begin(), g.end(), ghosts);
    if (send_idx && (int64_t)ls.size() <= send_cap) std::copy(ls.begin(), ls.end(), send_idx);
    return IRLS_OK;
}

irls_status create_csr_impl(irls_ctx **out, const irls_comm_desc *comm, int64_t n, const int64_t *row_ptr,
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

// One-rank CSR create with the preparation on the GPU (csr_prep.cu): the
// caller's arrays are uploaded once and every step of the host path —
// validation, duplicate merge (A7), exact symmetry, terminal split, c_st (A5),
// F, Prop. 1 / A8, SELL-64 — runs in kernels with the host path's results.
// Error codes follow the host path's priority (first offending entry, then
// self loops, then symmetry, then singularity).
static irls_status create_csr_gpu(irls_ctx **out, const irls_comm_desc *comm, int64_t n, const int64_t *row_ptr,
                                  const int32_t *col, const double *w, int64_t s_, int64_t t_, const irls_options *opt)
{
    const int64_t nnz = row_ptr[n], nr = n - 2;
    irls_ctx *c = new irls_ctx();
    irls_status st = common_setup(c, comm, opt);
    std::vector<void *> tmp;
    cudaStream_t S = c->stream;
    auto talloc = [&](size_t bytes) -> void * {
        void *p = nullptr;
        if (cudaMallocAsync(&p, std::max<size_t>(bytes, 16), S) != cudaSuccess) return nullptr;
        tmp.push_back(p);
        return p;
    };
    auto finish = [&](irls_status r) -> irls_status {
        for (void *p : tmp) cudaFreeAsync(p, S);
        cudaStreamSynchronize(S);
        if (r) {
            irls_mincut_destroy(c);
            return r;
        }
        *out = c;
        return IRLS_OK;
    };
    if (st) return finish(st);
    if (c->multi) return finish(IRLS_ERR_INVALID_ARGUMENT);  // (the caller routes communicators to the host path)
    int64_t *d_rp = (int64_t *)talloc(8 * (size_t)(n + 1));
    int32_t *d_col = (int32_t *)talloc(4 * (size_t)nnz), *d_scol = (int32_t *)talloc(4 * (size_t)nnz);
    double *d_w = (double *)talloc(8 * (size_t)nnz), *d_sw = (double *)talloc(8 * (size_t)nnz);
    int32_t *d_mcnt = (int32_t *)talloc(4 * (size_t)(n + 1)), *d_mptr = (int32_t *)talloc(4 * (size_t)(n + 1));
    int64_t *d_scan = (int64_t *)talloc(8 * (size_t)((n + 1 + 4095) / 4096 + 2 + (nr + 1 + 4095) / 4096 +
                                                     (nr / kSell + 4096) / 4096 + 8));
    unsigned long long *d_u64 = (unsigned long long *)talloc(8 * 4);  // first_bad, cnt, cmax, wmax
    int32_t *d_flags = (int32_t *)talloc(4 * 4);                      // selfloop, asym, lonely
    double *d_cst = (double *)talloc(8);
    if (!d_rp || !d_col || !d_scol || !d_w || !d_sw || !d_mcnt || !d_mptr || !d_scan || !d_u64 || !d_flags || !d_cst)
        return finish(fail(c, IRLS_ERR_OOM, "csr preparation buffers"));
    CK(cudaMemcpyAsync(d_rp, row_ptr, 8 * (size_t)(n + 1), cudaMemcpyHostToDevice, S));
    CK(cudaMemcpyAsync(d_col, col, 4 * (size_t)nnz, cudaMemcpyHostToDevice, S));
    CK(cudaMemcpyAsync(d_w, w, 8 * (size_t)nnz, cudaMemcpyHostToDevice, S));
    CK(cudaMemsetAsync(d_u64, 0, 8 * 4, S));
    CK(cudaMemsetAsync(d_u64, 0xff, 8, S));  // first_bad = none
    CK(cudaMemsetAsync(d_flags, 0, 4 * 4, S));
    csrp_check(d_rp, d_col, d_w, n, d_u64, d_flags, S);
    unsigned long long h_u64[4];
    int32_t h_flags[4];
    CK(cudaMemcpyAsync(h_u64, d_u64, sizeof(h_u64), cudaMemcpyDeviceToHost, S));
    CK(cudaMemcpyAsync(h_flags, d_flags, sizeof(h_flags), cudaMemcpyDeviceToHost, S));
    CK(cudaStreamSynchronize(S));
    if (h_u64[0] != ~0ull) {
        const int64_t e = (int64_t)h_u64[0];
        return finish(col[e] < 0 || col[e] >= n ? IRLS_ERR_INVALID_ARGUMENT : IRLS_ERR_BAD_CAPACITY);
    }
    if (h_flags[0]) return finish(IRLS_ERR_INVALID_ARGUMENT);
    // merge duplicates (A7) -> merged CSR (mptr, mcol = d_col, mw = d_w reused)
    int launches = 0;
    csrp_merge(d_rp, d_col, d_w, n, d_scol, d_sw, d_mcnt, S);
    CK(cudaMemsetAsync(d_mcnt + n, 0, 4, S));
    exclusive_scan_i32(d_mcnt, n + 1, d_mptr, d_scan, S, &launches);
    csrp_compact(d_rp, d_scol, d_sw, d_mptr, n, d_col, d_w, S);
    csrp_symmetry(d_mptr, d_col, d_w, n, d_flags + 1, S);
    CK(cudaMemcpyAsync(h_flags, d_flags, sizeof(h_flags), cudaMemcpyDeviceToHost, S));
    CK(cudaStreamSynchronize(S));
    if (h_flags[1]) return finish(IRLS_ERR_NOT_SYMMETRIC);
    // the context's sizes
    c->kind = 1;
    c->n_glob = nr;
    c->n_total = n;
    c->s_id = s_;
    c->t_id = t_;
    c->K = (int32_t)((nr + kChunk - 1) / kChunk);
    c->g0 = 0;
    c->g1 = kGroups;
    c->lo = 0;
    c->n_own = nr;
    c->chunk0 = 0;
    c->nchunks = (int32_t)((nr + kChunk - 1) / kChunk);
    c->n_fin = count_nonempty(c->K, 0, kGroups);
    c->npad_own = (int64_t)c->nchunks * kChunk;
    c->rank_lo = {0, nr};
    const int64_t gpad = (int64_t)c->K * kChunk;
    c->cs = dalloc<double>(c, gpad);
    c->ct = dalloc<double>(c, gpad);
    c->orig_dev = dalloc<int64_t>(c, std::max<int64_t>(nr, 1));
    int32_t *d_acnt = (int32_t *)talloc(4 * (size_t)(nr + 1)), *d_aptr = (int32_t *)talloc(4 * (size_t)(nr + 1));
    if (!c->cs || !c->ct || !c->orig_dev || !d_acnt || !d_aptr) return finish(fail(c, IRLS_ERR_OOM, "csr arrays"));
    csrp_reduce(d_mptr, d_col, d_w, nr, s_, t_, c->cs, c->ct, c->orig_dev, d_acnt, d_u64 + 1, d_u64 + 2, d_cst, S);
    CK(cudaMemsetAsync(d_acnt + nr, 0, 4, S));
    exclusive_scan_i32(d_acnt, nr + 1, d_aptr, d_scan, S, &launches);
    int32_t h_na = 0;
    double cst = 0.0;
    CK(cudaMemcpyAsync(&h_na, d_aptr + nr, 4, cudaMemcpyDeviceToHost, S));
    CK(cudaMemcpyAsync(&cst, d_cst, 8, cudaMemcpyDeviceToHost, S));
    CK(cudaMemcpyAsync(h_u64, d_u64, sizeof(h_u64), cudaMemcpyDeviceToHost, S));
    CK(cudaStreamSynchronize(S));
    int32_t *d_aidx = (int32_t *)talloc(4 * (size_t)std::max<int32_t>(h_na, 1));
    double *d_ac = (double *)talloc(8 * (size_t)std::max<int32_t>(h_na, 1));
    int32_t *d_par = (int32_t *)talloc(4 * (size_t)std::max<int64_t>(nr, 1));
    int32_t *d_root = (int32_t *)talloc(4 * (size_t)std::max<int64_t>(nr, 1));
    uint8_t *d_anc = (uint8_t *)talloc((size_t)std::max<int64_t>(nr, 1));
    if (!d_aidx || !d_ac || !d_par || !d_root || !d_anc) return finish(fail(c, IRLS_ERR_OOM, "csr arrays"));
    csrp_fill(d_mptr, d_col, d_w, c->orig_dev, d_aptr, nr, s_, t_, d_aidx, d_ac, S);
    if (nr > 0) csrp_components(d_aptr, d_aidx, c->cs, c->ct, nr, d_par, d_root, d_anc, d_flags + 2, S);
    c->comp_root.resize((size_t)std::max<int64_t>(nr, 1));
    if (nr > 0) CK(cudaMemcpyAsync(c->comp_root.data(), d_root, 4 * (size_t)nr, cudaMemcpyDeviceToHost, S));
    CK(cudaMemcpyAsync(h_flags, d_flags, sizeof(h_flags), cudaMemcpyDeviceToHost, S));
    CK(cudaStreamSynchronize(S));
    if (h_flags[2]) return finish(IRLS_ERR_SINGULAR);
    {
        double cmax;
        memcpy(&cmax, &h_u64[2], sizeof(double));
        cmax = std::max(cmax, cst);
        c->F = compute_F(cmax, (int64_t)h_u64[1] + (cst > 0.0 ? 1 : 0));
    }
    c->c_st = cst;
    c->n_links = h_na / 2;
    // SELL-64
    const int64_t nsl = (nr + kSell - 1) / kSell;
    int32_t *d_sw32 = (int32_t *)talloc(4 * (size_t)(nsl + 1)), *d_sp32 = (int32_t *)talloc(4 * (size_t)(nsl + 1));
    if (!d_sw32 || !d_sp32) return finish(fail(c, IRLS_ERR_OOM, "sell widths"));
    CK(cudaMemsetAsync(d_sw32, 0, 4 * (size_t)(nsl + 1), S));
    if (nsl > 0) csrp_sell_width(d_aptr, nr, d_sw32, d_u64 + 3, S);
    exclusive_scan_i32(d_sw32, nsl + 1, d_sp32, d_scan, S, &launches);
    int32_t nent32 = 0;
    CK(cudaMemcpyAsync(&nent32, d_sp32 + nsl, 4, cudaMemcpyDeviceToHost, S));
    CK(cudaMemcpyAsync(h_u64, d_u64, sizeof(h_u64), cudaMemcpyDeviceToHost, S));
    CK(cudaStreamSynchronize(S));
    const int64_t nent = nent32;
    c->n_entries = nent;
    c->sell_wmax = (int32_t)h_u64[3];
    st = alloc_solver(c, 0);
    if (st) return finish(st);
    c->slice_ptr = dalloc<int64_t>(c, nsl + 1);
    c->col = dalloc<int32_t>(c, nent);
    c->cap = dalloc<double>(c, nent);
    c->gsell = dalloc<double>(c, nent);
    if (!c->slice_ptr || !c->col || !c->cap || !c->gsell) return finish(fail(c, IRLS_ERR_OOM, "sell arrays"));
    csrp_i32_to_i64(d_sp32, nsl + 1, c->slice_ptr, S);
    CK(cudaMemsetAsync(c->col, 0xff, 4 * (size_t)std::max<int64_t>(nent, 1), S));  // padding: column -1
    CK(cudaMemsetAsync(c->cap, 0, 8 * (size_t)std::max<int64_t>(nent, 1), S));
    if (nr > 0) csrp_sell_fill(d_aptr, d_aidx, d_ac, c->slice_ptr, nr, c->col, c->cap, S);
    c->lslice_ptr = c->slice_ptr;
    c->lcol = c->col;
    c->lcap = c->cap;
    c->lg = c->gsell;
    c->lcs = c->cs;
    c->lct = c->ct;
    c->lwmax = c->sell_wmax;
    c->ln_entries = c->n_entries;
    st = last_launch(c, "csr preparation");
    if (!st) st = init_nccl(c, comm);
    return finish(st);
}

irls_status create_csr_impl(irls_ctx **out, const irls_comm_desc *comm, int64_t n, const int64_t *row_ptr,
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
    // one rank, no block preconditioner: the preparation runs on the GPU
    const bool gpu_prep = !vg && (!comm || (comm->world_size == 1 && !comm->nccl_unique_id)) &&
                          opt->block_size == 0 && nnz < ((int64_t)1 << 31) - 1 && !getenv("IRLS_HOST_CSR_PREP");
    if (gpu_prep) return create_csr_gpu(out, comm, n, row_ptr, col, w, s_, t_, opt);
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
    parallel_prefix(mptr.data(), n);
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
    // every entry is written by the parallel pass below (no serial zero fill)
    HostBuf<double> hcs(nr), hct(nr);
    HostBuf<int64_t> orig(nr);
    HostBuf<int64_t> aptr(nr + 1);
    aptr[0] = 0;
    double cst = 0.0;
    for (int64_t e = mptr[s_]; e < mptr[s_ + 1]; e++)
        if (mcol[e] == t_) cst = mw[e];
    parallel_for(nr, [&](int, int64_t a, int64_t b) {
        for (int64_t r = a; r < b; r++) {
            const int64_t u = orig_of(r);
            orig[r] = u;
            hcs[r] = 0.0;
            hct[r] = 0.0;
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
    parallel_prefix(aptr.data(), nr);
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
    {
        std::vector<int64_t> twmax(host_threads(nsl), 0);
        parallel_for(nsl, [&](int i, int64_t a, int64_t b) {
            for (int64_t sl = a; sl < b; sl++) {
                int64_t wmax = 0;
                for (int64_t r = sl * kSell; r < std::min<int64_t>(nr, sl * kSell + kSell); r++)
                    wmax = std::max(wmax, aptr[r + 1] - aptr[r]);
                sptr[sl + 1] = kSell * wmax;
                twmax[i] = std::max(twmax[i], wmax);
            }
        });
        parallel_prefix(sptr.data(), nsl);
        for (int64_t wm : twmax) sell_wmax = std::max(sell_wmax, wm);
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
        const int64_t lo = c->lo, hi = c->lo + c->n_own;
        std::vector<int32_t> ghosts;
        csr_strip_halo(aptr.data(), aidx.data(), c->rank_lo, c->rank, ghosts, c->recv_off, c->send_off, lsend);
        c->n_ghost = (int64_t)ghosts.size();
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
                                       : c->npad_own + (std::lower_bound(ghosts.begin(), ghosts.end(), (int32_t)v) -
                                                        ghosts.begin());
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
            if (e != cudaSuccess)
                st = fail(c, IRLS_ERR_CUDA, std::string("csr strip upload: ") + cudaGetErrorString(e));
        }
    }
    if (!st) st = block_setup_csr(c, aptr.data(), aidx.data(), c->multi ? lsptr.data() : sptr.data());
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

