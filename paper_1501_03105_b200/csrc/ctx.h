// ctx.h — host-side context of one rank (internal).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <string>
#include <vector>

#include "../../include/irls_mincut.h"
#include "kernels.h"

struct irls_vgroup;

// Page-locked host array (fast D2H of the coarse graph); grows, never shrinks.
template <class T>
struct PinnedBuf {
    T *p = nullptr;
    size_t n = 0, cap = 0;
    PinnedBuf() = default;
    PinnedBuf(const PinnedBuf &) = delete;
    PinnedBuf &operator=(const PinnedBuf &) = delete;
    ~PinnedBuf()
    {
        if (p) cudaFreeHost(p);
    }
    bool resize(size_t m)
    {
        if (m > cap) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            cap = 0;
            const size_t c2 = m + m / 4 + 16;
            if (cudaMallocHost((void **)&p, c2 * sizeof(T)) != cudaSuccess) return false;
            cap = c2;
        }
        n = m;
        return true;
    }
    size_t size() const { return n; }
    T *data() { return p; }
    const T *data() const { return p; }
    T &operator[](size_t i) { return p[i]; }
    const T &operator[](size_t i) const { return p[i]; }
};

struct irls_ctx {
    // ---- configuration
    int kind = 0;  // 0 stencil, 1 csr
    irls_options opt{};
    int world = 1, rank = 0, device = 0;
    bool multi = false;  // the multi-rank (NCCL) code path: world > 1, or a 1-rank communicator (self-test)
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    irls_device_alloc_fn dev_alloc = nullptr;  // caller's allocator (irls_comm_desc), or the pool
    irls_device_free_fn dev_free = nullptr;
    void *alloc_user = nullptr;
    ncclComm_t nccl = nullptr;
    std::string err;
    bool poisoned = false;
    int state = 0;  // 0 created, 1 potentials valid

    // ---- sizes (reduced ids)
    int64_t n_glob = 0;  // n~
    int64_t n_own = 0, lo = 0;
    int32_t K = 0, chunk0 = 0, nchunks = 0;
    int32_t g0 = 0, g1 = 8, n_fin = 0;
    int64_t n_links = 0;

    // ---- stencil geometry
    int32_t nx = 0, ny = 0, nz = 0, z0 = 0, z1 = 0;
    int64_t P = 0;
    bool lo_ghost = false, hi_ghost = false;

    // ---- csr bookkeeping
    int64_t n_total = 0, s_id = 0, t_id = 0;
    double c_st = 0.0;
    int64_t *orig_dev = nullptr;

    // ---- CSR multi-rank (id strips): the solve's local SELL (rows [lo, lo+n_own),
    // columns remapped: owned v -> v - lo, ghost -> npad_own + ghost index) and
    // the halo lists; aliases of the global arrays when the path is single-rank
    int64_t *lslice_ptr = nullptr;
    int32_t *lcol = nullptr;
    double *lcap = nullptr, *lg = nullptr, *lcs = nullptr, *lct = nullptr;
    int32_t lwmax = 0;
    int64_t ln_entries = 0;
    int64_t n_ghost = 0, npad_own = 0;       // ghost values at [npad_own, npad_own + n_ghost)
    std::vector<int64_t> send_off, recv_off;  // [world + 1]: per-peer ranges of send_idx / the ghost block
    int32_t *send_idx = nullptr;             // local ids packed for the peers (device)
    double *sendbuf = nullptr;
    std::vector<int64_t> rank_lo;            // [world + 1]: first reduced id owned by every rank
    std::vector<int32_t> comp_root;          // component (root id) of every non-terminal in G~ (host)

    // ---- block-Jacobi preconditioner (opt.block_size > 0, A32)
    irls::BlockArgs blk{};
    bool blk_on = false;  // this solve (mode) uses it: every IRLS solve; not lambda_2's (A30)

    // ---- sweep fixed point
    int32_t F = 0;

    // ---- device arrays
    std::vector<void *> allocs;
    double *x = nullptr, *z = nullptr, *p0 = nullptr, *p1 = nullptr;  // ghost arrays (offset)
    double *D = nullptr, *Dinv = nullptr, *r = nullptr, *q = nullptr;
    double *cx = nullptr, *cy = nullptr, *cz = nullptr, *cs = nullptr, *ct = nullptr;
    double *gx = nullptr, *gy = nullptr, *gz = nullptr;
    double *gs_diag = nullptr, *gt_diag = nullptr;
    int64_t *slice_ptr = nullptr;
    int32_t *col = nullptr;
    double *cap = nullptr, *gsell = nullptr;
    int64_t n_entries = 0;
    int32_t sell_wmax = 0;

    irls::DevCtrl *ctrl = nullptr;
    double *part = nullptr, *slots_local = nullptr, *slots_glob = nullptr;
    irls::DevReport *reports = nullptr;
    int max_reports = 0;
    int *h_done = nullptr;  // pinned

    // multi-GPU
    irls_halo hplan{};
    irls_vgroup *vg = nullptr;    // virtual group (one process drives every rank)
    double *x_full = nullptr;     // rank 0: gathered potentials
    void *msg_dev = nullptr;      // sweep result broadcast

    // Chronopoulos-Gear PCG (irls_options.cg_variant = IRLS_CG_CG)
    bool cgcg = false;
    double *cg_r2 = nullptr, *cg_w[2] = {nullptr, nullptr}, *cg_s[2] = {nullptr, nullptr};  // ghosted

    // peer-memory collectives (irls_options.p2p on a multi-rank context)
    bool p2p = false;
    double *p2p_buf = nullptr;    // [2][kMaxQ][8] slot sums by parity, then one u64 arrival counter
    double **d_pslots = nullptr;  // device [world]: every rank's p2p_buf
    unsigned long long **d_pcnt = nullptr;  // device [world]: every rank's arrival counter
    int32_t n_groups_all = 0;     // non-empty C3 groups over all ranks (arrivals per reduction)
    double *zpeer_lo = nullptr, *zpeer_hi = nullptr;  // neighbours' z ghost planes (z-slabs)
    double *wpeer_lo[2] = {nullptr, nullptr}, *wpeer_hi[2] = {nullptr, nullptr};  // CG-CG: neighbours' w ghost planes
    double *w_base[2] = {nullptr, nullptr};  // CG-CG w allocations (IPC export)
    double *z_base = nullptr;     // start of z's allocation (IPC export)
    // CSR strips with p2p: the z halo as peer stores (entry i of the send
    // lists goes to rank halo_peer[i] at offset halo_pos[i] of its z array)
    int32_t *halo_peer_dev = nullptr;
    int64_t *halo_pos_dev = nullptr;
    double **d_zpeers = nullptr;  // device [world]: every rank's z (owned start)
    std::vector<void *> raw_allocs;  // cudaMalloc'd, IPC-exportable (multi-process p2p)
    std::vector<void *> ipc_open;    // peers' allocations opened with cudaIpcOpenMemHandle

    // sweep
    irls::SweepBuffers sb{};
    int32_t *order_dev = nullptr;  // points into sb.vals / vals_alt after a sweep
    int32_t *order_out = nullptr;
    bool sweep_valid = false;
    int64_t sweep_k = 0;
    double sweep_cut = 0.0;
    int64_t sweep_sorted = 0;  // nodes the last sweep radix-sorted
    int32_t bb_skip = 0;       // sweeps left that skip the branch-and-bound attempt

    // two-level rounding (rank 0)
    irls::TLBuffers tl{};
    bool tl_valid = false;
    PinnedBuf<int32_t> h_cp, h_ccol;
    PinnedBuf<double> h_ccap;
    PinnedBuf<__int128> h_cqs, h_cqt;
    __int128 h_qst = 0;

    // ---- graphs
    cudaGraphExec_t gexec[4] = {nullptr, nullptr, nullptr, nullptr};  // by assemble mode
    cudaGraphExec_t gmulti[4] = {nullptr, nullptr, nullptr, nullptr};  // T reweight steps in one graph, by mode
    int64_t gm_fixed[4] = {0, 0, 0, 0};  // kernels per step of the multi-step graph (outside the CG body)
    cudaStream_t side_stream = nullptr, side_stream2 = nullptr;

    // ---- stats
    int64_t launches = 0, last_cg_iters = 0;
    int64_t gl_fixed[4] = {0, 0, 0, 0};  // kernels per solve graph outside the WHILE body
    int64_t gl_body = 0;              // kernels per CG iteration (WHILE body)
    bool graph_iters_pending = false;
};

// W ranks of one grid driven by one host thread on one device and one stream;
// the collectives are device copies (testing the multi-GPU data path).
struct irls_vgroup {
    std::vector<irls_ctx *> ranks;
    cudaStream_t stream = nullptr;
    double **src_slots = nullptr;  // device array of every rank's slots_local
    irls::DevCtrl **src_ctrl = nullptr;  // device array of every rank's control block
};
