// api_round.cu — rounding of x^(T): the GPU sweep cut, the
// two-level rounding with the host max-flow, the exact min cut
// (mu* for delta, Eq. 13), and the Cheeger-type lambda_2.
#include <chrono>

#include "api_internal.h"

// ---------------------------------------------------------------------------
// sweep cut
// ---------------------------------------------------------------------------
// Sweep buffers in two parts: what every sweep needs (flags, k, the k-th node,
// side[], the radix look-back words the candidates' sort reuses), and the
// n-sized arrays of the full sort (keys, ids, delta, order, tile scans), which
// the branch-and-bound sweep does not touch (3.2 GB on config 4).
static irls_status alloc_sweep_base(irls_ctx *c)
{
    SweepBuffers &b = c->sb;
    if (b.flags) return IRLS_OK;
    const int64_t n = c->n_glob, nt = sweep_ntiles(n);
    b.n = n;
    b.rank = nullptr;  // the sweep forms membership from x (two-level uses its own ranks)
    b.tile_hist = dalloc<int32_t>(c, 2 * 256 * nt);  // look-back words of radix tiles down to 2048 keys
    b.digit_hist = dalloc<unsigned long long>(c, 8 * 256);
    b.flags = dalloc<int32_t>(c, 4);
    b.k_out = dalloc<int64_t>(c, 1);
    b.lastv = dalloc<int32_t>(c, 1);
    b.side = dalloc<uint8_t>(c, c->n_total);
    if (!b.tile_hist || !b.digit_hist || !b.flags || !b.k_out || !b.lastv || !b.side)
        return fail(c, IRLS_ERR_OOM, "sweep buffers");
    return IRLS_OK;
}

static irls_status alloc_sweep(irls_ctx *c)
{
    irls_status s = alloc_sweep_base(c);
    if (s) return s;
    if (c->sb.keys) return IRLS_OK;
    SweepBuffers &b = c->sb;
    const int64_t n = c->n_glob, nt = sweep_ntiles(n);
    b.keys = dalloc<unsigned long long>(c, n);
    b.keys_alt = dalloc<unsigned long long>(c, n);
    b.vals = dalloc<int32_t>(c, n);
    b.vals_alt = dalloc<int32_t>(c, n);
    b.tile_off = dalloc<int32_t>(c, 256 * nt);
    b.scan_tmp = (int32_t *)dalloc<int64_t>(c, (256 * nt + 4095) / 4096 + 1);
    b.delta = dalloc<__int128>(c, n + 2);
    b.tile_sum = dalloc<__int128>(c, nt);
    b.tile_incl = dalloc<__int128>(c, nt);
    b.qcs_tile = dalloc<__int128>(c, nt);
    b.tile_min = dalloc<__int128>(c, nt);
    b.tile_argmin = dalloc<int64_t>(c, nt);
    c->order_out = dalloc<int32_t>(c, n);
    if (!b.keys || !b.keys_alt || !b.vals || !b.vals_alt || !b.tile_off || !b.scan_tmp || !b.delta || !b.tile_sum ||
        !b.tile_incl || !b.qcs_tile || !b.tile_min || !b.tile_argmin || !c->order_out)
        return fail(c, IRLS_ERR_OOM, "sweep buffers");
    return IRLS_OK;
}

// Rank 0 result of the sweep, broadcast so every rank returns the same values.
struct SweepResultMsg {
    int64_t status, k;
    double cut;
};

irls_status sweep_rank0(irls_ctx *c, const double *xfull, uint8_t *side, int32_t *order, int64_t *k,
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

// Branch-and-bound sweep (sweep_bb.cu) for callers that do not need the order:
// k and the k-th node (x*, v*) of the order, exactly as the full sort's scan
// finds them (k_out, lastv written on the device).  *done = false (nothing
// decided) when the bound prunes too little or a buffer is not available;
// the caller then runs the full sort.
static irls_status sweep_bb(irls_ctx *c, const double *xfull, int *launches, bool *done)
{
    *done = false;
    cudaStream_t st = c->stream;
    SweepBuffers &b = c->sb;
    const int64_t n = c->n_glob;
    const int32_t nb = 4096, ns = 16384;
    typedef unsigned long long u64;
    typedef __int128 i128;
    const int G = bb_num_ctas();
    std::vector<void *> tmp;
    auto talloc = [&](size_t bytes) -> void * {
        void *p = nullptr;
        if (cudaMallocAsync(&p, std::max<size_t>(bytes, 16), st) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        tmp.push_back(p);
        return p;
    };
    struct Free {
        std::vector<void *> *t;
        cudaStream_t s;
        ~Free() { for (void *p : *t) cudaFreeAsync(p, s); }
    } fr{&tmp, st};
    u64 *skey = (u64 *)talloc(8 * 2 * ns), *spk = (u64 *)talloc(8 * nb);
    int32_t *sid = (int32_t *)talloc(4 * (2 * ns + (size_t)ns * (ns / 1024))), *spi = (int32_t *)talloc(4 * nb);
    u64 *part = (u64 *)talloc(8 * 4 * (size_t)G * nb);
    void *table = talloc(bb_table_bytes());
    uint16_t *bkt = (uint16_t *)talloc(2 * (size_t)n + 16);
    i128 *pqcs = (i128 *)talloc(16 * (size_t)G);
    unsigned *cnt = (unsigned *)talloc(4 * nb);
    i128 *bsum = (i128 *)talloc(16 * nb), *bneg = (i128 *)talloc(16 * nb), *p0 = (i128 *)talloc(16);
    int16_t *slot_of = (int16_t *)talloc(2 * nb);
    if (!skey || !spk || !sid || !spi || !part || !table || !bkt || !pqcs || !cnt || !bsum || !bneg || !p0 || !slot_of)
        return IRLS_OK;
    // buckets, then one pass: counts, exact sums, negative bounds, P_0, NaN flag
    bb_sample_sort(xfull, n, ns, nb, skey, sid, spk, spi, table, st);
    if (c->kind == 0)
        bb_pass_stencil(stencil_args(c, true), n, c->F, xfull, spk, spi, table, nb, part, pqcs, b.flags, bkt, st);
    else bb_pass_sell(sell_args_full(c), c->F, xfull, spk, spi, table, nb, part, pqcs, b.flags, bkt, st);
    bb_reduce(part, pqcs, nb, qfix_host(c->c_st, c->F), cnt, bsum, bneg, p0, st);
    *launches += 7;  // sample, rank, rank scatter, splitters, table, pass, reduce
    std::vector<unsigned> hc(nb);
    std::vector<i128> hsum(nb), hneg(nb);
    i128 hp0 = 0;
    int32_t hflag = 0;
    CK(cudaMemcpyAsync(hc.data(), cnt, 4 * nb, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hsum.data(), bsum, 16 * nb, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hneg.data(), bneg, 16 * nb, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&hp0, p0, 16, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&hflag, b.flags, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (hflag) return fail(c, IRLS_ERR_BAD_POTENTIAL, "NaN in potentials");
    std::vector<int64_t> hs(nb + 1, 0);
    for (int i = 0; i < nb; i++) hs[i + 1] = hs[i] + hc[i];
    if (hs[nb] != n) return fail(c, IRLS_ERR_CUDA, "sweep buckets do not cover the nodes");
    // P at the bucket boundaries; the first minimum among them
    std::vector<i128> Pb(nb + 1);
    Pb[0] = hp0;
    for (int i = 0; i < nb; i++) Pb[i + 1] = Pb[i] + hsum[i];
    i128 best = Pb[0];
    int64_t barg = 0;
    int bi_best = 0;
    for (int i = 1; i <= nb; i++)
        if (Pb[i] < best) {  // equal values keep the earlier position
            best = Pb[i];
            barg = hs[i];
            bi_best = i;
        }
    // candidates: buckets whose lower bound reaches the best boundary value,
    // and the bucket holding position barg - 1 (for the k-th node)
    std::vector<int32_t> cand;
    int holder = -1;
    if (barg > 0)
        for (int i = bi_best - 1; i >= 0; i--)
            if (hc[i] > 0) {
                holder = i;
                break;
            }
    for (int i = 0; i < nb; i++)
        if ((hc[i] > 1 && Pb[i] + hneg[i] <= best) || i == holder) cand.push_back(i);
    const int32_t nc = (int32_t)cand.size();
    std::vector<int64_t> dst((size_t)nc + 1, 0), cpos(std::max(nc, 1));
    std::vector<u64> cur(std::max(nc, 1));
    std::vector<i128> cP(std::max(nc, 1));
    std::vector<int16_t> hslot(nb, -1);
    for (int j = 0; j < nc; j++) {
        dst[j + 1] = dst[j] + hc[cand[j]];
        cur[j] = (u64)dst[j];
        cpos[j] = hs[cand[j]];
        cP[j] = Pb[cand[j]];
        hslot[cand[j]] = (int16_t)j;
    }
    const int64_t C = dst[nc];
    // (IRLS_SWEEP_BB_MAX: a smaller limit on the candidates, for tests)
    const int64_t cmax = getenv("IRLS_SWEEP_BB_MAX") ? atoll(getenv("IRLS_SWEEP_BB_MAX")) : n / 4;
    if (C > cmax) {  // pruning failed: the full path, also for the next sweeps
        c->bb_skip = 8;
        return IRLS_OK;
    }
    const size_t Cs = (size_t)std::max<int64_t>(C, 1);
    u64 *ck = (u64 *)talloc(8 * Cs), *k1 = (u64 *)talloc(8 * Cs), *k2 = (u64 *)talloc(8 * Cs);
    u64 *cursor = (u64 *)talloc(8 * (size_t)std::max(nc, 1));
    int32_t *cid = (int32_t *)talloc(4 * Cs), *v1 = (int32_t *)talloc(4 * Cs), *v2 = (int32_t *)talloc(4 * Cs);
    i128 *cdel = (i128 *)talloc(16 * Cs);
    u64 *dh = (u64 *)talloc(2 * 8 * 8 * 256);
    int64_t *ddst = (int64_t *)talloc(8 * ((size_t)nc + 1)), *dpos = (int64_t *)talloc(8 * (size_t)std::max(nc, 1));
    i128 *dP = (i128 *)talloc(16 * (size_t)std::max(nc, 1)), *cmin = (i128 *)talloc(16 * (size_t)std::max(nc, 1));
    int64_t *carg = (int64_t *)talloc(8 * (size_t)std::max(nc, 1));
    if (!ck || !k1 || !k2 || !cursor || !cid || !v1 || !v2 || !cdel || !dh || !ddst || !dpos || !dP || !cmin || !carg)
        return IRLS_OK;
    CK(cudaMemcpyAsync(slot_of, hslot.data(), 2 * nb, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(cursor, cur.data(), 8 * (size_t)std::max(nc, 1), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(ddst, dst.data(), 8 * ((size_t)nc + 1), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dpos, cpos.data(), 8 * (size_t)std::max(nc, 1), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dP, cP.data(), 16 * (size_t)std::max(nc, 1), cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(dh, 0, 2 * 8 * 8 * 256, st));
    CK(cudaMemsetAsync(b.flags + 2, 0, sizeof(int32_t), st));
    int32_t *sorted = v1;
    if (nc > 0) {
        bb_extract(n, xfull, bkt, nb, slot_of, cursor, ck, cid, k1, v1, dh, st);
        // the radix sort of sweep.cu is stable on the key alone; ties must
        // leave in ascending id, so: (A) sort positions by id, (B) gather
        // the keys in that order and sort them (values: compact positions)
        SweepBuffers tb = b;
        tb.n = C;
        tb.keys = k1;
        tb.keys_alt = k2;
        tb.vals = v1;
        tb.vals_alt = v2;
        tb.digit_hist = dh;
        bool nan = false;
        const int32_t *perm = sweep_sort(tb, st, launches, &nan);
        if (c->kind == 0) bb_cdelta_stencil(stencil_args(c, true), c->F, xfull, cid, perm, C, cdel, st);
        else bb_cdelta_sell(sell_args_full(c), c->F, xfull, cid, perm, C, cdel, st);
        int32_t *pin = perm == v1 ? v2 : v1;  // the other value buffer; k1, k2 are free
        int32_t *spare = perm == v1 ? v1 : v2;
        bb_gather(ck, perm, C, k1, pin, dh + 8 * 256, st);
        tb.keys = k1;
        tb.keys_alt = k2;
        tb.vals = pin;
        tb.vals_alt = spare;
        tb.digit_hist = dh + 8 * 256;
        sorted = sweep_sort(tb, st, launches, &nan);
        bb_cand_scan(cdel, sorted, ddst, dpos, dP, nc, cmin, carg, st);
        *launches += 4;  // extract, deltas, gather, candidate scan
    }
    bb_finish(cmin, carg, nc, best, barg, ddst, dpos, sorted, cid, b.k_out, b.lastv, b.flags, st);
    *launches += 1;
    c->sweep_sorted = C;
    *done = true;
    return IRLS_OK;
}

irls_status sweep_rank0(irls_ctx *c, const double *xfull, uint8_t *side, int32_t *order, int64_t *k,
                               double *cut_value)
{
    cudaStream_t st = c->stream;
    const int64_t n = c->n_glob;
    irls_status s = alloc_sweep_base(c);
    if (s) return s;
    int launches = 0;
    c->launches = 0;
    SweepBuffers &b = c->sb;
    CK(cudaMemsetAsync(b.flags, 0, sizeof(int32_t) * 4, st));
    // without an order to return, large graphs take the branch-and-bound sweep
    bool bb_done = false;
    int32_t *ord = nullptr;
    c->sweep_sorted = 0;
    // (after a sweep whose bound pruned too little, the next 8 sweeps of this
    // context go straight to the full sort: the potentials of consecutive
    // solves are alike)
    const bool try_bb = !order && n >= (1 << 20) && !getenv("IRLS_SWEEP_FULL") && c->bb_skip == 0;
    if (!order && c->bb_skip > 0) c->bb_skip--;
    if (try_bb) {
        s = sweep_bb(c, xfull, &launches, &bb_done);
        if (s) return s;
    }
    if (!bb_done) {
        s = alloc_sweep(c);
        if (s) return s;
        CK(cudaMemsetAsync(b.flags, 0, sizeof(int32_t) * 4, st));
        CK(cudaMemsetAsync(b.digit_hist, 0, sizeof(unsigned long long) * 8 * 256, st));
        if (c->kind == 0) sweep_prep_stencil(stencil_args(c, true), n, c->F, xfull, b, st);
        else sweep_prep_sell(sell_args_full(c), c->F, xfull, b, st);
        launches++;
        bool nan = false;
        ord = sweep_sort(b, st, &launches, &nan);
        if (nan) return fail(c, IRLS_ERR_BAD_POTENTIAL, "NaN in potentials");
        sweep_scan_argmin(b, ord, qfix_host(c->c_st, c->F), st);
        launches += 3;
        c->sweep_sorted = n;
    }
    RedArgs ra;
    ra.part = c->part;
    ra.slots = c->slots_local;
    ra.ctrl = c->ctrl;
    ra.K = (int32_t)((n + kChunk - 1) / kChunk);
    ra.g0 = 0;
    ra.g1 = 8;
    ra.n_fin = count_nonempty(ra.K, 0, 8);
    if (c->kind == 0) {
        if (n > 0) sweep_side_cross_x_stencil(stencil_args(c, true), n, xfull, ord, b, ra, st);
        else {
            const uint8_t sd[2] = {1, 0};
            CK(cudaMemcpyAsync(b.side, sd, 2, cudaMemcpyHostToDevice, st));
        }
    } else {
        CK(cudaMemsetAsync(b.side, 0, c->n_total, st));
        sweep_side_cross_x_sell(sell_args_full(c), xfull, ord, c->orig_dev, b, ra, st);
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
    int32_t hf2 = 0;
    if (bb_done) CK(cudaMemcpyAsync(&hf2, b.flags + 2, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    if (order && n > 0) {
        sweep_order_out(ord, c->kind == 1 ? c->orig_dev : nullptr, c->order_out, n, st);
        launches++;
        CK(cudaMemcpyAsync(order, c->order_out, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
    }
    if (side) CK(cudaMemcpyAsync(side, b.side, c->n_total, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (hf2) return fail(c, IRLS_ERR_CUDA, "branch-and-bound sweep: the k-th node is in no candidate");
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
// Two-level rounding (include/irls_mincut.h, DESIGN.md §2 A25-A29)
// ---------------------------------------------------------------------------

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
irls_status two_level_rank0(irls_ctx *c, const double *xfull, uint8_t *side, irls_two_level_report *r,
                                   bool exact)
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
    if (!exact && !(r->gamma0 < r->gamma1)) {  // A26': crossing thresholds -> (c0, c1)
        r->gamma0 = h.c0;
        r->gamma1 = h.c1;
    }
    if (!exact && !(r->gamma0 < r->gamma1)) {
        // A26': still degenerate (c0 >= c1): the sweep cut of x
        int64_t k = 0;
        double cut = 0.0;
        s = sweep_rank0(c, xfull, side, nullptr, &k, &cut);
        if (s) return s;
        r->cut_value = cut;
        r->certified = 1;
        r->ms_total = (float)std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
        return IRLS_OK;
    }
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

// Two-level rounding (or, exact = true, the no-contraction mu*) on rank 0
// over the gathered x, its report broadcast to every rank.
static irls_status two_level_collective(irls_ctx *c, uint8_t *side, irls_two_level_report *rep, bool exact)
{
    double *xfull = nullptr;
    irls_status s = gather_x(c, &xfull);  // exact: only the length matters (every node is in Sc)
    if (s) return s;
    TwoLevelMsg msg;
    memset(&msg, 0, sizeof(msg));
    if (c->rank == 0) {
        s = two_level_rank0(c, xfull, side, &msg.rep, exact);
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

extern "C" irls_status irls_two_level_cut(irls_ctx *c, uint8_t *side, irls_two_level_report *rep)
{
    NvtxRange nvtx_("irls_two_level_cut");
    GUARD(c);
    if (c->state == 0) return fail(c, IRLS_ERR_STATE, "two-level rounding before solve");
    return two_level_collective(c, side, rep, false);
}

extern "C" irls_status irls_exact_min_cut(irls_ctx *c, uint8_t *side, irls_two_level_report *rep)
{
    NvtxRange nvtx_("irls_exact_min_cut");
    GUARD(c);
    if (!c->multi) {  // no solve needed: x only sizes the classification (every node is in Sc)
        irls_two_level_report r;
        irls_status s = two_level_rank0(c, c->x, side, &r, true);
        if (s) return s;
        if (rep) *rep = r;
        return IRLS_OK;
    }
    return two_level_collective(c, side, rep, true);
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
    if (!(cg_rtol >= 0.0) || cg_max_iter < 0 || (cg_norm != 0 && cg_norm != 1))
        return fail(c, IRLS_ERR_INVALID_ARGUMENT, "lambda2 CG options");
    cudaStream_t st = c->stream;
    const int64_t n = c->n_own;
    if (c->n_glob == 0) {  // only s and t: x = (1, -1), x^T L x = 4 c_st, C = 2 c_st
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
    if (n > 0) CK(cudaMemcpyAsync(xs, c->x, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
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
    // the quadratic form on rank 0 over the gathered v (P:L303's gather, as
    // the sweep; every rank holds the full capacities), broadcast to all
    double *full = c->x;
    if (!s && c->multi) s = gather_x(c, &full);
    const int64_t ng = c->n_glob;
    double msg[2 * kGroups + 1];  // status, then the two quantities' 8 group sums
    memset(msg, 0, sizeof(msg));
    if (!s && c->rank == 0) {
        RedArgs ra;
        ra.part = c->part;
        ra.slots = c->slots_local;
        ra.ctrl = c->ctrl;
        ra.K = (int32_t)((ng + kChunk - 1) / kChunk);
        ra.g0 = 0;
        ra.g1 = 8;
        ra.n_fin = count_nonempty(ra.K, 0, 8);
        if (c->kind == 0) launch_l2_quad_stencil(stencil_args(c, true), ng, full, ra, st);
        else launch_l2_quad_sell(sell_args_full(c), full, ra, st);
        s = last_launch(c, "lambda2 quadratic form");
        if (!s) CK(memcpy_sync(c, msg + 1, c->slots_local, sizeof(double) * 2 * kGroups, cudaMemcpyDeviceToHost));
        if (!s && x_out) CK(memcpy_sync(c, x_out, full, sizeof(double) * ng, cudaMemcpyDeviceToHost));
    }
    if (c->multi) {  // every rank returns rank 0's values (and its status)
        msg[0] = (double)s;
        double *dmsg = dalloc<double>(c, 2 * kGroups + 1);
        if (!dmsg) return fail(c, IRLS_ERR_OOM, "lambda2 msg");
        if (c->rank == 0) CK(cudaMemcpyAsync(dmsg, msg, sizeof(msg), cudaMemcpyHostToDevice, st));
        NK(ncclBroadcast(dmsg, dmsg, sizeof(msg), ncclUint8, 0, c->nccl, st));
        CK(cudaMemcpyAsync(msg, dmsg, sizeof(msg), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        CK(dfree(c, dmsg));
        if (!s && msg[0] != 0.0) s = fail(c, (irls_status)(int)msg[0], "lambda2 failed on rank 0");
    }
    double *slots = msg + 1;
    if (n > 0) CK(cudaMemcpyAsync(c->x, xs, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
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

