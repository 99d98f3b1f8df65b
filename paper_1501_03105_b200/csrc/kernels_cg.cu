// kernels_cg.cu — assembly, PCG and diagnostic kernels (stencil and SELL-32).
//
// One CTA of 256 threads owns one C3 chunk of 4096 consecutive node ids;
// thread t handles nodes base + 2t + 512j + e (j = 0..7, e = 0,1) in that
// order, so its running sums are exactly C3 step 2 and the block epilogue
// (common.cuh) completes steps 3-6.  Per-node arithmetic follows O1-O5 of
// DESIGN.md §2 operation for operation (no FMA: built with -fmad=false).
#include <algorithm>

#include "kernels.h"

namespace irls {

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------
struct Coord {
    int32_t x, y, z;
};

__device__ __forceinline__ Coord coord_of(const StencilArgs &s, int64_t ug)
{
    Coord c;
    const uint32_t u = (uint32_t)ug;
    const uint32_t t1 = fdiv(u, s.fd_nx);
    c.x = (int32_t)(u - t1 * (uint32_t)s.nx);
    const uint32_t zz = fdiv(t1, s.fd_ny);
    c.y = (int32_t)(t1 - zz * (uint32_t)s.ny);
    c.z = (int32_t)zz;
    return c;
}

__device__ __forceinline__ void set_cond(const CondArgs &cd, const DevCtrl *c)
{
    if (cd.use) cudaGraphSetConditional(cd.handle, c->done ? 0u : 1u);
}

#define FOR_CHUNK_NODES(...)                                                     \
    {                                                                             \
        const int64_t base__ = (int64_t)blockIdx.x * kChunk;                      \
        _Pragma("unroll 1") for (int j__ = 0; j__ < 8; j__++)                     \
        {                                                                         \
            _Pragma("unroll") for (int e__ = 0; e__ < 2; e__++)                   \
            {                                                                     \
                const int64_t u = base__ + 2 * (int64_t)threadIdx.x + 512 * j__ + e__; \
                if (u < v.n_own) { __VA_ARGS__ }                                         \
            }                                                                     \
        }                                                                         \
    }

// ---------------------------------------------------------------------------
// K1 / K2: reweight (Eq. 4) + assemble the reduced Laplacian (Eq. 7-8, O1),
// initial residual r0 = b - L~ x0, z0 = Dinv r0 and the START reductions.
// ---------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(kThreads) k_stencil_assemble(StencilArgs s, VecArgs v, RedArgs ra, CondArgs cd,
                                                               double eps2, double *gs_out, double *gt_out)
{
    if (v.frozen && *(const volatile int32_t *)v.frozen) return;  // fixed point: this step repeats the last one
    double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    const int64_t P = s.P;
    FOR_CHUNK_NODES({
        const Coord c = coord_of(s, s.lo + u);
        const bool hz = c.z > 0, hy = c.y > 0, hx = c.x > 0;
        const bool px = c.x < s.nx - 1, py = c.y < s.ny - 1, pz = c.z < s.nz - 1;
        double xu = 0.0, xmz = 0.0, xmy = 0.0, xmx = 0.0, xpx = 0.0, xpy = 0.0, xpz = 0.0;
        double gmz = 0.0, gmy = 0.0, gmx = 0.0, gpx = 0.0, gpy = 0.0, gpz = 0.0, gs, gt;
        if (MODE == ASM_INIT || MODE == ASM_LAMBDA2) {  // W^(0) = C: g = c
            if (hz) gmz = s.cz[u - P];
            if (hy) gmy = s.cy[u - s.nx];
            if (hx) gmx = s.cx[u - 1];
            if (px) gpx = s.cx[u];
            if (py) gpy = s.cy[u];
            if (pz) gpz = s.cz[u];
            gs = s.cs[u];
            gt = s.ct[u];
        } else {
            xu = v.x[u];
            if (hz) { xmz = v.x[u - P]; gmz = rw_g(s.cz[u - P], xmz - xu, eps2); }
            if (hy) { xmy = v.x[u - s.nx]; gmy = rw_g(s.cy[u - s.nx], xmy - xu, eps2); }
            if (hx) { xmx = v.x[u - 1]; gmx = rw_g(s.cx[u - 1], xmx - xu, eps2); }
            if (px) { xpx = v.x[u + 1]; gpx = rw_g(s.cx[u], xu - xpx, eps2); }
            if (py) { xpy = v.x[u + s.nx]; gpy = rw_g(s.cy[u], xu - xpy, eps2); }
            if (pz) { xpz = v.x[u + P]; gpz = rw_g(s.cz[u], xu - xpz, eps2); }
            gs = rw_g(s.cs[u], 1.0 - xu, eps2);  // A3: x_s = 1
            gt = rw_g(s.ct[u], xu, eps2);        // A3: x_t = 0
        }
        // O1: D = ((sum_asc g) + gs) + gt, ascending = (-z,-y,-x,+x,+y,+z)
        double a = 0.0;
        if (hz) a = a + gmz;
        if (hy) a = a + gmy;
        if (hx) a = a + gmx;
        if (px) a = a + gpx;
        if (py) a = a + gpy;
        if (pz) a = a + gpz;
        const double D = (a + gs) + gt;
        const double Dinv = 1.0 / D;
        s.gx[u] = gpx;
        s.gy[u] = gpy;
        s.gz[u] = gpz;
        if (s.lo_ghost && u < P) s.gz[u - P] = gmz;  // the -z edge of the first plane
        v.D[u] = D;
        v.Dinv[u] = Dinv;
        if (gs_out) { gs_out[u] = gs; gt_out[u] = gt; }
        double r;
        if (MODE == ASM_REWEIGHT_WARM) {  // r0 = b - L~ x^(l-1)  (O2 with p = x)
            double a2 = 0.0;
            if (hz) a2 = a2 + gmz * xmz;
            if (hy) a2 = a2 + gmy * xmy;
            if (hx) a2 = a2 + gmx * xmx;
            if (px) a2 = a2 + gpx * xpx;
            if (py) a2 = a2 + gpy * xpy;
            if (pz) a2 = a2 + gpz * xpz;
            r = gs - (D * xu - a2);
        } else {  // x0 = 0: r0 = b exactly
            r = MODE == ASM_LAMBDA2 ? gs - gt : gs;
        }
        const double zr = r * Dinv;
        v.r[u] = r;
        v.z[u] = zr;
        const double bu = MODE == ASM_LAMBDA2 ? gs - gt : gs;
        const double mb = bu * Dinv;
        acc[0] = acc[0] + r * zr;
        acc[1] = acc[1] + zr * zr;
        acc[2] = acc[2] + r * r;
        acc[3] = acc[3] + mb * mb;
        acc[4] = acc[4] + bu * bu;
    })
    if (c3_chunk_epilogue<5>(acc, v.chunk0 + (int32_t)blockIdx.x, ra) && cd.finalize && threadIdx.x == 0) {
        finalize_start(ra.ctrl, ra.slots);
        set_cond(cd, ra.ctrl);
    }
}

template <int MODE>
__global__ void __launch_bounds__(kThreads) k_sell_assemble(SellArgs s, VecArgs v, RedArgs ra, CondArgs cd,
                                                            double eps2, double *gs_out, double *gt_out)
{
    if (v.frozen && *(const volatile int32_t *)v.frozen) return;  // fixed point: this step repeats the last one
    double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    FOR_CHUNK_NODES({
        const int64_t sl = u / kSell;
        const int64_t e0 = s.slice_ptr[sl] + (u % kSell);
        const int32_t W = (int32_t)((s.slice_ptr[sl + 1] - s.slice_ptr[sl]) / kSell);
        const double xu = (MODE == ASM_INIT || MODE == ASM_LAMBDA2) ? 0.0 : v.x[u];
        double a = 0.0, a2 = 0.0;
        for (int32_t k = 0; k < W; k++) {
            const int64_t idx = e0 + kSell * (int64_t)k;
            const int32_t nb = s.col[idx];
            if (nb < 0) break;
            const double c = s.c[idx];
            double g;
            if (MODE == ASM_INIT || MODE == ASM_LAMBDA2) {
                g = c;
            } else {
                const double xv = v.x[nb];
                g = rw_g(c, xu - xv, eps2);
                if (MODE == ASM_REWEIGHT_WARM) a2 = a2 + g * xv;
            }
            s.g[idx] = g;
            a = a + g;
        }
        const double gs = (MODE == ASM_INIT || MODE == ASM_LAMBDA2) ? s.cs[u] : rw_g(s.cs[u], 1.0 - xu, eps2);
        const double gt = (MODE == ASM_INIT || MODE == ASM_LAMBDA2) ? s.ct[u] : rw_g(s.ct[u], xu, eps2);
        const double D = (a + gs) + gt;
        const double Dinv = 1.0 / D;
        v.D[u] = D;
        v.Dinv[u] = Dinv;
        if (gs_out) { gs_out[u] = gs; gt_out[u] = gt; }
        const double r = MODE == ASM_REWEIGHT_WARM ? gs - (D * xu - a2) : (MODE == ASM_LAMBDA2 ? gs - gt : gs);
        const double zr = r * Dinv;
        v.r[u] = r;
        v.z[u] = zr;
        const double bu = MODE == ASM_LAMBDA2 ? gs - gt : gs;
        const double mb = bu * Dinv;
        acc[0] = acc[0] + r * zr;
        acc[1] = acc[1] + zr * zr;
        acc[2] = acc[2] + r * r;
        acc[3] = acc[3] + mb * mb;
        acc[4] = acc[4] + bu * bu;
    })
    if (c3_chunk_epilogue<5>(acc, v.chunk0 + (int32_t)blockIdx.x, ra) && cd.finalize && threadIdx.x == 0) {
        finalize_start(ra.ctrl, ra.slots);
        set_cond(cd, ra.ctrl);
    }
}

// ---------------------------------------------------------------------------
// K3: p = z + beta p_old (p = z at k = 0, O9(i)), recomputed for the node and
// its neighbours (O9(ii)); lazy x += alpha_{k-1} p_{k-1}; q = L~ p (O2);
// PQ reduction.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_stencil_pspmv(StencilArgs s, VecArgs v, RedArgs ra, CondArgs cd,
                                                            bool w0)
{
    const DevCtrl *ctrl = ra.ctrl;
    if (w0 && ctrl->done) return;  // CG-CG's w0 pass after a START that stopped
    const int32_t k = ctrl->k;
    const bool first = (k == 0);
    const double beta = ctrl->beta, alpha = ctrl->alpha;
    const double *__restrict__ pold = (k & 1) ? v.p1 : v.p0;
    double *__restrict__ pnew = (k & 1) ? v.p0 : v.p1;
    const double *__restrict__ zv = v.z;
    const int64_t P = s.P;
    double acc[1] = {0.0};
#define PVAL(w) (first ? zv[w] : zv[w] + beta * pold[w])
    FOR_CHUNK_NODES({
        const Coord c = coord_of(s, s.lo + u);
        const double pu = PVAL(u);
        double a = 0.0;
        if (c.z > 0) a = a + s.gz[u - P] * PVAL(u - P);
        if (c.y > 0) a = a + s.gy[u - s.nx] * PVAL(u - s.nx);
        if (c.x > 0) a = a + s.gx[u - 1] * PVAL(u - 1);
        if (c.x < s.nx - 1) a = a + s.gx[u] * PVAL(u + 1);
        if (c.y < s.ny - 1) a = a + s.gy[u] * PVAL(u + s.nx);
        if (c.z < s.nz - 1) a = a + s.gz[u] * PVAL(u + P);
        const double qu = v.D[u] * pu - a;
        pnew[u] = pu;
        v.q[u] = qu;
        if (!first) v.x[u] = v.x[u] + alpha * pold[u];
        acc[0] = acc[0] + pu * qu;
    })
#undef PVAL
    if (c3_chunk_epilogue<1>(acc, v.chunk0 + (int32_t)blockIdx.x, ra) && cd.finalize && threadIdx.x == 0) {
        finalize_pq(ra.ctrl, ra.slots);
        if (w0) set_cond(cd, ra.ctrl);
    }
}

__global__ void __launch_bounds__(kThreads) k_sell_pspmv(SellArgs s, VecArgs v, RedArgs ra, CondArgs cd, bool w0)
{
    const DevCtrl *ctrl = ra.ctrl;
    if (w0 && ctrl->done) return;  // CG-CG's w0 pass after a START that stopped
    const int32_t k = ctrl->k;
    const bool first = (k == 0);
    const double beta = ctrl->beta, alpha = ctrl->alpha;
    const double *__restrict__ pold = (k & 1) ? v.p1 : v.p0;
    double *__restrict__ pnew = (k & 1) ? v.p0 : v.p1;
    const double *__restrict__ zv = v.z;
    double acc[1] = {0.0};
#define PVAL(w) (first ? zv[w] : zv[w] + beta * pold[w])
    FOR_CHUNK_NODES({
        const int64_t sl = u / kSell;
        const int64_t e0 = s.slice_ptr[sl] + (u % kSell);
        const int32_t W = (int32_t)((s.slice_ptr[sl + 1] - s.slice_ptr[sl]) / kSell);
        const double pu = PVAL(u);
        double a = 0.0;
        for (int32_t kk = 0; kk < W; kk++) {
            const int64_t idx = e0 + kSell * (int64_t)kk;
            const int32_t nb = s.col[idx];
            if (nb < 0) break;
            a = a + s.g[idx] * PVAL(nb);
        }
        const double qu = v.D[u] * pu - a;
        pnew[u] = pu;
        v.q[u] = qu;
        if (!first) v.x[u] = v.x[u] + alpha * pold[u];
        acc[0] = acc[0] + pu * qu;
    })
#undef PVAL
    if (c3_chunk_epilogue<1>(acc, v.chunk0 + (int32_t)blockIdx.x, ra) && cd.finalize && threadIdx.x == 0) {
        finalize_pq(ra.ctrl, ra.slots);
        if (w0) set_cond(cd, ra.ctrl);
    }
}

// Ghost planes of p (multi-GPU): the neighbour rank's boundary plane of p is
// maintained locally from the exchanged z with the same update.
__global__ void k_ghost_pupdate(VecArgs v, int64_t ghost_lo, int64_t ghost_hi, int64_t plane, const DevCtrl *ctrl)
{
    const int32_t k = ctrl->k;
    const bool first = (k == 0);
    const double beta = ctrl->beta;
    const double *pold = (k & 1) ? v.p1 : v.p0;
    double *pnew = (k & 1) ? v.p0 : v.p1;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nlo = ghost_lo ? plane : 0, nhi = ghost_hi ? plane : 0;
    if (i < nlo) {
        const int64_t w = i - plane;
        pnew[w] = first ? v.z[w] : v.z[w] + beta * pold[w];
    } else if (i < nlo + nhi) {
        const int64_t w = v.n_own + (i - nlo);
        pnew[w] = first ? v.z[w] : v.z[w] + beta * pold[w];
    }
}

// CSR strips: the ghost block [start, start + count) of p, same update.
__global__ void k_ghost_range_pupdate(VecArgs v, int64_t start, int64_t count, const DevCtrl *ctrl)
{
    const int32_t k = ctrl->k;
    const bool first = (k == 0);
    const double beta = ctrl->beta;
    const double *pold = (k & 1) ? v.p1 : v.p0;
    double *pnew = (k & 1) ? v.p0 : v.p1;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) {
        const int64_t w = start + i;
        pnew[w] = first ? v.z[w] : v.z[w] + beta * pold[w];
    }
}

__global__ void k_halo_pack(const double *arr, const int32_t *idx, int64_t n, double *out)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = arr[idx[i]];
}

void launch_ghost_range_pupdate(const VecArgs &v, int64_t start, int64_t count, DevCtrl *ctrl, cudaStream_t st)
{
    if (count <= 0) return;
    k_ghost_range_pupdate<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(v, start, count, ctrl);
}

void launch_halo_pack(const double *arr, const int32_t *idx, int64_t n, double *out, cudaStream_t st)
{
    if (n <= 0) return;
    k_halo_pack<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(arr, idx, n, out);
}

// ---------------------------------------------------------------------------
// K5: r = r - alpha q; z = r Dinv (Jacobi, A12); RZ reduction.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_axpy_jacobi(VecArgs v, RedArgs ra, CondArgs cd)
{
    DevCtrl *ctrl = ra.ctrl;
    if (ctrl->done) {  // breakdown flagged after q = A p
        if (blockIdx.x == 0 && threadIdx.x == 0) set_cond(cd, ctrl);
        return;
    }
    const double alpha = ctrl->alpha;
    double acc[3] = {0.0, 0.0, 0.0};
    FOR_CHUNK_NODES({
        const double r = v.r[u] - alpha * v.q[u];
        const double zr = r * v.Dinv[u];
        v.r[u] = r;
        v.z[u] = zr;
        acc[0] = acc[0] + r * zr;
        acc[1] = acc[1] + zr * zr;
        acc[2] = acc[2] + r * r;
    })
    if (c3_chunk_epilogue<3>(acc, v.chunk0 + (int32_t)blockIdx.x, ra) && cd.finalize && threadIdx.x == 0) {
        finalize_rz(ctrl, ra.slots);
        set_cond(cd, ctrl);
    }
}

// After the loop: the deferred x += alpha_{k-1} p_{k-1}; or v = 0 when b = 0.
__global__ void __launch_bounds__(kThreads) k_finish(VecArgs v, const DevCtrl *ctrl)
{
    const int32_t k = ctrl->k;
    const bool zero = ctrl->zero_x != 0;
    if (!zero && (k == 0 || ctrl->status != ST_OK)) return;
    const double alpha = ctrl->alpha;
    const double *pl = (k & 1) ? v.p1 : v.p0;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < v.n_own) v.x[i] = zero ? 0.0 : v.x[i] + alpha * pl[i];
}

__global__ void k_finalize(int phase, DevCtrl *ctrl, const double *slots, CondArgs cd, P2PWait pw)
{
    // phases whose producers did not run (as on one rank, where the skipped
    // kernel's fused finalize is skipped with it): a fixed-point step's
    // assembly, and K5 after a breakdown in the PQ phase
    if ((phase == PH_START && ctrl->frozen) || ((phase == PH_RZ || phase == PH_W0 || phase == PH_CG) && ctrl->done)) {
        set_cond(cd, ctrl);
        return;
    }
    if (pw.buf && !(slots = p2p_wait(ctrl, pw))) {
        set_cond(cd, ctrl);
        return;
    }
    if (phase == PH_START) finalize_start(ctrl, slots);
    else if (phase == PH_PQ || phase == PH_W0) finalize_pq(ctrl, slots);  // W0: alpha_0 = rho / <z, A z>
    else if (phase == PH_CG) finalize_cgcg(ctrl, slots);
    else finalize_rz(ctrl, slots);
    if (phase != PH_PQ) set_cond(cd, ctrl);
}

__global__ void k_report(DevCtrl *ctrl, DevReport *reports, int freeze)
{
    // A warm reweight step that stopped before its first CG iteration left x
    // unchanged (no update, b != 0): every later step of this solve reweights
    // from the same x and repeats it bit for bit, so they may be skipped.
    if (freeze && ctrl->k == 0 && ctrl->zero_x == 0 && ctrl->status == ST_OK) ctrl->frozen = 1;
    DevReport &R = reports[ctrl->step];
    const double ref = ctrl->ref;
    R.cg_iters = ctrl->k;
    R.status = ctrl->status;
    R.ref = ref;
    R.rel_res = ref > 0.0 ? ctrl->res / ref : 0.0;
    R.converged = ctrl->status == ST_OK && (ref == 0.0 || ctrl->res <= ctrl->rtol * ref);
    R.true_rel_res = R.S_eps = R.flow_value = R.current_s = 0.0;
    R.x_min = R.x_max = 0.0;
    R.t_end = global_ns();
    R.t_asm = ctrl->t_asm;
    ctrl->step = ctrl->step + 1;
    ctrl->xmin_key = ~0ull;
    ctrl->xmax_key = 0ull;
}

// ---------------------------------------------------------------------------
// record_trace diagnostics (O8): [S_eps, flow, current_s, ||res||^2] + range
// ---------------------------------------------------------------------------
__device__ __forceinline__ void range_update(DevCtrl *ctrl, double mn, double mx)
{
    // warp-aggregate then one atomic per warp
    unsigned long long kmin = dkey_asc(mn), kmax = dkey_asc(mx);
    for (int off = 16; off >= 1; off >>= 1) {
        unsigned long long o1 = __shfl_down_sync(0xffffffffu, kmin, off);
        unsigned long long o2 = __shfl_down_sync(0xffffffffu, kmax, off);
        kmin = o1 < kmin ? o1 : kmin;
        kmax = o2 > kmax ? o2 : kmax;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&ctrl->xmin_key, kmin);
        atomicMax(&ctrl->xmax_key, kmax);
    }
}

__global__ void __launch_bounds__(kThreads) k_stencil_diag(StencilArgs s, VecArgs v, RedArgs ra, double eps2,
                                                           int norm, const double *gsv, const double *gtv)
{
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    double mn = INFINITY, mx = -INFINITY;
    const int64_t P = s.P;
    FOR_CHUNK_NODES({
        const Coord c = coord_of(s, s.lo + u);
        const double xu = v.x[u];
        mn = fmin(mn, xu);
        mx = fmax(mx, xu);
        double Se = 0.0, fl = 0.0;
        // owned edges: +x, +y, +z (ascending), then s-link, t-link
        const bool px = c.x < s.nx - 1, py = c.y < s.ny - 1, pz = c.z < s.nz - 1;
        double xpx = 0.0, xpy = 0.0, xpz = 0.0;
        if (px) { xpx = v.x[u + 1]; const double cc = s.cx[u]; if (cc > 0.0) { const double a = cc * (xu - xpx); Se = Se + sqrt(a * a + eps2); const double d = xu - xpx; fl = fl + s.gx[u] * (d * d); } }
        if (py) { xpy = v.x[u + s.nx]; const double cc = s.cy[u]; if (cc > 0.0) { const double a = cc * (xu - xpy); Se = Se + sqrt(a * a + eps2); const double d = xu - xpy; fl = fl + s.gy[u] * (d * d); } }
        if (pz) { xpz = v.x[u + P]; const double cc = s.cz[u]; if (cc > 0.0) { const double a = cc * (xu - xpz); Se = Se + sqrt(a * a + eps2); const double d = xu - xpz; fl = fl + s.gz[u] * (d * d); } }
        if (s.cs[u] > 0.0) { const double a = s.cs[u] * (1.0 - xu); Se = Se + sqrt(a * a + eps2); }
        if (s.ct[u] > 0.0) { const double a = s.ct[u] * xu; Se = Se + sqrt(a * a + eps2); }
        const double ds = 1.0 - xu;
        fl = fl + gsv[u] * (ds * ds);
        fl = fl + gtv[u] * (xu * xu);
        // true residual b - L~ x
        double a2 = 0.0;
        if (c.z > 0) a2 = a2 + s.gz[u - P] * v.x[u - P];
        if (c.y > 0) a2 = a2 + s.gy[u - s.nx] * v.x[u - s.nx];
        if (c.x > 0) a2 = a2 + s.gx[u - 1] * v.x[u - 1];
        if (px) a2 = a2 + s.gx[u] * xpx;
        if (py) a2 = a2 + s.gy[u] * xpy;
        if (pz) a2 = a2 + s.gz[u] * xpz;
        const double rr = gsv[u] - (v.D[u] * xu - a2);
        const double tv = norm == 0 ? rr * v.Dinv[u] : rr;
        acc[0] = acc[0] + Se;
        acc[1] = acc[1] + fl;
        acc[2] = acc[2] + gsv[u] * (1.0 - xu);
        acc[3] = acc[3] + tv * tv;
    })
    range_update(ra.ctrl, mn, mx);
    c3_chunk_epilogue<4>(acc, v.chunk0 + (int32_t)blockIdx.x, ra);
}

__global__ void __launch_bounds__(kThreads) k_sell_diag(SellArgs s, VecArgs v, RedArgs ra, double eps2, int norm,
                                                        const double *gsv, const double *gtv)
{
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    double mn = INFINITY, mx = -INFINITY;
    FOR_CHUNK_NODES({
        const int64_t sl = u / kSell;
        const int64_t e0 = s.slice_ptr[sl] + (u % kSell);
        const int32_t W = (int32_t)((s.slice_ptr[sl + 1] - s.slice_ptr[sl]) / kSell);
        const double xu = v.x[u];
        mn = fmin(mn, xu);
        mx = fmax(mx, xu);
        double Se = 0.0, fl = 0.0, a2 = 0.0;
        for (int32_t k = 0; k < W; k++) {
            const int64_t idx = e0 + kSell * (int64_t)k;
            const int32_t nb = s.col[idx];
            if (nb < 0) break;
            const double xv = v.x[nb];
            a2 = a2 + s.g[idx] * xv;
            if (nb < s.gbase ? nb > u : nb - s.gbase >= s.glow) {  // owned edge: higher global id
                const double a = s.c[idx] * (xu - xv);
                Se = Se + sqrt(a * a + eps2);
                const double d = xu - xv;
                fl = fl + s.g[idx] * (d * d);
            }
        }
        if (s.cs[u] > 0.0) { const double a = s.cs[u] * (1.0 - xu); Se = Se + sqrt(a * a + eps2); }
        if (s.ct[u] > 0.0) { const double a = s.ct[u] * xu; Se = Se + sqrt(a * a + eps2); }
        const double ds = 1.0 - xu;
        fl = fl + gsv[u] * (ds * ds);
        fl = fl + gtv[u] * (xu * xu);
        const double rr = gsv[u] - (v.D[u] * xu - a2);
        const double tv = norm == 0 ? rr * v.Dinv[u] : rr;
        acc[0] = acc[0] + Se;
        acc[1] = acc[1] + fl;
        acc[2] = acc[2] + gsv[u] * (1.0 - xu);
        acc[3] = acc[3] + tv * tv;
    })
    range_update(ra.ctrl, mn, mx);
    c3_chunk_epilogue<4>(acc, v.chunk0 + (int32_t)blockIdx.x, ra);
}

__global__ void k_diag_finalize(DevCtrl *ctrl, const double *slots, DevReport *reports, int norm, P2PWait pw)
{
    DevReport &R = reports[ctrl->step - 1];
    if (pw.buf && !(slots = p2p_wait(ctrl, pw))) {
        R.status = ctrl->status;
        return;
    }
    R.S_eps = slot_total(slots, 0);
    R.flow_value = slot_total(slots, 1);
    R.current_s = slot_total(slots, 2);
    const double tr = sqrt(slot_total(slots, 3));
    R.true_rel_res = ctrl->ref > 0.0 ? tr / ctrl->ref : 0.0;
    R.x_min = dkey_inv(ctrl->xmin_key);
    R.x_max = dkey_inv(ctrl->xmax_key);
}

// ---------------------------------------------------------------------------
// Chronopoulos-Gear PCG (O5', A31): ONE kernel and ONE
// C3 reduction per iteration.  Node u at iteration k (alpha = alpha_k, beta =
// beta_k; k = 0: p = z, s = w):
//   s = w + beta s_old;  z = r Dinv;  p = z + beta p;  x += alpha p;
//   r' = r - alpha s;  z' = r' Dinv;  w' = D z' - sum_asc g z'_nbr   (O2)
// with every neighbour's z' recomputed from its r, w, s_old and Dinv by the
// same formulas (same bits as the owner's, O9 (ii)); quantities
// [<r',z'>, <z',w'>, <z',z'>, <r',r'>].
// ---------------------------------------------------------------------------
#define CG_SVAL(i) (first ? wk[i] : wk[i] + beta * so[i])
#define CG_ZNEW(i) ((rk[i] - alpha * CG_SVAL(i)) * di[i])
#define CG_NODE_TAIL()                                                            \
    const double su = CG_SVAL(u);                                                 \
    const double zu = rk[u] * di[u];                                              \
    const double pu = first ? zu : zu + beta * g.p[u];                            \
    const double ru = rk[u] - alpha * su;                                         \
    const double zn = ru * di[u];                                                 \
    const double wu = v.D[u] * zn - a;                                            \
    g.p[u] = pu;                                                                  \
    sn[u] = su;                                                                   \
    v.x[u] = v.x[u] + alpha * pu;                                                 \
    rn[u] = ru;                                                                   \
    wn[u] = wu;                                                                   \
    acc[0] = acc[0] + ru * zn;                                                    \
    acc[1] = acc[1] + zn * wu;                                                    \
    acc[2] = acc[2] + zn * zn;                                                    \
    acc[3] = acc[3] + ru * ru;

#define CG_PROLOGUE()                                                             \
    DevCtrl *ctrl = ra.ctrl;                                                      \
    if (ctrl->done) {                                                             \
        if (blockIdx.x == 0 && threadIdx.x == 0) set_cond(cd, ctrl);              \
        return;                                                                   \
    }                                                                             \
    const int32_t k = ctrl->k;                                                    \
    const bool first = (k == 0);                                                  \
    const double alpha = ctrl->alpha, beta = ctrl->beta;                          \
    const double *__restrict__ rk = g.r[k & 1];                                   \
    const double *__restrict__ wk = g.w[k & 1];                                   \
    const double *__restrict__ so = g.s[(k + 1) & 1];                             \
    double *__restrict__ rn = g.r[(k + 1) & 1];                                   \
    double *__restrict__ wn = g.w[(k + 1) & 1];                                   \
    double *__restrict__ sn = g.s[k & 1];                                         \
    const double *__restrict__ di = v.Dinv;                                       \
    double acc[4] = {0.0, 0.0, 0.0, 0.0};

#define CG_EPILOGUE()                                                             \
    if (c3_chunk_epilogue<4>(acc, v.chunk0 + (int32_t)blockIdx.x, ra) && cd.finalize && threadIdx.x == 0) { \
        finalize_cgcg(ra.ctrl, ra.slots);                                         \
        set_cond(cd, ra.ctrl);                                                    \
    }

__global__ void __launch_bounds__(kThreads) k_cgcg_stencil(StencilArgs s, VecArgs v, CgArgs g, RedArgs ra,
                                                           CondArgs cd)
{
    CG_PROLOGUE()
    const int64_t P = s.P;
    double *wl = g.wpeer_lo[(k + 1) & 1], *wh = g.wpeer_hi[(k + 1) & 1];
    bool peer = false;
    FOR_CHUNK_NODES({
        const Coord c = coord_of(s, s.lo + u);
        double a = 0.0;
        if (c.z > 0) a = a + s.gz[u - P] * CG_ZNEW(u - P);
        if (c.y > 0) a = a + s.gy[u - s.nx] * CG_ZNEW(u - s.nx);
        if (c.x > 0) a = a + s.gx[u - 1] * CG_ZNEW(u - 1);
        if (c.x < s.nx - 1) a = a + s.gx[u] * CG_ZNEW(u + 1);
        if (c.y < s.ny - 1) a = a + s.gy[u] * CG_ZNEW(u + s.nx);
        if (c.z < s.nz - 1) a = a + s.gz[u] * CG_ZNEW(u + P);
        CG_NODE_TAIL()
        if (wl && u < g.plane) { wl[u] = wu; peer = true; }  // fused w halo (p2p)
        if (wh && u >= v.n_own - g.plane) { wh[u - (v.n_own - g.plane)] = wu; peer = true; }
    })
    if (peer) __threadfence_system();
    CG_EPILOGUE()
}

__global__ void __launch_bounds__(kThreads) k_cgcg_sell(SellArgs s, VecArgs v, CgArgs g, RedArgs ra, CondArgs cd)
{
    CG_PROLOGUE()
    FOR_CHUNK_NODES({
        const int64_t sl = u / kSell;
        const int64_t e0 = s.slice_ptr[sl] + (u % kSell);
        const int32_t W = (int32_t)((s.slice_ptr[sl + 1] - s.slice_ptr[sl]) / kSell);
        double a = 0.0;
        for (int32_t kk = 0; kk < W; kk++) {
            const int64_t idx = e0 + kSell * (int64_t)kk;
            const int32_t nb = s.col[idx];
            if (nb < 0) break;
            a = a + s.g[idx] * CG_ZNEW(nb);
        }
        CG_NODE_TAIL()
    })
    CG_EPILOGUE()
}

// Ghost entries of a multi-rank context, in the phase of iteration k: the
// owner's s and r updates (the neighbour's w arrives by the halo).
__global__ void k_cgcg_ghost(CgArgs g, int64_t lo, int64_t n, const DevCtrl *ctrl)
{
    if (ctrl->done) return;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t k = ctrl->k;
    const bool first = (k == 0);
    const double alpha = ctrl->alpha, beta = ctrl->beta;
    const double *wk = g.w[k & 1], *so = g.s[(k + 1) & 1], *rk = g.r[k & 1];
    const int64_t u = lo + i;
    const double su = CG_SVAL(u);
    g.s[k & 1][u] = su;
    g.r[(k + 1) & 1][u] = rk[u] - alpha * su;
}
#undef CG_SVAL
#undef CG_ZNEW
#undef CG_NODE_TAIL
#undef CG_PROLOGUE
#undef CG_EPILOGUE

// After a CG-CG solve x is final (updated every iteration); only b = 0 needs x = 0.
__global__ void k_cgcg_finish(VecArgs v, const DevCtrl *ctrl)
{
    if (!ctrl->zero_x) return;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < v.n_own; i += (int64_t)gridDim.x * blockDim.x)
        v.x[i] = 0.0;
}

void launch_cgcg_finish(const VecArgs &v, const DevCtrl *ctrl, cudaStream_t st)
{
    const unsigned nb = (unsigned)std::min<int64_t>(std::max<int64_t>((v.n_own + 255) / 256, 1), 148 * 8);
    k_cgcg_finish<<<nb, 256, 0, st>>>(v, ctrl);
}

void launch_stencil_cgcg(const StencilArgs &s, const VecArgs &v, const CgArgs &g, const RedArgs &ra,
                         const CondArgs &cd, cudaStream_t st)
{
    if (s.nx % 2 == 0) return launch_pair_cgcg(s, v, g, ra, cd, st);
    k_cgcg_stencil<<<(unsigned)((v.n_own + kChunk - 1) / kChunk), kThreads, 0, st>>>(s, v, g, ra, cd);
}

void launch_sell_cgcg(const SellArgs &s, const VecArgs &v, const CgArgs &g, const RedArgs &ra, const CondArgs &cd,
                      cudaStream_t st)
{
    k_cgcg_sell<<<(unsigned)((v.n_own + kChunk - 1) / kChunk), kThreads, 0, st>>>(s, v, g, ra, cd);
}

void launch_cgcg_ghost(const CgArgs &g, int64_t lo, int64_t n, const DevCtrl *ctrl, cudaStream_t st)
{
    if (n > 0) k_cgcg_ghost<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(g, lo, n, ctrl);
}

// ---------------------------------------------------------------------------
// CSR strips with p2p: after K5 (which keeps its group sums local), the z
// values of the send lists are stored straight into the peers' ghost blocks,
// then one block publishes this rank's RZ group sums to every rank and bumps
// their arrival counters — so a peer sees the new ghost z before the arrival
// it waits on.  Both skip a finished solve (as K5 and the RZ finalize do).
// ---------------------------------------------------------------------------
__global__ void k_p2p_halo_store(const double *z, const int32_t *send_idx, const int32_t *peer, const int64_t *pos,
                                 int64_t n, double *const *zpeers, const DevCtrl *ctrl)
{
    if (ctrl->done) return;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        zpeers[peer[i]][pos[i]] = z[send_idx[i]];
    __threadfence_system();
}

__global__ void k_p2p_push(const double *slots, int nq, int g0, int g1, int32_t K, int n_fin,
                           double *const *pslots, unsigned long long *const *pcnt, int world, const DevCtrl *ctrl)
{
    if (ctrl->done || threadIdx.x != 0) return;
    __threadfence_system();
    const int off = (int)(ctrl->red_seq & 1u) * (kMaxQ * kGroups);
    for (int w = 0; w < world; w++)
        for (int q = 0; q < nq; q++)
            for (int g = g0; g < g1; g++)
                if (group_lo(g + 1, K) > group_lo(g, K))  // non-empty groups only (empty ones stay +0.0)
                    pslots[w][off + q * kGroups + g] = slots[q * kGroups + g];
    __threadfence_system();
    for (int w = 0; w < world; w++)
        if (n_fin > 0) atomicAdd_system(pcnt[w], (unsigned long long)n_fin);
}

void launch_p2p_halo_push(const double *z, const int32_t *send_idx, const int32_t *peer, const int64_t *pos,
                          int64_t n, double *const *zpeers, const double *slots, int nq, int g0, int g1, int32_t K,
                          int n_fin, double *const *pslots, unsigned long long *const *pcnt, int world,
                          const DevCtrl *ctrl, cudaStream_t st)
{
    if (n > 0) {
        const unsigned nb = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 4);
        k_p2p_halo_store<<<nb, 256, 0, st>>>(z, send_idx, peer, pos, n, zpeers, ctrl);
    }
    k_p2p_push<<<1, 32, 0, st>>>(slots, nq, g0, g1, K, n_fin, pslots, pcnt, world, ctrl);
}

// Virtual-group "allreduce": dst = sum over ranks (rank order) of src[r].
__global__ void k_vsum(const double *const *src, int W, int n, double *dst)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double acc = 0.0;
    for (int r = 0; r < W; r++) acc = acc + src[r][i];
    dst[i] = acc;
}

// Virtual-group min / max of the diagnostic x range over every rank.
__global__ void k_vminmax(DevCtrl *const *ctrl, int W)
{
    unsigned long long mn = ~0ull, mx = 0ull;
    for (int r = 0; r < W; r++) {
        mn = ctrl[r]->xmin_key < mn ? ctrl[r]->xmin_key : mn;
        mx = ctrl[r]->xmax_key > mx ? ctrl[r]->xmax_key : mx;
    }
    for (int r = 0; r < W; r++) {
        ctrl[r]->xmin_key = mn;
        ctrl[r]->xmax_key = mx;
    }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
void launch_vminmax(DevCtrl *const *ctrl, int W, cudaStream_t st) { k_vminmax<<<1, 1, 0, st>>>(ctrl, W); }

void launch_vsum(double *const *src, int W, int n, double *dst, cudaStream_t st)
{
    k_vsum<<<(n + 127) / 128, 128, 0, st>>>(src, W, n, dst);
}

static inline unsigned nblocks(int64_t n_own) { return (unsigned)((n_own + kChunk - 1) / kChunk); }

void launch_stencil_assemble(const StencilArgs &s, const VecArgs &v, const RedArgs &ra, const CondArgs &cd,
                             int mode, double eps, cudaStream_t st)
{
    launch_stencil_assemble_ex(s, v, ra, cd, mode, eps, nullptr, nullptr, st);
}

int launch_stencil_assemble_ex(const StencilArgs &s, const VecArgs &v, const RedArgs &ra, const CondArgs &cd,
                                int mode, double eps, double *gs_out, double *gt_out, cudaStream_t st)
{
    if (s.nx % 2 == 0) return launch_pair_assemble(s, v, ra, cd, mode, eps, gs_out, gt_out, st);
    const double eps2 = eps * eps;
    const unsigned nb = nblocks(v.n_own);
    if (mode == ASM_INIT) k_stencil_assemble<ASM_INIT><<<nb, kThreads, 0, st>>>(s, v, ra, cd, eps2, gs_out, gt_out);
    else if (mode == ASM_LAMBDA2)
        k_stencil_assemble<ASM_LAMBDA2><<<nb, kThreads, 0, st>>>(s, v, ra, cd, eps2, gs_out, gt_out);
    else if (mode == ASM_REWEIGHT_WARM)
        k_stencil_assemble<ASM_REWEIGHT_WARM><<<nb, kThreads, 0, st>>>(s, v, ra, cd, eps2, gs_out, gt_out);
    else k_stencil_assemble<ASM_REWEIGHT_COLD><<<nb, kThreads, 0, st>>>(s, v, ra, cd, eps2, gs_out, gt_out);
    return 1;
}

void launch_sell_assemble(const SellArgs &s, const VecArgs &v, const RedArgs &ra, const CondArgs &cd, int mode,
                          double eps, cudaStream_t st)
{
    launch_sell_assemble_ex(s, v, ra, cd, mode, eps, nullptr, nullptr, st);
}

int launch_sell_assemble_ex(const SellArgs &s, const VecArgs &v, const RedArgs &ra, const CondArgs &cd, int mode,
                             double eps, double *gs_out, double *gt_out, cudaStream_t st)
{
    if (launch_sellp_assemble(s, v, ra, cd, mode, eps, gs_out, gt_out, st)) return 1;
    const double eps2 = eps * eps;
    const unsigned nb = nblocks(v.n_own);
    if (mode == ASM_INIT) k_sell_assemble<ASM_INIT><<<nb, kThreads, 0, st>>>(s, v, ra, cd, eps2, gs_out, gt_out);
    else if (mode == ASM_LAMBDA2)
        k_sell_assemble<ASM_LAMBDA2><<<nb, kThreads, 0, st>>>(s, v, ra, cd, eps2, gs_out, gt_out);
    else if (mode == ASM_REWEIGHT_WARM)
        k_sell_assemble<ASM_REWEIGHT_WARM><<<nb, kThreads, 0, st>>>(s, v, ra, cd, eps2, gs_out, gt_out);
    else k_sell_assemble<ASM_REWEIGHT_COLD><<<nb, kThreads, 0, st>>>(s, v, ra, cd, eps2, gs_out, gt_out);
    return 1;
}

void launch_stencil_pspmv(const StencilArgs &s, const VecArgs &v, const RedArgs &ra, const CondArgs &cd,
                          cudaStream_t st, bool w0)
{
    if (s.nx % 2 == 0) return launch_pair_pspmv(s, v, ra, cd, st, w0);
    k_stencil_pspmv<<<nblocks(v.n_own), kThreads, 0, st>>>(s, v, ra, cd, w0);
}

void launch_sell_pspmv(const SellArgs &s, const VecArgs &v, const RedArgs &ra, const CondArgs &cd, cudaStream_t st,
                       bool w0)
{
    if (launch_sellp_pspmv(s, v, ra, cd, st, w0)) return;
    k_sell_pspmv<<<nblocks(v.n_own), kThreads, 0, st>>>(s, v, ra, cd, w0);
}

void launch_ghost_pupdate(const VecArgs &v, int64_t ghost_lo, int64_t ghost_hi, int64_t plane, DevCtrl *ctrl,
                          cudaStream_t st)
{
    const int64_t n = (ghost_lo ? plane : 0) + (ghost_hi ? plane : 0);
    if (n == 0) return;
    k_ghost_pupdate<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(v, ghost_lo, ghost_hi, plane, ctrl);
}

void launch_axpy_jacobi(const VecArgs &v, const RedArgs &ra, const CondArgs &cd, cudaStream_t st)
{
    launch_pair_axpy(v, ra, cd, st);
}

void launch_finish(const VecArgs &v, DevCtrl *ctrl, cudaStream_t st)
{
    launch_pair_finish(v, ctrl, st);
}

void launch_finalize(int phase, DevCtrl *ctrl, const double *slots, const CondArgs &cd, const P2PWait &pw,
                     cudaStream_t st)
{
    k_finalize<<<1, 1, 0, st>>>(phase, ctrl, slots, cd, pw);
}

__global__ void k_gate(const DevCtrl *ctrl, cudaGraphConditionalHandle h)
{
    cudaGraphSetConditional(h, ctrl->frozen ? 0u : 1u);
}

void launch_gate(const DevCtrl *ctrl, cudaGraphConditionalHandle h, cudaStream_t st)
{
    k_gate<<<1, 1, 0, st>>>(ctrl, h);
}

__global__ void k_mark(DevCtrl *ctrl) { ctrl->t_mark = global_ns(); }

__global__ void k_outer_init(DevCtrl *ctrl, cudaGraphConditionalHandle h, int count)
{
    ctrl->outer_left = count;
    ctrl->outer_end = ctrl->step + count;
    cudaGraphSetConditional(h, count > 0 ? 1u : 0u);
}

__global__ void k_outer_next(DevCtrl *ctrl, cudaGraphConditionalHandle h, int freeze_exit)
{
    const int left = ctrl->outer_left - 1;
    ctrl->outer_left = left;
    cudaGraphSetConditional(h, (left > 0 && !(freeze_exit && ctrl->frozen)) ? 1u : 0u);
}

// after a fixed-point exit: the skipped steps' reports are the frozen one's
__global__ void k_fill_reports(DevCtrl *ctrl, DevReport *reports)
{
    const int end = ctrl->outer_end;
    int step = ctrl->step;
    if (step <= 0) return;
    const DevReport last = reports[step - 1];
    for (; step < end; step++) reports[step] = last;
    ctrl->step = step;
}

void launch_mark(DevCtrl *ctrl, cudaStream_t st) { k_mark<<<1, 1, 0, st>>>(ctrl); }
void launch_outer_init(DevCtrl *ctrl, cudaGraphConditionalHandle h, int count, cudaStream_t st)
{
    k_outer_init<<<1, 1, 0, st>>>(ctrl, h, count);
}
void launch_outer_next(DevCtrl *ctrl, cudaGraphConditionalHandle h, int freeze_exit, cudaStream_t st)
{
    k_outer_next<<<1, 1, 0, st>>>(ctrl, h, freeze_exit);
}
void launch_fill_reports(DevCtrl *ctrl, DevReport *reports, cudaStream_t st)
{
    k_fill_reports<<<1, 1, 0, st>>>(ctrl, reports);
}

void launch_report(DevCtrl *ctrl, DevReport *reports, int freeze, cudaStream_t st)
{
    k_report<<<1, 1, 0, st>>>(ctrl, reports, freeze);
}

void launch_stencil_diag_ex(const StencilArgs &s, const VecArgs &v, const RedArgs &ra, double eps, int norm,
                            const double *gsv, const double *gtv, cudaStream_t st)
{
    k_stencil_diag<<<nblocks(v.n_own), kThreads, 0, st>>>(s, v, ra, eps * eps, norm, gsv, gtv);
}

void launch_sell_diag_ex(const SellArgs &s, const VecArgs &v, const RedArgs &ra, double eps, int norm,
                         const double *gsv, const double *gtv, cudaStream_t st)
{
    k_sell_diag<<<nblocks(v.n_own), kThreads, 0, st>>>(s, v, ra, eps * eps, norm, gsv, gtv);
}

void launch_diag_finalize(DevCtrl *ctrl, const double *slots, DevReport *reports, int norm, const P2PWait &pw,
                          cudaStream_t st)
{
    k_diag_finalize<<<1, 1, 0, st>>>(ctrl, slots, reports, norm, pw);
}

}  // namespace irls
