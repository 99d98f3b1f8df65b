// sell_pair.cu — CSR path (SELL-64, pair-interleaved) for graphs whose widest
// slice holds <= 8 neighbours (road-like graphs: <= 4).
//
// Thread t owns rows u0 = base + 2t + 512j and u0+1 (C3 mapping).  With slices
// of 64 rows stored column-major, the k-th neighbour slot of rows u0 and u0+1
// are adjacent: one int2 load for the two column ids and one 128-bit load for
// the two capacities / conductances.  Every load of an iteration (own vectors,
// all slots, then all neighbour gathers) is issued before the first use.
// Sums run over the slots in stored (= ascending neighbour id) order, padding
// slots (col = -1) contribute nothing (C2).
#include "kernels.h"

namespace irls {

__device__ __forceinline__ double2 ldp2(const double *__restrict__ a, int64_t i)
{
    return __ldg(reinterpret_cast<const double2 *>(a + i));
}
__device__ __forceinline__ void stp2(double *a, int64_t i, double2 v) { *reinterpret_cast<double2 *>(a + i) = v; }
__device__ __forceinline__ int2 ldi2(const int32_t *__restrict__ a, int64_t i)
{
    return __ldg(reinterpret_cast<const int2 *>(a + i));
}

__device__ __forceinline__ void set_cond3(const CondArgs &cd, const DevCtrl *c)
{
    if (cd.use) cudaGraphSetConditional(cd.handle, c->done ? 0u : 1u);
}

// Terminal conductances (same formula and bits as rw_g on each terminal).
__device__ __forceinline__ double term_g(double cs, double ct, double x, double eps2, double &gt)
{
    const bool s_first = cs > 0.0;
    const double g1 = rw_g(s_first ? cs : ct, s_first ? 1.0 - x : x, eps2);
    double gs = s_first ? g1 : 0.0;
    gt = s_first ? 0.0 : g1;
    if (s_first && ct > 0.0) gt = rw_g(ct, x, eps2);
    return gs;
}

template <int WMAX, int MODE, int MINB = 1, int HALF = WMAX>
__global__ void __launch_bounds__(kThreads, MINB) k_sellp_assemble(SellArgs s, VecArgs v, RedArgs ra, CondArgs cd,
                                                             double eps2, double *gs_out, double *gt_out)
{
    if (v.frozen && *(const volatile int32_t *)v.frozen) return;  // fixed point: this step repeats the last one
    constexpr bool WARM = MODE == ASM_REWEIGHT_WARM;
    constexpr bool INITG = MODE == ASM_INIT || MODE == ASM_LAMBDA2;  // g = c
    constexpr bool HASX = !INITG;
    const int64_t base = (int64_t)blockIdx.x * kChunk;
    double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll 1
    for (int j = 0; j < 8; j++) {
        const int64_t u0 = base + 2 * (int64_t)threadIdx.x + 512 * j;
        if (u0 >= v.n_own) break;
        const bool v1 = u0 + 1 < v.n_own;
        const int64_t sl = u0 / kSell;
        const int64_t e0 = s.slice_ptr[sl] + (u0 % kSell);
        const int32_t W = (int32_t)((s.slice_ptr[sl + 1] - s.slice_ptr[sl]) / kSell);
        // ---- loads: own, slots, then gathers
        const double2 x2 = HASX ? ldp2(v.x, u0) : make_double2(0.0, 0.0);
        const double2 cs2 = ldp2(s.cs, u0), ct2 = ldp2(s.ct, u0);
        // ---- conductances in slot order, HALF slots' loads at a time
        double a0 = 0.0, b0 = 0.0, a1 = 0.0, b1 = 0.0;
#pragma unroll
        for (int k0 = 0; k0 < WMAX; k0 += HALF) {
            int2 cl[HALF];
            double2 cc[HALF];
#pragma unroll
            for (int k = 0; k < HALF; k++) {
                if (k0 + k < W) {
                    cl[k] = ldi2(s.col, e0 + (int64_t)kSell * (k0 + k));
                    cc[k] = ldp2(s.c, e0 + (int64_t)kSell * (k0 + k));
                } else {
                    cl[k] = make_int2(-1, -1);
                    cc[k] = make_double2(0.0, 0.0);
                }
            }
            double xa[HALF], xb[HALF];
#pragma unroll
            for (int k = 0; k < HALF; k++) {
                xa[k] = (HASX && cl[k].x >= 0) ? __ldg(v.x + cl[k].x) : 0.0;
                xb[k] = (HASX && cl[k].y >= 0) ? __ldg(v.x + cl[k].y) : 0.0;
            }
#pragma unroll
            for (int k = 0; k < HALF; k++) {
                if (k0 + k < W) {
                    double g0 = 0.0, g1 = 0.0;
                    if (cl[k].x >= 0) {
                        g0 = INITG ? cc[k].x : rw_g(cc[k].x, x2.x - xa[k], eps2);
                        a0 = a0 + g0;
                        if (WARM) b0 = b0 + g0 * xa[k];
                    }
                    if (cl[k].y >= 0) {
                        g1 = INITG ? cc[k].y : rw_g(cc[k].y, x2.y - xb[k], eps2);
                        a1 = a1 + g1;
                        if (WARM) b1 = b1 + g1 * xb[k];
                    }
                    stp2(s.g, e0 + (int64_t)kSell * (k0 + k), make_double2(g0, g1));
                }
            }
        }
        double2 gs2, gt2;
        if (INITG) {
            gs2 = cs2;
            gt2 = ct2;
        } else {
            gs2.x = term_g(cs2.x, ct2.x, x2.x, eps2, gt2.x);
            gs2.y = term_g(cs2.y, ct2.y, x2.y, eps2, gt2.y);
        }
        const double D0 = (a0 + gs2.x) + gt2.x, D1 = (a1 + gs2.y) + gt2.y;
        const double Di0 = 1.0 / D0, Di1 = v1 ? 1.0 / D1 : 0.0;
        const double bb0 = MODE == ASM_LAMBDA2 ? gs2.x - gt2.x : gs2.x;
        const double bb1 = MODE == ASM_LAMBDA2 ? gs2.y - gt2.y : gs2.y;
        const double r0 = WARM ? gs2.x - (D0 * x2.x - b0) : bb0;
        const double r1 = v1 ? (WARM ? gs2.y - (D1 * x2.y - b1) : bb1) : 0.0;
        const double z0 = r0 * Di0, z1 = r1 * Di1;
        stp2(v.D, u0, make_double2(D0, v1 ? D1 : 0.0));
        stp2(v.Dinv, u0, make_double2(Di0, Di1));
        stp2(v.r, u0, make_double2(r0, r1));
        stp2(v.z, u0, make_double2(z0, z1));
        if (gs_out) {
            stp2(gs_out, u0, gs2);
            stp2(gt_out, u0, gt2);
        }
        const double mb0 = bb0 * Di0;
        acc[0] = acc[0] + r0 * z0;
        acc[1] = acc[1] + z0 * z0;
        acc[2] = acc[2] + r0 * r0;
        acc[3] = acc[3] + mb0 * mb0;
        acc[4] = acc[4] + bb0 * bb0;
        if (v1) {
            const double mb1 = bb1 * Di1;
            acc[0] = acc[0] + r1 * z1;
            acc[1] = acc[1] + z1 * z1;
            acc[2] = acc[2] + r1 * r1;
            acc[3] = acc[3] + mb1 * mb1;
            acc[4] = acc[4] + bb1 * bb1;
        }
    }
    if (c3_chunk_epilogue<5>(acc, v.chunk0 + (int32_t)blockIdx.x, ra) && cd.finalize && threadIdx.x == 0) {
        finalize_start(ra.ctrl, ra.slots);
        set_cond3(cd, ra.ctrl);
    }
}

template <int WMAX, int MINB, bool W0, int HALF = WMAX>
__global__ void __launch_bounds__(kThreads, MINB) k_sellp_pspmv(SellArgs s, VecArgs v, RedArgs ra, CondArgs cd)
{
    const DevCtrl *ctrl = ra.ctrl;
    if (W0 && ctrl->done) return;  // CG-CG's w0 pass after a START that stopped
    const int32_t it = ctrl->k;
    const bool first = (it == 0);
    const double beta = ctrl->beta, alpha = ctrl->alpha;
    const double *__restrict__ pold = (it & 1) ? v.p1 : v.p0;
    double *__restrict__ pnew = (it & 1) ? v.p0 : v.p1;
    const double *__restrict__ zv = v.z;
    const int64_t base = (int64_t)blockIdx.x * kChunk;
    double acc[1] = {0.0};
#pragma unroll 1
    for (int j = 0; j < 8; j++) {
        const int64_t u0 = base + 2 * (int64_t)threadIdx.x + 512 * j;
        if (u0 >= v.n_own) break;
        const bool v1 = u0 + 1 < v.n_own;
        const int64_t sl = u0 / kSell;
        const int64_t e0 = s.slice_ptr[sl] + (u0 % kSell);
        const int32_t W = (int32_t)((s.slice_ptr[sl + 1] - s.slice_ptr[sl]) / kSell);
        const double2 z2 = ldp2(zv, u0);
        const double2 po = first ? make_double2(0.0, 0.0) : ldp2(pold, u0);
        const double2 D2 = ldp2(v.D, u0);
        double2 x2 = make_double2(0.0, 0.0);
        if (!first) x2 = *reinterpret_cast<const double2 *>(v.x + u0);
        const double p0 = first ? z2.x : z2.x + beta * po.x;
        const double p1 = first ? z2.y : z2.y + beta * po.y;
        double a = 0.0, b = 0.0;
        // slots in groups of HALF (loads of a group in flight together; fewer
        // live registers than all WMAX at once)
#pragma unroll
        for (int k0 = 0; k0 < WMAX; k0 += HALF) {
            int2 cl[HALF];
            double2 gg[HALF];
#pragma unroll
            for (int k = 0; k < HALF; k++)
                cl[k] = k0 + k < W ? ldi2(s.col, e0 + (int64_t)kSell * (k0 + k)) : make_int2(-1, -1);
#pragma unroll
            for (int k = 0; k < HALF; k++)  // padding slots of both rows: no conductance load
                gg[k] = (cl[k].x >= 0 || cl[k].y >= 0) ? ldp2(s.g, e0 + (int64_t)kSell * (k0 + k))
                                                        : make_double2(0.0, 0.0);
            double za[HALF], zb[HALF], pa[HALF], pb[HALF];
#pragma unroll
            for (int k = 0; k < HALF; k++) {
                za[k] = cl[k].x >= 0 ? __ldg(zv + cl[k].x) : 0.0;
                zb[k] = cl[k].y >= 0 ? __ldg(zv + cl[k].y) : 0.0;
                pa[k] = (!first && cl[k].x >= 0) ? __ldg(pold + cl[k].x) : 0.0;
                pb[k] = (!first && cl[k].y >= 0) ? __ldg(pold + cl[k].y) : 0.0;
            }
#pragma unroll
            for (int k = 0; k < HALF; k++) {
                if (cl[k].x >= 0) a = a + gg[k].x * (first ? za[k] : za[k] + beta * pa[k]);
                if (cl[k].y >= 0) b = b + gg[k].y * (first ? zb[k] : zb[k] + beta * pb[k]);
            }
        }
        const double q0 = D2.x * p0 - a, q1 = v1 ? D2.y * p1 - b : 0.0;
        stp2(pnew, u0, make_double2(p0, v1 ? p1 : 0.0));
        stp2(v.q, u0, make_double2(q0, q1));
        if (!first) stp2(v.x, u0, make_double2(x2.x + alpha * po.x, x2.y + alpha * po.y));
        acc[0] = acc[0] + p0 * q0;
        if (v1) acc[0] = acc[0] + p1 * q1;
    }
    if (c3_chunk_epilogue<1>(acc, v.chunk0 + (int32_t)blockIdx.x, ra) && cd.finalize && threadIdx.x == 0) {
        finalize_pq(ra.ctrl, ra.slots);
        if (W0) set_cond3(cd, ra.ctrl);
    }
}

static inline unsigned nblk3(int64_t n) { return (unsigned)((n + kChunk - 1) / kChunk); }

template <int WMAX>
static void asm_w(const SellArgs &s, const VecArgs &v, const RedArgs &ra, const CondArgs &cd, int mode, double eps2,
                  double *gs_out, double *gt_out, cudaStream_t st)
{
    const unsigned nb = nblk3(v.n_own);
    // reweight steps at 3 CTAs/SM: config 3 0.62 ms vs 0.72 ms at 1, 2 or 4
    // (per-slot loads at 4 CTAs/SM measured 0.676 ms and two slots at a time
    // 0.682 ms against 0.622 ms for all slots' loads first at 3 CTAs/SM)
    if (WMAX == 4 && mode == ASM_REWEIGHT_WARM) {
        k_sellp_assemble<WMAX, ASM_REWEIGHT_WARM, 3><<<nb, kThreads, 0, st>>>(s, v, ra, cd, eps2, gs_out, gt_out);
        return;
    }
    if (WMAX == 4 && mode == ASM_REWEIGHT_COLD) {
        k_sellp_assemble<WMAX, ASM_REWEIGHT_COLD, 3><<<nb, kThreads, 0, st>>>(s, v, ra, cd, eps2, gs_out, gt_out);
        return;
    }
    if (mode == ASM_INIT) k_sellp_assemble<WMAX, ASM_INIT><<<nb, kThreads, 0, st>>>(s, v, ra, cd, eps2, gs_out, gt_out);
    else if (mode == ASM_LAMBDA2)
        k_sellp_assemble<WMAX, ASM_LAMBDA2><<<nb, kThreads, 0, st>>>(s, v, ra, cd, eps2, gs_out, gt_out);
    else if (mode == ASM_REWEIGHT_WARM)
        k_sellp_assemble<WMAX, ASM_REWEIGHT_WARM><<<nb, kThreads, 0, st>>>(s, v, ra, cd, eps2, gs_out, gt_out);
    else k_sellp_assemble<WMAX, ASM_REWEIGHT_COLD><<<nb, kThreads, 0, st>>>(s, v, ra, cd, eps2, gs_out, gt_out);
}

bool launch_sellp_assemble(const SellArgs &s, const VecArgs &v, const RedArgs &ra, const CondArgs &cd, int mode,
                           double eps, double *gs_out, double *gt_out, cudaStream_t st)
{
    const double eps2 = eps * eps;
    if (s.wmax <= 4) asm_w<4>(s, v, ra, cd, mode, eps2, gs_out, gt_out, st);
    else if (s.wmax <= 8) asm_w<8>(s, v, ra, cd, mode, eps2, gs_out, gt_out, st);
    else return false;
    return true;
}

bool launch_sellp_pspmv(const SellArgs &s, const VecArgs &v, const RedArgs &ra, const CondArgs &cd, cudaStream_t st,
                        bool w0)
{
    // WMAX 4: one slot at a time (HALF = 1: 64 registers, no spill, 4 CTAs/SM;
    // the unrolled slot loop still keeps the loads in flight): config 3
    // 0.431 ms against 0.517 ms for all four slots' loads first at 3 CTAs/SM
    // (80 registers, 48 B spilled) and 0.450 ms for two at a time (same box)
    if (s.wmax <= 4 && w0) k_sellp_pspmv<4, 4, true, 1><<<nblk3(v.n_own), kThreads, 0, st>>>(s, v, ra, cd);
    else if (s.wmax <= 4) k_sellp_pspmv<4, 4, false, 1><<<nblk3(v.n_own), kThreads, 0, st>>>(s, v, ra, cd);
    else if (s.wmax <= 8 && w0) k_sellp_pspmv<8, 1, true><<<nblk3(v.n_own), kThreads, 0, st>>>(s, v, ra, cd);
    else if (s.wmax <= 8) k_sellp_pspmv<8, 1, false><<<nblk3(v.n_own), kThreads, 0, st>>>(s, v, ra, cd);
    else return false;
    return true;
}

}  // namespace irls
