// stencil_pair.cu — pair-vectorised stencil kernels (nx even).
//
// Same C3 mapping as kernels_cg.cu (thread t owns nodes base + 2t + 512j + e),
// but each thread moves its node pair (u0, u0+1) with 128-bit loads/stores
// and takes the +-x neighbours from the adjacent lanes by warp shuffle.  With
// nx even a pair never straddles a row, so both nodes share (y, z).
//
// K1 is split in two passes:
//   K1a  edge pass: the conductance of every owned +x/+y/+z edge (Eq. 4, 8)
//        -> gx, gy, gz  (3 sqrt+div per node instead of 6 in one pass)
//   K1b  node pass: terminal conductances, D, Dinv (O1), r0 = b - L~ x0,
//        z0 = Dinv r0 and the START reductions.
// Absent neighbours contribute exact +0.0 products, which leaves every sum
// bitwise unchanged (the accumulators are never -0.0), so these kernels give
// the same bits as the scalar ones and as the oracle.
#include <algorithm>
#include <cstdlib>
#include "kernels.h"

namespace irls {

__device__ __forceinline__ double2 ldp(const double *__restrict__ a, int64_t i)
{
    return __ldg(reinterpret_cast<const double2 *>(a + i));
}
__device__ __forceinline__ double2 ldp_cg(const double *a, int64_t i)
{
    return *reinterpret_cast<const double2 *>(a + i);
}
__device__ __forceinline__ void stp(double *a, int64_t i, double2 v) { *reinterpret_cast<double2 *>(a + i) = v; }

struct PairCoord {
    int32_t x0, y, z;
};

__device__ __forceinline__ PairCoord pair_coord(const StencilArgs &s, int64_t ug0)
{
    PairCoord c;
    const uint32_t u = (uint32_t)ug0;
    const uint32_t t1 = fdiv(u, s.fd_nx);
    c.x0 = (int32_t)(u - t1 * (uint32_t)s.nx);
    const uint32_t zz = fdiv(t1, s.fd_ny);
    c.y = (int32_t)(t1 - zz * (uint32_t)s.ny);
    c.z = (int32_t)zz;
    return c;
}

// Terminal conductances gs = rw(cs, 1 - x), gt = rw(ct, x) (Eq. 4/8, A3).
// Most nodes have exactly one positive terminal capacity; computing that one
// first keeps the warp convergent (one sqrt + div for every lane) and the
// second pair only runs for nodes with both.  Same formula, same bits.
__device__ __forceinline__ double terminal_g(double cs, double ct, double x, double eps2, double &gt)
{
    const bool s_first = cs > 0.0;
    const double g1 = rw_g(s_first ? cs : ct, s_first ? 1.0 - x : x, eps2);
    double gs = s_first ? g1 : 0.0;
    gt = s_first ? 0.0 : g1;
    if (s_first && ct > 0.0) gt = rw_g(ct, x, eps2);
    return gs;
}

__device__ __forceinline__ void set_cond2(const CondArgs &cd, const DevCtrl *c)
{
    if (cd.use) cudaGraphSetConditional(cd.handle, c->done ? 0u : 1u);
}

// ---------------------------------------------------------------------------
// K1a: owned edge conductances
// ---------------------------------------------------------------------------
template <bool INIT>
__global__ void __launch_bounds__(kThreads) k_pair_edges(StencilArgs s, VecArgs v, double eps2)
{
    if (v.frozen && *(const volatile int32_t *)v.frozen) return;  // fixed point: this step repeats the last one
    const int lane = threadIdx.x & 31;
    const int64_t base = (int64_t)blockIdx.x * kChunk;
    const int64_t P = s.P;
    const double2 zero2 = make_double2(0.0, 0.0);
#pragma unroll 1
    for (int j = 0; j < 8; j++) {
        const int64_t u0 = base + 2 * (int64_t)threadIdx.x + 512 * j;
        const bool valid = u0 < v.n_own;
        const PairCoord c = pair_coord(s, s.lo + u0);
        const bool hasr = c.x0 + 1 < s.nx - 1;  // node u0+1 has a +x edge
        const bool py = valid && c.y < s.ny - 1, pz = valid && c.z < s.nz - 1;
        const bool gh = valid && s.lo_ghost && u0 < P;
        // ---- loads first
        const double2 x2 = INIT ? zero2 : ldp(v.x, u0);
        const double2 cx2 = valid ? ldp(s.cx, u0) : zero2;
        const double2 cy2 = py ? ldp(s.cy, u0) : zero2;
        const double2 cz2 = pz ? ldp(s.cz, u0) : zero2;
        const double2 xpy = (!INIT && py) ? ldp(v.x, u0 + s.nx) : zero2;
        const double2 xpz = (!INIT && pz) ? ldp(v.x, u0 + P) : zero2;
        const double2 czm = gh ? ldp(s.cz, u0 - P) : zero2;
        const double2 xmz = (!INIT && gh) ? ldp(v.x, u0 - P) : zero2;
        double xe = 0.0;
        if (!INIT && valid && lane == 31 && hasr) xe = __ldg(v.x + u0 + 2);
        double xr = __shfl_down_sync(0xffffffffu, x2.x, 1);
        if (!valid) continue;
        if (lane == 31) xr = xe;
        double2 gx2, gy2, gz2;
        if (INIT) {
            gx2 = make_double2(cx2.x, hasr ? cx2.y : 0.0);
            gy2 = cy2;
            gz2 = cz2;
        } else {
            gx2.x = rw_g(cx2.x, x2.x - x2.y, eps2);
            gx2.y = hasr ? rw_g(cx2.y, x2.y - xr, eps2) : 0.0;
            gy2 = py ? make_double2(rw_g(cy2.x, x2.x - xpy.x, eps2), rw_g(cy2.y, x2.y - xpy.y, eps2)) : zero2;
            gz2 = pz ? make_double2(rw_g(cz2.x, x2.x - xpz.x, eps2), rw_g(cz2.y, x2.y - xpz.y, eps2)) : zero2;
        }
        stp(s.gx, u0, gx2);
        stp(s.gy, u0, gy2);
        stp(s.gz, u0, gz2);
        if (gh)  // the -z edge of the first owned plane (ghost slot)
            stp(s.gz, u0 - P, INIT ? czm
                                   : make_double2(rw_g(czm.x, xmz.x - x2.x, eps2), rw_g(czm.y, xmz.y - x2.y, eps2)));
    }
}

// ---------------------------------------------------------------------------
// K1b: terminals, D, Dinv, r0, z0, START reductions
// ---------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(kThreads) k_pair_nodes(StencilArgs s, VecArgs v, RedArgs ra, CondArgs cd,
                                                         double eps2, double *gs_out, double *gt_out)
{
    if (v.frozen && *(const volatile int32_t *)v.frozen) return;  // fixed point: this step repeats the last one
    const int lane = threadIdx.x & 31;
    const int64_t base = (int64_t)blockIdx.x * kChunk;
    const int64_t P = s.P;
    const double2 zero2 = make_double2(0.0, 0.0);
    constexpr bool WARM = MODE == ASM_REWEIGHT_WARM;
    constexpr bool INITG = MODE == ASM_INIT || MODE == ASM_LAMBDA2;  // g = c
    constexpr bool HASX = !INITG;
    double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll 1
    for (int j = 0; j < 8; j++) {
        const int64_t u0 = base + 2 * (int64_t)threadIdx.x + 512 * j;
        const bool valid = u0 < v.n_own;
        const PairCoord c = pair_coord(s, s.lo + u0);
        const bool hx = c.x0 > 0, hr = c.x0 + 1 < s.nx - 1;
        const bool hy = valid && c.y > 0, py = valid && c.y < s.ny - 1;
        const bool hz = valid && c.z > 0, pz = valid && c.z < s.nz - 1;
        // ---- loads first
        const double2 gx2 = ldp(s.gx, u0);
        const double2 x2 = HASX ? ldp(v.x, u0) : zero2;
        const double2 gy2 = valid ? ldp(s.gy, u0) : zero2, gz2 = valid ? ldp(s.gz, u0) : zero2;
        const double2 gym = hy ? ldp(s.gy, u0 - s.nx) : zero2;
        const double2 gzm = hz ? ldp(s.gz, u0 - P) : zero2;
        const double2 cs2 = valid ? ldp(s.cs, u0) : zero2, ct2 = valid ? ldp(s.ct, u0) : zero2;
        const double2 xmz = (WARM && hz) ? ldp(v.x, u0 - P) : zero2;
        const double2 xmy = (WARM && hy) ? ldp(v.x, u0 - s.nx) : zero2;
        const double2 xpy = (WARM && py) ? ldp(v.x, u0 + s.nx) : zero2;
        const double2 xpz = (WARM && pz) ? ldp(v.x, u0 + P) : zero2;
        double gxe = 0.0, xle = 0.0, xre = 0.0;
        if (valid && lane == 0 && hx) {
            gxe = __ldg(s.gx + u0 - 1);
            if (WARM) xle = __ldg(v.x + u0 - 1);
        }
        if (WARM && valid && lane == 31 && hr) xre = __ldg(v.x + u0 + 2);
        double gxl = __shfl_up_sync(0xffffffffu, gx2.y, 1);
        double xl = __shfl_up_sync(0xffffffffu, x2.y, 1);
        double xr = __shfl_down_sync(0xffffffffu, x2.x, 1);
        if (!valid) continue;
        if (lane == 0) { gxl = gxe; xl = xle; }
        if (lane == 31) xr = xre;
        if (!hx) { gxl = 0.0; xl = 0.0; }
        if (!hr) xr = 0.0;
        double2 gs2, gt2;
        if (INITG) {
            gs2 = cs2;
            gt2 = ct2;
        } else {
            gs2.x = terminal_g(cs2.x, ct2.x, x2.x, eps2, gt2.x);
            gs2.y = terminal_g(cs2.y, ct2.y, x2.y, eps2, gt2.y);
        }
        // O1, ascending (-z, -y, -x, +x, +y, +z); absent terms are +0.0
        const double D0 = ((((((0.0 + gzm.x) + gym.x) + gxl) + gx2.x) + gy2.x) + gz2.x + gs2.x) + gt2.x;
        const double D1 = ((((((0.0 + gzm.y) + gym.y) + gx2.x) + gx2.y) + gy2.y) + gz2.y + gs2.y) + gt2.y;
        const double Di0 = 1.0 / D0, Di1 = 1.0 / D1;
        double r0, r1;
        if (WARM) {
            double a = 0.0;
            a = a + gzm.x * xmz.x;
            a = a + gym.x * xmy.x;
            a = a + gxl * xl;
            a = a + gx2.x * x2.y;
            a = a + gy2.x * xpy.x;
            a = a + gz2.x * xpz.x;
            r0 = gs2.x - (D0 * x2.x - a);
            double b = 0.0;
            b = b + gzm.y * xmz.y;
            b = b + gym.y * xmy.y;
            b = b + gx2.x * x2.x;
            b = b + gx2.y * xr;
            b = b + gy2.y * xpy.y;
            b = b + gz2.y * xpz.y;
            r1 = gs2.y - (D1 * x2.y - b);
        } else {
            r0 = MODE == ASM_LAMBDA2 ? gs2.x - gt2.x : gs2.x;
            r1 = MODE == ASM_LAMBDA2 ? gs2.y - gt2.y : gs2.y;
        }
        const double z0 = r0 * Di0, z1 = r1 * Di1;
        stp(v.D, u0, make_double2(D0, D1));
        stp(v.Dinv, u0, make_double2(Di0, Di1));
        stp(v.r, u0, make_double2(r0, r1));
        stp(v.z, u0, make_double2(z0, z1));
        if (gs_out) {
            stp(gs_out, u0, gs2);
            stp(gt_out, u0, gt2);
        }
        const double b0 = MODE == ASM_LAMBDA2 ? gs2.x - gt2.x : gs2.x;
        const double b1 = MODE == ASM_LAMBDA2 ? gs2.y - gt2.y : gs2.y;
        const double mb0 = b0 * Di0, mb1 = b1 * Di1;
        acc[0] = acc[0] + r0 * z0;
        acc[1] = acc[1] + z0 * z0;
        acc[2] = acc[2] + r0 * r0;
        acc[3] = acc[3] + mb0 * mb0;
        acc[4] = acc[4] + b0 * b0;
        acc[0] = acc[0] + r1 * z1;
        acc[1] = acc[1] + z1 * z1;
        acc[2] = acc[2] + r1 * r1;
        acc[3] = acc[3] + mb1 * mb1;
        acc[4] = acc[4] + b1 * b1;
    }
    if (c3_chunk_epilogue<5>(acc, v.chunk0 + (int32_t)blockIdx.x, ra) && cd.finalize && threadIdx.x == 0) {
        finalize_start(ra.ctrl, ra.slots);
        set_cond2(cd, ra.ctrl);
    }
}


// ---------------------------------------------------------------------------
// K1 fused (reweight steps, nx a multiple of 512): one pass per chunk.  With
// nx = 512 m, thread t's pair of iteration j has its -y neighbour pair in
// iteration j - m of the SAME thread (same x), so the -y conductance comes
// from a thread-private shared-memory ring (no barrier); -x comes from the
// adjacent lane by shuffle (lane 0 recomputes it); -z (another chunk) and -y
// of the first m iterations are recomputed.  Same formula and operand order
// as the owner's computation, so the bits equal K1a + K1b and the oracle.
// 104 B/node of compulsory traffic instead of 136.
// ---------------------------------------------------------------------------
template <int MODE, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_pair_fused(StencilArgs s, VecArgs v, RedArgs ra, CondArgs cd,
                                                            double eps2, double *gs_out, double *gt_out)
{
    if (v.frozen && *(const volatile int32_t *)v.frozen) return;  // fixed point: this step repeats the last one
    __shared__ double2 ring[8][kThreads];
    const int lane = threadIdx.x & 31;
    const int64_t base = (int64_t)blockIdx.x * kChunk;
    const int64_t P = s.P;
    const int m = s.nx >> 9;
    const double2 zero2 = make_double2(0.0, 0.0);
    constexpr bool WARM = MODE == ASM_REWEIGHT_WARM;
    double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll 1
    for (int j = 0; j < 8; j++) {
        const int64_t u0 = base + 2 * (int64_t)threadIdx.x + 512 * j;
        const bool valid = u0 < v.n_own;
        const PairCoord c = pair_coord(s, s.lo + u0);
        const bool hx = c.x0 > 0, hr = c.x0 + 1 < s.nx - 1;
        const bool hy = valid && c.y > 0, py = valid && c.y < s.ny - 1;
        const bool hz = valid && c.z > 0, pz = valid && c.z < s.nz - 1;
        const bool ring_y = j >= m;  // -y pair computed by this thread in iteration j - m
        // ---- loads first
        const double2 x2 = valid ? ldp(v.x, u0) : zero2;
        const double2 cx2 = valid ? ldp(s.cx, u0) : zero2;
        const double2 cy2 = py ? ldp(s.cy, u0) : zero2, cz2 = pz ? ldp(s.cz, u0) : zero2;
        const double2 cs2 = valid ? ldp(s.cs, u0) : zero2, ct2 = valid ? ldp(s.ct, u0) : zero2;
        const double2 xpy = py ? ldp(v.x, u0 + s.nx) : zero2, xpz = pz ? ldp(v.x, u0 + P) : zero2;
        const double2 xmz = hz ? ldp(v.x, u0 - P) : zero2, czm = hz ? ldp(s.cz, u0 - P) : zero2;
        const double2 xmy = (hy && (WARM || !ring_y)) ? ldp(v.x, u0 - s.nx) : zero2;
        const double2 cym = (hy && !ring_y) ? ldp(s.cy, u0 - s.nx) : zero2;
        double xle = 0.0, cxle = 0.0, xre = 0.0;
        if (valid && lane == 0 && hx) {
            xle = __ldg(v.x + u0 - 1);
            cxle = __ldg(s.cx + u0 - 1);
        }
        if (valid && lane == 31 && hr) xre = __ldg(v.x + u0 + 2);
        double xl = __shfl_up_sync(0xffffffffu, x2.y, 1);
        double xr = __shfl_down_sync(0xffffffffu, x2.x, 1);
        if (lane == 0) xl = xle;
        if (lane == 31) xr = xre;
        if (!hx) xl = 0.0;
        if (!hr) xr = 0.0;
        // ---- owned edges (K1a)
        double2 gx2;
        gx2.x = valid ? rw_g(cx2.x, x2.x - x2.y, eps2) : 0.0;
        gx2.y = (valid && hr) ? rw_g(cx2.y, x2.y - xr, eps2) : 0.0;
        double gxl = __shfl_up_sync(0xffffffffu, gx2.y, 1);
        if (!valid) continue;
        if (lane == 0) gxl = hx ? rw_g(cxle, xl - x2.x, eps2) : 0.0;
        if (!hx) gxl = 0.0;
        const double2 gy2 = py ? make_double2(rw_g(cy2.x, x2.x - xpy.x, eps2), rw_g(cy2.y, x2.y - xpy.y, eps2)) : zero2;
        const double2 gz2 = pz ? make_double2(rw_g(cz2.x, x2.x - xpz.x, eps2), rw_g(cz2.y, x2.y - xpz.y, eps2)) : zero2;
        // ---- lower-neighbour edges: ring (-y), recompute (-z, first rows' -y)
        double2 gym = zero2;
        if (hy) gym = ring_y ? ring[j - m][threadIdx.x]
                             : make_double2(rw_g(cym.x, xmy.x - x2.x, eps2), rw_g(cym.y, xmy.y - x2.y, eps2));
        ring[j][threadIdx.x] = gy2;
        const double2 gzm = hz ? make_double2(rw_g(czm.x, xmz.x - x2.x, eps2), rw_g(czm.y, xmz.y - x2.y, eps2)) : zero2;
        stp(s.gx, u0, gx2);
        stp(s.gy, u0, gy2);
        stp(s.gz, u0, gz2);
        if (s.lo_ghost && u0 < P) stp(s.gz, u0 - P, gzm);  // the -z edge of the first owned plane (ghost slot)
        // ---- terminals, D, Dinv, r0, z0 (K1b)
        double2 gs2, gt2;
        gs2.x = terminal_g(cs2.x, ct2.x, x2.x, eps2, gt2.x);
        gs2.y = terminal_g(cs2.y, ct2.y, x2.y, eps2, gt2.y);
        const double D0 = ((((((0.0 + gzm.x) + gym.x) + gxl) + gx2.x) + gy2.x) + gz2.x + gs2.x) + gt2.x;
        const double D1 = ((((((0.0 + gzm.y) + gym.y) + gx2.x) + gx2.y) + gy2.y) + gz2.y + gs2.y) + gt2.y;
        const double Di0 = 1.0 / D0, Di1 = 1.0 / D1;
        double r0, r1;
        if (WARM) {
            double a = 0.0;
            a = a + gzm.x * xmz.x;
            a = a + gym.x * xmy.x;
            a = a + gxl * xl;
            a = a + gx2.x * x2.y;
            a = a + gy2.x * xpy.x;
            a = a + gz2.x * xpz.x;
            r0 = gs2.x - (D0 * x2.x - a);
            double b = 0.0;
            b = b + gzm.y * xmz.y;
            b = b + gym.y * xmy.y;
            b = b + gx2.x * x2.x;
            b = b + gx2.y * xr;
            b = b + gy2.y * xpy.y;
            b = b + gz2.y * xpz.y;
            r1 = gs2.y - (D1 * x2.y - b);
        } else {
            r0 = gs2.x;
            r1 = gs2.y;
        }
        const double z0 = r0 * Di0, z1 = r1 * Di1;
        stp(v.D, u0, make_double2(D0, D1));
        stp(v.Dinv, u0, make_double2(Di0, Di1));
        stp(v.r, u0, make_double2(r0, r1));
        stp(v.z, u0, make_double2(z0, z1));
        if (gs_out) {
            stp(gs_out, u0, gs2);
            stp(gt_out, u0, gt2);
        }
        const double mb0 = gs2.x * Di0, mb1 = gs2.y * Di1;
        acc[0] = acc[0] + r0 * z0;
        acc[1] = acc[1] + z0 * z0;
        acc[2] = acc[2] + r0 * r0;
        acc[3] = acc[3] + mb0 * mb0;
        acc[4] = acc[4] + gs2.x * gs2.x;
        acc[0] = acc[0] + r1 * z1;
        acc[1] = acc[1] + z1 * z1;
        acc[2] = acc[2] + r1 * r1;
        acc[3] = acc[3] + mb1 * mb1;
        acc[4] = acc[4] + gs2.y * gs2.y;
    }
    if (c3_chunk_epilogue<5>(acc, v.chunk0 + (int32_t)blockIdx.x, ra) && cd.finalize && threadIdx.x == 0) {
        finalize_start(ra.ctrl, ra.slots);
        set_cond2(cd, ra.ctrl);
    }
}

// ---------------------------------------------------------------------------
// K1 fused, TMA-fed (nx = 512, ny a multiple of 8: config 4's rows).  A chunk
// is 8 whole rows, iteration j = row y0 + j.  Instead of every thread loading
// its pair's operands into registers, one thread streams the rows the CTA
// needs into shared memory with 1-D bulk copies (cp.async.bulk, 4 KB per
// row) completing on mbarriers, up to two iterations ahead: per iteration x
// of row j+1 (kept in a 4-row ring, so the +-y neighbours' x come from the
// rows of the neighbouring iterations), x of the planes above and below, cx,
// cy, cz, cz of the plane below (cs, ct, used last, are plain loads).  The threads read their operands from shared
// memory (the -x / +x neighbours too: a row is self-contained) and compute
// exactly what k_pair_fused computes, in the same order (same bits).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity)
{
    // bounded: a phase that never completes (a byte-count bug) traps instead
    // of hanging the device
    for (long long spin = 0;; spin++) {
        uint32_t ok;
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n"
            "}\n"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (ok) return;
        if (spin > (1ll << 26)) __trap();
    }
}
__device__ __forceinline__ void bulk_row(double *dst, const double *src, uint64_t *bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(smem_u32(bar))
                 : "memory");
}

constexpr int kTR = 512;  // row length (doubles) of the TMA-fed K1

template <bool ZM>
struct K1Smem {
    double xr[4][kTR];             // x rows, slot (row + 1) & 3, rows -1 .. 8
    double st[2][6][kTR];          // per stage: xu, xd, cx, cy, cz, czd
    double cym0[kTR];              // cy of row -1 (iteration 0's -y conductance)
    double gzr[ZM ? 8 : 1][kTR];   // ZM: the previous plane's +z conductances (this plane's -z)
    unsigned long long bar[3];     // full[0], full[1], prologue
};

// ZM (z-march): CTA (chunk column, segment of zp planes) takes the chunks of
// its column plane after plane; the -z conductance of a node is the +z
// conductance the same thread computed for the node below in the previous
// chunk (kept in shared memory), so it is recomputed only in the segment's
// first plane.  Every chunk keeps its own C3 epilogue.
template <int MODE, int MINB, bool ZM>
__global__ void __launch_bounds__(kThreads, MINB) k_pair_fused_tma(StencilArgs s, VecArgs v, RedArgs ra, CondArgs cd,
                                                              double eps2, double *gs_out, double *gt_out, int zp)
{
    if (v.frozen && *(const volatile int32_t *)v.frozen) return;  // fixed point: this step repeats the last one
    extern __shared__ __align__(128) unsigned char k1_dyn[];
    K1Smem<ZM> &S = *reinterpret_cast<K1Smem<ZM> *>(k1_dyn);
    const int lane = threadIdx.x & 31, t = threadIdx.x;
    const int64_t P = s.P;
    const double2 zero2 = make_double2(0.0, 0.0);
    constexpr bool WARM = MODE == ASM_REWEIGHT_WARM;
    const int32_t Pc = ZM ? (int32_t)(P / kChunk) : 1;
    const int32_t cxi = ZM ? (int32_t)blockIdx.x % Pc : (int32_t)blockIdx.x;
    const int32_t zl0 = ZM ? ((int32_t)blockIdx.x / Pc) * zp : 0;
    const int32_t zl1 = ZM ? min(zl0 + zp, (int32_t)(v.n_own / P)) : 1;
    uint64_t *full = reinterpret_cast<uint64_t *>(S.bar);
    uint64_t *pro = full + 2;
    struct Geo {
        int64_t base;
        bool hz, pz, ylo, yhi, zr;
    };
    auto geo = [&](int32_t zl_) {
        Geo g;
        g.base = (int64_t)(ZM ? zl_ * Pc + cxi : cxi) * kChunk;
        // the chunk's rows: y0 .. y0 + 7 of plane z (global coordinates)
        const PairCoord c0 = pair_coord(s, s.lo + g.base);
        g.hz = c0.z > 0;
        g.pz = c0.z < s.nz - 1;
        g.ylo = c0.y > 0;
        g.yhi = c0.y + 8 < s.ny;
        g.zr = ZM && zl_ > zl0;  // -z conductances from the previous chunk of this CTA
        return g;
    };
    auto issue = [&](const Geo &g, int j) {  // stage j: x row j+1 and the per-iteration rows of row j
        const int b = j & 1;
        const int64_t r = g.base + (int64_t)kTR * j;
        const bool xnext = j < 7 || g.yhi;
        const bool czd = g.hz && !g.zr;
        const unsigned n = 3 + (xnext ? 1 : 0) + (g.pz ? 1 : 0) + (g.hz ? 1 : 0) + (czd ? 1 : 0);  // cx cy cz + optional
        mbar_expect_tx(&full[b], 4096u * n);
        if (xnext) bulk_row(S.xr[(j + 2) & 3], v.x + r + kTR, &full[b]);
        if (g.pz) bulk_row(S.st[b][0], v.x + r + P, &full[b]);
        if (g.hz) bulk_row(S.st[b][1], v.x + r - P, &full[b]);
        if (czd) bulk_row(S.st[b][5], s.cz + r - P, &full[b]);
        bulk_row(S.st[b][2], s.cx + r, &full[b]);
        bulk_row(S.st[b][3], s.cy + r, &full[b]);
        bulk_row(S.st[b][4], s.cz + r, &full[b]);
    };
    auto start = [&](const Geo &g) {  // the chunk's prologue rows and its first two stages
        mbar_expect_tx(pro, 4096u * (g.ylo ? 3u : 1u));
        bulk_row(S.xr[1], v.x + g.base, pro);
        if (g.ylo) {
            bulk_row(S.xr[0], v.x + g.base - kTR, pro);
            bulk_row(S.cym0, s.cy + g.base - kTR, pro);
        }
        issue(g, 0);
        issue(g, 1);
    };
    if (t == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        mbar_init(pro, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        start(geo(zl0));
    }
    __syncthreads();
#pragma unroll 1
    for (int32_t zl = zl0; zl < zl1; zl++) {
    const Geo G = geo(zl);
    const int32_t chunk = ZM ? zl * Pc + cxi : cxi;
    const int64_t base = G.base;
    const bool zr = G.zr, hz = G.hz, pz = G.pz, ylo = G.ylo, yhi = G.yhi;
    double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    double2 gyprev = zero2;  // gy2 of the previous iteration (the -y conductance of this one)
    mbar_wait(pro, (unsigned)(zl - zl0) & 1u);
#pragma unroll 1
    for (int j = 0; j < 8; j++) {
        const int64_t u0 = base + 2 * (int64_t)t + kTR * j;
        // the terminal capacities straight to registers (used last)
        const double2 cs2 = ldp(s.cs, u0), ct2 = ldp(s.ct, u0);
        mbar_wait(&full[j & 1], (j >> 1) & 1);
        const int b = j & 1;
        const bool hx = t > 0, hr = t < kThreads - 1;
        const bool hy = ylo || j > 0, py = yhi || j < 7;
        const double *xrow = S.xr[(j + 1) & 3];
        const double2 x2 = *reinterpret_cast<const double2 *>(xrow + 2 * t);
        const double2 cx2 = *reinterpret_cast<const double2 *>(S.st[b][2] + 2 * t);
        const double2 cy2 = py ? *reinterpret_cast<const double2 *>(S.st[b][3] + 2 * t) : zero2;
        const double2 cz2 = pz ? *reinterpret_cast<const double2 *>(S.st[b][4] + 2 * t) : zero2;
        const double2 xpy = py ? *reinterpret_cast<const double2 *>(S.xr[(j + 2) & 3] + 2 * t) : zero2;
        const double2 xpz = pz ? *reinterpret_cast<const double2 *>(S.st[b][0] + 2 * t) : zero2;
        const double2 xmz = hz ? *reinterpret_cast<const double2 *>(S.st[b][1] + 2 * t) : zero2;
        const double2 czm = (hz && !zr) ? *reinterpret_cast<const double2 *>(S.st[b][5] + 2 * t) : zero2;
        const double2 xmy = (hy && (WARM || j == 0)) ? *reinterpret_cast<const double2 *>(S.xr[j & 3] + 2 * t) : zero2;
        const double2 cym = (hy && j == 0) ? *reinterpret_cast<const double2 *>(S.cym0 + 2 * t) : zero2;
        const double xl = hx ? xrow[2 * t - 1] : 0.0;
        const double xr = hr ? xrow[2 * t + 2] : 0.0;
        const double cxl = hx ? S.st[b][2][2 * t - 1] : 0.0;
        // ---- owned edges (K1a)
        double2 gx2;
        gx2.x = rw_g(cx2.x, x2.x - x2.y, eps2);
        gx2.y = hr ? rw_g(cx2.y, x2.y - xr, eps2) : 0.0;
        double gxl = __shfl_up_sync(0xffffffffu, gx2.y, 1);
        if (lane == 0) gxl = hx ? rw_g(cxl, xl - x2.x, eps2) : 0.0;
        if (!hx) gxl = 0.0;
        const double2 gy2 = py ? make_double2(rw_g(cy2.x, x2.x - xpy.x, eps2), rw_g(cy2.y, x2.y - xpy.y, eps2)) : zero2;
        const double2 gz2 = pz ? make_double2(rw_g(cz2.x, x2.x - xpz.x, eps2), rw_g(cz2.y, x2.y - xpz.y, eps2)) : zero2;
        // ---- lower-neighbour edges: previous iteration (-y), recompute (-z, row 0's -y)
        double2 gym = zero2;
        if (hy) gym = j > 0 ? gyprev : make_double2(rw_g(cym.x, xmy.x - x2.x, eps2), rw_g(cym.y, xmy.y - x2.y, eps2));
        gyprev = gy2;
        double2 gzm = zero2;
        if (hz)
            gzm = zr ? *reinterpret_cast<const double2 *>(S.gzr[ZM ? j : 0] + 2 * t)
                     : make_double2(rw_g(czm.x, xmz.x - x2.x, eps2), rw_g(czm.y, xmz.y - x2.y, eps2));
        if (ZM) *reinterpret_cast<double2 *>(S.gzr[ZM ? j : 0] + 2 * t) = gz2;
        stp(s.gx, u0, gx2);
        stp(s.gy, u0, gy2);
        stp(s.gz, u0, gz2);
        if (s.lo_ghost && u0 < P) stp(s.gz, u0 - P, gzm);  // the -z edge of the first owned plane (ghost slot)
        // ---- terminals, D, Dinv, r0, z0 (K1b)
        double2 gs2, gt2;
        gs2.x = terminal_g(cs2.x, ct2.x, x2.x, eps2, gt2.x);
        gs2.y = terminal_g(cs2.y, ct2.y, x2.y, eps2, gt2.y);
        const double D0 = ((((((0.0 + gzm.x) + gym.x) + gxl) + gx2.x) + gy2.x) + gz2.x + gs2.x) + gt2.x;
        const double D1 = ((((((0.0 + gzm.y) + gym.y) + gx2.x) + gx2.y) + gy2.y) + gz2.y + gs2.y) + gt2.y;
        const double Di0 = 1.0 / D0, Di1 = 1.0 / D1;
        double r0, r1;
        if (WARM) {
            double a = 0.0;
            a = a + gzm.x * xmz.x;
            a = a + gym.x * xmy.x;
            a = a + gxl * xl;
            a = a + gx2.x * x2.y;
            a = a + gy2.x * xpy.x;
            a = a + gz2.x * xpz.x;
            r0 = gs2.x - (D0 * x2.x - a);
            double bb = 0.0;
            bb = bb + gzm.y * xmz.y;
            bb = bb + gym.y * xmy.y;
            bb = bb + gx2.x * x2.x;
            bb = bb + gx2.y * xr;
            bb = bb + gy2.y * xpy.y;
            bb = bb + gz2.y * xpz.y;
            r1 = gs2.y - (D1 * x2.y - bb);
        } else {
            r0 = gs2.x;
            r1 = gs2.y;
        }
        const double z0 = r0 * Di0, z1 = r1 * Di1;
        stp(v.D, u0, make_double2(D0, D1));
        stp(v.Dinv, u0, make_double2(Di0, Di1));
        stp(v.r, u0, make_double2(r0, r1));
        stp(v.z, u0, make_double2(z0, z1));
        if (gs_out) {
            stp(gs_out, u0, gs2);
            stp(gt_out, u0, gt2);
        }
        const double mb0 = gs2.x * Di0, mb1 = gs2.y * Di1;
        acc[0] = acc[0] + r0 * z0;
        acc[1] = acc[1] + z0 * z0;
        acc[2] = acc[2] + r0 * r0;
        acc[3] = acc[3] + mb0 * mb0;
        acc[4] = acc[4] + gs2.x * gs2.x;
        acc[0] = acc[0] + r1 * z1;
        acc[1] = acc[1] + z1 * z1;
        acc[2] = acc[2] + r1 * r1;
        acc[3] = acc[3] + mb1 * mb1;
        acc[4] = acc[4] + gs2.y * gs2.y;
        if (j + 2 < 8) {
            __syncthreads();  // stage j's buffers and x row j-1 are free
            if (t == 0) issue(G, j + 2);
        }
    }
    if (ZM && zl + 1 < zl1) {  // the next chunk's rows while this one reduces (-2% against after it)
        __syncthreads();  // every thread is done with this chunk's staging buffers
        if (t == 0) start(geo(zl + 1));
    }
    if (c3_chunk_epilogue<5>(acc, v.chunk0 + chunk, ra) && cd.finalize && threadIdx.x == 0) {
        finalize_start(ra.ctrl, ra.slots);
        set_cond2(cd, ra.ctrl);
    }
    }
}

// ---------------------------------------------------------------------------
// K3: p = z + beta p_old (recomputed for neighbours), lazy x update, q = L~ p
// ---------------------------------------------------------------------------
// W0: CG-CG's w0 = A z0 pass (k = 0), which runs after the START stopping
// test: it returns at once when that test already stopped the solve, and its
// fused finalize also sets the loop condition (alpha_0 breakdown).
template <bool W0>
__global__ void __launch_bounds__(kThreads) k_pair_pspmv(StencilArgs s, VecArgs v, RedArgs ra, CondArgs cd)
{
    const DevCtrl *ctrl = ra.ctrl;
    if (W0 && ctrl->done) return;
    const int32_t k = ctrl->k;
    const bool first = (k == 0);
    const double beta = ctrl->beta, alpha = ctrl->alpha;
    const double *__restrict__ pold = (k & 1) ? v.p1 : v.p0;
    double *__restrict__ pnew = (k & 1) ? v.p0 : v.p1;
    const double *__restrict__ zv = v.z;
    const int lane = threadIdx.x & 31;
    const int64_t base = (int64_t)blockIdx.x * kChunk;
    const int64_t P = s.P;
    const double2 zero2 = make_double2(0.0, 0.0);
    double acc[1] = {0.0};
#pragma unroll 1
    for (int j = 0; j < 8; j++) {
        const int64_t u0 = base + 2 * (int64_t)threadIdx.x + 512 * j;
        const bool valid = u0 < v.n_own;
        const PairCoord c = pair_coord(s, s.lo + u0);
        const bool hx = c.x0 > 0, hr = c.x0 + 1 < s.nx - 1;
        const bool hy = valid && c.y > 0, py = valid && c.y < s.ny - 1;
        const bool hz = valid && c.z > 0, pz = valid && c.z < s.nz - 1;
        // ---- issue every load of this pair first (memory-level parallelism)
        const double2 z2 = ldp(zv, u0);
        const double2 zmz = hz ? ldp(zv, u0 - P) : zero2;
        const double2 zmy = hy ? ldp(zv, u0 - s.nx) : zero2;
        const double2 zpy = py ? ldp(zv, u0 + s.nx) : zero2;
        const double2 zpz = pz ? ldp(zv, u0 + P) : zero2;
        double2 po = zero2, pmz = zero2, pmy = zero2, ppy = zero2, ppz = zero2;
        if (!first) {
            po = ldp(pold, u0);
            if (hz) pmz = ldp(pold, u0 - P);
            if (hy) pmy = ldp(pold, u0 - s.nx);
            if (py) ppy = ldp(pold, u0 + s.nx);
            if (pz) ppz = ldp(pold, u0 + P);
        }
        const double2 gx2 = ldp(s.gx, u0);
        const double2 gy2 = valid ? ldp(s.gy, u0) : zero2, gz2 = valid ? ldp(s.gz, u0) : zero2;
        const double2 gym = hy ? ldp(s.gy, u0 - s.nx) : zero2;
        const double2 gzm = hz ? ldp(s.gz, u0 - P) : zero2;
        const double2 D2 = valid ? ldp(v.D, u0) : zero2;
        double2 x2 = zero2;
        if (!first && valid) x2 = ldp_cg(v.x, u0);
        double zl = 0.0, pol = 0.0, gxe = 0.0, zr = 0.0, por = 0.0;
        if (valid && lane == 0 && hx) {
            zl = __ldg(zv + u0 - 1);
            gxe = __ldg(s.gx + u0 - 1);
            if (!first) pol = __ldg(pold + u0 - 1);
        }
        if (valid && lane == 31 && hr) {
            zr = __ldg(zv + u0 + 2);
            if (!first) por = __ldg(pold + u0 + 2);
        }
        // ---- p = z + beta p_old
        double2 p2 = z2;
        if (!first) p2 = make_double2(z2.x + beta * po.x, z2.y + beta * po.y);
        double pl = __shfl_up_sync(0xffffffffu, p2.y, 1);
        double pr = __shfl_down_sync(0xffffffffu, p2.x, 1);
        double gxl = __shfl_up_sync(0xffffffffu, gx2.y, 1);
        if (!valid) continue;
        if (lane == 0) { pl = first ? zl : zl + beta * pol; gxl = gxe; }
        if (lane == 31) pr = first ? zr : zr + beta * por;
        if (!hx) { pl = 0.0; gxl = 0.0; }
        if (!hr) pr = 0.0;
        double2 qmz = zmz, qmy = zmy, qpy = zpy, qpz = zpz;
        if (!first) {
            qmz = make_double2(zmz.x + beta * pmz.x, zmz.y + beta * pmz.y);
            qmy = make_double2(zmy.x + beta * pmy.x, zmy.y + beta * pmy.y);
            qpy = make_double2(zpy.x + beta * ppy.x, zpy.y + beta * ppy.y);
            qpz = make_double2(zpz.x + beta * ppz.x, zpz.y + beta * ppz.y);
        }
        double a = 0.0;
        a = a + gzm.x * qmz.x;
        a = a + gym.x * qmy.x;
        a = a + gxl * pl;
        a = a + gx2.x * p2.y;
        a = a + gy2.x * qpy.x;
        a = a + gz2.x * qpz.x;
        double b = 0.0;
        b = b + gzm.y * qmz.y;
        b = b + gym.y * qmy.y;
        b = b + gx2.x * p2.x;
        b = b + gx2.y * pr;
        b = b + gy2.y * qpy.y;
        b = b + gz2.y * qpz.y;
        const double q0 = D2.x * p2.x - a, q1 = D2.y * p2.y - b;
        stp(pnew, u0, p2);
        stp(v.q, u0, make_double2(q0, q1));
        if (!first) stp(v.x, u0, make_double2(x2.x + alpha * po.x, x2.y + alpha * po.y));
        acc[0] = acc[0] + p2.x * q0;
        acc[0] = acc[0] + p2.y * q1;
    }
    if (c3_chunk_epilogue<1>(acc, v.chunk0 + (int32_t)blockIdx.x, ra) && cd.finalize && threadIdx.x == 0) {
        finalize_pq(ra.ctrl, ra.slots);
        if (W0) set_cond2(cd, ra.ctrl);
    }
}

// ---------------------------------------------------------------------------
// K5 (vectorised; any graph): r -= alpha q, z = Dinv r, RZ reductions.
// Requires n_own even or arrays padded (they are padded to whole chunks).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_pair_axpy(VecArgs v, RedArgs ra, CondArgs cd)
{
    DevCtrl *ctrl = ra.ctrl;
    if (ctrl->done) {
        if (blockIdx.x == 0 && threadIdx.x == 0) set_cond2(cd, ctrl);
        return;
    }
    const double alpha = ctrl->alpha;
    const int64_t base = (int64_t)blockIdx.x * kChunk;
    double acc[3] = {0.0, 0.0, 0.0};
    bool peer = false;
#pragma unroll 2
    for (int j = 0; j < 8; j++) {
        const int64_t u0 = base + 2 * (int64_t)threadIdx.x + 512 * j;
        if (u0 >= v.n_own) break;
        const double2 r2 = ldp_cg(v.r, u0), q2 = ldp(v.q, u0), d2 = ldp(v.Dinv, u0);
        const double r0 = r2.x - alpha * q2.x, r1 = r2.y - alpha * q2.y;
        const double z0 = r0 * d2.x, z1 = r1 * d2.y;
        stp(v.r, u0, make_double2(r0, r1));
        stp(v.z, u0, make_double2(z0, z1));
        if (v.zpeer_lo && u0 < v.plane) {  // fused halo: first owned plane -> lower neighbour
            v.zpeer_lo[u0] = z0;
            if (u0 + 1 < v.plane) v.zpeer_lo[u0 + 1] = z1;
            peer = true;
        }
        if (v.zpeer_hi && u0 + 1 >= v.n_own - v.plane) {  // last owned plane -> upper neighbour
            const int64_t b = v.n_own - v.plane;
            if (u0 >= b) v.zpeer_hi[u0 - b] = z0;
            if (u0 + 1 < v.n_own) v.zpeer_hi[u0 + 1 - b] = z1;
            peer = true;
        }
        acc[0] = acc[0] + r0 * z0;
        acc[1] = acc[1] + z0 * z0;
        acc[2] = acc[2] + r0 * r0;
        if (u0 + 1 < v.n_own) {
            acc[0] = acc[0] + r1 * z1;
            acc[1] = acc[1] + z1 * z1;
            acc[2] = acc[2] + r1 * r1;
        }
    }
    // the peer stores are visible system-wide before this block's partial
    // (and so before the group's arrival at any peer) is published
    if (peer) __threadfence_system();
    if (c3_chunk_epilogue<3>(acc, v.chunk0 + (int32_t)blockIdx.x, ra) && cd.finalize && threadIdx.x == 0) {
        finalize_rz(ctrl, ra.slots);
        set_cond2(cd, ctrl);
    }
}

// ---------------------------------------------------------------------------
// Chronopoulos-Gear iteration on node pairs (nx even; O5', A31): the
// kernels_cg.cu k_cgcg_stencil arithmetic with K3's data movement — every
// load of the pair first, -x / +x neighbours' new z by shuffle (lanes 0 / 31
// recompute theirs), -y / +y / -z / +z recomputed from r, w, s_old, Dinv.
// ---------------------------------------------------------------------------
struct CgNb {
    double2 r, w, s, d;
};

template <int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_cgcg_pair(StencilArgs s, VecArgs v, CgArgs g, RedArgs ra,
                                                           CondArgs cd)
{
    DevCtrl *ctrl = ra.ctrl;
    if (ctrl->done) {
        if (blockIdx.x == 0 && threadIdx.x == 0) set_cond2(cd, ctrl);
        return;
    }
    const int32_t k = ctrl->k;
    const bool first = (k == 0);
    const double alpha = ctrl->alpha, beta = ctrl->beta;
    const double *__restrict__ rk = g.r[k & 1];
    const double *__restrict__ wk = g.w[k & 1];
    const double *__restrict__ so = g.s[(k + 1) & 1];
    double *__restrict__ rn = g.r[(k + 1) & 1];
    double *__restrict__ wn = g.w[(k + 1) & 1];
    double *__restrict__ sn = g.s[k & 1];
    const double *__restrict__ di = v.Dinv;
    const int lane = threadIdx.x & 31;
    const int64_t base = (int64_t)blockIdx.x * kChunk;
    const int64_t P = s.P;
    const double2 zero2 = make_double2(0.0, 0.0);
    auto ldnb = [&](bool has, int64_t i) {
        CgNb n{zero2, zero2, zero2, zero2};
        if (has) {
            n.r = ldp(rk, i);
            n.w = ldp(wk, i);
            if (!first) n.s = ldp(so, i);
            n.d = ldp(di, i);
        }
        return n;
    };
    // new z of a neighbour: (r - alpha (w | w + beta s_old)) Dinv
    auto znew = [&](double r, double w, double so_, double d) {
        const double sv = first ? w : w + beta * so_;
        return (r - alpha * sv) * d;
    };
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    double *wl = g.wpeer_lo[(k + 1) & 1], *wh = g.wpeer_hi[(k + 1) & 1];
    bool peer = false;
#pragma unroll 1
    for (int j = 0; j < 8; j++) {
        const int64_t u0 = base + 2 * (int64_t)threadIdx.x + 512 * j;
        const bool valid = u0 < v.n_own;
        const PairCoord c = pair_coord(s, s.lo + u0);
        const bool hx = c.x0 > 0, hr = c.x0 + 1 < s.nx - 1;
        const bool hy = valid && c.y > 0, py = valid && c.y < s.ny - 1;
        const bool hz = valid && c.z > 0, pz = valid && c.z < s.nz - 1;
        // ---- own pair first: s, z, p, x, r', z'
        const CgNb own = ldnb(valid, u0);
        const double2 po = (valid && !first) ? ldp(g.p, u0) : zero2;
        const double2 gx2 = valid ? ldp(s.gx, u0) : zero2;
        const double2 x2 = valid ? ldp_cg(v.x, u0) : zero2;
        double el_r = 0.0, el_w = 0.0, el_s = 0.0, el_d = 0.0, gxe = 0.0;
        double er_r = 0.0, er_w = 0.0, er_s = 0.0, er_d = 0.0;
        if (valid && lane == 0 && hx) {
            el_r = __ldg(rk + u0 - 1);
            el_w = __ldg(wk + u0 - 1);
            if (!first) el_s = __ldg(so + u0 - 1);
            el_d = __ldg(di + u0 - 1);
            gxe = __ldg(s.gx + u0 - 1);
        }
        if (valid && lane == 31 && hr) {
            er_r = __ldg(rk + u0 + 2);
            er_w = __ldg(wk + u0 + 2);
            if (!first) er_s = __ldg(so + u0 + 2);
            er_d = __ldg(di + u0 + 2);
        }
        const double s0 = first ? own.w.x : own.w.x + beta * own.s.x;
        const double s1 = first ? own.w.y : own.w.y + beta * own.s.y;
        const double z0 = own.r.x * own.d.x, z1 = own.r.y * own.d.y;
        const double p0 = first ? z0 : z0 + beta * po.x;
        const double p1 = first ? z1 : z1 + beta * po.y;
        const double r0 = own.r.x - alpha * s0, r1 = own.r.y - alpha * s1;
        const double zn0 = r0 * own.d.x, zn1 = r1 * own.d.y;
        double zl = __shfl_up_sync(0xffffffffu, zn1, 1);
        double zr = __shfl_down_sync(0xffffffffu, zn0, 1);
        double gxl = __shfl_up_sync(0xffffffffu, gx2.y, 1);
        if (!valid) continue;
        if (lane == 0) { zl = znew(el_r, el_w, el_s, el_d); gxl = gxe; }
        if (lane == 31) zr = znew(er_r, er_w, er_s, er_d);
        if (!hx) { zl = 0.0; gxl = 0.0; }
        if (!hr) zr = 0.0;
        // ---- w' = D z' - sum_asc g z'_nbr (O2: -z, -y, -x, +x, +y, +z), one
        // neighbour direction at a time (keeps the live state small)
        auto zpair = [&](const CgNb &n) {
            return make_double2(znew(n.r.x, n.w.x, n.s.x, n.d.x), znew(n.r.y, n.w.y, n.s.y, n.d.y));
        };
        double a = 0.0, b = 0.0;
        {
            const double2 gzm = hz ? ldp(s.gz, u0 - P) : zero2;
            const double2 zz = zpair(ldnb(hz, u0 - P));
            a = a + gzm.x * zz.x;
            b = b + gzm.y * zz.y;
        }
        {
            const double2 gym = hy ? ldp(s.gy, u0 - s.nx) : zero2;
            const double2 zz = zpair(ldnb(hy, u0 - s.nx));
            a = a + gym.x * zz.x;
            b = b + gym.y * zz.y;
        }
        a = a + gxl * zl;
        a = a + gx2.x * zn1;
        b = b + gx2.x * zn0;
        b = b + gx2.y * zr;
        {
            const double2 gy2 = ldp(s.gy, u0);
            const double2 zz = zpair(ldnb(py, u0 + s.nx));
            a = a + gy2.x * zz.x;
            b = b + gy2.y * zz.y;
        }
        {
            const double2 gz2 = ldp(s.gz, u0);
            const double2 zz = zpair(ldnb(pz, u0 + P));
            a = a + gz2.x * zz.x;
            b = b + gz2.y * zz.y;
        }
        const double2 D2 = ldp(v.D, u0);
        const double w0 = D2.x * zn0 - a, w1 = D2.y * zn1 - b;
        stp(g.p, u0, make_double2(p0, p1));
        stp(sn, u0, make_double2(s0, s1));
        stp(v.x, u0, make_double2(x2.x + alpha * p0, x2.y + alpha * p1));
        stp(rn, u0, make_double2(r0, r1));
        stp(wn, u0, make_double2(w0, w1));
        if (wl && u0 < g.plane) {  // fused w halo (p2p): first owned plane -> lower neighbour
            wl[u0] = w0;
            wl[u0 + 1] = w1;
            peer = true;
        }
        if (wh && u0 >= v.n_own - g.plane) {  // last owned plane -> upper neighbour
            wh[u0 - (v.n_own - g.plane)] = w0;
            wh[u0 + 1 - (v.n_own - g.plane)] = w1;
            peer = true;
        }
        acc[0] = acc[0] + r0 * zn0;
        acc[1] = acc[1] + zn0 * w0;
        acc[2] = acc[2] + zn0 * zn0;
        acc[3] = acc[3] + r0 * r0;
        acc[0] = acc[0] + r1 * zn1;
        acc[1] = acc[1] + zn1 * w1;
        acc[2] = acc[2] + zn1 * zn1;
        acc[3] = acc[3] + r1 * r1;
    }
    if (peer) __threadfence_system();
    if (c3_chunk_epilogue<4>(acc, v.chunk0 + (int32_t)blockIdx.x, ra) && cd.finalize && threadIdx.x == 0) {
        finalize_cgcg(ctrl, ra.slots);
        set_cond2(cd, ctrl);
    }
}

// After the loop: x += alpha_{k-1} p_{k-1} (or 0 when b = 0); grid-stride over
// pairs with a small grid, so an idle call (k = 0) costs one short launch.
__global__ void __launch_bounds__(256) k_pair_finish(VecArgs v, const DevCtrl *ctrl)
{
    const int32_t k = ctrl->k;
    const bool zero = ctrl->zero_x != 0;
    if (!zero && (k == 0 || ctrl->status != ST_OK)) return;
    const double alpha = ctrl->alpha;
    const double *pl = (k & 1) ? v.p1 : v.p0;
    const int64_t npairs = (v.n_own + 1) / 2;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npairs; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t u0 = 2 * i;
        if (zero) {
            stp(v.x, u0, make_double2(0.0, 0.0));
        } else {
            const double2 x2 = ldp_cg(v.x, u0), p2 = ldp(pl, u0);
            stp(v.x, u0, make_double2(x2.x + alpha * p2.x, x2.y + alpha * p2.y));
        }
    }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
static inline unsigned nblk(int64_t n_own) { return (unsigned)((n_own + kChunk - 1) / kChunk); }

int launch_pair_assemble(const StencilArgs &s, const VecArgs &v, const RedArgs &ra, const CondArgs &cd, int mode,
                          double eps, double *gs_out, double *gt_out, cudaStream_t st)
{
    const double eps2 = eps * eps;
    const unsigned nb = nblk(v.n_own);
    if (mode == ASM_INIT || mode == ASM_LAMBDA2) {
        k_pair_edges<true><<<nb, kThreads, 0, st>>>(s, v, eps2);
        if (mode == ASM_INIT) k_pair_nodes<ASM_INIT><<<nb, kThreads, 0, st>>>(s, v, ra, cd, eps2, gs_out, gt_out);
        else k_pair_nodes<ASM_LAMBDA2><<<nb, kThreads, 0, st>>>(s, v, ra, cd, eps2, gs_out, gt_out);
    } else if (s.nx % 512 == 0 && s.nx <= 4096) {  // fused single pass
        // 3 CTAs/SM (80 registers): measured on config 4 1.57 ms vs 1.64 (two
        // passes), 1.90 (4 CTAs/SM, spills) and 1.70 (2 CTAs/SM); a z-cluster
        // variant (8 CTAs, -z conductances from the CTA below via DSMEM after a
        // cluster barrier) measured 2.40 ms (round 2)
        // TMA-fed variant for rows of exactly 512 in whole 8-row chunks
        const bool tma = s.nx == 512 && s.ny % 8 == 0 && v.n_own % kChunk == 0 && !getenv("IRLS_K1_NOTMA");
        if (tma) {
            // 2 CTAs/SM (108 registers, 68 KB of staging each): config 4 1.485 ms
            // against 1.55-1.57 ms for k_pair_fused; at 3 CTAs/SM (85
            // registers) it spills: 1.73 ms
            static bool attr = false;
            if (!attr) {
                cudaFuncSetAttribute(k_pair_fused_tma<ASM_REWEIGHT_WARM, 2, false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(K1Smem<false>));
                cudaFuncSetAttribute(k_pair_fused_tma<ASM_REWEIGHT_COLD, 2, false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(K1Smem<false>));
                cudaFuncSetAttribute(k_pair_fused_tma<ASM_REWEIGHT_WARM, 2, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(K1Smem<true>));
                cudaFuncSetAttribute(k_pair_fused_tma<ASM_REWEIGHT_COLD, 2, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(K1Smem<true>));
                attr = true;
            }
            // z-march segments of 8 planes (2,048 CTAs on config 4): 1.42 ms against
            // 1.50 ms per chunk (same box); 4 planes 1.46 ms, 16 1.52-1.54, 32 1.59
            // (fewer CTAs than 7 waves of 296 leave a tail); IRLS_K1_ZP overrides
            static const int zp_env = getenv("IRLS_K1_ZP") ? atoi(getenv("IRLS_K1_ZP")) : 8;
            const int64_t nzl = v.n_own / s.P;
            const bool zm = zp_env > 1 && v.n_own % s.P == 0 && nzl > 1;
            if (zm) {
                const int zp = (int)std::min<int64_t>(zp_env, nzl);
                const unsigned g = (unsigned)((s.P / kChunk) * ((nzl + zp - 1) / zp));
                if (mode == ASM_REWEIGHT_WARM)
                    k_pair_fused_tma<ASM_REWEIGHT_WARM, 2, true><<<g, kThreads, sizeof(K1Smem<true>), st>>>(
                        s, v, ra, cd, eps2, gs_out, gt_out, zp);
                else
                    k_pair_fused_tma<ASM_REWEIGHT_COLD, 2, true><<<g, kThreads, sizeof(K1Smem<true>), st>>>(
                        s, v, ra, cd, eps2, gs_out, gt_out, zp);
            } else if (mode == ASM_REWEIGHT_WARM)
                k_pair_fused_tma<ASM_REWEIGHT_WARM, 2, false><<<nb, kThreads, sizeof(K1Smem<false>), st>>>(
                    s, v, ra, cd, eps2, gs_out, gt_out, 1);
            else
                k_pair_fused_tma<ASM_REWEIGHT_COLD, 2, false><<<nb, kThreads, sizeof(K1Smem<false>), st>>>(
                    s, v, ra, cd, eps2, gs_out, gt_out, 1);
        } else if (mode == ASM_REWEIGHT_WARM)
            k_pair_fused<ASM_REWEIGHT_WARM, 3><<<nb, kThreads, 0, st>>>(s, v, ra, cd, eps2, gs_out, gt_out);
        else
            k_pair_fused<ASM_REWEIGHT_COLD, 3><<<nb, kThreads, 0, st>>>(s, v, ra, cd, eps2, gs_out, gt_out);
        return 1;
    } else {
        k_pair_edges<false><<<nb, kThreads, 0, st>>>(s, v, eps2);
        if (mode == ASM_REWEIGHT_WARM)
            k_pair_nodes<ASM_REWEIGHT_WARM><<<nb, kThreads, 0, st>>>(s, v, ra, cd, eps2, gs_out, gt_out);
        else
            k_pair_nodes<ASM_REWEIGHT_COLD><<<nb, kThreads, 0, st>>>(s, v, ra, cd, eps2, gs_out, gt_out);
    }
    return 2;
}

void launch_pair_pspmv(const StencilArgs &s, const VecArgs &v, const RedArgs &ra, const CondArgs &cd,
                       cudaStream_t st, bool w0)
{
    if (w0) k_pair_pspmv<true><<<nblk(v.n_own), kThreads, 0, st>>>(s, v, ra, cd);
    else k_pair_pspmv<false><<<nblk(v.n_own), kThreads, 0, st>>>(s, v, ra, cd);
}

void launch_pair_axpy(const VecArgs &v, const RedArgs &ra, const CondArgs &cd, cudaStream_t st)
{
    k_pair_axpy<<<nblk(v.n_own), kThreads, 0, st>>>(v, ra, cd);
}

void launch_pair_cgcg(const StencilArgs &s, const VecArgs &v, const CgArgs &g, const RedArgs &ra, const CondArgs &cd,
                      cudaStream_t st)
{
    // 3 CTAs/SM (80 registers): config 4 282.8 ms per step vs 293.9 (2 CTAs/SM)
    // and 379.6 (1 CTA/SM, 180 registers); the generic per-node kernel 326.5
    k_cgcg_pair<3><<<nblk(v.n_own), kThreads, 0, st>>>(s, v, g, ra, cd);
}

void launch_pair_finish(const VecArgs &v, DevCtrl *ctrl, cudaStream_t st)
{
    const int64_t npairs = (v.n_own + 1) / 2;
    const unsigned nb = (unsigned)std::min<int64_t>((npairs + 255) / 256, 148 * 8);
    k_pair_finish<<<nb > 0 ? nb : 1, 256, 0, st>>>(v, ctrl);
}

}  // namespace irls
