// block_jacobi.cu — block-Jacobi preconditioner kernels (reading A32;
// SURVEY §8(f) NEXT #2; the paper's block Jacobi with exact "LU" blocks,
// P:L235-242).
//
// M = blockdiag(A_B): the blocks are BFS patches of at most B nodes inside
// one C3 group (built on the host, api_block.cu), A_B = L~ restricted to a
// block in block order.  Per IRLS step KF factors every block as
// A_B = L D L^T; per CG iteration KB applies z = M^-1 r.  The arithmetic is
// the oracle's written definition (C1: no FMA, IEEE '/'), every sum in the
// definition's order:
//   L_ij = (A_ij - sum_{k asc} (L_ik * L_jk) * d_k) / d_j
//   d_i  =  A_ii - sum_{k asc} (L_ik * L_ik) * d_k
//   forward  y_i = r_i - sum_{k asc} L_ik * y_k ;  w_i = y_i / d_i
//   backward z_k = w_k - sum_{i desc} L_ik * z_i
// executed literally by rows, one thread per block, the 32 blocks of a warp
// stored interleaved (one 256-byte access per band element).  Row i is
// stored over [rowF, i), the union of the warp's 32 envelopes; the entries
// outside a block's own envelope are exact zeros of the dense algorithm (A32:
// every update with them is a bitwise no-op), so the bits are the dense
// definition's, i.e. the oracle's.  For blocks of at most 16 nodes the
// right-hand sides live in registers (fully unrolled recurrences).
//
// KR then forms the C3 reductions of the solve (START: <r,z>, <z,z>, <r,r>,
// <M^-1 b, M^-1 b>, <b,b>; per iteration: <r,z>, <z,z>, <r,r>) in the
// standard chunk mapping, so the finalizers are K1's / K5's.
#include <algorithm>
#include "kernels.h"

namespace irls {

struct Lane {
    int32_t p0, m;
    int64_t R0;
    double *L;   // &band[G][0][l]
    double *Dd;  // &pivots[G][0][l]
};

__device__ __forceinline__ Lane lane_of(const BlockArgs &b, int64_t blk)
{
    Lane t;
    const int64_t G = blk >> 5, l = blk & 31;
    t.p0 = b.bptr[blk];
    t.m = b.bptr[blk + 1] - t.p0;
    t.R0 = b.gR[G];
    t.L = b.L + 32 * b.gL[G] + l;
    t.Dd = b.Dd + 32 * t.R0 + l;
    return t;
}

// row i of the lane's block: element (i, k) at row[32 k]
__device__ __forceinline__ double *band_row(const BlockArgs &b, const Lane &t, int i, int32_t &F)
{
    F = b.rowF[t.R0 + i];
    return t.L + 32 * ((int64_t)b.rowOff[t.R0 + i] - F);
}

// KF: factor every block (one thread per block).  D: the assembled diagonal.
__global__ void __launch_bounds__(128) k_block_factor(BlockArgs b, const double *__restrict__ D, const int32_t *frozen)
{
    if (frozen && *(const volatile int32_t *)frozen) return;
    const int64_t blk = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (blk >= b.nblk) return;
    const Lane t = lane_of(b, blk);
    for (int i = 0; i < t.m; i++) {
        int32_t F;
        double *Li = band_row(b, t, i, F);
        for (int k = F; k < i; k++) Li[32 * k] = 0.0;
        for (int32_t e = b.eptr[t.p0 + i]; e < b.eptr[t.p0 + i + 1]; e++) Li[32 * b.ecol[e]] = -*b.eg[e];
        for (int j = F; j < i; j++) {
            int32_t Fj;
            const double *Lj = band_row(b, t, j, Fj);
            double s = Li[32 * j];
            for (int k = max(F, Fj); k < j; k++) {
                const double p = Li[32 * k] * Lj[32 * k];
                s = s - p * t.Dd[32 * k];
            }
            Li[32 * j] = s / t.Dd[32 * j];
        }
        double s = D[b.bnode[t.p0 + i]];
        for (int k = F; k < i; k++) {
            const double p = Li[32 * k] * Li[32 * k];
            s = s - p * t.Dd[32 * k];
        }
        t.Dd[32 * i] = s;
    }
}

// Forward + diagonal + backward on y (and y2 when TWO).  MAXM <= 16: fully
// unrolled (registers); larger: runtime loops (local memory).
template <bool TWO, int MAXM>
__device__ __forceinline__ void block_apply(const BlockArgs &b, const Lane &t, double (&y)[MAXM], double (&y2)[MAXM])
{
    constexpr bool UNROLL = MAXM <= 16;
#pragma unroll
    for (int i = 0; i < (UNROLL ? MAXM : t.m); i++) {
        if (i < t.m) {
            int32_t F;
            const double *Li = band_row(b, t, i, F);
            double a = y[i], a2 = TWO ? y2[i] : 0.0;
#pragma unroll
            for (int k = (UNROLL ? 0 : F); k < (UNROLL ? MAXM : i); k++) {
                if (k >= F && k < i) {
                    const double l = __ldcs(Li + 32 * k);
                    a = a - l * y[k];
                    if (TWO) a2 = a2 - l * y2[k];
                }
            }
            y[i] = a;
            if (TWO) y2[i] = a2;
        }
    }
#pragma unroll
    for (int i = 0; i < (UNROLL ? MAXM : t.m); i++) {  // w = D^-1 y
        if (i < t.m) {
            const double d = t.Dd[32 * i];
            y[i] = y[i] / d;
            if (TWO) y2[i] = y2[i] / d;
        }
    }
#pragma unroll
    for (int i = (UNROLL ? MAXM : t.m) - 1; i >= 0; i--) {
        if (i < t.m) {
            int32_t F;
            const double *Li = band_row(b, t, i, F);
            const double zi = y[i], zi2 = TWO ? y2[i] : 0.0;
#pragma unroll
            for (int k = (UNROLL ? 0 : F); k < (UNROLL ? MAXM : i); k++) {
                if (k >= F && k < i) {
                    const double l = __ldcs(Li + 32 * k);
                    y[k] = y[k] - l * zi;
                    if (TWO) y2[k] = y2[k] - l * zi2;
                }
            }
        }
    }
}

// KB0 (START): z0 = M^-1 r0 and mb = M^-1 b (b = gs), two right-hand sides.
template <int MAXM>
__global__ void __launch_bounds__(128) k_block_solve_start(BlockArgs b, VecArgs v, const double *__restrict__ gs)
{
    if (v.frozen && *(const volatile int32_t *)v.frozen) return;
    const int64_t blk = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (blk >= b.nblk) return;
    const Lane t = lane_of(b, blk);
    double y[MAXM], y2[MAXM];
#pragma unroll
    for (int i = 0; i < MAXM; i++) {
        if (i < t.m) {
            const int32_t u = b.bnode[t.p0 + i];
            y[i] = v.r[u];
            y2[i] = gs[u];
        }
    }
    block_apply<true, MAXM>(b, t, y, y2);
#pragma unroll
    for (int i = 0; i < MAXM; i++) {
        if (i < t.m) {
            const int32_t u = b.bnode[t.p0 + i];
            v.z[u] = y[i];
            b.mb[u] = y2[i];
        }
    }
}

// KB (iteration): r = r - alpha q (K5's update, same operation), z = M^-1 r.
template <int MAXM>
__global__ void __launch_bounds__(128) k_block_solve_iter(BlockArgs b, VecArgs v, const DevCtrl *ctrl)
{
    if (ctrl->done) return;  // breakdown after q = A p: KR sets the condition
    const int64_t blk = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (blk >= b.nblk) return;
    const double alpha = ctrl->alpha;
    const Lane t = lane_of(b, blk);
    double y[MAXM], y2[MAXM];
#pragma unroll
    for (int i = 0; i < MAXM; i++) {
        if (i < t.m) {
            const int32_t u = b.bnode[t.p0 + i];
            const double r = v.r[u] - alpha * v.q[u];
            v.r[u] = r;
            y[i] = r;
        }
    }
    block_apply<false, MAXM>(b, t, y, y2);
#pragma unroll
    for (int i = 0; i < MAXM; i++)
        if (i < t.m) v.z[b.bnode[t.p0 + i]] = y[i];
}

__device__ __forceinline__ void set_cond_b(const CondArgs &cd, const DevCtrl *c)
{
    if (cd.use) cudaGraphSetConditional(cd.handle, c->done ? 0u : 1u);
}

#define FOR_CHUNK_NODES_B(...)                                                    \
    {                                                                             \
        const int64_t base__ = (int64_t)blockIdx.x * kChunk;                      \
        _Pragma("unroll 1") for (int j__ = 0; j__ < 8; j__++)                     \
        {                                                                         \
            _Pragma("unroll") for (int e__ = 0; e__ < 2; e__++)                   \
            {                                                                     \
                const int64_t u = base__ + 2 * (int64_t)threadIdx.x + 512 * j__ + e__; \
                if (u < v.n_own) { __VA_ARGS__ }                                  \
            }                                                                     \
        }                                                                         \
    }

// KR0: START reductions [<r,z>, <z,z>, <r,r>, <mb,mb>, <b,b>] (K1's order).
__global__ void __launch_bounds__(kThreads) k_block_reduce_start(VecArgs v, const double *mb, const double *gs,
                                                               RedArgs ra, CondArgs cd)
{
    if (v.frozen && *(const volatile int32_t *)v.frozen) return;
    double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    FOR_CHUNK_NODES_B({
        const double r = v.r[u], z = v.z[u], m = mb[u], bb = gs[u];
        acc[0] = acc[0] + r * z;
        acc[1] = acc[1] + z * z;
        acc[2] = acc[2] + r * r;
        acc[3] = acc[3] + m * m;
        acc[4] = acc[4] + bb * bb;
    })
    if (c3_chunk_epilogue<5>(acc, v.chunk0 + (int32_t)blockIdx.x, ra) && cd.finalize && threadIdx.x == 0) {
        finalize_start(ra.ctrl, ra.slots);
        set_cond_b(cd, ra.ctrl);
    }
}

// KR: iteration reductions [<r,z>, <z,z>, <r,r>] (K5's order).
__global__ void __launch_bounds__(kThreads) k_block_reduce_iter(VecArgs v, RedArgs ra, CondArgs cd)
{
    DevCtrl *ctrl = ra.ctrl;
    if (ctrl->done) {
        if (blockIdx.x == 0 && threadIdx.x == 0) set_cond_b(cd, ctrl);
        return;
    }
    double acc[3] = {0.0, 0.0, 0.0};
    FOR_CHUNK_NODES_B({
        const double r = v.r[u], z = v.z[u];
        acc[0] = acc[0] + r * z;
        acc[1] = acc[1] + z * z;
        acc[2] = acc[2] + r * r;
    })
    if (c3_chunk_epilogue<3>(acc, v.chunk0 + (int32_t)blockIdx.x, ra) && cd.finalize && threadIdx.x == 0) {
        finalize_rz(ctrl, ra.slots);
        set_cond_b(cd, ctrl);
    }
}

static unsigned blk_grid(const BlockArgs &b) { return (unsigned)((b.nblk + 127) / 128); }

int launch_block_factor(const BlockArgs &b, const double *D, const int32_t *frozen, cudaStream_t st)
{
    if (b.nblk == 0) return 0;
    k_block_factor<<<blk_grid(b), 128, 0, st>>>(b, D, frozen);
    return 1;
}

#define BLK_DISPATCH(KERNEL, ...)                                                        \
    do {                                                                                 \
        if (b.m_max <= 8) KERNEL<8><<<blk_grid(b), 128, 0, st>>>(__VA_ARGS__);           \
        else if (b.m_max <= 16) KERNEL<16><<<blk_grid(b), 128, 0, st>>>(__VA_ARGS__);    \
        else if (b.m_max <= 64) KERNEL<64><<<blk_grid(b), 128, 0, st>>>(__VA_ARGS__);    \
        else KERNEL<256><<<blk_grid(b), 128, 0, st>>>(__VA_ARGS__);                      \
    } while (0)

int launch_block_start(const BlockArgs &b, const VecArgs &v, const double *gs, const RedArgs &ra,
                       const CondArgs &cd, cudaStream_t st)
{
    int n = 0;
    if (b.nblk > 0) {
        BLK_DISPATCH(k_block_solve_start, b, v, gs);
        n++;
    }
    const unsigned nb = (unsigned)((v.n_own + kChunk - 1) / kChunk);
    if (nb > 0) {
        k_block_reduce_start<<<nb, kThreads, 0, st>>>(v, b.mb, gs, ra, cd);
        n++;
    }
    return n;
}

int launch_block_iter(const BlockArgs &b, const VecArgs &v, const RedArgs &ra, const CondArgs &cd, cudaStream_t st)
{
    int n = 0;
    if (b.nblk > 0) {
        BLK_DISPATCH(k_block_solve_iter, b, v, ra.ctrl);
        n++;
    }
    const unsigned nb = (unsigned)((v.n_own + kChunk - 1) / kChunk);
    if (nb > 0) {
        k_block_reduce_iter<<<nb, kThreads, 0, st>>>(v, ra, cd);
        n++;
    }
    return n;
}

}  // namespace irls
