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
// executed column by column (right-looking) by the lanes of one warp per
// block: entry (i, j) receives its updates in ascending step order, which is
// the definition's order.  Entries outside a row's envelope [f_i, i) are
// exact zeros of the dense algorithm and are skipped (bitwise no-ops).
// The envelope first columns f_i are non-decreasing in block order (a BFS
// node's first in-block neighbour is the node that discovered it), so the
// rows touched by step k are the contiguous range (k, l_k].
//
// KR then forms the C3 reductions of the solve (START: <r,z>, <z,z>, <r,r>,
// <M^-1 b, M^-1 b>, <b,b>; per iteration: <r,z>, <z,z>, <r,r>) in the
// standard chunk mapping, so the finalizers are K1's / K5's.
#include <algorithm>
#include "kernels.h"

namespace irls {

// Dynamic shared memory per warp: [env_max doubles][m_max doubles (d or acc)]
// [m_max doubles (acc2)] [m_max int32 (f)] [m_max int32 (row offsets)].
__host__ __device__ inline size_t blk_warp_bytes(const BlockArgs &b)
{
    return sizeof(double) * ((size_t)b.env_max + 2 * (size_t)b.m_max) + sizeof(int32_t) * 2 * (size_t)b.m_max;
}

struct WarpSmem {
    double *env, *a0, *a1;
    int32_t *f, *ro;
};

__device__ __forceinline__ WarpSmem warp_smem(const BlockArgs &b, unsigned char *dyn, int w)
{
    unsigned char *p = dyn + (size_t)w * ((blk_warp_bytes(b) + 15) & ~(size_t)15);
    WarpSmem s;
    s.env = reinterpret_cast<double *>(p);
    s.a0 = s.env + b.env_max;
    s.a1 = s.a0 + b.m_max;
    s.f = reinterpret_cast<int32_t *>(s.a1 + b.m_max);
    s.ro = s.f + b.m_max;
    return s;
}

// KF: factor every block (one warp per block).  D: the assembled diagonal.
__global__ void k_block_factor(BlockArgs b, const double *__restrict__ D, const int32_t *frozen)
{
    if (frozen && *(const volatile int32_t *)frozen) return;
    extern __shared__ __align__(16) unsigned char blk_dyn[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t blk = (int64_t)blockIdx.x * (blockDim.x >> 5) + w;
    if (blk >= b.nblk) return;
    const WarpSmem s = warp_smem(b, blk_dyn, w);
    const int32_t p0 = b.bptr[blk], m = b.bptr[blk + 1] - p0;
    const int64_t e0 = b.boff[p0];
    const int32_t ne = (int32_t)(b.boff[p0 + m] - e0);
    for (int e = lane; e < ne; e += 32) s.env[e] = 0.0;
    for (int i = lane; i < m; i += 32) {
        const int32_t fi = b.bfirst[p0 + i];
        s.f[i] = fi;
        s.ro[i] = (int32_t)(b.boff[p0 + i] - e0) - fi;  // env index of (i, j) = ro[i] + j
        s.a0[i] = D[b.bnode[p0 + i]];
    }
    __syncwarp();
    for (int i = lane; i < m; i += 32)  // A_ij = -g_uv for the in-block lower neighbours
        for (int32_t e = b.eptr[p0 + i]; e < b.eptr[p0 + i + 1]; e++) s.env[s.ro[i] + b.ecol[e]] = -*b.eg[e];
    __syncwarp();
    for (int j = 0; j < m; j++) {
        const double dj = s.a0[j];  // final: every step k < j has updated it
        for (int i = j + 1 + lane; i < m; i += 32)
            if (s.f[i] <= j) s.env[s.ro[i] + j] = s.env[s.ro[i] + j] / dj;  // L_ij
        __syncwarp();
        for (int i = j + 1 + lane; i < m; i += 32) {
            if (s.f[i] > j) continue;
            const double lij = s.env[s.ro[i] + j];
            double *row = s.env + s.ro[i];
            for (int k = j + 1; k < i; k++) {  // f_k <= f_i <= j: L_kj inside k's envelope
                const double t = lij * s.env[s.ro[k] + j];
                row[k] = row[k] - t * dj;
            }
            const double t = lij * lij;
            s.a0[i] = s.a0[i] - t * dj;
        }
        __syncwarp();
    }
    for (int e = lane; e < ne; e += 32) b.L[e0 + e] = s.env[e];
    for (int i = lane; i < m; i += 32) b.Dd[p0 + i] = s.a0[i];
}

// Forward + diagonal + backward on acc (and acc2 when TWO), in shared memory.
template <bool TWO>
__device__ __forceinline__ void block_apply(const WarpSmem &s, const double *__restrict__ Dd, int m, int lane)
{
    for (int k = 0; k < m; k++) {
        __syncwarp();
        const double yk = s.a0[k];
        const double yk2 = TWO ? s.a1[k] : 0.0;
        for (int i = k + 1 + lane; i < m; i += 32) {
            if (s.f[i] > k) break;  // f non-decreasing: no later row reaches column k
            const double l = s.env[s.ro[i] + k];
            s.a0[i] = s.a0[i] - l * yk;
            if (TWO) s.a1[i] = s.a1[i] - l * yk2;
        }
    }
    __syncwarp();
    for (int i = lane; i < m; i += 32) {
        const double d = Dd[i];
        s.a0[i] = s.a0[i] / d;
        if (TWO) s.a1[i] = s.a1[i] / d;
    }
    for (int i = m - 1; i >= 0; i--) {
        __syncwarp();
        const double zi = s.a0[i];
        const double zi2 = TWO ? s.a1[i] : 0.0;
        const double *row = s.env + s.ro[i];
        for (int k = s.f[i] + lane; k < i; k += 32) {
            const double l = row[k];
            s.a0[k] = s.a0[k] - l * zi;
            if (TWO) s.a1[k] = s.a1[k] - l * zi2;
        }
    }
    __syncwarp();
}

__device__ __forceinline__ void block_load(const BlockArgs &b, const WarpSmem &s, int32_t p0, int m, int lane)
{
    const int64_t e0 = b.boff[p0];
    const int32_t ne = (int32_t)(b.boff[p0 + m] - e0);
    for (int e = lane; e < ne; e += 32) s.env[e] = __ldcs(b.L + e0 + e);
    for (int i = lane; i < m; i += 32) {
        const int32_t fi = b.bfirst[p0 + i];
        s.f[i] = fi;
        s.ro[i] = (int32_t)(b.boff[p0 + i] - e0) - fi;
    }
}

// KB0 (START): z0 = M^-1 r0 and mb = M^-1 b (b = gs), two right-hand sides.
__global__ void k_block_solve_start(BlockArgs b, VecArgs v, const double *__restrict__ gs)
{
    if (v.frozen && *(const volatile int32_t *)v.frozen) return;
    extern __shared__ __align__(16) unsigned char blk_dyn[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t blk = (int64_t)blockIdx.x * (blockDim.x >> 5) + w;
    if (blk >= b.nblk) return;
    const WarpSmem s = warp_smem(b, blk_dyn, w);
    const int32_t p0 = b.bptr[blk], m = b.bptr[blk + 1] - p0;
    block_load(b, s, p0, m, lane);
    for (int i = lane; i < m; i += 32) {
        const int32_t u = b.bnode[p0 + i];
        s.a0[i] = v.r[u];
        s.a1[i] = gs[u];
    }
    block_apply<true>(s, b.Dd + p0, m, lane);
    for (int i = lane; i < m; i += 32) {
        const int32_t u = b.bnode[p0 + i];
        v.z[u] = s.a0[i];
        b.mb[u] = s.a1[i];
    }
}

// KB (iteration): r = r - alpha q (K5's update, same operation), z = M^-1 r.
__global__ void k_block_solve_iter(BlockArgs b, VecArgs v, const DevCtrl *ctrl)
{
    if (ctrl->done) return;  // breakdown after q = A p: KR sets the condition
    extern __shared__ __align__(16) unsigned char blk_dyn[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t blk = (int64_t)blockIdx.x * (blockDim.x >> 5) + w;
    if (blk >= b.nblk) return;
    const double alpha = ctrl->alpha;
    const WarpSmem s = warp_smem(b, blk_dyn, w);
    const int32_t p0 = b.bptr[blk], m = b.bptr[blk + 1] - p0;
    block_load(b, s, p0, m, lane);
    for (int i = lane; i < m; i += 32) {
        const int32_t u = b.bnode[p0 + i];
        const double r = v.r[u] - alpha * v.q[u];
        v.r[u] = r;
        s.a0[i] = r;
    }
    block_apply<false>(s, b.Dd + p0, m, lane);
    for (int i = lane; i < m; i += 32) v.z[b.bnode[p0 + i]] = s.a0[i];
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

static int blk_warps(const BlockArgs &b)
{
    const size_t per = (blk_warp_bytes(b) + 15) & ~(size_t)15;
    int w = (int)std::min<size_t>(8, (200 * 1024) / std::max<size_t>(per, 1));
    return std::max(w, 1);
}

size_t block_smem_per_cta(const BlockArgs &b)
{
    return (size_t)blk_warps(b) * ((blk_warp_bytes(b) + 15) & ~(size_t)15);
}

void block_prepare(const BlockArgs &b)
{
    const int smem = (int)block_smem_per_cta(b);
    cudaFuncSetAttribute(k_block_factor, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_block_solve_start, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_block_solve_iter, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}

static unsigned blk_grid(const BlockArgs &b)
{
    const int w = blk_warps(b);
    return (unsigned)((b.nblk + w - 1) / w);
}

int launch_block_factor(const BlockArgs &b, const double *D, const int32_t *frozen, cudaStream_t st)
{
    if (b.nblk == 0) return 0;
    k_block_factor<<<blk_grid(b), 32 * blk_warps(b), block_smem_per_cta(b), st>>>(b, D, frozen);
    return 1;
}

int launch_block_start(const BlockArgs &b, const VecArgs &v, const double *gs, const RedArgs &ra,
                       const CondArgs &cd, cudaStream_t st)
{
    int n = 0;
    if (b.nblk > 0) {
        k_block_solve_start<<<blk_grid(b), 32 * blk_warps(b), block_smem_per_cta(b), st>>>(b, v, gs);
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
        k_block_solve_iter<<<blk_grid(b), 32 * blk_warps(b), block_smem_per_cta(b), st>>>(b, v, ra.ctrl);
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
