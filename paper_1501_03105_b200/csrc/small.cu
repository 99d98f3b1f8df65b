// small.cu — the whole Jacobi-PCG loop of one solve in ONE thread block, for
// graphs of at most one C3 chunk (n~ <= 4096, e.g. config 1's 1,024 nodes).
// Such solves are latency-bound (config 1: ~112k CG iterations of a 1k-node
// system): two grid-wide kernels per iteration cost ~14 us; here an
// iteration is a few block barriers on shared memory.  The block performs
// exactly the K3 / K5 arithmetic (p = z + beta p_old, the lazy x += alpha
// p_old, q = D p - sum_asc g p_nbr (O2, C2), r -= alpha q, z = Dinv r) and
// the C3 reductions of a single chunk (per-thread sums over elements
// 2t + 512j + e, the warp and 8-warp trees, the chunk as the only non-empty
// group, the 8-leaf tree), and every thread applies the same finalizers
// (finalize_pq_t / finalize_rz_t) to a register copy of the control block —
// so every bit matches the multi-block kernels and the oracle.  x, r, z, p
// live in shared memory for the solve; q stays in registers between the two
// halves of an iteration.
#include "kernels.h"

namespace irls {

template <int KIND>  // 0 stencil, 1 SELL
__device__ __forceinline__ double small_nbr_sum(const StencilArgs &s, const SellArgs &sl, const double *p, int64_t u)
{
    double a = 0.0;
    if (KIND == 0) {
        const uint32_t uu = (uint32_t)u;
        const uint32_t t1 = fdiv(uu, s.fd_nx);
        const int32_t x = (int32_t)(uu - t1 * (uint32_t)s.nx);
        const uint32_t zz = fdiv(t1, s.fd_ny);
        const int32_t y = (int32_t)(t1 - zz * (uint32_t)s.ny), z = (int32_t)zz;
        if (z > 0) a = a + __ldg(s.gz + u - s.P) * p[u - s.P];
        if (y > 0) a = a + __ldg(s.gy + u - s.nx) * p[u - s.nx];
        if (x > 0) a = a + __ldg(s.gx + u - 1) * p[u - 1];
        if (x < s.nx - 1) a = a + __ldg(s.gx + u) * p[u + 1];
        if (y < s.ny - 1) a = a + __ldg(s.gy + u) * p[u + s.nx];
        if (z < s.nz - 1) a = a + __ldg(s.gz + u) * p[u + s.P];
    } else {
        const int64_t sli = u / kSell;
        const int64_t e0 = sl.slice_ptr[sli] + (u % kSell);
        const int32_t W = (int32_t)((sl.slice_ptr[sli + 1] - sl.slice_ptr[sli]) / kSell);
        for (int32_t k = 0; k < W; k++) {
            const int64_t idx = e0 + kSell * (int64_t)k;
            const int32_t nb = __ldg(sl.col + idx);
            if (nb < 0) break;
            a = a + __ldg(sl.g + idx) * p[nb];
        }
    }
    return a;
}

// 8 group slots of a one-chunk reduction: the chunk's partial in its group
// (the last group starting at chunk 0), +0.0 elsewhere, the 8-leaf tree.
__device__ __forceinline__ double small_total(double partial, int g1)
{
    double s[kGroups];
#pragma unroll
    for (int g = 0; g < kGroups; g++) s[g] = g == g1 ? partial : 0.0;
    return tree8(s);
}

template <int KIND>
__global__ void __launch_bounds__(kThreads, 1) k_small_cg(StencilArgs s, SellArgs sl, VecArgs v, DevCtrl *ctrl)
{
    extern __shared__ double sm[];  // p | x | r | z, kChunk each
    double *sp = sm, *sx = sm + kChunk, *sr = sm + 2 * kChunk, *sz = sm + 3 * kChunk;
    __shared__ double red[kMaxQ * 8];
    __shared__ double bcast[3];
    const int64_t n = v.n_own;
    int g1 = 0;
    for (int gg = 1; gg < kGroups; gg++)
        if (0 >= group_lo(gg, 1)) g1 = gg;
    DevCtrl cl = *ctrl;  // register copy: every thread runs the finalizers identically
    for (int64_t u = threadIdx.x; u < n; u += blockDim.x) {
        sx[u] = v.x[u];
        sr[u] = v.r[u];
        sz[u] = v.z[u];
    }
    double q[16];
    while (!cl.done) {
        const bool first = cl.k == 0;
        const double beta = cl.beta, alpha = cl.alpha;
        __syncthreads();
        // phase A (own elements): p = z + beta p_old, x += alpha p_old
#pragma unroll
        for (int j = 0; j < 8; j++)
#pragma unroll
            for (int e = 0; e < 2; e++) {
                const int64_t u = 2 * (int64_t)threadIdx.x + 512 * j + e;
                if (u < n) {
                    if (first) {
                        sp[u] = sz[u];
                    } else {
                        const double po = sp[u];
                        sx[u] = sx[u] + alpha * po;
                        sp[u] = sz[u] + beta * po;
                    }
                }
            }
        __syncthreads();
        // phase B: q = D p - sum_asc g p_nbr; pi partials in C3 order
        double a1[1] = {0.0};
#pragma unroll
        for (int j = 0; j < 8; j++)
#pragma unroll
            for (int e = 0; e < 2; e++) {
                const int64_t u = 2 * (int64_t)threadIdx.x + 512 * j + e;
                q[2 * j + e] = 0.0;
                if (u < n) {
                    const double a = small_nbr_sum<KIND>(s, sl, sp, u);
                    const double qu = __ldg(v.D + u) * sp[u] - a;
                    q[2 * j + e] = qu;
                    a1[0] = a1[0] + sp[u] * qu;
                }
            }
        c3_block_sum<1>(a1, red);
        if (threadIdx.x == 0) bcast[0] = a1[0];
        __syncthreads();
        finalize_pq_t(&cl, small_total(bcast[0], g1));
        if (cl.status != ST_OK) break;
        const double al = cl.alpha;
        // phase C (own elements): r -= alpha q; z = Dinv r; rz, zz, rr partials
        double a3[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int j = 0; j < 8; j++)
#pragma unroll
            for (int e = 0; e < 2; e++) {
                const int64_t u = 2 * (int64_t)threadIdx.x + 512 * j + e;
                if (u < n) {
                    const double r = sr[u] - al * q[2 * j + e];
                    const double z = r * __ldg(v.Dinv + u);
                    sr[u] = r;
                    sz[u] = z;
                    a3[0] = a3[0] + r * z;
                    a3[1] = a3[1] + z * z;
                    a3[2] = a3[2] + r * r;
                }
            }
        __syncthreads();  // bcast reuse
        c3_block_sum<3>(a3, red);
        if (threadIdx.x == 0) {
            bcast[0] = a3[0];
            bcast[1] = a3[1];
            bcast[2] = a3[2];
        }
        __syncthreads();
        finalize_rz_t(&cl, small_total(bcast[0], g1), small_total(bcast[1], g1), small_total(bcast[2], g1));
    }
    __syncthreads();
    // write back the solve state; the finish kernel reads p[k & 1]
    double *plast = (cl.k & 1) ? v.p1 : v.p0;
    for (int64_t u = threadIdx.x; u < n; u += blockDim.x) {
        v.x[u] = sx[u];
        v.r[u] = sr[u];
        v.z[u] = sz[u];
        if (cl.k > 0) plast[u] = sp[u];
    }
    if (threadIdx.x == 0) *ctrl = cl;
}

// Grids of at most 512 NJ nodes (config 1: 1,024 = NJ 2): the same loop with
// each thread's nodes (u = 2t + 512j + e, j < NJ) resolved once per solve —
// neighbour offsets, conductances in ascending order (C2), D and Dinv held
// in registers — so an iteration is shared-memory arithmetic, the two C3
// reductions and the (replicated) scalar finalizers.  Same operations in
// the same order as k_small_cg<0>.
template <int NJ>
__global__ void __launch_bounds__(kThreads, 1) k_small_cg_grid(StencilArgs s, VecArgs v, DevCtrl *ctrl)
{
    constexpr int NS = 2 * NJ;
    extern __shared__ double sm[];  // p | x | r | z, kChunk each
    double *sp = sm, *sx = sm + kChunk, *sr = sm + 2 * kChunk, *sz = sm + 3 * kChunk;
    __shared__ double red[kMaxQ * 8];
    __shared__ double bcast[3];
    const int64_t n = v.n_own;
    int g1 = 0;
    for (int gg = 1; gg < kGroups; gg++)
        if (0 >= group_lo(gg, 1)) g1 = gg;
    DevCtrl cl = *ctrl;
    for (int64_t u = threadIdx.x; u < n; u += blockDim.x) {
        sx[u] = v.x[u];
        sr[u] = v.r[u];
        sz[u] = v.z[u];
    }
    // per-solve operator of this thread's nodes
    int32_t uu[NS], off[NS][6];
    unsigned mask[NS];
    double gg6[NS][6], Dd[NS], Di[NS];
#pragma unroll
    for (int i = 0; i < NS; i++) {
        const int32_t u = 2 * (int32_t)threadIdx.x + 512 * (i >> 1) + (i & 1);
        uu[i] = u;
        mask[i] = 0u;
        Dd[i] = Di[i] = 0.0;
#pragma unroll
        for (int d = 0; d < 6; d++) { off[i][d] = u; gg6[i][d] = 0.0; }
        if (u < n) {
            const uint32_t t1 = fdiv((uint32_t)u, s.fd_nx);
            const int32_t x = (int32_t)((uint32_t)u - t1 * (uint32_t)s.nx);
            const uint32_t zz = fdiv(t1, s.fd_ny);
            const int32_t y = (int32_t)(t1 - zz * (uint32_t)s.ny), z = (int32_t)zz;
            const int32_t P = (int32_t)s.P;
            const bool has[6] = {z > 0, y > 0, x > 0, x < s.nx - 1, y < s.ny - 1, z < s.nz - 1};
            const int32_t o[6] = {u - P, u - s.nx, u - 1, u + 1, u + s.nx, u + P};
            const int32_t gi[6] = {u - P, u - s.nx, u - 1, u, u, u};
            const double *ga[6] = {s.gz, s.gy, s.gx, s.gx, s.gy, s.gz};
#pragma unroll
            for (int d = 0; d < 6; d++)
                if (has[d]) {
                    mask[i] |= 1u << d;
                    off[i][d] = o[d];
                    gg6[i][d] = ga[d][gi[d]];
                }
            mask[i] |= 1u << 6;  // valid node
            Dd[i] = v.D[u];
            Di[i] = v.Dinv[u];
        }
    }
    double q[NS];
    while (!cl.done) {
        const bool first = cl.k == 0;
        const double beta = cl.beta, alpha = cl.alpha;
        __syncthreads();
#pragma unroll
        for (int i = 0; i < NS; i++)
            if (mask[i] >> 6) {
                const int32_t u = uu[i];
                if (first) {
                    sp[u] = sz[u];
                } else {
                    const double po = sp[u];
                    sx[u] = sx[u] + alpha * po;
                    sp[u] = sz[u] + beta * po;
                }
            }
        __syncthreads();
        double a1[1] = {0.0};
#pragma unroll
        for (int i = 0; i < NS; i++) {
            q[i] = 0.0;
            if (mask[i] >> 6) {
                double a = 0.0;
#pragma unroll
                for (int d = 0; d < 6; d++)
                    if (mask[i] & (1u << d)) a = a + gg6[i][d] * sp[off[i][d]];
                const double pu = sp[uu[i]];
                const double qu = Dd[i] * pu - a;
                q[i] = qu;
                a1[0] = a1[0] + pu * qu;
            }
        }
        c3_block_sum<1>(a1, red);
        if (threadIdx.x == 0) bcast[0] = a1[0];
        __syncthreads();
        finalize_pq_t(&cl, small_total(bcast[0], g1));
        if (cl.status != ST_OK) break;
        const double al = cl.alpha;
        double a3[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int i = 0; i < NS; i++)
            if (mask[i] >> 6) {
                const int32_t u = uu[i];
                const double r = sr[u] - al * q[i];
                const double z = r * Di[i];
                sr[u] = r;
                sz[u] = z;
                a3[0] = a3[0] + r * z;
                a3[1] = a3[1] + z * z;
                a3[2] = a3[2] + r * r;
            }
        __syncthreads();  // bcast reuse
        c3_block_sum<3>(a3, red);
        if (threadIdx.x == 0) {
            bcast[0] = a3[0];
            bcast[1] = a3[1];
            bcast[2] = a3[2];
        }
        __syncthreads();
        finalize_rz_t(&cl, small_total(bcast[0], g1), small_total(bcast[1], g1), small_total(bcast[2], g1));
    }
    __syncthreads();
    double *plast = (cl.k & 1) ? v.p1 : v.p0;
    for (int64_t u = threadIdx.x; u < n; u += blockDim.x) {
        v.x[u] = sx[u];
        v.r[u] = sr[u];
        v.z[u] = sz[u];
        if (cl.k > 0) plast[u] = sp[u];
    }
    if (threadIdx.x == 0) *ctrl = cl;
}

static constexpr size_t kSmallSmem = 4 * sizeof(double) * kChunk;

void small_cg_prepare()
{
    cudaFuncSetAttribute(k_small_cg<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmallSmem);
    cudaFuncSetAttribute(k_small_cg<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmallSmem);
    cudaFuncSetAttribute(k_small_cg_grid<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmallSmem);
    cudaFuncSetAttribute(k_small_cg_grid<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmallSmem);
}

void launch_small_cg(int kind, const StencilArgs &s, const SellArgs &sl, const VecArgs &v, DevCtrl *ctrl,
                     double *slots, cudaStream_t st)
{
    (void)slots;
    if (kind == 0 && v.n_own <= 512) k_small_cg_grid<1><<<1, kThreads, kSmallSmem, st>>>(s, v, ctrl);
    else if (kind == 0 && v.n_own <= 1024) k_small_cg_grid<2><<<1, kThreads, kSmallSmem, st>>>(s, v, ctrl);
    else if (kind == 0) k_small_cg<0><<<1, kThreads, kSmallSmem, st>>>(s, sl, v, ctrl);
    else k_small_cg<1><<<1, kThreads, kSmallSmem, st>>>(s, sl, v, ctrl);
}

}  // namespace irls
