// lambda2.cu — the quadratic form of the Cheeger-type diagnostic (
// P:L543-551; reading A30): per node u, the owned terms of x^T L x on the
// capacities c with x_s = 1, x_t = -1, and the owned capacities for
// C = 2 sum_e c_e, both reduced by C3:
//   own_u = sum_{v > u, asc} c_uv (d d) [d = x_u - x_v] + cs_u (ds ds) [ds = 1 - x_u]
//           + ct_u (dt dt) [dt = x_u + 1]
//   cap_u = (sum_{v > u, asc} c_uv + cs_u) + ct_u
#include "kernels.h"

namespace irls {

__global__ void __launch_bounds__(kThreads) k_l2_quad_stencil(StencilArgs s, int64_t N, const double *x, RedArgs ra)
{
    double acc[2] = {0.0, 0.0};
    const int64_t base = (int64_t)blockIdx.x * kChunk;
    for (int j = 0; j < 8; j++)
        for (int e = 0; e < 2; e++) {
            const int64_t u = base + 2 * (int64_t)threadIdx.x + 512 * j + e;
            if (u >= N) continue;
            const uint32_t uv = (uint32_t)u;
            const uint32_t t1 = fdiv(uv, s.fd_nx);
            const int32_t xx = (int32_t)(uv - t1 * (uint32_t)s.nx);
            const uint32_t zz = fdiv(t1, s.fd_ny);
            const int32_t y = (int32_t)(t1 - zz * (uint32_t)s.ny), z = (int32_t)zz;
            const double xu = x[u];
            double q = 0.0, c = 0.0;
            if (xx < s.nx - 1) {
                const double cc = s.cx[u], d = xu - x[u + 1];
                q = q + cc * (d * d);
                c = c + cc;
            }
            if (y < s.ny - 1) {
                const double cc = s.cy[u], d = xu - x[u + s.nx];
                q = q + cc * (d * d);
                c = c + cc;
            }
            if (z < s.nz - 1) {
                const double cc = s.cz[u], d = xu - x[u + s.P];
                q = q + cc * (d * d);
                c = c + cc;
            }
            const double ds = 1.0 - xu, dt = xu + 1.0;
            q = q + s.cs[u] * (ds * ds);
            q = q + s.ct[u] * (dt * dt);
            acc[0] = acc[0] + q;
            acc[1] = acc[1] + ((c + s.cs[u]) + s.ct[u]);
        }
    c3_chunk_epilogue<2>(acc, (int32_t)blockIdx.x, ra);
}

__global__ void __launch_bounds__(kThreads) k_l2_quad_sell(SellArgs s, const double *x, RedArgs ra)
{
    double acc[2] = {0.0, 0.0};
    const int64_t base = (int64_t)blockIdx.x * kChunk;
    for (int j = 0; j < 8; j++)
        for (int e = 0; e < 2; e++) {
            const int64_t u = base + 2 * (int64_t)threadIdx.x + 512 * j + e;
            if (u >= s.n) continue;
            const int64_t sl = u / kSell;
            const int64_t e0 = s.slice_ptr[sl] + (u % kSell);
            const int32_t W = (int32_t)((s.slice_ptr[sl + 1] - s.slice_ptr[sl]) / kSell);
            const double xu = x[u];
            double q = 0.0, c = 0.0;
            for (int32_t k = 0; k < W; k++) {
                const int64_t idx = e0 + kSell * (int64_t)k;
                const int32_t nb = s.col[idx];
                if (nb < 0) break;
                if (nb < u) continue;
                const double cc = s.c[idx], d = xu - x[nb];
                q = q + cc * (d * d);
                c = c + cc;
            }
            const double ds = 1.0 - xu, dt = xu + 1.0;
            q = q + s.cs[u] * (ds * ds);
            q = q + s.ct[u] * (dt * dt);
            acc[0] = acc[0] + q;
            acc[1] = acc[1] + ((c + s.cs[u]) + s.ct[u]);
        }
    c3_chunk_epilogue<2>(acc, (int32_t)blockIdx.x, ra);
}

void launch_l2_quad_stencil(const StencilArgs &s, int64_t N, const double *x, const RedArgs &ra, cudaStream_t st)
{
    if (N == 0) return;
    k_l2_quad_stencil<<<(unsigned)((N + kChunk - 1) / kChunk), kThreads, 0, st>>>(s, N, x, ra);
}

void launch_l2_quad_sell(const SellArgs &s, const double *x, const RedArgs &ra, cudaStream_t st)
{
    if (s.n == 0) return;
    k_l2_quad_sell<<<(unsigned)((s.n + kChunk - 1) / kChunk), kThreads, 0, st>>>(s, x, ra);
}

}  // namespace irls
