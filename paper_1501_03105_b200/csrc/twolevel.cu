// twolevel.cu — GPU part of the two-level rounding ("A two-level
// rounding procedure"; readings A25-A29 in DESIGN.md §2).
//
//   kmeans    Lloyd k = 2 on x^(T) (non-terminals + x_s = 1, x_t = 0), initial
//             centres 0.1 / 0.9; one launch per round, the C3 sums
//             of the two clusters and the member count; the last block
//             computes the new centres and the stop flag on the device
//   classify  S0 (x <= gamma0) / S1 (x >= gamma1) / Sc, the coarse degree of
//             every Sc node, and the fixed-point s_c-t_c partials per tile
//   (scan)    coarse ids and coarse row offsets (exclusive scans)
//   fill      coarse CSR (ascending coarse ids) with the capacities, and the
//             coarse s_c / t_c links in exact 128-bit fixed point
//   lift      pseudo-rank (0 = source side) so the sweep's side/cut kernel
//             recomputes the cut on G by C3
// The exact max-flow on G_c runs on the host (maxflow.cu), as the paper's
// second level does, and is timed separately.
#include "kernels.h"

namespace irls {

typedef __int128 i128;

constexpr int kTlTile = 4096;  // nodes per block in classify / fill (256 x 16)

__device__ __forceinline__ int tl_class(double x, double g0, double g1) { return x <= g0 ? 0 : (x >= g1 ? 1 : 2); }

// ---------------------------------------------------------------------------
// K-means round (A25)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_tl_kmeans(const double *x, int64_t n, TLState *st, RedArgs ra)
{
    if (*(volatile int32_t *)&st->done) return;  // converged in an earlier launch of this batch
    const double c0 = st->c0, c1 = st->c1;
    double acc[3] = {0.0, 0.0, 0.0};
    const int64_t base = (int64_t)blockIdx.x * kChunk;
#pragma unroll
    for (int j = 0; j < 8; j++)
#pragma unroll
        for (int e = 0; e < 2; e++) {
            const int64_t v = base + 2 * (int64_t)threadIdx.x + 512 * j + e;
            if (v < n) {
                const double xv = x[v];
                const bool in1 = fabs(xv - c1) < fabs(xv - c0);
                acc[0] = acc[0] + (in1 ? 0.0 : xv);
                acc[1] = acc[1] + (in1 ? xv : 0.0);
                acc[2] = acc[2] + (in1 ? 1.0 : 0.0);
            }
        }
    if (!c3_chunk_epilogue<3>(acc, (int32_t)blockIdx.x, ra)) return;
    if (threadIdx.x != 0) return;
    double s0 = slot_total(ra.slots, 0), s1 = slot_total(ra.slots, 1);
    int64_t n1 = (int64_t)slot_total(ra.slots, 2);
    const double xt[2] = {1.0, 0.0};  // x_s, x_t
    for (int i = 0; i < 2; i++) {
        if (fabs(xt[i] - c1) < fabs(xt[i] - c0)) {
            s1 = s1 + xt[i];
            n1++;
        } else {
            s0 = s0 + xt[i];
        }
    }
    const int64_t n0 = n + 2 - n1;
    const double d0 = n0 > 0 ? s0 / (double)n0 : c0;
    const double d1 = n1 > 0 ? s1 / (double)n1 : c1;
    const bool same = (d0 == c0) && (d1 == c1);
    st->c0 = d0;
    st->c1 = d1;
    st->rounds = st->rounds + 1;
    __threadfence();
    st->done = (same || st->rounds >= 100) ? 1 : 0;
}

// Partition of the block's tile of int128 values into one block total.
__device__ __forceinline__ void tl_block_sum_i128(i128 v, i128 *out, int32_t cnt, int32_t *cnt_out)
{
    __shared__ unsigned long long sm[2][8];
    __shared__ int32_t sc[8];
    for (int off = 16; off >= 1; off >>= 1) cnt += __shfl_down_sync(0xffffffffu, cnt, off);
    if ((threadIdx.x & 31) == 0) sc[threadIdx.x >> 5] = cnt;
    for (int off = 16; off >= 1; off >>= 1) {
        unsigned long long lo = (unsigned long long)v, hi = (unsigned long long)(v >> 64);
        lo = __shfl_down_sync(0xffffffffu, lo, off);
        hi = __shfl_down_sync(0xffffffffu, hi, off);
        v += ((i128)hi << 64) | (i128)lo;
    }
    if ((threadIdx.x & 31) == 0) {
        sm[0][threadIdx.x >> 5] = (unsigned long long)v;
        sm[1][threadIdx.x >> 5] = (unsigned long long)(v >> 64);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        i128 s = 0;
        int32_t c = 0;
        for (int i = 0; i < 8; i++) {
            s += ((i128)sm[1][i] << 64) | (i128)sm[0][i];
            c += sc[i];
        }
        *out = s;
        *cnt_out = c;
    }
}

// ---------------------------------------------------------------------------
// classify + coarse degree + s_c-t_c partials
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_tl_classify_stencil(StencilArgs s, int64_t N, const double *x, double g0,
                                                             double g1, int32_t F, int8_t *cls, int32_t *flag,
                                                             int32_t *deg, i128 *tile_a, int32_t *tile_n1)
{
    i128 a = 0;
    int32_t n1 = 0;
    const int64_t base = (int64_t)blockIdx.x * kTlTile;
    for (int r = 0; r < 16; r++) {
        const int64_t v = base + r * 256 + threadIdx.x;
        if (v >= N) break;
        const int cv = tl_class(x[v], g0, g1);
        cls[v] = (int8_t)cv;
        flag[v] = cv == 2;
        const uint32_t uv = (uint32_t)v;
        const uint32_t t1 = fdiv(uv, s.fd_nx);
        const int32_t xx = (int32_t)(uv - t1 * (uint32_t)s.nx);
        const uint32_t zz = fdiv(t1, s.fd_ny);
        const int32_t y = (int32_t)(t1 - zz * (uint32_t)s.ny), z = (int32_t)zz;
        int d = 0;
        i128 q0 = 0;  // S1 node: fixed-point capacity to S0 neighbours
#define NB(cond, w, cap)                                                  \
    if (cond) {                                                           \
        const double c_ = (cap);                                          \
        if (c_ > 0.0) {                                                   \
            const int cw = tl_class(x[w], g0, g1);                        \
            if (cv == 2) d += cw == 2;                                    \
            else if (cv == 1 && cw == 0) q0 += qfix(c_, F);               \
        }                                                                 \
    }
        if (cv != 0) {
            NB(z > 0, v - s.P, s.cz[v - s.P]);
            NB(y > 0, v - s.nx, s.cy[v - s.nx]);
            NB(xx > 0, v - 1, s.cx[v - 1]);
            NB(xx < s.nx - 1, v + 1, s.cx[v]);
            NB(y < s.ny - 1, v + s.nx, s.cy[v]);
            NB(z < s.nz - 1, v + s.P, s.cz[v]);
        }
#undef NB
        deg[v] = d;
        n1 += cv == 1;
        if (cv == 1) a += q0 + qfix(s.ct[v], F);
        else if (cv == 0) a += qfix(s.cs[v], F);
    }
    tl_block_sum_i128(a, tile_a + blockIdx.x, n1, tile_n1 + blockIdx.x);
}

__global__ void __launch_bounds__(256) k_tl_classify_sell(SellArgs s, const double *x, double g0, double g1,
                                                          int32_t F, int8_t *cls, int32_t *flag, int32_t *deg,
                                                          i128 *tile_a, int32_t *tile_n1)
{
    i128 a = 0;
    int32_t n1 = 0;
    const int64_t base = (int64_t)blockIdx.x * kTlTile;
    for (int r = 0; r < 16; r++) {
        const int64_t v = base + r * 256 + threadIdx.x;
        if (v >= s.n) break;
        const int cv = tl_class(x[v], g0, g1);
        cls[v] = (int8_t)cv;
        flag[v] = cv == 2;
        int d = 0;
        i128 q0 = 0;
        if (cv != 0) {
            const int64_t sl = v / kSell;
            const int64_t e0 = s.slice_ptr[sl] + (v % kSell);
            const int32_t W = (int32_t)((s.slice_ptr[sl + 1] - s.slice_ptr[sl]) / kSell);
            for (int32_t k = 0; k < W; k++) {
                const int64_t idx = e0 + kSell * (int64_t)k;
                const int32_t nb = s.col[idx];
                if (nb < 0) break;
                const double c_ = s.c[idx];
                if (c_ > 0.0) {
                    const int cw = tl_class(x[nb], g0, g1);
                    if (cv == 2) d += cw == 2;
                    else if (cv == 1 && cw == 0) q0 += qfix(c_, F);
                }
            }
        }
        deg[v] = d;
        n1 += cv == 1;
        if (cv == 1) a += q0 + qfix(s.ct[v], F);
        else if (cv == 0) a += qfix(s.cs[v], F);
    }
    tl_block_sum_i128(a, tile_a + blockIdx.x, n1, tile_n1 + blockIdx.x);
}

// ---------------------------------------------------------------------------
// fill: coarse CSR rows of the Sc nodes
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_tl_fill_stencil(StencilArgs s, int64_t N, int32_t F, const int8_t *cls,
                                                         const int32_t *cid, const int32_t *eoff, int32_t *cp,
                                                         int32_t *ccol, double *ccap, i128 *cqs, i128 *cqt)
{
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= N || cls[v] != 2) return;
    const uint32_t uv = (uint32_t)v;
    const uint32_t t1 = fdiv(uv, s.fd_nx);
    const int32_t xx = (int32_t)(uv - t1 * (uint32_t)s.nx);
    const uint32_t zz = fdiv(t1, s.fd_ny);
    const int32_t y = (int32_t)(t1 - zz * (uint32_t)s.ny), z = (int32_t)zz;
    const int32_t me = cid[v];
    int32_t e = eoff[v];
    cp[me] = e;
    i128 qs = 0, qt = 0;
#define NB(cond, w, cap)                                       \
    if (cond) {                                                \
        const double c_ = (cap);                               \
        if (c_ > 0.0) {                                        \
            const int cw = cls[w];                             \
            if (cw == 2) {                                     \
                ccol[e] = cid[w];                              \
                ccap[e] = c_;                                  \
                e++;                                           \
            } else if (cw == 1) {                              \
                qs += qfix(c_, F);                             \
            } else {                                           \
                qt += qfix(c_, F);                             \
            }                                                  \
        }                                                      \
    }
    NB(z > 0, v - s.P, s.cz[v - s.P]);
    NB(y > 0, v - s.nx, s.cy[v - s.nx]);
    NB(xx > 0, v - 1, s.cx[v - 1]);
    NB(xx < s.nx - 1, v + 1, s.cx[v]);
    NB(y < s.ny - 1, v + s.nx, s.cy[v]);
    NB(z < s.nz - 1, v + s.P, s.cz[v]);
#undef NB
    cqs[me] = qs + qfix(s.cs[v], F);
    cqt[me] = qt + qfix(s.ct[v], F);
}

__global__ void __launch_bounds__(256) k_tl_fill_sell(SellArgs s, const int8_t *cls, const int32_t *cid,
                                                      const int32_t *eoff, int32_t F, int32_t *cp, int32_t *ccol,
                                                      double *ccap, i128 *cqs, i128 *cqt)
{
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= s.n || cls[v] != 2) return;
    const int32_t me = cid[v];
    int32_t e = eoff[v];
    cp[me] = e;
    i128 qs = 0, qt = 0;
    const int64_t sl = v / kSell;
    const int64_t e0 = s.slice_ptr[sl] + (v % kSell);
    const int32_t W = (int32_t)((s.slice_ptr[sl + 1] - s.slice_ptr[sl]) / kSell);
    for (int32_t k = 0; k < W; k++) {
        const int64_t idx = e0 + kSell * (int64_t)k;
        const int32_t nb = s.col[idx];
        if (nb < 0) break;
        const double c_ = s.c[idx];
        if (c_ > 0.0) {
            const int cw = cls[nb];
            if (cw == 2) {
                ccol[e] = cid[nb];
                ccap[e] = c_;
                e++;
            } else if (cw == 1) {
                qs += qfix(c_, F);
            } else {
                qt += qfix(c_, F);
            }
        }
    }
    cqs[me] = qs + qfix(s.cs[v], F);
    cqt[me] = qt + qfix(s.ct[v], F);
}

// lift: pseudo-rank 0 = source side ({s} + S1 + source side of G_c)
__global__ void k_tl_lift(const int8_t *cls, const int32_t *cid, const uint8_t *src, int64_t n, int32_t *prank)
{
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const int c = cls[v];
    prank[v] = (c == 1 || (c == 2 && src[cid[v]])) ? 0 : 1;
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
int64_t tl_ntiles(int64_t n) { return (n + kTlTile - 1) / kTlTile; }

void tl_kmeans_round(const double *x, int64_t n, TLState *st, const RedArgs &ra, cudaStream_t stream)
{
    k_tl_kmeans<<<(unsigned)((n + kChunk - 1) / kChunk), kThreads, 0, stream>>>(x, n, st, ra);
}

void tl_classify_stencil(const StencilArgs &s, int64_t N, const double *x, double g0, double g1, int32_t F,
                         TLBuffers &b, cudaStream_t st)
{
    k_tl_classify_stencil<<<(unsigned)tl_ntiles(N), 256, 0, st>>>(s, N, x, g0, g1, F, b.cls, b.flag, b.deg,
                                                                   b.tile_a, b.tile_n1);
}

void tl_classify_sell(const SellArgs &s, const double *x, double g0, double g1, int32_t F, TLBuffers &b,
                      cudaStream_t st)
{
    k_tl_classify_sell<<<(unsigned)tl_ntiles(s.n), 256, 0, st>>>(s, x, g0, g1, F, b.cls, b.flag, b.deg, b.tile_a,
                                                                b.tile_n1);
}

void tl_fill_stencil(const StencilArgs &s, int64_t N, int32_t F, TLBuffers &b, cudaStream_t st)
{
    k_tl_fill_stencil<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(s, N, F, b.cls, b.cid, b.eoff, b.cp, b.ccol,
                                                                    b.ccap, b.cqs, b.cqt);
}

void tl_fill_sell(const SellArgs &s, int32_t F, TLBuffers &b, cudaStream_t st)
{
    k_tl_fill_sell<<<(unsigned)((s.n + 255) / 256), 256, 0, st>>>(s, b.cls, b.cid, b.eoff, F, b.cp, b.ccol, b.ccap,
                                                                   b.cqs, b.cqt);
}

void tl_lift(TLBuffers &b, cudaStream_t st)
{
    if (b.n == 0) return;
    k_tl_lift<<<(unsigned)((b.n + 255) / 256), 256, 0, st>>>(b.cls, b.cid, b.src, b.n, b.prank);
}

}  // namespace irls
