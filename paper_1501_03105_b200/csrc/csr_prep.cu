// csr_prep.cu — create-time preparation of a CSR graph on the GPU (a1 of
// validate, merge duplicates (A7), exact symmetry, split the
// terminal edges, c_st (A5), Prop. 1 (A8), the SELL-64 layout).
//
// The same results as the host preparation in api_create.cu, entry for
// entry: rows are sorted by column with a stable insertion sort and equal
// columns summed in their CSR order (the host's stable_sort + sequential
// sum), so the merged capacities carry the same bits; every other output is
// integer or a copy.  Connected components for A8 by the lock-free
// union-find of the host path (link the larger root below the smaller with
// compare-and-swap; the components do not depend on the order).
#include <algorithm>
#include "kernels.h"

namespace irls {

typedef unsigned long long u64;

// First offending entry (column out of range, or c < 0 / NaN / Inf) and any
// self loop.  Thread per row.
__global__ void k_csr_check(const int64_t *rp, const int32_t *col, const double *w, int64_t n, u64 *first_bad,
                            int32_t *selfloop)
{
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n) return;
    for (int64_t e = rp[u]; e < rp[u + 1]; e++) {
        const int32_t c = col[e];
        const double x = w[e];
        if (c < 0 || c >= n || !(x >= 0.0) || isinf(x)) {
            atomicMin(first_bad, (u64)e);
            break;
        }
        if (c == u) *selfloop = 1;
    }
}

// Stable insertion sort of row u by column in the scratch copy (at the row's
// own offset), then duplicates merged in place by summation in CSR order.
__global__ void k_csr_merge_rows(const int64_t *rp, const int32_t *col, const double *w, int64_t n, int32_t *scol,
                                 double *sw, int32_t *mcnt)
{
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n) return;
    const int64_t a = rp[u], b = rp[u + 1];
    for (int64_t e = a; e < b; e++) {
        const int32_t c = col[e];
        const double x = w[e];
        int64_t i = e;
        while (i > a && scol[i - 1] > c) {  // strict: equal columns keep their CSR order
            scol[i] = scol[i - 1];
            sw[i] = sw[i - 1];
            i--;
        }
        scol[i] = c;
        sw[i] = x;
    }
    int64_t m = a;
    for (int64_t e = a; e < b; e++) {
        if (e > a && scol[e] == scol[m - 1]) {
            sw[m - 1] = sw[m - 1] + sw[e];
        } else {
            scol[m] = scol[e];
            sw[m] = sw[e];
            m++;
        }
    }
    mcnt[u] = (int32_t)(m - a);
}

__global__ void k_csr_compact(const int64_t *rp, const int32_t *scol, const double *sw, const int32_t *mptr, int64_t n,
                              int32_t *mcol, double *mw)
{
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n) return;
    const int64_t a = rp[u];
    for (int32_t k = 0; k < mptr[u + 1] - mptr[u]; k++) {
        mcol[mptr[u] + k] = scol[a + k];
        mw[mptr[u] + k] = sw[a + k];
    }
}

// Exact symmetry: (u, v, c) needs (v, u, c) with the same bits.
__global__ void k_csr_symmetry(const int32_t *mptr, const int32_t *mcol, const double *mw, int64_t n, int32_t *asym)
{
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n) return;
    for (int32_t e = mptr[u]; e < mptr[u + 1]; e++) {
        const int32_t v = mcol[e];
        int32_t lo = mptr[v], hi = mptr[v + 1];
        while (lo < hi) {
            const int32_t mid = (lo + hi) >> 1;
            if (mcol[mid] < u) lo = mid + 1;
            else hi = mid;
        }
        if (lo == mptr[v + 1] || mcol[lo] != u || mw[lo] != mw[e]) {
            *asym = 1;
            return;
        }
    }
}

// Reduced row r (original id u): terminal capacities, the n-link count
// (c > 0, neither terminal), and the inputs of the fixed-point scale F (the
// count and maximum of the positive capacities, each n-link once).
__global__ void k_csr_reduce_rows(const int32_t *mptr, const int32_t *mcol, const double *mw, int64_t nr, int64_t s,
                                  int64_t t, double *cs, double *ct, int64_t *orig, int32_t *acnt, u64 *cnt,
                                  u64 *cmax_bits)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    u64 cn = 0;
    double cm = 0.0;
    if (r < nr) {
        const int64_t lo2 = min(s, t), hi2 = max(s, t);
        int64_t u = r;
        if (u >= lo2) u++;
        if (u >= hi2) u++;
        orig[r] = u;
        double a = 0.0, b = 0.0;
        int32_t k = 0;
        for (int32_t e = mptr[u]; e < mptr[u + 1]; e++) {
            const int64_t v = mcol[e];
            const double x = mw[e];
            if (v == s) a = x;
            else if (v == t) b = x;
            else if (x > 0.0) {
                k++;
                if (v > u) { cn++; cm = fmax(cm, x); }
            }
        }
        cs[r] = a;
        ct[r] = b;
        acnt[r] = k;
        if (a > 0.0) { cn++; cm = fmax(cm, a); }
        if (b > 0.0) { cn++; cm = fmax(cm, b); }
    }
    // one atomic per warp (integer count; maximum: c >= 0, so bit order = value order)
    u64 bits = (u64)__double_as_longlong(cm);
    for (int off = 16; off >= 1; off >>= 1) {
        cn += __shfl_down_sync(0xffffffffu, cn, off);
        bits = max(bits, (u64)__shfl_down_sync(0xffffffffu, bits, off));
    }
    if ((threadIdx.x & 31) == 0) {
        if (cn) atomicAdd(cnt, cn);
        if (bits) atomicMax(cmax_bits, bits);
    }
}

__global__ void k_csr_reduce_fill(const int32_t *mptr, const int32_t *mcol, const double *mw, const int64_t *orig,
                                  const int32_t *aptr, int64_t nr, int64_t s, int64_t t, int32_t *aidx, double *ac)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nr) return;
    const int64_t u = orig[r];
    int32_t k = aptr[r];
    for (int32_t e = mptr[u]; e < mptr[u + 1]; e++) {
        const int64_t v = mcol[e];
        if (v == s || v == t || !(mw[e] > 0.0)) continue;
        aidx[k] = (int32_t)(v - (v > s) - (v > t));
        ac[k] = mw[e];
        k++;
    }
}

__global__ void k_csr_cst(const int32_t *mptr, const int32_t *mcol, const double *mw, int64_t s, int64_t t, double *out)
{
    double c = 0.0;
    for (int32_t e = mptr[s]; e < mptr[s + 1]; e++)
        if (mcol[e] == t) c = mw[e];
    *out = c;
}

// ---- union-find (A8)
__device__ __forceinline__ int32_t uf_find(int32_t *par, int32_t x)
{
    volatile int32_t *vp = par;
    for (;;) {
        const int32_t p = vp[x];
        if (p == x) return x;
        const int32_t gp = vp[p];
        if (gp != p) atomicCAS(par + x, p, gp);  // path halving
        x = gp;
    }
}

__global__ void k_uf_init(int32_t *par, int64_t nr)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < nr) par[r] = (int32_t)r;
}

__global__ void k_uf_link(const int32_t *aptr, const int32_t *aidx, int64_t nr, int32_t *par)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nr) return;
    for (int32_t e = aptr[r]; e < aptr[r + 1]; e++) {
        if (aidx[e] < r) continue;
        int32_t x = (int32_t)r, y = aidx[e];
        for (;;) {
            x = uf_find(par, x);
            y = uf_find(par, y);
            if (x == y) break;
            if (x < y) { const int32_t tmp = x; x = y; y = tmp; }  // link the larger root below the smaller
            if (atomicCAS(par + x, x, y) == x) break;
        }
    }
}

__global__ void k_uf_roots(int32_t *par, const double *cs, const double *ct, int64_t nr, int32_t *root,
                           uint8_t *anchored)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nr) return;
    const int32_t q = uf_find(par, (int32_t)r);
    root[r] = q;
    if (cs[r] > 0.0 || ct[r] > 0.0) anchored[q] = 1;
}

__global__ void k_uf_lonely(const int32_t *root, const uint8_t *anchored, int64_t nr, int32_t *lonely)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < nr && !anchored[root[r]]) *lonely = 1;
}

// ---- SELL-64: slice widths, then the fill (padding: column -1, capacity 0)
__global__ void k_sell_width(const int32_t *aptr, int64_t nr, int32_t *sw, u64 *wmax)
{
    const int64_t sl = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nsl = (nr + kSell - 1) / kSell;
    if (sl >= nsl) return;
    int32_t m = 0;
    for (int64_t r = sl * kSell; r < min(nr, sl * kSell + kSell); r++) m = max(m, aptr[r + 1] - aptr[r]);
    sw[sl] = kSell * m;
    atomicMax(wmax, (u64)m);
}

__global__ void k_i32_to_i64(const int32_t *in, int64_t n, int64_t *out)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = in[i];
}

__global__ void k_sell_fill(const int32_t *aptr, const int32_t *aidx, const double *ac, const int64_t *sptr, int64_t nr,
                            int32_t *scol, double *scap)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nr) return;
    const int64_t sl = r / kSell, ln = r % kSell;
    for (int32_t k = 0; k < aptr[r + 1] - aptr[r]; k++) {
        scol[sptr[sl] + kSell * (int64_t)k + ln] = aidx[aptr[r] + k];
        scap[sptr[sl] + kSell * (int64_t)k + ln] = ac[aptr[r] + k];
    }
}

static inline unsigned g256(int64_t n) { return (unsigned)std::max<int64_t>((n + 255) / 256, 1); }

void csrp_check(const int64_t *rp, const int32_t *col, const double *w, int64_t n, u64 *first_bad, int32_t *selfloop,
                cudaStream_t st)
{
    k_csr_check<<<g256(n), 256, 0, st>>>(rp, col, w, n, first_bad, selfloop);
}
void csrp_merge(const int64_t *rp, const int32_t *col, const double *w, int64_t n, int32_t *scol, double *sw,
                int32_t *mcnt, cudaStream_t st)
{
    k_csr_merge_rows<<<g256(n), 256, 0, st>>>(rp, col, w, n, scol, sw, mcnt);
}
void csrp_compact(const int64_t *rp, const int32_t *scol, const double *sw, const int32_t *mptr, int64_t n,
                  int32_t *mcol, double *mw, cudaStream_t st)
{
    k_csr_compact<<<g256(n), 256, 0, st>>>(rp, scol, sw, mptr, n, mcol, mw);
}
void csrp_symmetry(const int32_t *mptr, const int32_t *mcol, const double *mw, int64_t n, int32_t *asym,
                   cudaStream_t st)
{
    k_csr_symmetry<<<g256(n), 256, 0, st>>>(mptr, mcol, mw, n, asym);
}
void csrp_reduce(const int32_t *mptr, const int32_t *mcol, const double *mw, int64_t nr, int64_t s, int64_t t,
                 double *cs, double *ct, int64_t *orig, int32_t *acnt, u64 *cnt, u64 *cmax_bits, double *cst,
                 cudaStream_t st)
{
    k_csr_reduce_rows<<<g256(nr), 256, 0, st>>>(mptr, mcol, mw, nr, s, t, cs, ct, orig, acnt, cnt, cmax_bits);
    k_csr_cst<<<1, 1, 0, st>>>(mptr, mcol, mw, s, t, cst);
}
void csrp_fill(const int32_t *mptr, const int32_t *mcol, const double *mw, const int64_t *orig, const int32_t *aptr,
               int64_t nr, int64_t s, int64_t t, int32_t *aidx, double *ac, cudaStream_t st)
{
    k_csr_reduce_fill<<<g256(nr), 256, 0, st>>>(mptr, mcol, mw, orig, aptr, nr, s, t, aidx, ac);
}
void csrp_components(const int32_t *aptr, const int32_t *aidx, const double *cs, const double *ct, int64_t nr,
                     int32_t *par, int32_t *root, uint8_t *anchored, int32_t *lonely, cudaStream_t st)
{
    k_uf_init<<<g256(nr), 256, 0, st>>>(par, nr);
    k_uf_link<<<g256(nr), 256, 0, st>>>(aptr, aidx, nr, par);
    cudaMemsetAsync(anchored, 0, (size_t)std::max<int64_t>(nr, 1), st);
    k_uf_roots<<<g256(nr), 256, 0, st>>>(par, cs, ct, nr, root, anchored);
    k_uf_lonely<<<g256(nr), 256, 0, st>>>(root, anchored, nr, lonely);
}
void csrp_sell_width(const int32_t *aptr, int64_t nr, int32_t *sw, u64 *wmax, cudaStream_t st)
{
    k_sell_width<<<g256((nr + kSell - 1) / kSell), 256, 0, st>>>(aptr, nr, sw, wmax);
}
void csrp_i32_to_i64(const int32_t *in, int64_t n, int64_t *out, cudaStream_t st)
{
    k_i32_to_i64<<<g256(n), 256, 0, st>>>(in, n, out);
}
void csrp_sell_fill(const int32_t *aptr, const int32_t *aidx, const double *ac, const int64_t *sptr, int64_t nr,
                    int32_t *scol, double *scap, cudaStream_t st)
{
    k_sell_fill<<<g256(nr), 256, 0, st>>>(aptr, aidx, ac, sptr, nr, scol, scap);
}

}  // namespace irls
