// validate.cu — create-time checks of stencil capacities on the device:
// finite and >= 0 (A6), the count of zero interior n-links and of
// positive terminal edges (quick Prop. 1 test, A8), and max / count of the
// positive capacities for the sweep's fixed-point scale F (A15).
#include <algorithm>
#include "kernels.h"

namespace irls {

struct ValidateOut {
    unsigned long long bad, zero_nlinks, pos_terms, cnt_pos, cmax_bits, nlinks_pos;
};

__device__ __forceinline__ void vcheck(double c, bool present, unsigned long long &bad, unsigned long long &zero,
                                       unsigned long long &cnt, double &cmax, bool nlink)
{
    if (!present) return;
    if (!(c >= 0.0) || isinf(c)) { bad++; return; }
    if (c > 0.0) {
        cnt++;
        cmax = fmax(cmax, c);
    } else if (nlink) {
        zero++;
    }
}

__global__ void k_validate_stencil(int32_t nx, int32_t ny, int32_t nz, FastDiv fdx, FastDiv fdy, const double *cx,
                                   const double *cy, const double *cz, const double *cs, const double *ct, int64_t N,
                                   ValidateOut *out)
{
    unsigned long long bad = 0, zero = 0, cnt = 0, pt = 0, nl = 0;
    double cmax = 0.0;
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < N; u += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t uu = (uint32_t)u;
        const uint32_t t1 = fdiv(uu, fdx);
        const int32_t x = (int32_t)(uu - t1 * (uint32_t)nx);
        const uint32_t zz = fdiv(t1, fdy);
        const int32_t y = (int32_t)(t1 - zz * (uint32_t)ny), z = (int32_t)zz;
        const unsigned long long cb = cnt;
        vcheck(cx[u], x < nx - 1, bad, zero, cnt, cmax, true);
        vcheck(cy[u], y < ny - 1, bad, zero, cnt, cmax, true);
        vcheck(cz[u], z < nz - 1, bad, zero, cnt, cmax, true);
        nl += cnt - cb;
        const unsigned long long c0 = cnt;
        vcheck(cs[u], true, bad, zero, cnt, cmax, false);
        vcheck(ct[u], true, bad, zero, cnt, cmax, false);
        if (cnt > c0) pt++;
    }
    for (int off = 16; off >= 1; off >>= 1) {
        bad += __shfl_down_sync(0xffffffffu, bad, off);
        zero += __shfl_down_sync(0xffffffffu, zero, off);
        cnt += __shfl_down_sync(0xffffffffu, cnt, off);
        pt += __shfl_down_sync(0xffffffffu, pt, off);
        nl += __shfl_down_sync(0xffffffffu, nl, off);
        cmax = fmax(cmax, __shfl_down_sync(0xffffffffu, cmax, off));
    }
    if ((threadIdx.x & 31) == 0) {
        if (bad) atomicAdd(&out->bad, bad);
        if (zero) atomicAdd(&out->zero_nlinks, zero);
        if (cnt) atomicAdd(&out->cnt_pos, cnt);
        if (pt) atomicAdd(&out->pos_terms, pt);
        if (nl) atomicAdd(&out->nlinks_pos, nl);
        atomicMax(&out->cmax_bits, (unsigned long long)__double_as_longlong(cmax));  // cmax >= 0
    }
}

// returns 0 on success (host results in out_host[5])
int validate_stencil(int32_t nx, int32_t ny, int32_t nz, const double *cx, const double *cy, const double *cz,
                     const double *cs, const double *ct, unsigned long long *out_host, cudaStream_t st)
{
    ValidateOut *d = nullptr;
    if (cudaMallocAsync((void **)&d, sizeof(ValidateOut), st) != cudaSuccess) return 1;
    cudaMemsetAsync(d, 0, sizeof(ValidateOut), st);
    const int64_t N = (int64_t)nx * ny * nz;
    const FastDiv fdx = make_fastdiv((uint32_t)nx), fdy = make_fastdiv((uint32_t)ny);
    const int64_t nb = std::min<int64_t>((N + 255) / 256, 148 * 16);
    k_validate_stencil<<<(unsigned)nb, 256, 0, st>>>(nx, ny, nz, fdx, fdy, cx, cy, cz, cs, ct, N, d);
    ValidateOut h;
    cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(d, st);
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return 2;
    out_host[0] = h.bad;
    out_host[1] = h.zero_nlinks;
    out_host[2] = h.pos_terms;
    out_host[3] = h.cnt_pos;
    out_host[4] = h.cmax_bits;
    out_host[5] = h.nlinks_pos;
    return 0;
}

}  // namespace irls
