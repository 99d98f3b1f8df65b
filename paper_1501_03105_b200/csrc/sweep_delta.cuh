// sweep_delta.cuh — the per-node quantities of the sweep (A14, A15), shared by
// the full sort (sweep.cu) and the branch-and-bound sweep (sweep_bb.cu):
//   key(v)   order-preserving 64-bit key, ascending key = x descending
//   delta_v  sum over neighbours u of (u after v ? +Q(c_uv) : -Q(c_uv)) +
//            Q(ct_v) - Q(cs_v), exact 128-bit fixed point (Q(c) = rint(c 2^F))
// where "u after v" in the total order (x desc, id asc, A14) is
// x_u < x_v || (x_u == x_v && u > v) — rank_u > rank_v, evaluated from the
// potentials, so delta needs no rank array.
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace irls {

__device__ __forceinline__ double canon(double x) { return x == 0.0 ? 0.0 : x; }  // -0.0 -> +0.0

__device__ __forceinline__ bool after(double xu, int64_t u, double xv, int64_t v)
{
    return xu < xv || (xu == xv && u > v);
}

__device__ __forceinline__ unsigned long long sweep_key(double xv) { return ~dkey_asc(xv); }

// delta_v of stencil node v (xv = canon(x[v])); qs = Q(cs_v) (for P_0)
__device__ __forceinline__ void delta_stencil(const StencilArgs &s, int32_t F, const double *x, int64_t v, double xv,
                                              __int128 &d, __int128 &qs)
{
    const uint32_t uv = (uint32_t)v;
    const uint32_t t1 = fdiv(uv, s.fd_nx);
    const int32_t xx = (int32_t)(uv - t1 * (uint32_t)s.nx);
    const uint32_t zz = fdiv(t1, s.fd_ny);
    const int32_t y = (int32_t)(t1 - zz * (uint32_t)s.ny), z = (int32_t)zz;
    d = 0;
#define NB(cond, w, cap)                                                           \
    if (cond) {                                                                    \
        const __int128 q = qfix(cap, F);                                           \
        d += after(canon(x[w]), w, xv, v) ? q : -q;                                \
    }
    NB(z > 0, v - s.P, s.cz[v - s.P]);
    NB(y > 0, v - s.nx, s.cy[v - s.nx]);
    NB(xx > 0, v - 1, s.cx[v - 1]);
    NB(xx < s.nx - 1, v + 1, s.cx[v]);
    NB(y < s.ny - 1, v + s.nx, s.cy[v]);
    NB(z < s.nz - 1, v + s.P, s.cz[v]);
#undef NB
    qs = qfix(s.cs[v], F);
    d += qfix(s.ct[v], F);
    d -= qs;
}

// delta_v of SELL-64 row v
__device__ __forceinline__ void delta_sell(const SellArgs &s, int32_t F, const double *x, int64_t v, double xv,
                                           __int128 &d, __int128 &qs)
{
    const int64_t sl = v / kSell;
    const int64_t e0 = s.slice_ptr[sl] + (v % kSell);
    const int32_t W = (int32_t)((s.slice_ptr[sl + 1] - s.slice_ptr[sl]) / kSell);
    d = 0;
    for (int32_t k = 0; k < W; k++) {
        const int64_t idx = e0 + kSell * (int64_t)k;
        const int32_t u = s.col[idx];
        if (u < 0) break;
        const __int128 q = qfix(s.c[idx], F);
        d += after(canon(x[u]), u, xv, v) ? q : -q;
    }
    qs = qfix(s.cs[v], F);
    d += qfix(s.ct[v], F);
    d -= qs;
}

}  // namespace irls
