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

// delta_v of stencil node v (xv = canon(x[v])); qs = Q(cs_v) (for P_0).
// Every load is issued up front from clamped indices (absent neighbours read
// the node itself and get capacity 0, contributing +-Q(0) = 0), so the 15
// loads of a node are in flight together.
__device__ __forceinline__ void delta_stencil(const StencilArgs &s, int32_t F, const double *x, int64_t v, double xv,
                                              __int128 &d, __int128 &qs)
{
    const uint32_t uv = (uint32_t)v;
    const uint32_t t1 = fdiv(uv, s.fd_nx);
    const int32_t xx = (int32_t)(uv - t1 * (uint32_t)s.nx);
    const uint32_t zz = fdiv(t1, s.fd_ny);
    const int32_t y = (int32_t)(t1 - zz * (uint32_t)s.ny), z = (int32_t)zz;
    const bool hz0 = z > 0, hy0 = y > 0, hx0 = xx > 0, hx1 = xx < s.nx - 1, hy1 = y < s.ny - 1, hz1 = z < s.nz - 1;
    const int64_t wz0 = hz0 ? v - s.P : v, wy0 = hy0 ? v - s.nx : v, wx0 = hx0 ? v - 1 : v;
    const int64_t wx1 = hx1 ? v + 1 : v, wy1 = hy1 ? v + s.nx : v, wz1 = hz1 ? v + s.P : v;
    const double c0 = s.cz[wz0], c1 = s.cy[wy0], c2 = s.cx[wx0], c3 = s.cx[v], c4 = s.cy[v], c5 = s.cz[v];
    const double x0 = x[wz0], x1 = x[wy0], x2 = x[wx0], x3 = x[wx1], x4 = x[wy1], x5 = x[wz1];
    const double cs = s.cs[v], ct = s.ct[v];
    d = 0;
#define NB(has, w, xw, cap)                                                            {                                                                                      const __int128 q = qfix((has) ? (cap) : 0.0, F);                                   d += after(canon(xw), w, xv, v) ? q : -q;                                      }
    NB(hz0, wz0, x0, c0);
    NB(hy0, wy0, x1, c1);
    NB(hx0, wx0, x2, c2);
    NB(hx1, wx1, x3, c3);
    NB(hy1, wy1, x4, c4);
    NB(hz1, wz1, x5, c5);
#undef NB
    qs = qfix(cs, F);
    d += qfix(ct, F);
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
