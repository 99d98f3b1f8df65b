// sweep.cu — GPU sweep cut ("sorting the nodes according to x^(T)";
// O7 / A14 / A15 in DESIGN.md §2).
//
//   keys      order-preserving 64-bit key of x (descending), ids as values
//   sort      stable LSD radix sort, 8-bit digits; constant-digit passes skipped
//   rank      rank[order[i]] = i
//   delta     delta_v = sum_u (+-Q(c_uv)) + Q(ct_v) - Q(cs_v) in exact 128-bit
//             fixed point (Q(c) = rint(c 2^F)), written at position rank[v]
//   scan      P_i = P_0 + delta_0 + ... + delta_{i-1}; exact integer sums, so
//             any parallel order equals the sequential definition
//   argmin    first i in 0..n minimising P_i
//   side/cut  side[v] = rank[v] < k; cut value recomputed by C3 (+ c_st)
#include <algorithm>
#include "kernels.h"
#include "sweep_delta.cuh"

namespace irls {

typedef unsigned long long u64;
typedef __int128 i128;

constexpr int kTile = 4096;  // keys per tile (256 threads x 16)

int64_t sweep_ntiles(int64_t n) { return (n + kTile - 1) / kTile; }


__int128 qfix_host(double c, int32_t F)
{
    if (c == 0.0) return 0;
    const double v = rint(ldexp(c, F));
    return (__int128)v;
}

__device__ __forceinline__ i128 shfl_up_i128(i128 v, int off)
{
    u64 lo = (u64)v, hi = (u64)(v >> 64);
    lo = __shfl_up_sync(0xffffffffu, lo, off);
    hi = __shfl_up_sync(0xffffffffu, hi, off);
    return ((i128)hi << 64) | (i128)lo;
}
__device__ __forceinline__ i128 shfl_down_i128(i128 v, int off)
{
    u64 lo = (u64)v, hi = (u64)(v >> 64);
    lo = __shfl_down_sync(0xffffffffu, lo, off);
    hi = __shfl_down_sync(0xffffffffu, hi, off);
    return ((i128)hi << 64) | (i128)lo;
}

__device__ __forceinline__ void tile_sum_i128(i128 v, i128 *out)
{
    __shared__ i128 sm[8];
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v += shfl_down_i128(v, off);
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        i128 s = 0;
        for (int i = 0; i < 8; i++) s += sm[i];
        *out = s;
    }
}

// ---------------------------------------------------------------------------
// prep: keys, ids, the exact delta_v in id order (sweep_delta.cuh), global
// digit histograms; delta is written coalesced in id order (the scan gathers it)
// ---------------------------------------------------------------------------
template <class NB>
__device__ __forceinline__ void prep_tile(int64_t N, int32_t F, const double *x, u64 *keys, int32_t *vals,
                                          i128 *delta, u64 *digit_hist, i128 *qcs_tile, int32_t *flags, NB nb)
{
    __shared__ unsigned h[8][256];
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) (&h[0][0])[i] = 0u;
    __syncthreads();
    i128 qcs = 0;
    bool nan = false;
    const int64_t base = (int64_t)blockIdx.x * kTile;
    for (int r = 0; r < 16; r++) {
        const int64_t v = base + r * 256 + threadIdx.x;
        if (v >= N) break;
        const double xr = x[v];
        nan |= isnan(xr);
        const double xv = canon(xr);
        const u64 key = sweep_key(xv);  // ascending key order = x descending
        keys[v] = key;
        vals[v] = (int32_t)v;           // ties keep ascending id (stable sort)
#pragma unroll
        for (int d = 0; d < 8; d++) atomicAdd(&h[d][(key >> (8 * d)) & 255u], 1u);
        i128 d = 0, qs = 0;
        nb(v, xv, d, qs);
        qcs += qs;
        delta[v] = d;
    }
    if (nan) flags[0] = 1;
    __syncthreads();
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) {
        const unsigned c = (&h[0][0])[i];
        if (c) atomicAdd(&digit_hist[i], (u64)c);
    }
    tile_sum_i128(qcs, qcs_tile + blockIdx.x);
}

__global__ void __launch_bounds__(256) k_sweep_prep_stencil(StencilArgs s, int64_t N, int32_t F, const double *x,
                                                            u64 *keys, int32_t *vals, i128 *delta, u64 *digit_hist,
                                                            i128 *qcs_tile, int32_t *flags)
{
    prep_tile(N, F, x, keys, vals, delta, digit_hist, qcs_tile, flags,
              [&](int64_t v, double xv, i128 &d, i128 &qs) { delta_stencil(s, F, x, v, xv, d, qs); });
}

__global__ void __launch_bounds__(256) k_sweep_prep_sell(SellArgs s, int32_t F, const double *x, u64 *keys,
                                                         int32_t *vals, i128 *delta, u64 *digit_hist, i128 *qcs_tile,
                                                         int32_t *flags)
{
    prep_tile(s.n, F, x, keys, vals, delta, digit_hist, qcs_tile, flags,
              [&](int64_t v, double xv, i128 &d, i128 &qs) { delta_sell(s, F, x, v, xv, d, qs); });
}

// ---------------------------------------------------------------------------
// radix sort: stable LSD, 8-bit digits, one kernel per pass ("onesweep"):
// tiles taken in ticket order publish their digit counts and find their
// global offsets by decoupled look-back over the earlier tiles
// ---------------------------------------------------------------------------
constexpr uint32_t kStAgg = 1u << 30, kStIncl = 2u << 30, kStMask = (1u << 30) - 1u;

struct GStart {
    int32_t g[256];  // global start of every digit's bucket in this pass
};

// Stable scatter of one tile.  Warp w owns keys [base + 512 w, +512) in 16
// rounds of 32; ranking in ONE pass: per round, the lanes holding the same
// digit find each other (match_any); the lowest of them advances the warp's
// counter of that digit with a shared-memory atomic whose old value,
// broadcast to the group, is the group's start — so every key gets its rank
// among the warp's keys of its digit, in key order.  Then the tile's digit
// counts are published (aggregate), the exclusive prefix over earlier tiles
// found by look-back (inclusive prefix published), the per-warp digit starts
// formed (digit-major, warp-minor: stable), the keys staged in shared memory
// in digit order and written out so that consecutive threads write
// consecutive positions of a bucket.
template <int KPT, int MINB>
__global__ void __launch_bounds__(256, MINB) k_onesweep(const u64 *keys, const int32_t *vals, u64 *okeys,
                                                     int32_t *ovals, int64_t n, int shift, GStart gs, uint32_t *state,
                                                     int32_t *ticket)
{
    constexpr int RT = 256 * KPT;      // keys per tile
    __shared__ int32_t wh[8][256];     // per-warp digit counts, then per-warp tile starts
    __shared__ int32_t gdelta[256];    // global start of the bucket minus its tile-local start
    __shared__ int32_t s_tile;
    extern __shared__ __align__(16) unsigned char radix_dyn[];  // RT keys + RT values
    u64 *skey = reinterpret_cast<u64 *>(radix_dyn);
    int32_t *sval = reinterpret_cast<int32_t *>(radix_dyn + sizeof(u64) * RT);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1);
    for (int i = threadIdx.x; i < 8 * 256; i += 256) (&wh[0][0])[i] = 0;
    __syncthreads();
    const int32_t tile = s_tile;
    const int64_t tbase = (int64_t)tile * RT;
    const int64_t base = tbase + w * 32 * KPT;
    u64 k[KPT];
    int32_t vv[KPT];
    uint32_t dr[KPT];  // digit << 16 | rank within (warp, digit); 0xffffffff past n
#pragma unroll
    for (int r = 0; r < KPT; r++) {
        const int64_t i = base + r * 32 + lane;
        if (i < n) {
            k[r] = __ldcs(keys + i);
            vv[r] = __ldcs(vals + i);
        } else {
            k[r] = 0;
            vv[r] = 0;
        }
    }
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int r = 0; r < KPT; r++) {
        const int64_t i = base + r * 32 + lane;
        const int d = i < n ? (int)((k[r] >> shift) & 255u) : 256 + lane;  // past n: a group of one
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const int leader = __ffs(peers) - 1;
        int old = 0;
        if (lane == leader && d < 256) old = atomicAdd(&wh[w][d], __popc(peers));
        old = __shfl_sync(0xffffffffu, old, leader);
        dr[r] = d < 256 ? ((uint32_t)d << 16) | (uint32_t)(old + __popc(peers & lt)) : 0xffffffffu;
    }
    __syncthreads();
    // digit d (one per thread): tile total, published; look-back; exclusive
    // scan over digits; per-warp starts
    const int d = threadIdx.x;
    int32_t tot = 0;
#pragma unroll
    for (int w2 = 0; w2 < 8; w2++) tot += wh[w2][d];
    volatile uint32_t *vst = state;
    vst[(int64_t)tile * 256 + d] = (tile == 0 ? kStIncl : kStAgg) | (uint32_t)tot;
    int32_t excl = 0;
    if (tile > 0) {
        // four predecessors per round (independent loads): the ready prefix
        // is consumed up to the first inclusive prefix
        int64_t t = tile - 1;
        for (bool done = false; !done;) {
            uint32_t wv[4];
#pragma unroll
            for (int q = 0; q < 4; q++) wv[q] = t - q >= 0 ? vst[(t - q) * 256 + d] : (2u << 30);  // (below tile 0: an empty inclusive prefix)
            int q = 0;
            for (; q < 4; q++) {
                if ((wv[q] & ~kStMask) == 0u) break;
                excl += (int32_t)(wv[q] & kStMask);
                if ((wv[q] & ~kStMask) == kStIncl) {
                    done = true;
                    break;
                }
            }
            if (done) break;
            if (q == 0) __nanosleep(32);
            t -= q;
        }
        vst[(int64_t)tile * 256 + d] = kStIncl | (uint32_t)(excl + tot);
    }
    {
        int32_t inc = tot;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int32_t o = __shfl_up_sync(0xffffffffu, inc, off);
            if (lane >= off) inc += o;
        }
        __shared__ int32_t wsum[8];
        if (lane == 31) wsum[w] = inc;
        __syncthreads();
        int32_t pre = 0;
        for (int i = 0; i < w; i++) pre += wsum[i];
        const int32_t ex = pre + inc - tot;
        gdelta[d] = gs.g[d] + excl - ex;
        int32_t run = ex;
#pragma unroll
        for (int w2 = 0; w2 < 8; w2++) {
            const int32_t c = wh[w2][d];
            wh[w2][d] = run;
            run += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < KPT; r++) {
        if (dr[r] != 0xffffffffu) {
            const int32_t pos = wh[w][dr[r] >> 16] + (int32_t)(dr[r] & 0xffffu);
            skey[pos] = k[r];
            sval[pos] = vv[r];
        }
    }
    __syncthreads();
    const int32_t cnt = (int32_t)(n - tbase < RT ? n - tbase : RT);
    for (int i = threadIdx.x; i < cnt; i += 256) {
        const u64 key = skey[i];
        const int dd = (int)((key >> shift) & 255u);
        const int64_t g = (int64_t)gdelta[dd] + i;
        okeys[g] = key;
        ovals[g] = sval[i];
    }
}

// Exclusive scan of int32 counts (length m) -> out, via 4096-element blocks.
__device__ __forceinline__ int64_t block_exscan_i64(int64_t v, int64_t *smem, int64_t &total)
{
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int64_t inc = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int64_t o = __shfl_up_sync(0xffffffffu, inc, off);
        if (lane >= off) inc += o;
    }
    if (lane == 31) smem[w] = inc;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t run = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); i++) {
            const int64_t c = smem[i];
            smem[i] = run;
            run += c;
        }
        smem[32] = run;
    }
    __syncthreads();
    const int64_t ex = smem[w] + inc - v;
    total = smem[32];
    __syncthreads();
    return ex;
}

__global__ void __launch_bounds__(256) k_scan_reduce(const int32_t *in, int64_t m, int64_t *bsum)
{
    __shared__ int64_t sm[33];
    int64_t acc = 0;
    const int64_t base = (int64_t)blockIdx.x * kTile;
    for (int r = 0; r < 16; r++) {
        const int64_t i = base + r * 256 + threadIdx.x;
        if (i < m) acc += in[i];
    }
    int64_t tot;
    block_exscan_i64(acc, sm, tot);
    if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(256) k_scan_top(int64_t *bsum, int64_t nb)
{
    __shared__ int64_t sm[33];
    int64_t carry = 0;
    for (int64_t b0 = 0; b0 < nb; b0 += 256) {
        const int64_t i = b0 + threadIdx.x;
        const int64_t v = i < nb ? bsum[i] : 0;
        int64_t tot;
        const int64_t ex = block_exscan_i64(v, sm, tot);
        if (i < nb) bsum[i] = carry + ex;
        carry += tot;
    }
}

__global__ void __launch_bounds__(256) k_scan_down(const int32_t *in, int64_t m, const int64_t *bsum,
                                                   int32_t *out)
{
    __shared__ int64_t sm[33];
    int64_t carry = bsum[blockIdx.x];
    const int64_t base = (int64_t)blockIdx.x * kTile;
    for (int r = 0; r < 16; r++) {
        const int64_t i = base + r * 256 + threadIdx.x;
        const int64_t v = i < m ? in[i] : 0;
        int64_t tot;
        const int64_t ex = block_exscan_i64(v, sm, tot);
        if (i < m) out[i] = (int32_t)(carry + ex);
        carry += tot;
    }
}

void exclusive_scan_i32(const int32_t *in, int64_t m, int32_t *out, int64_t *tmp, cudaStream_t st,
                        int *launches)
{
    const int64_t nb = (m + kTile - 1) / kTile;
    k_scan_reduce<<<(unsigned)nb, 256, 0, st>>>(in, m, tmp);
    k_scan_top<<<1, 256, 0, st>>>(tmp, nb);
    k_scan_down<<<(unsigned)nb, 256, 0, st>>>(in, m, tmp, out);
    *launches += 3;
}

void sweep_prep_stencil(const StencilArgs &s, int64_t N, int32_t F, const double *x, SweepBuffers &b,
                        cudaStream_t st)
{
    if (N == 0) return;
    k_sweep_prep_stencil<<<(unsigned)sweep_ntiles(N), 256, 0, st>>>(s, N, F, x, b.keys, b.vals, b.delta, b.digit_hist,
                                                                    b.qcs_tile, b.flags);
}

void sweep_prep_sell(const SellArgs &s, int32_t F, const double *x, SweepBuffers &b, cudaStream_t st)
{
    if (s.n == 0) return;
    k_sweep_prep_sell<<<(unsigned)sweep_ntiles(s.n), 256, 0, st>>>(s, F, x, b.keys, b.vals, b.delta, b.digit_hist,
                                                                  b.qcs_tile, b.flags);
}

int32_t *sweep_sort(SweepBuffers &b, cudaStream_t st, int *launches, bool *nan)
{
    const int64_t n = b.n;
    *nan = false;
    if (n == 0) return b.vals;
    const int64_t nt = sweep_ntiles(n);
    // one host round trip: the digit histograms (constant-digit passes are
    // skipped; the others' bucket starts) and the NaN flag of the prep kernel
    u64 h[8 * 256];
    int32_t hflag = 0;
    cudaMemcpyAsync(h, b.digit_hist, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&hflag, b.flags, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    if (hflag) {
        *nan = true;
        return b.vals;
    }
    u64 *ka = b.keys, *kb = b.keys_alt;
    int32_t *va = b.vals, *vb = b.vals_alt;
    uint32_t *state = reinterpret_cast<uint32_t *>(b.tile_hist);  // [ntiles][256] look-back words
    int32_t *ticket = b.flags + 1;
    // keys per thread: 16 (tiles of 4096, 3 CTAs/SM; measured 9.5 ms per sweep on
    // config 4 against 11.4 ms with IRLS_SORT_KPT=8: tiles of 2048 at 4 CTAs/SM)
    static const int kpt = getenv("IRLS_SORT_KPT") && atoi(getenv("IRLS_SORT_KPT")) == 8 ? 8 : 16;
    const int64_t rt = 256 * (int64_t)kpt, ntr = (n + rt - 1) / rt;
    const int dyn = (int)((sizeof(u64) + sizeof(int32_t)) * rt);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_onesweep<16, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 4096);
        cudaFuncSetAttribute(k_onesweep<8, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 2048);
        attr = true;
    }
    for (int d = 0; d < 8; d++) {
        bool run = true;
        for (int i = 0; i < 256; i++)
            if (h[d * 256 + i] == (u64)n) run = false;
        if (!run) continue;
        GStart gs;
        int64_t acc = 0;
        for (int i = 0; i < 256; i++) {
            gs.g[i] = (int32_t)acc;
            acc += (int64_t)h[d * 256 + i];
        }
        cudaMemsetAsync(state, 0, sizeof(uint32_t) * 256 * ntr, st);
        cudaMemsetAsync(ticket, 0, sizeof(int32_t), st);
        if (kpt == 16) k_onesweep<16, 3><<<(unsigned)ntr, 256, dyn, st>>>(ka, va, kb, vb, n, 8 * d, gs, state, ticket);
        else k_onesweep<8, 4><<<(unsigned)ntr, 256, dyn, st>>>(ka, va, kb, vb, n, 8 * d, gs, state, ticket);
        *launches += 1;
        std::swap(ka, kb);
        std::swap(va, vb);
    }
    return va;
}

// ---------------------------------------------------------------------------
// scan + argmin
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool lex_less(i128 a, int64_t ia, i128 b, int64_t ib)
{
    return a < b || (a == b && ia < ib);
}

// P_0 = Q(c_st) + sum of the prep kernel's per-tile Q(cs) sums (one block).
__global__ void __launch_bounds__(256) k_p0(const i128 *qcs_tile, int64_t nt, i128 qcst, i128 *p0_out)
{
    __shared__ i128 sm[256];
    i128 q = 0;
    for (int64_t i = threadIdx.x; i < nt; i += 256) q += qcs_tile[i];
    sm[threadIdx.x] = q;
    __syncthreads();
    if (threadIdx.x == 0) {
        i128 p0 = qcst;
        for (int i = 0; i < 256; i++) p0 += sm[i];
        *p0_out = p0;
    }
}

// Single pass over the sweep order: tile t (ticket order) gathers its 4096
// deltas (id order, through ord), publishes its sum, finds the exclusive
// prefix by decoupled look-back (exact integers: any association gives the
// same P_i), then forms P_{i+1} = P_0 + delta_0 + ... + delta_i and the
// tile's first minimum.  look[t] = 0 (nothing), 1 (aggregate in agg[t]),
// 2 (inclusive prefix in incl[t]); values are written before their flag.
__global__ void __launch_bounds__(256) k_scan_argmin(const i128 *delta, const int32_t *ord, int64_t n,
                                                     const i128 *p0, i128 *agg, i128 *incl, int32_t *look,
                                                     int32_t *ticket, i128 *tile_min, int64_t *tile_arg)
{
    __shared__ i128 wsum[8];
    __shared__ i128 smin[8];
    __shared__ int64_t sarg[8];
    __shared__ i128 s_excl;
    __shared__ int32_t s_tile;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1);
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t t0 = tile * kTile + 16 * (int64_t)threadIdx.x;
    int32_t id[16];
#pragma unroll
    for (int q = 0; q < 16; q++) id[q] = t0 + q < n ? ord[t0 + q] : -1;
    i128 own = 0, dl[16];
#pragma unroll
    for (int q = 0; q < 16; q++) {
        dl[q] = id[q] >= 0 ? delta[id[q]] : (i128)0;
        own += dl[q];
    }
    i128 inc = own;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const i128 o = shfl_up_i128(inc, off);
        if (lane >= off) inc += o;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    i128 wpre = 0;
    for (int k = 0; k < w; k++) wpre += wsum[k];
    if (w == 0) {  // warp 0: publish the tile sum, then look back 32 tiles at a time
        i128 T = 0;
        for (int k = 0; k < 8; k++) T += wsum[k];
        volatile int32_t *vlook = look;
        i128 ex = 0;
        if (tile == 0) {
            ex = *p0;
        } else {
            if (lane == 0) {
                agg[tile] = T;
                __threadfence();
                vlook[tile] = 1;
            }
            for (int64_t hi = tile - 1;;) {
                const int64_t t = hi - lane;  // lane 0: the nearest predecessor
                const int32_t f = t >= 0 ? vlook[t] : 2;
                const unsigned ready = __ballot_sync(0xffffffffu, f != 0);
                const unsigned incl_m = __ballot_sync(0xffffffffu, f == 2);
                int upto = -1;  // lanes 0..upto are summed
                if (incl_m) {
                    const int first = __ffs(incl_m) - 1;
                    const unsigned need = first == 31 ? 0xffffffffu : ((2u << first) - 1u);
                    if ((ready & need) == need) upto = first;
                } else if (ready == 0xffffffffu) {
                    upto = 31;
                }
                if (upto < 0) {
                    __nanosleep(32);
                    continue;
                }
                __threadfence();
                i128 v = 0;
                if (lane <= upto && t >= 0) v = (f == 2) ? *(volatile i128 *)(incl + t) : *(volatile i128 *)(agg + t);
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) v += shfl_down_i128(v, off);
                ex += v;  // lane 0 holds the window's sum
                if (incl_m && upto == __ffs(incl_m) - 1) break;
                hi -= 32;
            }
        }
        if (lane == 0) {
            incl[tile] = ex + T;
            __threadfence();
            vlook[tile] = 2;
            s_excl = ex;
        }
    }
    __syncthreads();
    i128 P = s_excl + wpre + inc - own;  // P_{t0}
    i128 best = (i128)(((unsigned __int128)1 << 127) - 1);  // +infinity
    int64_t barg = INT64_MAX;
#pragma unroll
    for (int q = 0; q < 16; q++) {
        const int64_t i = t0 + q;
        if (i < n) {
            P += dl[q];  // P_{i+1}
            if (lex_less(P, i + 1, best, barg)) { best = P; barg = i + 1; }
        }
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        const i128 ob = shfl_down_i128(best, off);
        const int64_t oa = __shfl_down_sync(0xffffffffu, barg, off);
        if (lex_less(ob, oa, best, barg)) { best = ob; barg = oa; }
    }
    if (lane == 0) { smin[w] = best; sarg[w] = barg; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < 8; k++)
            if (lex_less(smin[k], sarg[k], best, barg)) { best = smin[k]; barg = sarg[k]; }
        tile_min[tile] = best;
        tile_arg[tile] = barg;
    }
}

__global__ void __launch_bounds__(256) k_final_argmin(const i128 *tile_min, const int64_t *tile_arg, int64_t nt,
                                                      const i128 *p0, int64_t *k_out, i128 *pk_out)
{
    __shared__ i128 smin[256];
    __shared__ int64_t sarg[256];
    i128 best = *p0;
    int64_t barg = 0;
    for (int64_t i = threadIdx.x; i < nt; i += 256)
        if (lex_less(tile_min[i], tile_arg[i], best, barg)) { best = tile_min[i]; barg = tile_arg[i]; }
    smin[threadIdx.x] = best;
    sarg[threadIdx.x] = barg;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < 256; k++)
            if (lex_less(smin[k], sarg[k], best, barg)) { best = smin[k]; barg = sarg[k]; }
        *k_out = barg;
        *pk_out = best;
    }
}

void sweep_scan_argmin(SweepBuffers &b, const int32_t *ord, __int128 qcst, cudaStream_t st)
{
    const int64_t n = b.n, nt = sweep_ntiles(n);
    i128 *p0 = b.delta + n;        // two spare slots at the end of delta
    i128 *pk = b.delta + n + 1;
    int32_t *look = b.tile_hist;   // the radix passes are done with it
    k_p0<<<1, 256, 0, st>>>(b.qcs_tile, nt, qcst, p0);
    if (nt > 0) {
        cudaMemsetAsync(look, 0, sizeof(int32_t) * nt, st);
        cudaMemsetAsync(b.flags + 1, 0, sizeof(int32_t), st);
        k_scan_argmin<<<(unsigned)nt, 256, 0, st>>>(b.delta, ord, n, p0, b.tile_sum, b.tile_incl, look, b.flags + 1,
                                                    b.tile_min, b.tile_argmin);
    }
    k_final_argmin<<<1, 256, 0, st>>>(b.tile_min, b.tile_argmin, nt, p0, b.k_out, pk);
}

// ---------------------------------------------------------------------------
// side + directly recomputed cut value (O7 step 7), C3 over cross_v
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_side_cross_stencil(StencilArgs s, int64_t N, const int32_t *rank,
                                                                 const int64_t *kptr, uint8_t *side, RedArgs ra)
{
    const int64_t k = *kptr;
    double acc[1] = {0.0};
    const int64_t base = (int64_t)blockIdx.x * kChunk;
    for (int j = 0; j < 8; j++)
        for (int e = 0; e < 2; e++) {
            const int64_t v = base + 2 * (int64_t)threadIdx.x + 512 * j + e;
            if (v >= N) continue;
            const bool in = rank[v] < k;
            side[v] = in ? 1 : 0;
            double cr;
            if (in) {
                const uint32_t uv = (uint32_t)v;
                const uint32_t t1 = fdiv(uv, s.fd_nx);
                const int32_t x = (int32_t)(uv - t1 * (uint32_t)s.nx);
                const uint32_t zz = fdiv(t1, s.fd_ny);
                const int32_t y = (int32_t)(t1 - zz * (uint32_t)s.ny), z = (int32_t)zz;
                double a = 0.0;
                if (z > 0 && rank[v - s.P] >= k) a = a + s.cz[v - s.P];
                if (y > 0 && rank[v - s.nx] >= k) a = a + s.cy[v - s.nx];
                if (x > 0 && rank[v - 1] >= k) a = a + s.cx[v - 1];
                if (x < s.nx - 1 && rank[v + 1] >= k) a = a + s.cx[v];
                if (y < s.ny - 1 && rank[v + s.nx] >= k) a = a + s.cy[v];
                if (z < s.nz - 1 && rank[v + s.P] >= k) a = a + s.cz[v];
                cr = a + s.ct[v];
            } else {
                cr = s.cs[v];
            }
            acc[0] = acc[0] + cr;
        }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        side[N] = 1;
        side[N + 1] = 0;
    }
    c3_chunk_epilogue<1>(acc, (int32_t)blockIdx.x, ra);
}

__global__ void __launch_bounds__(kThreads) k_side_cross_sell(SellArgs s, const int32_t *rank, const int64_t *kptr,
                                                              const int64_t *orig, uint8_t *side, RedArgs ra)
{
    const int64_t k = *kptr;
    double acc[1] = {0.0};
    const int64_t base = (int64_t)blockIdx.x * kChunk;
    for (int j = 0; j < 8; j++)
        for (int e = 0; e < 2; e++) {
            const int64_t v = base + 2 * (int64_t)threadIdx.x + 512 * j + e;
            if (v >= s.n) continue;
            const bool in = rank[v] < k;
            side[orig[v]] = in ? 1 : 0;
            double cr;
            if (in) {
                const int64_t sl = v / kSell;
                const int64_t e0 = s.slice_ptr[sl] + (v % kSell);
                const int32_t W = (int32_t)((s.slice_ptr[sl + 1] - s.slice_ptr[sl]) / kSell);
                double a = 0.0;
                for (int32_t kk = 0; kk < W; kk++) {
                    const int64_t idx = e0 + kSell * (int64_t)kk;
                    const int32_t nb = s.col[idx];
                    if (nb < 0) break;
                    if (rank[nb] >= k) a = a + s.c[idx];
                }
                cr = a + s.ct[v];
            } else {
                cr = s.cs[v];
            }
            acc[0] = acc[0] + cr;
        }
    c3_chunk_epilogue<1>(acc, (int32_t)blockIdx.x, ra);
}

// The sweep's own side / cut pass: membership straight from the potentials —
// v is among the first k of the order iff (x_v, v) precedes or equals the
// k-th element (x*, v*): x_v > x* || (x_v == x* && v <= v*) — no rank array.
__device__ __forceinline__ bool in_first_k(double xv, int64_t v, bool any, double xs, int64_t vs)
{
    return any && (xv > xs || (xv == xs && v <= vs));
}

__global__ void __launch_bounds__(kThreads) k_side_cross_x_stencil(StencilArgs s, int64_t N, const double *x,
                                                                   const int32_t *ord, const int32_t *lastv,
                                                                   const int64_t *kptr, uint8_t *side, RedArgs ra)
{
    const int64_t k = *kptr;
    const bool any = k > 0;
    const int64_t vs = any ? (ord ? ord[k - 1] : *lastv) : 0;
    const double xs = any ? canon(x[vs]) : 0.0;
    double acc[1] = {0.0};
    const int64_t base = (int64_t)blockIdx.x * kChunk;
    for (int j = 0; j < 8; j++)
        for (int e = 0; e < 2; e++) {
            const int64_t v = base + 2 * (int64_t)threadIdx.x + 512 * j + e;
            if (v >= N) continue;
            const bool in = in_first_k(canon(x[v]), v, any, xs, vs);
            side[v] = in ? 1 : 0;
            double cr;
            if (in) {
                const uint32_t uv = (uint32_t)v;
                const uint32_t t1 = fdiv(uv, s.fd_nx);
                const int32_t xx = (int32_t)(uv - t1 * (uint32_t)s.nx);
                const uint32_t zz = fdiv(t1, s.fd_ny);
                const int32_t y = (int32_t)(t1 - zz * (uint32_t)s.ny), z = (int32_t)zz;
                double a = 0.0;
#define OUT(w) (!in_first_k(canon(x[w]), (w), any, xs, vs))
                if (z > 0 && OUT(v - s.P)) a = a + s.cz[v - s.P];
                if (y > 0 && OUT(v - s.nx)) a = a + s.cy[v - s.nx];
                if (xx > 0 && OUT(v - 1)) a = a + s.cx[v - 1];
                if (xx < s.nx - 1 && OUT(v + 1)) a = a + s.cx[v];
                if (y < s.ny - 1 && OUT(v + s.nx)) a = a + s.cy[v];
                if (z < s.nz - 1 && OUT(v + s.P)) a = a + s.cz[v];
#undef OUT
                cr = a + s.ct[v];
            } else {
                cr = s.cs[v];
            }
            acc[0] = acc[0] + cr;
        }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        side[N] = 1;
        side[N + 1] = 0;
    }
    c3_chunk_epilogue<1>(acc, (int32_t)blockIdx.x, ra);
}

__global__ void __launch_bounds__(kThreads) k_side_cross_x_sell(SellArgs s, const double *x, const int32_t *ord,
                                                                const int32_t *lastv, const int64_t *kptr,
                                                                const int64_t *orig, uint8_t *side, RedArgs ra)
{
    const int64_t k = *kptr;
    const bool any = k > 0;
    const int64_t vs = any ? (ord ? ord[k - 1] : *lastv) : 0;
    const double xs = any ? canon(x[vs]) : 0.0;
    double acc[1] = {0.0};
    const int64_t base = (int64_t)blockIdx.x * kChunk;
    for (int j = 0; j < 8; j++)
        for (int e = 0; e < 2; e++) {
            const int64_t v = base + 2 * (int64_t)threadIdx.x + 512 * j + e;
            if (v >= s.n) continue;
            const bool in = in_first_k(canon(x[v]), v, any, xs, vs);
            side[orig[v]] = in ? 1 : 0;
            double cr;
            if (in) {
                const int64_t sl = v / kSell;
                const int64_t e0 = s.slice_ptr[sl] + (v % kSell);
                const int32_t W = (int32_t)((s.slice_ptr[sl + 1] - s.slice_ptr[sl]) / kSell);
                double a = 0.0;
                for (int32_t kk = 0; kk < W; kk++) {
                    const int64_t idx = e0 + kSell * (int64_t)kk;
                    const int32_t u = s.col[idx];
                    if (u < 0) break;
                    if (!in_first_k(canon(x[u]), u, any, xs, vs)) a = a + s.c[idx];
                }
                cr = a + s.ct[v];
            } else {
                cr = s.cs[v];
            }
            acc[0] = acc[0] + cr;
        }
    c3_chunk_epilogue<1>(acc, (int32_t)blockIdx.x, ra);
}

void sweep_side_cross_x_stencil(const StencilArgs &s, int64_t N, const double *x, const int32_t *ord, SweepBuffers &b,
                                const RedArgs &ra, cudaStream_t st)
{
    k_side_cross_x_stencil<<<(unsigned)((N + kChunk - 1) / kChunk), kThreads, 0, st>>>(s, N, x, ord, b.lastv,
                                                                                      b.k_out, b.side, ra);
}

void sweep_side_cross_x_sell(const SellArgs &s, const double *x, const int32_t *ord, const int64_t *orig,
                             SweepBuffers &b, const RedArgs &ra, cudaStream_t st)
{
    if (s.n == 0) return;
    k_side_cross_x_sell<<<(unsigned)((s.n + kChunk - 1) / kChunk), kThreads, 0, st>>>(s, x, ord, b.lastv, b.k_out,
                                                                                     orig, b.side, ra);
}

void sweep_side_cross_stencil(const StencilArgs &s, int64_t N, SweepBuffers &b, const RedArgs &ra, cudaStream_t st)
{
    k_side_cross_stencil<<<(unsigned)((N + kChunk - 1) / kChunk), kThreads, 0, st>>>(s, N, b.rank, b.k_out, b.side,
                                                                                    ra);
}

void sweep_side_cross_sell(const SellArgs &s, const int64_t *orig, int64_t n_total, SweepBuffers &b,
                           const RedArgs &ra, cudaStream_t st)
{
    (void)n_total;
    if (s.n == 0) return;
    k_side_cross_sell<<<(unsigned)((s.n + kChunk - 1) / kChunk), kThreads, 0, st>>>(s, b.rank, b.k_out, orig,
                                                                                   b.side, ra);
}

__global__ void k_order_out(const int32_t *order, const int64_t *orig, int32_t *out, int64_t n)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = orig ? (int32_t)orig[order[i]] : order[i];
}

void sweep_order_out(const int32_t *order, const int64_t *orig, int32_t *out, int64_t n, cudaStream_t st)
{
    if (n == 0) return;
    k_order_out<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(order, orig, out, n);
}

}  // namespace irls
