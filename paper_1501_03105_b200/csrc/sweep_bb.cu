// sweep_bb.cu — the sweep cut without sorting every node (O7, A14,
// A15): the same k, cut value and side[] as the full sort (sweep.cu), for
// callers that do not ask for the order itself.
//
// P_i = P_0 + delta_0 + ... + delta_{i-1} over the order (x desc, id asc) is
// an exact integer sequence (A15).  The nodes are cut into B = 4096 ordered
// buckets by splitters drawn from a sorted sample of (key, id) pairs (so the
// buckets are ranges of the total order).  One pass over the graph computes
// every delta_v in registers (sweep_delta.cuh) and accumulates per bucket, in
// shared memory, the count, the exact sum of the deltas and a lower bound of
// the sum of the negative deltas — nothing per node is written.  That gives P
// exactly at every bucket boundary and a lower bound P_start + sum(delta < 0)
// of P anywhere inside a bucket.  The first minimum of P can only lie in a
// bucket whose bound does not exceed the best boundary value, so only those
// candidate buckets are extracted (a second pass over x), sorted (the radix
// sort of sweep.cu) and scanned; every value compared is exact, so k is the
// one the full scan finds.  On config 4 a few dozen of 4096 buckets survive.
//
// Exact bucket sums with two 64-bit shared-memory atomics per node: delta =
// hi 2^64 + lo (hi = delta >> 64 signed, lo unsigned); lo is added to the
// bucket's low word, and hi plus the carry out of that addition (detected from
// the returned old value) to its high word, so (high, low) is the exact
// 128-bit sum (F is chosen so that sum |delta_v| < 2^125, A15: no overflow).
// The negative bound sums floor(delta / 2^63) over delta < 0 (each term <=
// delta / 2^63, so 2^63 times the sum is <= the true sum: conservative).
// The bucket of a node: a table over 8192 equal cells of the splitters' key
// range gives the few splitters that can share its cell; a binary search
// over those finishes it.
#include <algorithm>
#include "kernels.h"
#include "sweep_delta.cuh"

namespace irls {

typedef unsigned long long u64;
typedef __int128 i128;

constexpr int kBbThreads = 1024;

__device__ __forceinline__ bool kless(u64 ka, int32_t ia, u64 kb, int32_t ib)
{
    return ka < kb || (ka == kb && ia < ib);
}

constexpr int kCells = 8192;

struct BbMeta {
    u64 kmin;   // smallest splitter key
    u64 shift;  // cell of key k >= kmin: (k - kmin) >> shift
};

// bucket of (key, v): the number of splitters <= (key, v)
__device__ __forceinline__ int bucket_fast(u64 key, int32_t v, const u64 *sk, const int32_t *si, const uint32_t *tabp,
                                           u64 kmin, int sh, int nb)
{
    if (key < kmin) return 0;
    const u64 c = (key - kmin) >> sh;
    if (c >= (u64)kCells) return nb - 1;
    const uint32_t p = tabp[c];
    int lo = (int)(p & 0xffffu), hi = (int)(p >> 16);
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (kless(key, v, sk[mid], si[mid])) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

// the cell table: tabp[c] = lb(c) | lb(c + 1) << 16, lb(c) = the number of
// splitters whose key is below the start of cell c
__global__ void k_bb_table(const u64 *spk, int nb, uint32_t *tabp, BbMeta *meta)
{
    const u64 kmin = spk[0], kmax = spk[nb - 2];
    int sh = 0;
    while (((kmax - kmin) >> sh) >= (u64)kCells) sh++;
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c == 0) {
        meta->kmin = kmin;
        meta->shift = (u64)sh;
    }
    if (c >= kCells) return;
    uint32_t lb[2];
    for (int q = 0; q < 2; q++) {
        const unsigned __int128 st = (unsigned __int128)kmin + ((unsigned __int128)(c + q) << sh);
        int lo = 0, hi = nb - 1;  // first splitter with key >= st
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if ((unsigned __int128)spk[mid] < st) lo = mid + 1;
            else hi = mid;
        }
        lb[q] = (uint32_t)lo;
    }
    tabp[c] = lb[0] | (lb[1] << 16);
}

__global__ void k_bb_sample(const double *x, int64_t n, int32_t ns, u64 *skey, int32_t *sid)
{
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= ns) return;
    const int64_t v = (int64_t)j * n / ns;
    skey[j] = sweep_key(canon(x[v]));
    sid[j] = (int32_t)v;
}

// Sample sort by rank: sample i goes to position #{j : (key_j, id_j) <
// (key_i, id_i)} (the ids are distinct, so the ranks are a permutation).
// ns^2 comparisons: block (bx, by) counts, for its 256 samples, the samples
// of slice by (1024 of them, staged in shared memory) below each; the
// scatter adds the slices' counts.
constexpr int kRankSlice = 1024;

__global__ void __launch_bounds__(256) k_bb_rank_samples(const u64 *skey, const int32_t *sid, int32_t ns,
                                                         int32_t *prank)
{
    __shared__ u64 tk[kRankSlice];
    __shared__ int32_t ti[kRankSlice];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int t0 = blockIdx.y * kRankSlice;
    for (int j = threadIdx.x; j < kRankSlice; j += blockDim.x) {
        tk[j] = t0 + j < ns ? skey[t0 + j] : ~0ull;
        ti[j] = t0 + j < ns ? sid[t0 + j] : 0x7fffffff;
    }
    __syncthreads();
    if (i >= ns) return;
    const u64 ki = skey[i];
    const int32_t ii = sid[i];
    int r = 0;
#pragma unroll 16
    for (int j = 0; j < kRankSlice; j++) r += kless(tk[j], ti[j], ki, ii) ? 1 : 0;
    prank[(int64_t)blockIdx.y * ns + i] = r;
}

__global__ void k_bb_rank_scatter(const u64 *skey, const int32_t *sid, const int32_t *prank, int32_t ns,
                                  int32_t nslices, u64 *okey, int32_t *oid)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ns) return;
    int r = 0;
    for (int q = 0; q < nslices; q++) r += prank[(int64_t)q * ns + i];
    okey[r] = skey[i];
    oid[r] = sid[i];
}

// splitter j (j = 1 .. nb - 1) = sorted sample j * ns / nb
__global__ void k_bb_splitters(const u64 *okey, const int32_t *oid, int32_t ns, int32_t nb, u64 *spk, int32_t *spi)
{
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= nb - 1) return;
    const int s = (int)(((int64_t)(j + 1) * ns) / nb);
    spk[j] = okey[s];
    spi[j] = oid[s];
}

__device__ __forceinline__ void load_splitters(const u64 *spk, const int32_t *spi, int nb, u64 *sk, int32_t *si)
{
    for (int i = threadIdx.x; i < nb - 1; i += blockDim.x) {
        sk[i] = spk[i];
        si[i] = spi[i];
    }
}

// The bucket pass (persistent: one CTA of 1024 threads per SM).  Partials
// per CTA g: part[(f * G + g) * nb + b] for the fields f = count, low word,
// high word, negative bound; pqcs[g] = the CTA's sum of Q(cs_v); bkt[v] = the
// bucket of v (2 bytes per node, read back by the extraction).
template <class DL>
__device__ __forceinline__ void bb_pass(int64_t N, const double *x, const u64 *spk, const int32_t *spi,
                                        const uint32_t *tabp_g, const BbMeta *meta, int nb, u64 *part, i128 *pqcs,
                                        int32_t *flags, uint16_t *bkt, DL dl)
{
    extern __shared__ __align__(16) unsigned char bb_dyn[];
    u64 *alo = reinterpret_cast<u64 *>(bb_dyn);              // [nb]
    u64 *ahi = alo + nb;                                      // [nb]
    u64 *aneg = ahi + nb;                                     // [nb]
    u64 *sk = aneg + nb;                                      // [nb - 1]
    int32_t *si = reinterpret_cast<int32_t *>(sk + nb);       // [nb - 1]
    unsigned *acnt = reinterpret_cast<unsigned *>(si + nb);   // [nb]
    uint32_t *tabp = acnt + nb;                               // [kCells]
    __shared__ i128 wq[32];
    for (int i = threadIdx.x; i < nb; i += blockDim.x) {
        alo[i] = ahi[i] = aneg[i] = 0ull;
        acnt[i] = 0u;
    }
    for (int i = threadIdx.x; i < kCells; i += blockDim.x) tabp[i] = tabp_g[i];
    load_splitters(spk, spi, nb, sk, si);
    const u64 kmin = meta->kmin;
    const int sh = (int)meta->shift;
    __syncthreads();
    i128 qcs = 0;
    bool nan = false;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < N; v += stride) {
        const double xr = x[v];
        nan |= isnan(xr);
        const double xv = canon(xr);
        i128 d, qs;
        dl(v, xv, d, qs);
        qcs += qs;
        const int b = bucket_fast(sweep_key(xv), (int32_t)v, sk, si, tabp, kmin, sh, nb);
        bkt[v] = (uint16_t)b;
        const u64 lo = (u64)d;
        atomicAdd(&acnt[b], 1u);
        const u64 old = atomicAdd(&alo[b], lo);
        atomicAdd(&ahi[b], (u64)(long long)(d >> 64) + (old + lo < old ? 1ull : 0ull));
        if (d < 0) atomicAdd(&aneg[b], (u64)(long long)(d >> 63));
    }
    if (nan) flags[0] = 1;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        const u64 l = __shfl_down_sync(0xffffffffu, (u64)qcs, off);
        const u64 h = __shfl_down_sync(0xffffffffu, (u64)(qcs >> 64), off);
        qcs += ((i128)h << 64) | (i128)l;
    }
    if ((threadIdx.x & 31) == 0) wq[threadIdx.x >> 5] = qcs;
    __syncthreads();
    if (threadIdx.x == 0) {
        i128 t = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); i++) t += wq[i];
        pqcs[blockIdx.x] = t;
    }
    const int G = gridDim.x;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) {
        part[((int64_t)0 * G + blockIdx.x) * nb + b] = acnt[b];
        part[((int64_t)1 * G + blockIdx.x) * nb + b] = alo[b];
        part[((int64_t)2 * G + blockIdx.x) * nb + b] = ahi[b];
        part[((int64_t)3 * G + blockIdx.x) * nb + b] = aneg[b];
    }
}

__global__ void __launch_bounds__(kBbThreads, 1) k_bb_pass_stencil(StencilArgs s, int64_t N, int32_t F,
                                                                   const double *x, const u64 *spk,
                                                                   const int32_t *spi, const uint32_t *tabp,
                                                                   const BbMeta *meta, int nb, u64 *part, i128 *pqcs,
                                                                   int32_t *flags, uint16_t *bkt)
{
    bb_pass(N, x, spk, spi, tabp, meta, nb, part, pqcs, flags, bkt,
            [&](int64_t v, double xv, i128 &d, i128 &qs) { delta_stencil(s, F, x, v, xv, d, qs); });
}

__global__ void __launch_bounds__(kBbThreads, 1) k_bb_pass_sell(SellArgs s, int32_t F, const double *x,
                                                                const u64 *spk, const int32_t *spi,
                                                                const uint32_t *tabp, const BbMeta *meta, int nb,
                                                                u64 *part, i128 *pqcs, int32_t *flags, uint16_t *bkt)
{
    bb_pass(s.n, x, spk, spi, tabp, meta, nb, part, pqcs, flags, bkt,
            [&](int64_t v, double xv, i128 &d, i128 &qs) { delta_sell(s, F, x, v, xv, d, qs); });
}

// per bucket: count, exact sum, negative bound; P_0 = Q(c_st) + sum Q(cs).
// A block takes 32 buckets; its 8 warps split the G partials.
__global__ void __launch_bounds__(256) k_bb_reduce(const u64 *part, const i128 *pqcs, int G, int nb, i128 qcst,
                                                   unsigned *cnt, i128 *bsum, i128 *bneg, i128 *p0)
{
    __shared__ u64 sc[8][32], sn[8][32];
    __shared__ i128 ss[8][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int b = blockIdx.x * 32 + lane;
    u64 c = 0, ng = 0;
    i128 sum = 0;
    if (b < nb)
        for (int k = w; k < G; k += 8) {
            c += part[((int64_t)0 * G + k) * nb + b];
            sum += (i128)part[((int64_t)1 * G + k) * nb + b];
            sum += (i128)(long long)part[((int64_t)2 * G + k) * nb + b] << 64;
            ng += part[((int64_t)3 * G + k) * nb + b];
        }
    sc[w][lane] = c;
    sn[w][lane] = ng;
    ss[w][lane] = sum;
    __syncthreads();
    if (w == 0 && b < nb) {
        for (int q = 1; q < 8; q++) {
            c += sc[q][lane];
            ng += sn[q][lane];
            sum += ss[q][lane];
        }
        cnt[b] = (unsigned)c;
        bsum[b] = sum;
        bneg[b] = (i128)(long long)ng << 63;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        i128 t = qcst;
        for (int k = 0; k < G; k++) t += pqcs[k];
        *p0 = t;
    }
}

// Candidate extraction (second pass, over the bucket ids: 2 bytes per node,
// eight per thread and load): nodes whose bucket has a slot get (key, id) at
// their slot's cursor, plus stage A of the candidates' sort (by id: key = id,
// value = compact position) and its digit histograms.  Their deltas follow
// in k_bb_cdelta_* over the candidates in id order (after stage A).
__global__ void __launch_bounds__(kBbThreads, 1) k_bb_extract(int64_t N, const double *x, const uint16_t *bkt, int nb,
                                                              const int16_t *slot_of, u64 *cursor, u64 *ck,
                                                              int32_t *cid, u64 *ida, int32_t *posa, u64 *digit_hist)
{
    extern __shared__ __align__(16) unsigned char bb_dyn[];
    int16_t *sl = reinterpret_cast<int16_t *>(bb_dyn);  // [nb]
    __shared__ unsigned h[4 * 256];
    for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) h[i] = 0u;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) sl[i] = slot_of[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    unsigned nmine = 0;
    const int64_t ng = (N + 7) / 8;  // groups of 8 nodes
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t g0 = (int64_t)blockIdx.x * blockDim.x; g0 < ng; g0 += stride) {
        const int64_t g = g0 + threadIdx.x;
        uint16_t bb[8];
        if (g < ng && 8 * g + 8 <= N) {
            const uint4 w = __ldcs(reinterpret_cast<const uint4 *>(bkt) + g);
            const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int q = 0; q < 4; q++) {
                bb[2 * q] = (uint16_t)(ww[q] & 0xffffu);
                bb[2 * q + 1] = (uint16_t)(ww[q] >> 16);
            }
        } else {
#pragma unroll
            for (int q = 0; q < 8; q++) bb[q] = (g < ng && 8 * g + q < N) ? bkt[8 * g + q] : (uint16_t)0xffffu;
        }
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const int64_t v = 8 * g + q;
            const int slot = bb[q] != 0xffffu ? (int)sl[bb[q]] : -1;
            if (__any_sync(0xffffffffu, slot >= 0)) {
                const unsigned peers = __match_any_sync(0xffffffffu, slot);
                if (slot >= 0) {
                    const int leader = __ffs(peers) - 1;
                    u64 p0 = 0;
                    if (lane == leader) p0 = atomicAdd(&cursor[slot], (u64)__popc(peers));
                    p0 = __shfl_sync(peers, p0, leader);
                    const int64_t p = (int64_t)p0 + __popc(peers & ((1u << lane) - 1u));
                    ck[p] = sweep_key(canon(x[v]));
                    cid[p] = (int32_t)v;
                    ida[p] = (u64)(uint32_t)v;
                    posa[p] = (int32_t)p;
#pragma unroll
                    for (int b = 0; b < 4; b++) atomicAdd(&h[b * 256 + (((uint32_t)v >> (8 * b)) & 255u)], 1u);
                    nmine++;
                }
            }
        }
    }
    // the upper id digits are all zero
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) nmine += __shfl_down_sync(0xffffffffu, nmine, off);
    __syncthreads();
    if (lane == 0 && nmine)
        for (int q = 4; q < 8; q++) atomicAdd(&digit_hist[q * 256], (u64)nmine);
    for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x)
        if (h[i]) atomicAdd(&digit_hist[i], (u64)h[i]);
}

// delta of every candidate (packed: full warps), in ascending id order
// (perm = stage A's sorted compact positions: neighbouring threads read
// neighbouring graph data)
__global__ void __launch_bounds__(256) k_bb_cdelta_stencil(StencilArgs s, int32_t F, const double *x, const int32_t *cid,
                                                           const int32_t *perm, int64_t C, i128 *cdel)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= C) return;
    const int64_t p = perm[r];
    const int64_t v = cid[p];
    i128 d, qs;
    delta_stencil(s, F, x, v, canon(x[v]), d, qs);
    cdel[p] = d;
}

__global__ void __launch_bounds__(256) k_bb_cdelta_sell(SellArgs s, int32_t F, const double *x, const int32_t *cid,
                                                        const int32_t *perm, int64_t C, i128 *cdel)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= C) return;
    const int64_t p = perm[r];
    const int64_t v = cid[p];
    i128 d, qs;
    delta_sell(s, F, x, v, canon(x[v]), d, qs);
    cdel[p] = d;
}

// Stage B input: the candidates in ascending id order (perm = stage A's
// sorted positions), value = compact position; the keys' digit histograms.
__global__ void __launch_bounds__(256) k_bb_gather(const u64 *ck, const int32_t *perm, int64_t C, u64 *kb,
                                                   int32_t *jb, u64 *digit_hist)
{
    __shared__ unsigned sh[8 * 256];
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) sh[i] = 0u;
    __syncthreads();
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < C; r += (int64_t)gridDim.x * blockDim.x) {
        const int32_t j = perm[r];
        const u64 key = ck[j];
        kb[r] = key;
        jb[r] = j;
#pragma unroll
        for (int d = 0; d < 8; d++) atomicAdd(&sh[d * 256 + ((key >> (8 * d)) & 255u)], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x)
        if (sh[i]) atomicAdd(&digit_hist[i], (u64)sh[i]);
}

__device__ __forceinline__ i128 shfl_up_i128b(i128 v, int off)
{
    u64 lo = (u64)v, hi = (u64)(v >> 64);
    lo = __shfl_up_sync(0xffffffffu, lo, off);
    hi = __shfl_up_sync(0xffffffffu, hi, off);
    return ((i128)hi << 64) | (i128)lo;
}

__device__ __forceinline__ i128 shfl_down_i128b(i128 v, int off)
{
    u64 lo = (u64)v, hi = (u64)(v >> 64);
    lo = __shfl_down_sync(0xffffffffu, lo, off);
    hi = __shfl_down_sync(0xffffffffu, hi, off);
    return ((i128)hi << 64) | (i128)lo;
}

__device__ __forceinline__ bool lexl(i128 a, int64_t ia, i128 b, int64_t ib) { return a < b || (a == b && ia < ib); }

// One CTA per candidate bucket, its elements sorted (compact positions):
// P at every position inside (and at its end), exact; the first minimum.
__global__ void __launch_bounds__(1024) k_bb_cand_scan(const i128 *cdel, const int32_t *sorted, const int64_t *cdst,
                                                       const int64_t *cpos, const i128 *cP, i128 *cmin,
                                                       int64_t *carg)
{
    __shared__ i128 wsum[32], smin[32];
    __shared__ int64_t sarg[32];
    __shared__ i128 carry;
    const int c = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int64_t a = cdst[c], len = cdst[c + 1] - cdst[c], pos0 = cpos[c];
    if (threadIdx.x == 0) carry = cP[c];
    __syncthreads();
    i128 best = (i128)(((unsigned __int128)1 << 127) - 1);
    int64_t barg = INT64_MAX;
    for (int64_t t0 = 0; t0 < len; t0 += blockDim.x) {
        const int64_t t = t0 + threadIdx.x;
        const i128 d = t < len ? cdel[sorted[a + t]] : (i128)0;
        i128 inc = d;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const i128 o = shfl_up_i128b(inc, off);
            if (lane >= off) inc += o;
        }
        if (lane == 31) wsum[w] = inc;
        __syncthreads();
        i128 pre = carry;
        for (int k2 = 0; k2 < w; k2++) pre += wsum[k2];
        const i128 P = pre + inc;  // P at position pos0 + t + 1
        if (t < len && lexl(P, pos0 + t + 1, best, barg)) {
            best = P;
            barg = pos0 + t + 1;
        }
        __syncthreads();
        if (threadIdx.x == 0)
            for (int k2 = 0; k2 < nw; k2++) carry += wsum[k2];
        __syncthreads();
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        const i128 ob = shfl_down_i128b(best, off);
        const int64_t oa = __shfl_down_sync(0xffffffffu, barg, off);
        if (lexl(ob, oa, best, barg)) {
            best = ob;
            barg = oa;
        }
    }
    if (lane == 0) {
        smin[w] = best;
        sarg[w] = barg;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k2 = 1; k2 < nw; k2++)
            if (lexl(smin[k2], sarg[k2], best, barg)) {
                best = smin[k2];
                barg = sarg[k2];
            }
        cmin[c] = best;
        carg[c] = barg;
    }
}

// k = the first minimiser over the boundary minimum (bP, bpos) and the
// candidates' minima; the k-th node of the order (position k - 1) from the
// candidate that holds it (the host makes sure one does when k > 0;
// flags[2] = 1 if not).
__global__ void k_bb_finish(const i128 *cmin, const int64_t *carg, int32_t nc, i128 bP, int64_t bpos,
                            const int64_t *cdst, const int64_t *cpos, const int32_t *sorted, const int32_t *cid,
                            int64_t *k_out, int32_t *lastv, int32_t *flags)
{
    if (threadIdx.x != 0) return;
    i128 best = bP;
    int64_t barg = bpos;
    for (int j = 0; j < nc; j++)
        if (lexl(cmin[j], carg[j], best, barg)) {
            best = cmin[j];
            barg = carg[j];
        }
    *k_out = barg;
    int32_t lv = 0;
    bool found = barg == 0;
    if (barg > 0) {
        const int64_t pos = barg - 1;
        for (int j = 0; j < nc; j++) {
            const int64_t len = cdst[j + 1] - cdst[j];
            if (pos >= cpos[j] && pos < cpos[j] + len) {
                lv = cid[sorted[cdst[j] + (pos - cpos[j])]];
                found = true;
                break;
            }
        }
    }
    *lastv = lv;
    if (!found) flags[2] = 1;
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
int bb_num_ctas()
{
    static int g = 0;
    if (!g) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g, cudaDevAttrMultiProcessorCount, dev);
        if (g <= 0) g = 148;
    }
    return g;
}

// scratch of the bucket stage: splitters, cell table, meta
size_t bb_table_bytes() { return sizeof(uint32_t) * kCells + sizeof(BbMeta); }

void bb_sample_sort(const double *x, int64_t n, int32_t ns, int32_t nb, u64 *skey, int32_t *sid, u64 *spk,
                    int32_t *spi, void *table, cudaStream_t st)
{
    // skey / sid hold 2 ns entries (the samples, then the sorted samples);
    // sid also ns * (ns / kRankSlice) slice ranks after them
    const int nsl = (ns + kRankSlice - 1) / kRankSlice;
    int32_t *prank = sid + 2 * ns;
    k_bb_sample<<<(ns + 255) / 256, 256, 0, st>>>(x, n, ns, skey, sid);
    k_bb_rank_samples<<<dim3((ns + 255) / 256, nsl), 256, 0, st>>>(skey, sid, ns, prank);
    k_bb_rank_scatter<<<(ns + 255) / 256, 256, 0, st>>>(skey, sid, prank, ns, nsl, skey + ns, sid + ns);
    k_bb_splitters<<<(nb + 255) / 256, 256, 0, st>>>(skey + ns, sid + ns, ns, nb, spk, spi);
    uint32_t *tabp = reinterpret_cast<uint32_t *>(table);
    BbMeta *meta = reinterpret_cast<BbMeta *>(tabp + kCells);
    k_bb_table<<<kCells / 256, 256, 0, st>>>(spk, nb, tabp, meta);
}

static size_t pass_smem(int nb) { return (size_t)nb * (3 * 8 + 8 + 4 + 4) + sizeof(uint32_t) * kCells; }

template <class K>
static void set_smem(K kern, size_t bytes)
{
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

static inline const uint32_t *tab_of(const void *t) { return reinterpret_cast<const uint32_t *>(t); }
static inline const BbMeta *meta_of(const void *t)
{
    return reinterpret_cast<const BbMeta *>(reinterpret_cast<const uint32_t *>(t) + kCells);
}

void bb_pass_stencil(const StencilArgs &s, int64_t N, int32_t F, const double *x, const u64 *spk, const int32_t *spi,
                     const void *table, int32_t nb, u64 *part, i128 *pqcs, int32_t *flags, uint16_t *bkt,
                     cudaStream_t st)
{
    set_smem(k_bb_pass_stencil, pass_smem(nb));
    k_bb_pass_stencil<<<bb_num_ctas(), kBbThreads, pass_smem(nb), st>>>(s, N, F, x, spk, spi, tab_of(table),
                                                                        meta_of(table), nb, part, pqcs, flags, bkt);
}

void bb_pass_sell(const SellArgs &s, int32_t F, const double *x, const u64 *spk, const int32_t *spi,
                  const void *table, int32_t nb, u64 *part, i128 *pqcs, int32_t *flags, uint16_t *bkt,
                  cudaStream_t st)
{
    set_smem(k_bb_pass_sell, pass_smem(nb));
    k_bb_pass_sell<<<bb_num_ctas(), kBbThreads, pass_smem(nb), st>>>(s, F, x, spk, spi, tab_of(table),
                                                                     meta_of(table), nb, part, pqcs, flags, bkt);
}

void bb_reduce(const u64 *part, const i128 *pqcs, int32_t nb, i128 qcst, unsigned *cnt, i128 *bsum, i128 *bneg,
               i128 *p0, cudaStream_t st)
{
    k_bb_reduce<<<(nb + 31) / 32, 256, 0, st>>>(part, pqcs, bb_num_ctas(), nb, qcst, cnt, bsum, bneg, p0);
}

void bb_extract(int64_t N, const double *x, const uint16_t *bkt, int32_t nb, const int16_t *slot_of, u64 *cursor,
                u64 *ck, int32_t *cid, u64 *ida, int32_t *posa, u64 *digit_hist, cudaStream_t st)
{
    k_bb_extract<<<bb_num_ctas(), kBbThreads, sizeof(int16_t) * nb, st>>>(N, x, bkt, nb, slot_of, cursor, ck, cid, ida,
                                                                         posa, digit_hist);
}

void bb_cdelta_stencil(const StencilArgs &s, int32_t F, const double *x, const int32_t *cid, const int32_t *perm,
                       int64_t C, i128 *cdel, cudaStream_t st)
{
    if (C > 0) k_bb_cdelta_stencil<<<(unsigned)((C + 255) / 256), 256, 0, st>>>(s, F, x, cid, perm, C, cdel);
}

void bb_cdelta_sell(const SellArgs &s, int32_t F, const double *x, const int32_t *cid, const int32_t *perm, int64_t C,
                    i128 *cdel, cudaStream_t st)
{
    if (C > 0) k_bb_cdelta_sell<<<(unsigned)((C + 255) / 256), 256, 0, st>>>(s, F, x, cid, perm, C, cdel);
}

void bb_gather(const u64 *ck, const int32_t *perm, int64_t C, u64 *kb, int32_t *jb, u64 *digit_hist, cudaStream_t st)
{
    if (C == 0) return;
    k_bb_gather<<<(unsigned)std::min<int64_t>((C + 1023) / 1024, 296), 256, 0, st>>>(ck, perm, C, kb, jb,
                                                                                     digit_hist);
}

void bb_cand_scan(const i128 *cdel, const int32_t *sorted, const int64_t *cdst, const int64_t *cpos, const i128 *cP,
                  int32_t ncand, i128 *cmin, int64_t *carg, cudaStream_t st)
{
    if (ncand == 0) return;
    k_bb_cand_scan<<<ncand, 1024, 0, st>>>(cdel, sorted, cdst, cpos, cP, cmin, carg);
}

void bb_finish(const i128 *cmin, const int64_t *carg, int32_t nc, i128 bP, int64_t bpos, const int64_t *cdst,
               const int64_t *cpos, const int32_t *sorted, const int32_t *cid, int64_t *k_out, int32_t *lastv,
               int32_t *flags, cudaStream_t st)
{
    k_bb_finish<<<1, 32, 0, st>>>(cmin, carg, nc, bP, bpos, cdst, cpos, sorted, cid, k_out, lastv, flags);
}

}  // namespace irls
