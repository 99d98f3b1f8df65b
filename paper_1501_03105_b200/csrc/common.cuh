// common.cuh — device-side building blocks shared by the IRLS kernels.
//
// Arithmetic contract: C1 no FMA (the library is compiled with
// -fmad=false and uses plain IEEE '+', '*', '/', sqrt); C2 per-node sums in
// ascending neighbour id; C3 the fixed reduction tree implemented by
// c3_block_sum() + the group epilogue below.  Nothing here is shared with the
// CPU oracle: both implement the same written specification.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace irls {

constexpr int kChunk = 4096;    // C3 chunk: 256 threads x 8 rounds x double2
constexpr int kThreads = 256;
constexpr int kGroups = 8;
constexpr int kMaxQ = 5;
constexpr int kSell = 64;     // SELL slice height: thread t's rows 2t, 2t+1 hold adjacent slots

// ---------------------------------------------------------------------------
// Fast unsigned division for n < 2^31, d < 2^31: q = (n * m) >> sh with
// sh = 31 + ceil(log2 d), m = ceil(2^sh / d)  (exact; n*m < 2^64).
// ---------------------------------------------------------------------------
struct FastDiv {
    uint64_t m;
    uint32_t sh, d;
};

static inline FastDiv make_fastdiv(uint32_t d)
{
    FastDiv f;
    uint32_t l = 0;
    while ((1ull << l) < d) l++;
    f.sh = 31 + l;
    f.m = (uint64_t)(((__uint128_t)1 << f.sh) + d - 1) / d;
    f.d = d;
    return f;
}

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv &f)
{
    return (uint32_t)(((unsigned long long)n * f.m) >> f.sh);
}

// ---------------------------------------------------------------------------
// Control block of one CG solve (device memory).  Scalars follow O5.
// ---------------------------------------------------------------------------
struct DevCtrl {
    double rho, alpha, beta, ref, res, rtol;
    int32_t k, max_iter, norm, done;
    int32_t status, zero_x, step, frozen;  // frozen: fixed point reached (fixed_point_exit)
    unsigned grp_cnt[kGroups];
    unsigned fin_cnt;
    int32_t outer_left;  // IRLS steps left in a multi-step graph
    int32_t outer_end;   // report index one past its last step
    uint32_t red_seq;    // peer-memory collectives: reductions consumed so far (slot parity, arrival target)
    unsigned long long xmin_key, xmax_key;
    unsigned long long t_mark;  // %globaltimer (ns) at the start of a solve sequence
    unsigned long long t_asm;   // %globaltimer (ns) at the last START finalize (end of the assembly)
};

__device__ __forceinline__ unsigned long long global_ns()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

enum { ST_OK = 0, ST_BREAKDOWN = 6 };

// Reduction bookkeeping for one kernel family (one "phase").
struct RedArgs {
    double *part;        // [NQ][K] chunk partials, global chunk index
    double *slots;       // [NQ][8] group sums of the groups this rank owns (others stay 0)
    DevCtrl *ctrl;
    int32_t K;           // global chunk count
    int32_t g0, g1;      // owned groups [g0, g1)
    int32_t n_fin;       // non-empty owned groups
    // peer-memory slot collective (irls_options.p2p, world > 1; nullptr: local
    // slots + an allreduce afterwards): the owner block of a group stores its
    // sums straight into every rank's slot buffer (parity red_seq & 1) and
    // bumps every rank's arrival counter
    double *const *pslots = nullptr;            // [world] -> [2][kMaxQ][8]
    unsigned long long *const *pcnt = nullptr;  // [world] -> arrival counter
    int32_t world = 0;
};

// ---------------------------------------------------------------------------
// C3 steps 3-4: warp tree (offsets 16,8,4,2,1; lane i += lane i+off) and the
// 8-warp tree ((w0+w4)+(w2+w6))+((w1+w5)+(w3+w7)).  Result valid in thread 0.
// smem: >= NQ*8 doubles.
// ---------------------------------------------------------------------------
template <int NQ>
__device__ __forceinline__ void c3_block_sum(double (&v)[NQ], double *smem)
{
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < NQ; q++) {
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) v[q] = v[q] + __shfl_down_sync(0xffffffffu, v[q], off);
        if (lane == 0) smem[q * 8 + w] = v[q];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < NQ; q++) {
            const double *s = smem + q * 8;
            v[q] = ((s[0] + s[4]) + (s[2] + s[6])) + ((s[1] + s[5]) + (s[3] + s[7]));
        }
    }
    __syncthreads();
}

__device__ __forceinline__ double tree8(const double *s)
{
    return ((s[0] + s[4]) + (s[2] + s[6])) + ((s[1] + s[5]) + (s[3] + s[7]));
}

__host__ __device__ __forceinline__ int32_t group_lo(int g, int32_t K) { return (int32_t)(((int64_t)g * K) / kGroups); }

// C3 step 5: the list a[q*K + lo .. lo+m) of each quantity, reduced chunk by
// chunk (the chunk procedure of steps 2-4), repeated until one value remains.
// Called by a whole block; in-place on the partial buffer.  Result in thread 0.
template <int NQ>
__device__ void c3_list_sum(double *part, int32_t K, int32_t lo, int32_t m, double (&out)[NQ], double *smem)
{
    while (m > 1) {
        const int32_t nk = (m + kChunk - 1) / kChunk;
        for (int32_t kk = 0; kk < nk; kk++) {
            double acc[NQ];
#pragma unroll
            for (int q = 0; q < NQ; q++) acc[q] = 0.0;
            const int32_t base = kk * kChunk;
#pragma unroll
            for (int j = 0; j < 8; j++)
#pragma unroll
                for (int e = 0; e < 2; e++) {
                    const int32_t i = base + 2 * (int)threadIdx.x + 512 * j + e;
                    if (i < m) {
#pragma unroll
                        for (int q = 0; q < NQ; q++) acc[q] = acc[q] + __ldcg(part + (int64_t)q * K + lo + i);
                    }
                }
            c3_block_sum<NQ>(acc, smem);
            if (threadIdx.x == 0) {
#pragma unroll
                for (int q = 0; q < NQ; q++) part[(int64_t)q * K + lo + kk] = acc[q];
            }
            __threadfence_block();
            __syncthreads();
        }
        m = nk;
    }
    if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < NQ; q++) out[q] = m == 1 ? __ldcg(part + (int64_t)q * K + lo) : 0.0;
    }
}

// Chunk epilogue: v holds each thread's sequential sums (C3 step 2).  Writes
// the chunk partial; the last chunk of a group reduces the group into its
// slot; the last group of this rank returns true (all threads of that block),
// after which slots[] hold every owned group sum.
template <int NQ>
__device__ bool c3_chunk_epilogue(double (&v)[NQ], int32_t chunk, const RedArgs &ra)
{
    __shared__ double smem[kMaxQ * 8];
    __shared__ int s_flag;
    c3_block_sum<NQ>(v, smem);
    int g = 0;
#pragma unroll
    for (int gg = 1; gg < kGroups; gg++)
        if (chunk >= group_lo(gg, ra.K)) g = gg;
    const int32_t glo = group_lo(g, ra.K), ghi = group_lo(g + 1, ra.K);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < NQ; q++) ra.part[(int64_t)q * ra.K + chunk] = v[q];
        __threadfence();
        const unsigned prev = atomicAdd(&ra.ctrl->grp_cnt[g], 1u);
        s_flag = (prev == (unsigned)(ghi - glo - 1));
    }
    __syncthreads();
    if (!s_flag) return false;
    __threadfence();
    double gsum[NQ];
    c3_list_sum<NQ>(ra.part, ra.K, glo, ghi - glo, gsum, smem);
    if (threadIdx.x == 0) {
        if (ra.pslots) {  // fused collective: push the group sum to every rank over peer memory
            const int off = (int)(ra.ctrl->red_seq & 1u) * (kMaxQ * kGroups) + g;
            for (int w = 0; w < ra.world; w++)
#pragma unroll
                for (int q = 0; q < NQ; q++) ra.pslots[w][off + q * kGroups] = gsum[q];
            __threadfence_system();
            for (int w = 0; w < ra.world; w++) atomicAdd_system(ra.pcnt[w], 1ull);
        } else {
#pragma unroll
            for (int q = 0; q < NQ; q++) ra.slots[q * kGroups + g] = gsum[q];
        }
        ra.ctrl->grp_cnt[g] = 0u;
        __threadfence();
        const unsigned prev = atomicAdd(&ra.ctrl->fin_cnt, 1u);
        s_flag = (prev == (unsigned)(ra.n_fin - 1));
        if (s_flag) ra.ctrl->fin_cnt = 0u;
    }
    __syncthreads();
    if (s_flag) __threadfence();
    return s_flag;
}

// ---------------------------------------------------------------------------
// Scalar finalizers (one thread).  slots = [NQ][8] global group sums.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double ldslot(const double *s, int q, int g) { return __ldcg(s + q * kGroups + g); }

__device__ __forceinline__ double slot_total(const double *slots, int q)
{
    double s[kGroups];
#pragma unroll
    for (int g = 0; g < kGroups; g++) s[g] = ldslot(slots, q, g);
    return tree8(s);
}

// Peer-memory slot collective, consumer side (one thread): wait until every
// non-empty group of this reduction has arrived (counter >= (red_seq + 1) *
// n_groups), consume it (red_seq + 1) and return its parity buffer.  A wait
// longer than 120 s (a peer died or the ranks fell out of step; ranks may
// legitimately enter a solve seconds apart) sets status
// ST_P2P_TIMEOUT, ends the solve and returns nullptr.
enum { ST_P2P_TIMEOUT = 10 };  // = IRLS_ERR_NCCL (a collective failed)
struct P2PWait {
    const double *buf;               // this rank's [2][kMaxQ][8] slot buffer (nullptr: not in use)
    const unsigned long long *cnt;   // this rank's arrival counter
    int32_t n_groups;                // non-empty groups over all ranks
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ inline const double *p2p_wait(DevCtrl *c, const P2PWait &pw)
{
    const unsigned long long target = ((unsigned long long)c->red_seq + 1ull) * (unsigned long long)pw.n_groups;
    if (ld_acquire_sys(pw.cnt) < target) {
        const unsigned long long t0 = global_ns();
        while (ld_acquire_sys(pw.cnt) < target) {
            if (global_ns() - t0 > 120000000000ull) {
                c->status = ST_P2P_TIMEOUT;
                c->done = 1;
                return nullptr;
            }
            __nanosleep(64);
        }
    }
    const double *slots = pw.buf + (c->red_seq & 1u) * (kMaxQ * kGroups);
    c->red_seq = c->red_seq + 1u;
    return slots;
}

// After assembly (phase START): quantities [rz, zz, rr, mbmb, bb].
__device__ __forceinline__ void finalize_start(DevCtrl *c, const double *slots)
{
    c->t_asm = global_ns();
    const double rz = slot_total(slots, 0), zz = slot_total(slots, 1), rr = slot_total(slots, 2);
    const double mbmb = slot_total(slots, 3), bb = slot_total(slots, 4);
    const double ref = sqrt(c->norm == 0 ? mbmb : bb);
    c->ref = ref;
    c->rho = rz;
    c->k = 0;
    c->status = ST_OK;
    c->alpha = 0.0;
    c->beta = 0.0;
    if (ref == 0.0) {  // b = 0 => v = 0
        c->zero_x = 1;
        c->res = 0.0;
        c->done = 1;
        return;
    }
    c->zero_x = 0;
    c->res = sqrt(c->norm == 0 ? zz : rr);
    c->done = (c->res <= c->rtol * ref) || (c->max_iter == 0);
}

// After q = A p (phase PQ): quantity [pq].
// (the _t forms take the totals; C = DevCtrl or a register copy of it)
template <class C>
__device__ __forceinline__ void finalize_pq_t(C *c, double pi)
{
    if (!(pi > 0.0) || isinf(pi)) {
        c->status = ST_BREAKDOWN;
        c->done = 1;
        return;
    }
    c->alpha = c->rho / pi;
}

__device__ __forceinline__ void finalize_pq(DevCtrl *c, const double *slots) { finalize_pq_t(c, slot_total(slots, 0)); }

// After r -= alpha q, z = M^-1 r (phase RZ): quantities [rz, zz, rr].
template <class C>
__device__ __forceinline__ void finalize_rz_t(C *c, double rz, double zz, double rr)
{
    const double res = sqrt(c->norm == 0 ? zz : rr);
    const double beta = rz / c->rho;
    c->res = res;
    c->beta = beta;
    c->rho = rz;
    c->k = c->k + 1;
    if (!isfinite(c->alpha) || !isfinite(beta) || !isfinite(res)) {
        c->status = ST_BREAKDOWN;
        c->done = 1;
        return;
    }
    c->done = (res <= c->rtol * c->ref) || (c->k == c->max_iter);
}

__device__ __forceinline__ void finalize_rz(DevCtrl *c, const double *slots)
{
    finalize_rz_t(c, slot_total(slots, 0), slot_total(slots, 1), slot_total(slots, 2));
}

// Chronopoulos-Gear PCG (O5', A31): after iteration k, quantities
// [gamma = <r,z>, delta = <z,w>, <z,z>, <r,r>] of the new r, z, w.
template <class C>
__device__ __forceinline__ void finalize_cgcg_t(C *c, double gamma, double delta, double zz, double rr)
{
    const double res = sqrt(c->norm == 0 ? zz : rr);
    const double alpha = c->alpha;
    const double beta = gamma / c->rho;
    double t = beta * gamma;
    t = t / alpha;
    const double den = delta - t;
    c->res = res;
    c->beta = beta;
    c->rho = gamma;
    c->k = c->k + 1;
    if (!isfinite(alpha) || !isfinite(beta) || !isfinite(res)) {
        c->status = ST_BREAKDOWN;
        c->done = 1;
        return;
    }
    c->done = (res <= c->rtol * c->ref) || (c->k == c->max_iter);
    if (!c->done) {
        if (!(den > 0.0) || isinf(den)) {
            c->status = ST_BREAKDOWN;
            c->done = 1;
            return;
        }
        c->alpha = gamma / den;
    }
}

__device__ __forceinline__ void finalize_cgcg(DevCtrl *c, const double *slots)
{
    finalize_cgcg_t(c, slot_total(slots, 0), slot_total(slots, 1), slot_total(slots, 2), slot_total(slots, 3));
}

// Order-preserving 64-bit key of a double (ascending).
__device__ __forceinline__ unsigned long long dkey_asc(double x)
{
    unsigned long long b = (unsigned long long)__double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dkey_inv(unsigned long long k)
{
    unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double((long long)b);
}

// Eq. 4 + Eq. 8 (O3): conductance c^2 / sqrt((c d)^2 + eps^2); c = 0 is an
// absent edge with conductance 0 (A6; identical bits to 0/w).
__device__ __forceinline__ double rw_g(double c, double d, double eps2)
{
    if (c == 0.0) return 0.0;
    const double a = c * d;
    const double w = sqrt(a * a + eps2);
    return (c * c) / w;
}

// A15 fixed point: Q(c) = rint(c 2^F) as an exact 128-bit integer (c >= 0,
// finite).  Integer arithmetic on the bits of c: c = m 2^(e - 1075) (m with
// its implicit bit; subnormals e = 1, no implicit bit), so c 2^F = m 2^sh,
// sh = e - 1075 + F.  sh >= 0: the exact left shift (F is chosen so the
// result stays below 2^124).  sh < 0: m / 2^-sh rounded half to even — the
// value rint gives for the exact product c 2^F (a power-of-two scaling,
// exact in double unless it underflows, where both give 0).  c = 0 gives 0.
__device__ __forceinline__ __int128 qfix(double c, int32_t F)
{
    const unsigned long long bits = (unsigned long long)__double_as_longlong(c);
    const int e = (int)(bits >> 52) & 0x7ff;
    const unsigned long long m = (bits & 0xfffffffffffffull) | (e ? (1ull << 52) : 0ull);
    const int sh = (e ? e : 1) - 1075 + F;
    if (sh >= 0) return (__int128)m << sh;
    const int k = -sh;
    if (k >= 64) return 0;
    const unsigned long long q = m >> k, rem = m & ((1ull << k) - 1ull), half = 1ull << (k - 1);
    return (__int128)(q + ((rem > half || (rem == half && (q & 1ull))) ? 1ull : 0ull));
}

}  // namespace irls
