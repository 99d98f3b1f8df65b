// api_block.cu — host setup of the block-Jacobi preconditioner (reading A32;
// SURVEY §8(f) NEXT #2): the partition of this rank's
// C3 groups into BFS blocks, each block row's envelope and in-block edge
// list, uploaded once at create.  The kernels are in block_jacobi.cu.
//
// A32 partition: for each owned C3 group in order and each of its ids
// ascending, an unassigned id opens a block; the earliest node of the block
// not yet expanded is expanded — its neighbours (ascending id, c > 0) inside
// the group and unassigned are appended in that order — until the block
// holds B nodes or every node of it is expanded.  The groups are independent
// (blocks never leave a group), so each is built on its own host thread.
#include "api_internal.h"

using namespace irls;

namespace {

struct GroupOut {
    std::vector<int32_t> nodes;   // local ids in block order
    std::vector<int32_t> starts;  // block starts (index into nodes)
};

// nbr(u, f): calls f(v, gptr) for every neighbour v of local node u (ascending
// id, c > 0) with gptr the device address of the edge's conductance; v may be
// outside [0, n_own) (then it is outside every group of this rank).
template <class NB>
irls_status build_blocks(irls_ctx *c, NB nbr)
{
    const int32_t B = c->opt.block_size;
    const int64_t n = c->n_own;
    std::vector<std::pair<int64_t, int64_t>> gr;
    for (int g = c->g0; g < c->g1; g++) {
        const int64_t lo = std::min<int64_t>((int64_t)group_lo(g, c->K) * kChunk, c->n_glob) - c->lo;
        const int64_t hi = std::min<int64_t>((int64_t)group_lo(g + 1, c->K) * kChunk, c->n_glob) - c->lo;
        gr.push_back({std::max<int64_t>(lo, 0), std::min<int64_t>(hi, n)});
    }
    std::vector<uint8_t> used((size_t)std::max<int64_t>(n, 1), 0);
    std::vector<GroupOut> out(gr.size());
    {
        std::vector<std::thread> th;
        for (size_t gi = 0; gi < gr.size(); gi++)
            th.emplace_back([&, gi]() {
                const int64_t lo = gr[gi].first, hi = gr[gi].second;
                GroupOut &o = out[gi];
                o.nodes.reserve((size_t)std::max<int64_t>(hi - lo, 0));
                for (int64_t u = lo; u < hi; u++) {
                    if (used[u]) continue;
                    const size_t start = o.nodes.size();
                    size_t head = start;
                    o.starts.push_back((int32_t)start);
                    o.nodes.push_back((int32_t)u);
                    used[u] = 1;
                    while (head < o.nodes.size() && (int64_t)(o.nodes.size() - start) < B) {
                        const int64_t v = o.nodes[head++];
                        nbr(v, [&](int64_t w, const double *) {
                            if ((int64_t)(o.nodes.size() - start) >= B || w < lo || w >= hi || used[w]) return;
                            used[w] = 1;
                            o.nodes.push_back((int32_t)w);
                        });
                    }
                }
            });
        for (auto &t : th) t.join();
    }
    // concatenate in group order
    std::vector<int32_t> bptr, bnode;
    bnode.reserve((size_t)n);
    for (auto &o : out) {
        const int32_t base = (int32_t)bnode.size();
        for (int32_t s : o.starts) bptr.push_back(base + s);
        bnode.insert(bnode.end(), o.nodes.begin(), o.nodes.end());
    }
    if ((int64_t)bnode.size() != n) return fail(c, IRLS_ERR_CUDA, "block partition does not cover the rank");
    const int64_t nblk = (int64_t)bptr.size();
    bptr.push_back((int32_t)n);
    {   // storage order: decreasing block size (the blocks are independent, so
        // their order changes no bit); a warp's blocks are then alike
        std::vector<int32_t> order((size_t)nblk);
        for (int64_t b = 0; b < nblk; b++) order[b] = (int32_t)b;
        std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b2) {
            return bptr[a + 1] - bptr[a] > bptr[b2 + 1] - bptr[b2];
        });
        std::vector<int32_t> sp((size_t)nblk + 1, 0), sn;
        sn.reserve((size_t)n);
        for (int64_t b = 0; b < nblk; b++) {
            sn.insert(sn.end(), bnode.begin() + bptr[order[b]], bnode.begin() + bptr[order[b] + 1]);
            sp[b + 1] = (int32_t)sn.size();
        }
        bptr.swap(sp);
        bnode.swap(sn);
    }
    std::vector<int32_t> pos((size_t)std::max<int64_t>(n, 1)), blk((size_t)std::max<int64_t>(n, 1));
    for (int64_t b = 0; b < nblk; b++)
        for (int32_t i = bptr[b]; i < bptr[b + 1]; i++) {
            pos[bnode[i]] = i;
            blk[bnode[i]] = (int32_t)b;
        }
    // envelopes and in-block lower-neighbour entries, per position
    std::vector<int32_t> bfirst((size_t)std::max<int64_t>(n, 1)), ecount((size_t)n + 1, 0);
    parallel_for(nblk, [&](int, int64_t a, int64_t bb) {
        for (int64_t b = a; b < bb; b++)
            for (int32_t i = bptr[b]; i < bptr[b + 1]; i++) {
                int32_t f = i, cnt = 0;
                nbr(bnode[i], [&](int64_t w, const double *) {
                    if (w < 0 || w >= n || blk[w] != b) return;
                    if (pos[w] < i) cnt++;
                    f = std::min(f, pos[w]);
                });
                bfirst[i] = f - bptr[b];
                ecount[i + 1] = cnt;
            }
    });
    int32_t m_max = 0;
    for (int64_t b = 0; b < nblk; b++) {
        for (int32_t i = bptr[b] + 1; i < bptr[b + 1]; i++)
            if (bfirst[i] < bfirst[i - 1])
                return fail(c, IRLS_ERR_CUDA, "block envelope not monotone (A32 partition broken)");
        m_max = std::max(m_max, bptr[b + 1] - bptr[b]);
    }
    // lane groups of 32 consecutive blocks: row i of group G spans the union
    // [min over the lanes of f_i, i) of their envelopes
    const int64_t nG = (nblk + 31) / 32;
    std::vector<int64_t> gL((size_t)nG + 1, 0), gR((size_t)nG + 1, 0);
    std::vector<int32_t> rowF, rowOff;
    for (int64_t G = 0; G < nG; G++) {
        const int64_t bl0 = 32 * G, bl1 = std::min<int64_t>(nblk, 32 * G + 32);
        int32_t M = 0;
        for (int64_t b = bl0; b < bl1; b++) M = std::max(M, bptr[b + 1] - bptr[b]);
        int64_t off = 0;
        for (int32_t i = 0; i < M; i++) {
            int32_t F = i;
            for (int64_t b = bl0; b < bl1; b++)
                if (i < bptr[b + 1] - bptr[b]) F = std::min(F, bfirst[bptr[b] + i]);
            rowF.push_back(F);
            rowOff.push_back((int32_t)off);
            off += i - F;
        }
        gR[G + 1] = gR[G] + M;
        gL[G + 1] = gL[G] + off;
    }
    std::vector<int32_t> eptr((size_t)n + 1, 0);
    for (int64_t i = 0; i < n; i++) eptr[i + 1] = eptr[i] + ecount[i + 1];
    std::vector<int32_t> ecol((size_t)std::max<int32_t>(eptr[n], 1));
    std::vector<const double *> eg((size_t)std::max<int32_t>(eptr[n], 1));
    parallel_for(nblk, [&](int, int64_t a, int64_t bb) {
        for (int64_t b = a; b < bb; b++)
            for (int32_t i = bptr[b]; i < bptr[b + 1]; i++) {
                int32_t e = eptr[i];
                nbr(bnode[i], [&](int64_t w, const double *gp) {
                    if (w < 0 || w >= n || blk[w] != b || pos[w] >= i) return;
                    ecol[e] = pos[w] - bptr[b];
                    eg[e] = gp;
                    e++;
                });
            }
    });
    BlockArgs &A = c->blk;
    A.nblk = nblk;
    A.m_max = m_max;
    if (m_max > 256) return fail(c, IRLS_ERR_INVALID_ARGUMENT, "block larger than 256 nodes");
    const int32_t ne = std::max<int32_t>(eptr[n], 1);
    int32_t *d_bptr = dalloc<int32_t>(c, nblk + 1), *d_bnode = dalloc<int32_t>(c, n);
    int32_t *d_eptr = dalloc<int32_t>(c, n + 1), *d_ecol = dalloc<int32_t>(c, ne);
    const double **d_eg = dalloc<const double *>(c, ne);
    int64_t *d_gL = dalloc<int64_t>(c, nG + 1), *d_gR = dalloc<int64_t>(c, nG + 1);
    int32_t *d_rowF = dalloc<int32_t>(c, std::max<int64_t>((int64_t)rowF.size(), 1));
    int32_t *d_rowOff = dalloc<int32_t>(c, std::max<int64_t>((int64_t)rowOff.size(), 1));
    A.L = dalloc<double>(c, 32 * std::max<int64_t>(gL[nG], 1));
    A.Dd = dalloc<double>(c, 32 * std::max<int64_t>(gR[nG], 1));
    A.mb = dalloc<double>(c, n);
    if (!c->gs_diag) c->gs_diag = dalloc<double>(c, (int64_t)c->nchunks * kChunk);
    if (!c->gt_diag) c->gt_diag = dalloc<double>(c, (int64_t)c->nchunks * kChunk);
    if (!d_bptr || !d_bnode || !d_eptr || !d_ecol || !d_eg || !d_gL || !d_gR || !d_rowF || !d_rowOff || !A.L ||
        !A.Dd || !A.mb || !c->gs_diag || !c->gt_diag)
        return fail(c, IRLS_ERR_OOM, "block preconditioner arrays");
    cudaError_t e = cudaSuccess;
    auto up = [&](void *dst, const void *src, size_t bytes) {
        if (e == cudaSuccess && bytes > 0) e = memcpy_sync(c, dst, src, bytes, cudaMemcpyHostToDevice);
    };
    up(d_bptr, bptr.data(), sizeof(int32_t) * (nblk + 1));
    up(d_bnode, bnode.data(), sizeof(int32_t) * n);
    up(d_eptr, eptr.data(), sizeof(int32_t) * (n + 1));
    up(d_ecol, ecol.data(), sizeof(int32_t) * eptr[n]);
    up(d_eg, eg.data(), sizeof(const double *) * eptr[n]);
    up(d_gL, gL.data(), sizeof(int64_t) * (nG + 1));
    up(d_gR, gR.data(), sizeof(int64_t) * (nG + 1));
    up(d_rowF, rowF.data(), sizeof(int32_t) * rowF.size());
    up(d_rowOff, rowOff.data(), sizeof(int32_t) * rowOff.size());
    if (e != cudaSuccess) return fail(c, IRLS_ERR_CUDA, std::string("block upload: ") + cudaGetErrorString(e));
    A.bptr = d_bptr;
    A.bnode = d_bnode;
    A.eptr = d_eptr;
    A.ecol = d_ecol;
    A.eg = d_eg;
    A.gL = d_gL;
    A.gR = d_gR;
    A.rowF = d_rowF;
    A.rowOff = d_rowOff;
    return IRLS_OK;
}

}  // namespace

// Grids: neighbours in ascending id (-z, -y, -x, +x, +y, +z) with c > 0 on
// the host copies of the capacities; conductances in gx / gy / gz (the +axis
// edge is owned by the lower node; gz has a ghost plane below).
irls_status block_setup_stencil(irls_ctx *c, const double *cx, const double *cy, const double *cz)
{
    if (c->opt.block_size <= 0) return IRLS_OK;
    const int64_t nx = c->nx, ny = c->ny, nz = c->nz, P = c->P, lo = c->lo;
    double *gx = c->gx, *gy = c->gy, *gz = c->gz;
    auto nbr = [&](int64_t u, auto &&f) {
        const int64_t gu = u + lo;
        const int64_t x = gu % nx, y = (gu / nx) % ny, z = gu / P;
        if (z > 0 && cz[gu - P] > 0.0) f(u - P, gz + (u - P));
        if (y > 0 && cy[gu - nx] > 0.0) f(u - nx, gy + (u - nx));
        if (x > 0 && cx[gu - 1] > 0.0) f(u - 1, gx + (u - 1));
        if (x < nx - 1 && cx[gu] > 0.0) f(u + 1, gx + u);
        if (y < ny - 1 && cy[gu] > 0.0) f(u + nx, gy + u);
        if (z < nz - 1 && cz[gu] > 0.0) f(u + P, gz + u);
    };
    return build_blocks(c, nbr);
}

// CSR: the reduced adjacency (ascending, c > 0) of the host preparation; the
// conductance of row r's k-th neighbour is slot sptr[r/64] + 64k + r%64 of
// the (local) SELL's g array.
irls_status block_setup_csr(irls_ctx *c, const int64_t *aptr, const int32_t *aidx, const int64_t *lsptr)
{
    if (c->opt.block_size <= 0) return IRLS_OK;
    const int64_t lo = c->lo;
    double *g = c->lg;
    auto nbr = [&](int64_t r, auto &&f) {
        const int64_t gr = r + lo, sl = r / kSell, ln = r % kSell;
        for (int64_t k = 0; k < aptr[gr + 1] - aptr[gr]; k++)
            f((int64_t)aidx[aptr[gr] + k] - lo, g + lsptr[sl] + kSell * k + ln);
    };
    return build_blocks(c, nbr);
}
