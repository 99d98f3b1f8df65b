// maxflow.cu — exact max-flow / min-cut on the coarse graph G_c of the
// two-level rounding (host code; "solve the undirected s-t min-cut
// problem on the coarsened graph G_c using a combinatorial max-flow/min-cut
// solver, e.g. [Boykov-Kolmogorov]"; the paper runs it sequentially on the
// root, and the north_star keeps it off the GPU hot path).
//
// Algorithm: Boykov-Kolmogorov augmenting paths with two search trees (grown
// from s_c and t_c; orphans re-adopted after each augmentation; the
// timestamp/distance heuristic for choosing parents).  Capacities are the
// exact 128-bit fixed-point integers of A15/A27, so the flow is exact.
// After termination the source side is recomputed as the set reachable from
// s_c in the residual graph (the minimal minimum cut, unique, A28) and the
// cut value of that set is compared with the flow value (strong duality is
// the certificate of optimality).
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <climits>
#include <thread>
#include <vector>

#include "kernels.h"

namespace irls {

typedef __int128 i128;

namespace {

constexpr int32_t kNone = -1, kTerm = -2, kOrphan = -3;

// FIFO of node ids with capacity n (a node is in each queue at most once)
struct Fifo {
    std::vector<int32_t> buf;
    size_t head = 0, tail = 0, cnt = 0;
    void init(int32_t n) { buf.assign((size_t)std::max(n, 1), 0); }
    bool empty() const { return cnt == 0; }
    int32_t front() const { return buf[head]; }
    void push(int32_t v)
    {
        buf[tail] = v;
        tail = tail + 1 == buf.size() ? 0 : tail + 1;
        cnt++;
    }
    void pop()
    {
        head = head + 1 == buf.size() ? 0 : head + 1;
        cnt--;
    }
};

// per-node search state, packed (one cache line touch per node visit)
struct NodeSt {
    int32_t parent, ts, dist;
    uint8_t tree, in_active, pad0, pad1;
};

struct BK {
    int32_t n;
    const int32_t *first, *head;
    std::vector<int32_t> sister;
    std::vector<i128> rc, tr;
    std::vector<NodeSt> nd;
    Fifo active, orphans;
    int32_t time = 0;
    i128 flow = 0;
    int64_t n_aug = 0, n_orphan = 0;

    void activate(int32_t i)
    {
        if (!nd[i].in_active) {
            nd[i].in_active = 1;
            active.push(i);
        }
    }
    void make_orphan(int32_t k)
    {
        nd[k].parent = kOrphan;
        orphans.push(k);
        n_orphan++;
    }

    // Growth stage: returns an arc from an S node to a T node with residual
    // capacity, or -1 when no active node can grow (maximum flow reached).
    int32_t grow()
    {
        while (!active.empty()) {
            const int32_t i = active.front();
            NodeSt &ni = nd[i];
            if (ni.tree == 0) {
                active.pop();
                ni.in_active = 0;
                continue;
            }
            for (int32_t a = first[i]; a < first[i + 1]; a++) {
                const int32_t j = head[a];
                NodeSt &nj = nd[j];
                if (ni.tree == 1) {
                    if (rc[a] == 0) continue;
                    if (nj.tree == 0) {
                        nj.tree = 1;
                        nj.parent = sister[a];
                        nj.ts = ni.ts;
                        nj.dist = ni.dist + 1;
                        activate(j);
                    } else if (nj.tree == 2) {
                        return a;
                    } else if (nj.ts <= ni.ts && nj.dist > ni.dist) {
                        nj.parent = sister[a];
                        nj.ts = ni.ts;
                        nj.dist = ni.dist + 1;
                    }
                } else {
                    const int32_t sa = sister[a];
                    if (rc[sa] == 0) continue;
                    if (nj.tree == 0) {
                        nj.tree = 2;
                        nj.parent = sa;
                        nj.ts = ni.ts;
                        nj.dist = ni.dist + 1;
                        activate(j);
                    } else if (nj.tree == 1) {
                        return sa;
                    } else if (nj.ts <= ni.ts && nj.dist > ni.dist) {
                        nj.parent = sa;
                        nj.ts = ni.ts;
                        nj.dist = ni.dist + 1;
                    }
                }
            }
            active.pop();
            ni.in_active = 0;
        }
        return -1;
    }

    // Augmentation along s_c -> ... -> i -a-> j -> ... -> t_c.
    void augment(int32_t a)
    {
        const int32_t i = head[sister[a]], j = head[a];
        i128 b = rc[a];
        for (int32_t k = i;;) {
            const int32_t p = nd[k].parent;
            if (p == kTerm) {
                if (tr[k] < b) b = tr[k];
                break;
            }
            if (rc[sister[p]] < b) b = rc[sister[p]];
            k = head[p];
        }
        for (int32_t k = j;;) {
            const int32_t p = nd[k].parent;
            if (p == kTerm) {
                if (-tr[k] < b) b = -tr[k];
                break;
            }
            if (rc[p] < b) b = rc[p];
            k = head[p];
        }
        rc[a] -= b;
        rc[sister[a]] += b;
        for (int32_t k = i;;) {
            const int32_t p = nd[k].parent;
            if (p == kTerm) {
                tr[k] -= b;
                if (tr[k] == 0) make_orphan(k);
                break;
            }
            const int32_t arc = sister[p], nxt = head[p];
            rc[arc] -= b;
            rc[p] += b;
            if (rc[arc] == 0) make_orphan(k);
            k = nxt;
        }
        for (int32_t k = j;;) {
            const int32_t p = nd[k].parent;
            if (p == kTerm) {
                tr[k] += b;
                if (tr[k] == 0) make_orphan(k);
                break;
            }
            const int32_t nxt = head[p];
            rc[p] -= b;
            rc[sister[p]] += b;
            if (rc[p] == 0) make_orphan(k);
            k = nxt;
        }
        flow += b;
        n_aug++;
    }

    // Adoption stage: every orphan finds a parent in its own tree whose
    // path reaches the terminal, or becomes free.
    void adopt()
    {
        while (!orphans.empty()) {
            const int32_t i = orphans.front();
            orphans.pop();
            const int t = nd[i].tree;
            int32_t best = kNone, dmin = INT_MAX;
            for (int32_t a0 = first[i]; a0 < first[i + 1]; a0++) {
                const int32_t j = head[a0];
                if (nd[j].tree != t) continue;
                if (!(t == 1 ? rc[sister[a0]] > 0 : rc[a0] > 0)) continue;
                int32_t d = 0, k = j;
                bool valid;
                for (;;) {
                    if (nd[k].ts == time) {
                        d += nd[k].dist;
                        valid = true;
                        break;
                    }
                    const int32_t p = nd[k].parent;
                    d++;
                    if (p == kTerm) {
                        nd[k].ts = time;
                        nd[k].dist = 1;
                        valid = true;
                        break;
                    }
                    if (p < 0) {  // orphan
                        valid = false;
                        break;
                    }
                    k = head[p];
                }
                if (!valid) continue;
                if (d < dmin) {
                    best = a0;
                    dmin = d;
                }
                for (k = j; nd[k].ts != time; k = head[nd[k].parent]) {
                    nd[k].ts = time;
                    nd[k].dist = d--;
                }
            }
            if (best != kNone) {
                nd[i].parent = best;
                nd[i].ts = time;
                nd[i].dist = dmin + 1;
                continue;
            }
            for (int32_t a0 = first[i]; a0 < first[i + 1]; a0++) {
                const int32_t j = head[a0];
                if (nd[j].tree != t) continue;
                if (t == 1 ? rc[sister[a0]] > 0 : rc[a0] > 0) activate(j);
                const int32_t p = nd[j].parent;
                if (p >= 0 && head[p] == i) make_orphan(j);
            }
            nd[i].tree = 0;
            nd[i].parent = kNone;
        }
    }
};

}  // namespace

static i128 maxflow_bk_one(int32_t nc, const int32_t *ptr, const int32_t *col, const i128 *cap, const i128 *qs,
                           const i128 *qt, uint8_t *src, int64_t *stats)
{
    BK g;
    g.n = nc;
    g.first = ptr;
    g.head = col;
    const int32_t m = ptr[nc];
    g.sister.assign(m, -1);
    g.rc.assign(cap, cap + m);
    g.tr.resize(nc);
    g.nd.assign(nc, NodeSt{kNone, 0, 0, 0, 0, 0, 0});
    g.active.init(nc);
    g.orphans.init(nc);
    // sister arcs: rows are sorted, so the entries (v, u) with u < v are the
    // leading entries of row v in ascending u
    {
        std::vector<int32_t> fill(ptr, ptr + nc);
        for (int32_t u = 0; u < nc; u++)
            for (int32_t a = ptr[u]; a < ptr[u + 1]; a++) {
                const int32_t v = col[a];
                if (v <= u) continue;
                const int32_t s = fill[v]++;
                if (s >= ptr[v + 1] || col[s] != u) {  // not symmetric
                    if (stats) stats[0] = -1;
                    return -1;
                }
                g.sister[a] = s;
                g.sister[s] = a;
            }
    }
    for (int32_t u = 0; u < nc; u++) {
        const i128 a = qs[u], b = qt[u];
        g.flow += a < b ? a : b;
        g.tr[u] = a - b;
    }
    // greedy length-3 paths s_c -> u -> v -> t_c over every arc (each push
    // keeps conservation) before the search trees start: 1.5x fewer
    // augmentations' worth of time on the config-2 coarse graph
    for (int32_t u = 0; u < nc; u++) {
        if (g.tr[u] <= 0) continue;
        for (int32_t a = ptr[u]; a < ptr[u + 1] && g.tr[u] > 0; a++) {
            const int32_t v = col[a];
            if (g.tr[v] >= 0 || g.rc[a] == 0) continue;
            i128 b = g.tr[u];
            if (g.rc[a] < b) b = g.rc[a];
            if (-g.tr[v] < b) b = -g.tr[v];
            g.tr[u] -= b;
            g.tr[v] += b;
            g.rc[a] -= b;
            g.rc[g.sister[a]] += b;
            g.flow += b;
        }
    }
    for (int32_t u = 0; u < nc; u++) {
        if (g.tr[u] != 0) {
            g.nd[u].tree = g.tr[u] > 0 ? 1 : 2;
            g.nd[u].parent = kTerm;
            g.nd[u].dist = 1;
            g.activate(u);
        }
    }
    for (;;) {
        const int32_t a = g.grow();
        if (a < 0) break;
        g.time++;
        g.augment(a);
        g.adopt();
    }
    // minimal source side: residual reachability from s_c
    std::vector<int32_t> q;
    q.reserve(nc);
    for (int32_t u = 0; u < nc; u++) {
        src[u] = g.tr[u] > 0;
        if (src[u]) q.push_back(u);
    }
    for (size_t h = 0; h < q.size(); h++) {
        const int32_t u = q[h];
        for (int32_t a = ptr[u]; a < ptr[u + 1]; a++)
            if (g.rc[a] > 0 && !src[col[a]]) {
                src[col[a]] = 1;
                q.push_back(col[a]);
            }
    }
    // certificate: cut(src) on the original capacities == flow value
    i128 cut = 0;
    for (int32_t u = 0; u < nc; u++) {
        cut += src[u] ? qt[u] : qs[u];
        if (src[u])
            for (int32_t a = ptr[u]; a < ptr[u + 1]; a++)
                if (!src[col[a]]) cut += cap[a];
    }
    if (stats) {
        stats[0] = cut == g.flow ? 1 : 0;
        stats[1] = g.n_aug;
        stats[2] = g.n_orphan;
    }
    return g.flow;
}

}  // namespace irls

namespace irls {

// The connected components of G_c (coarse n-links only) are independent
// max-flow problems joined by s_c and t_c: their flows add and their minimal
// source sides unite.  Components are solved by host threads, largest first;
// the result does not depend on the thread count.
i128 maxflow_bk(int32_t nc, const int32_t *ptr, const int32_t *col, const i128 *cap, const i128 *qs, const i128 *qt,
                uint8_t *src, int64_t *stats)
{
    if (nc <= 0) {
        if (stats) stats[0] = 1, stats[1] = 0, stats[2] = 0;
        return 0;
    }
    // components by BFS
    std::vector<int32_t> comp(nc, -1), order;
    order.reserve(nc);
    std::vector<int64_t> cstart;
    int32_t ncomp = 0;
    for (int32_t r = 0; r < nc; r++) {
        if (comp[r] >= 0) continue;
        cstart.push_back((int64_t)order.size());
        comp[r] = ncomp;
        order.push_back(r);
        for (size_t h = cstart.back(); h < order.size(); h++) {
            const int32_t u = order[h];
            for (int32_t a = ptr[u]; a < ptr[u + 1]; a++)
                if (comp[col[a]] < 0) {
                    comp[col[a]] = ncomp;
                    order.push_back(col[a]);
                }
        }
        ncomp++;
    }
    cstart.push_back(nc);
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    int64_t largest = 0;
    for (int32_t k = 0; k < ncomp; k++) largest = std::max<int64_t>(largest, cstart[k + 1] - cstart[k]);
    // one dominant component (or a small graph): no parallelism to gain
    static const int64_t par_min = [] {
        const char *e = getenv("IRLS_MAXFLOW_PAR_MIN");  // test hook: threaded path on small graphs
        return e ? atoll(e) : (int64_t)100000;
    }();
    if (ncomp == 1 || hw == 1 || nc < par_min || largest * 10 > (int64_t)nc * 9)
        return maxflow_bk_one(nc, ptr, col, cap, qs, qt, src, stats);
    // local ids: ascending original id inside each component (rows stay sorted)
    for (int32_t k = 0; k < ncomp; k++) std::sort(order.begin() + cstart[k], order.begin() + cstart[k + 1]);
    std::vector<int32_t> lid(nc);
    for (int32_t k = 0; k < ncomp; k++)
        for (int64_t i = cstart[k]; i < cstart[k + 1]; i++) lid[order[i]] = (int32_t)(i - cstart[k]);
    std::vector<int32_t> byk(ncomp);
    for (int32_t k = 0; k < ncomp; k++) byk[k] = k;
    std::sort(byk.begin(), byk.end(), [&](int32_t a, int32_t b) {
        return cstart[a + 1] - cstart[a] > cstart[b + 1] - cstart[b];
    });
    std::vector<i128> flows(ncomp, 0);
    std::vector<int64_t> st(3 * (size_t)ncomp, 0);
    std::atomic<int32_t> next{0};
    auto worker = [&]() {
        std::vector<int32_t> lp, lc;
        std::vector<i128> lcap, lqs, lqt;
        std::vector<uint8_t> lsrc;
        for (;;) {
            const int32_t j = next.fetch_add(1);
            if (j >= ncomp) return;
            const int32_t k = byk[j];
            const int64_t b0 = cstart[k], m = cstart[k + 1] - b0;
            lp.assign(m + 1, 0);
            lc.clear();
            lcap.clear();
            lqs.resize(m);
            lqt.resize(m);
            for (int64_t i = 0; i < m; i++) {
                const int32_t u = order[b0 + i];
                for (int32_t a = ptr[u]; a < ptr[u + 1]; a++) {
                    lc.push_back(lid[col[a]]);
                    lcap.push_back(cap[a]);
                }
                lp[i + 1] = (int32_t)lc.size();
                lqs[i] = qs[u];
                lqt[i] = qt[u];
            }
            lsrc.assign(m, 0);
            flows[k] = maxflow_bk_one((int32_t)m, lp.data(), lc.data(), lcap.data(), lqs.data(), lqt.data(),
                                      lsrc.data(), &st[3 * (size_t)k]);
            for (int64_t i = 0; i < m; i++) src[order[b0 + i]] = lsrc[i];
        }
    };
    const unsigned nt = std::min<unsigned>(hw, (unsigned)ncomp);
    std::vector<std::thread> th;
    for (unsigned i = 0; i < nt; i++) th.emplace_back(worker);
    for (auto &t : th) t.join();
    i128 flow = 0;
    int64_t cert = 1, aug = 0, orph = 0;
    for (int32_t k = 0; k < ncomp; k++) {
        flow += flows[k];
        cert = std::min<int64_t>(cert, st[3 * (size_t)k]);
        aug += st[3 * (size_t)k + 1];
        orph += st[3 * (size_t)k + 2];
    }
    if (stats) {
        stats[0] = cert;
        stats[1] = aug;
        stats[2] = orph;
    }
    return flow;
}

}  // namespace irls
