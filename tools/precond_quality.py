"""Cut quality vs CG accuracy and preconditioner strength on a mid-scale
config-3 analogue (road_graph(side), numpy/scipy float64, NOT the contract
arithmetic): IRLS (eps 1e-6, T = 50, warm, preconditioned-norm rtol) with
point Jacobi (prec_m = 1) or a Jacobi-Neumann polynomial preconditioner of
degree prec_m - 1 (M^-1 = sum_{k<m} (I - D^-1 L)^k D^-1, SPD for odd m),
then the sweep; delta against the exact min cut (scipy maximum_flow on
2^-20-scaled integer capacities).  Evidence for DESIGN.md §9 (NEXT #2).

usage: python tools/precond_quality.py [side]     (default 400)
"""
import sys, time
import numpy as np
import scipy.sparse as sp
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from synthetic import generators as gen

side = int(sys.argv[1]) if len(sys.argv) > 1 else 400
spec = gen.road_graph(side, seed=2, knn=1000)
n = spec["n"]; s = spec["s"]; t = spec["t"]
rp, col, w = spec["row_ptr"], spec["col"], spec["w"]
A = sp.csr_matrix((w, col, rp), shape=(n, n))
keep = np.ones(n, bool); keep[[s, t]] = False
idx = np.nonzero(keep)[0]
C = A[idx][:, idx].tocsr()          # n-links among non-terminals
cs = np.asarray(A[idx, s].todense()).ravel()
ct = np.asarray(A[idx, t].todense()).ravel()
C.sum_duplicates()
E = sp.triu(C, 1).tocoo()
eu, ev, ec = E.row, E.col, E.data
m = len(ec); nn = len(idx)
print("n", nn, "links", m, flush=True)
eps = 1e-6

def lap(g, gs, gt):
    L = sp.coo_matrix((np.concatenate([-g, -g]), (np.concatenate([eu, ev]), np.concatenate([ev, eu]))), shape=(nn, nn)).tocsr()
    D = np.bincount(eu, g, nn) + np.bincount(ev, g, nn) + gs + gt
    return L + sp.diags(D), D

def pcg(L, D, b, x0, prec_m, rtol=1e-3, cap=50):
    Dinv = 1.0 / D
    def M(r):
        z = Dinv * r; y = z.copy()
        for _ in range(prec_m - 1):
            y = z + y - Dinv * (L @ y)    # y <- D^-1 r + (I - D^-1 L) y
        return y
    x = x0.copy(); r = b - L @ x; z = M(r); p = z.copy(); rho = r @ z
    ref = np.linalg.norm(M(b)); k = 0
    while True:
        res = np.linalg.norm(z)
        if res <= rtol * ref or k == cap: break
        q = L @ p; a = rho / (p @ q); x += a * p; r -= a * q; z = M(r)
        rn = r @ z; p = z + (rn / rho) * p; rho = rn; k += 1
    return x, k

def sweep(x):
    order = np.lexsort((np.arange(nn), -x))
    rank = np.empty(nn, np.int64); rank[order] = np.arange(nn)
    # delta_v = sum_u (rank_u > rank_v ? +c : -c) + ct - cs
    d = ct - cs
    a_first = rank[eu] < rank[ev]
    np.add.at(d, np.where(a_first, ev, eu), -ec)   # later node: edge to earlier loses
    np.add.at(d, np.where(a_first, eu, ev), ec)
    P = cs.sum() + np.concatenate([[0.0], np.cumsum(d[order])])
    return P.min()

def run(prec_m, cap, rtol):
    x = np.zeros(nn); tot = 0
    g, gs, gt = ec.copy(), cs.copy(), ct.copy()
    L, D = lap(g, gs, gt); x, k = pcg(L, D, gs, x, prec_m, rtol=rtol, cap=cap); tot += k
    for l in range(50):
        dd = x[eu] - x[ev]; g = ec * ec / np.sqrt((ec * dd) ** 2 + eps ** 2)
        gs = cs * cs / np.sqrt((cs * (1 - x)) ** 2 + eps ** 2); gt = ct * ct / np.sqrt((ct * x) ** 2 + eps ** 2)
        L, D = lap(g, gs, gt); x, k = pcg(L, D, gs, x, prec_m, rtol=rtol, cap=cap); tot += k
    return sweep(x), tot

def mincut():
    from scipy.sparse.csgraph import maximum_flow
    scale = 2 ** 20
    N2 = nn + 2
    rows = np.concatenate([eu, ev, np.full(nn, nn), np.arange(nn)])
    cols = np.concatenate([ev, eu, np.arange(nn), np.full(nn, nn + 1)])
    cap = np.concatenate([ec, ec, cs, ct])
    ci = np.rint(cap * scale).astype(np.int64)
    assert ci.max() < 2 ** 31
    G = sp.csr_matrix((ci.astype(np.int32), (rows, cols)), shape=(N2, N2))
    return maximum_flow(G, nn, nn + 1).flow_value / scale

t0 = time.time(); mu = mincut(); print("mu*", mu, f"{time.time()-t0:.1f}s", flush=True)
for pm, cap, rtol in [(1, 50, 1e-3), (3, 50, 1e-3), (5, 50, 1e-3), (1, 150, 1e-3), (1, 1000, 1e-5), (1, 1000, 1e-8)]:
    t0 = time.time(); c, tot = run(pm, cap, rtol)
    print(f"prec_m={pm} cap={cap} rtol={rtol:g}: cut {c:.4f} delta {(c-mu)/mu:.4f} cg_iters {tot} spmv {tot*pm} ({time.time()-t0:.0f}s)", flush=True)
