"""Probe for SURVEY §8(f) NEXT #2 (block-Jacobi preconditioning, P:L235-242,
P:L365) on a mid-scale config-3 analogue (road_graph(side)) and a config-2/4
style blob grid: IRLS (eps 1e-6, T = 50, warm, rtol 1e-3 preconditioned
norm, cap 50) with M = point Jacobi, block Jacobi with exact block solves
(scipy splu) over contiguous id blocks of a given size, and block Jacobi with
red-black ILU(0) blocks (bipartite graphs).  numpy/scipy float64, NOT the
contract arithmetic.  Reports the sweep's delta against the exact min cut.

usage: python tools/precond_blocks_probe.py road|blob [side]
"""
import sys, time
import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from synthetic import generators as gen

kind = sys.argv[1] if len(sys.argv) > 1 else "road"
side = int(sys.argv[2]) if len(sys.argv) > 2 else 400
if kind == "road":
    spec = gen.road_graph(side, seed=2, knn=1000)
else:
    spec = gen.stencil_to_csr(gen.blob_grid(side, side, side // 2, seed=1, sigma=(side / 25.0, side / 6.0)))
n = spec["n"]; s = spec["s"]; t = spec["t"]
rp, col, w = spec["row_ptr"], spec["col"], spec["w"]
A = sp.csr_matrix((w, col, rp), shape=(n, n))
keep = np.ones(n, bool); keep[[s, t]] = False
idx = np.nonzero(keep)[0]
Cm = A[idx][:, idx].tocsr()
cs = np.asarray(A[idx, s].todense()).ravel()
ct = np.asarray(A[idx, t].todense()).ravel()
Cm.sum_duplicates()
E = sp.triu(Cm, 1).tocoo()
eu, ev, ec = E.row, E.col, E.data
nn = len(idx)
print(kind, "n", nn, "links", len(ec), flush=True)
eps = 1e-6
# 2-colouring by BFS (bipartite check)
from scipy.sparse.csgraph import breadth_first_order
colour = -np.ones(nn, np.int64)
G = (Cm != 0).astype(np.int8).tocsr()
for r0 in range(nn):
    if colour[r0] >= 0: continue
    order, pred = breadth_first_order(G, r0, directed=False, return_predecessors=True)
    colour[r0] = 0
    for v in order[1:]:
        colour[v] = 1 - colour[pred[v]]
bip = not np.any(colour[eu] == colour[ev])
print("bipartite", bip, flush=True)

def lap(g, gs, gt):
    L = sp.coo_matrix((np.concatenate([-g, -g]), (np.concatenate([eu, ev]), np.concatenate([ev, eu]))), shape=(nn, nn)).tocsr()
    D = np.bincount(eu, g, nn) + np.bincount(ev, g, nn) + gs + gt
    return (L + sp.diags(D)).tocsr(), D

_bfs_cache = {}


def bfs_blocks(bs):
    """Blocks grown by BFS from the lowest unassigned id, at most bs nodes
    each (a cheap planar-graph partition standing in for ParMETIS)."""
    if bs in _bfs_cache:
        return _bfs_cache[bs]
    from collections import deque
    blk = -np.ones(nn, np.int64)
    ptr, nb = G.indptr, G.indices
    b = 0
    for r0 in range(nn):
        if blk[r0] >= 0:
            continue
        q = deque([r0]); blk[r0] = b; cnt = 1
        while q and cnt < bs:
            u = q.popleft()
            for v in nb[ptr[u]:ptr[u + 1]]:
                if blk[v] < 0 and cnt < bs:
                    blk[v] = b; cnt += 1; q.append(v)
        b += 1
    _bfs_cache[bs] = blk
    return blk


def make_prec(L, D, kind, bs):
    if kind == "jacobi":
        Dinv = 1.0 / D
        return lambda r: Dinv * r
    if kind == "lubfs":
        blk = bfs_blocks(bs)
        kind = "lu"
    else:
        blk = np.arange(nn) // bs
    same = blk[L.tocoo().row] == blk[L.tocoo().col]
    Lc = L.tocoo()
    Lb = sp.csr_matrix((Lc.data[same], (Lc.row[same], Lc.col[same])), shape=(nn, nn))
    if kind == "lu":
        lu = spla.splu(Lb.tocsc())
        return lambda r: lu.solve(r)
    if kind == "rbilu":   # ILU(0) of each block in red-black order (exact closed form for 2-cyclic blocks)
        red = colour == 0
        Dinv = 1.0 / D
        Lo = Lb - sp.diags(Lb.diagonal())           # off-diagonal, within blocks
        Abr = Lo.multiply(np.outer(~red, red) if nn < 0 else 1).tocsr()
        # masks per row/col
        R = sp.diags(red.astype(float)); B = sp.diags((~red).astype(float))
        Abr = B @ Lo @ R; Arb = R @ Lo @ B
        # S_b = D_b - diag(A_br D_r^-1 A_rb)
        Sb = D - np.asarray((Abr.multiply(Abr) @ (Dinv * red))).ravel() * 0  # placeholder
        Sb = D - np.asarray(Abr.multiply(Abr) @ (Dinv * red)).ravel()  # sum_j a_bj^2 / d_j over red j
        Sinv = 1.0 / Sb
        def apply(r):
            y = r.copy()
            y[~red] = r[~red] - (Abr @ (Dinv * red * r))[~red]
            z = np.zeros_like(r)
            z[~red] = Sinv[~red] * y[~red]
            z[red] = Dinv[red] * (y[red] - (Arb @ z)[red])
            return z
        return apply
    raise ValueError(kind)

def pcg(L, D, b, x0, M, rtol=1e-3, cap=50):
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
    d = ct - cs
    a_first = rank[eu] < rank[ev]
    np.add.at(d, np.where(a_first, ev, eu), -ec)
    np.add.at(d, np.where(a_first, eu, ev), ec)
    P = cs.sum() + np.concatenate([[0.0], np.cumsum(d[order])])
    return P.min()

def run(pk, bs, cap=50, rtol=1e-3):
    x = np.zeros(nn); its = []
    g, gs, gt = ec.copy(), cs.copy(), ct.copy()
    for l in range(51):
        if l:
            dd = x[eu] - x[ev]; g = ec * ec / np.sqrt((ec * dd) ** 2 + eps ** 2)
            gs = cs * cs / np.sqrt((cs * (1 - x)) ** 2 + eps ** 2); gt = ct * ct / np.sqrt((ct * x) ** 2 + eps ** 2)
        L, D = lap(g, gs, gt)
        x, k = pcg(L, D, gs, x, make_prec(L, D, pk, bs), rtol=rtol, cap=cap); its.append(k)
    return sweep(x), its

def mincut():
    from scipy.sparse.csgraph import maximum_flow
    scale = 2 ** 20 if kind == "road" else 2 ** 16
    N2 = nn + 2
    rows = np.concatenate([eu, ev, np.full(nn, nn), np.arange(nn)])
    cols = np.concatenate([ev, eu, np.arange(nn), np.full(nn, nn + 1)])
    cap = np.concatenate([ec, ec, cs, ct])
    ci = np.rint(cap * scale).astype(np.int64)
    Gm = sp.csr_matrix((ci.astype(np.int32), (rows, cols)), shape=(N2, N2))
    return maximum_flow(Gm, nn, nn + 1).flow_value / scale

t0 = time.time(); mu = mincut(); print("mu*", mu, f"{time.time()-t0:.1f}s", flush=True)
cases = [("jacobi", 1)]
if bip:
    cases += [("rbilu", 4096), ("rbilu", nn // 8 + 1), ("rbilu", nn)]
cases += [("lu", 256), ("lu", 4096), ("lubfs", 64), ("lubfs", 256), ("lubfs", 1024), ("lubfs", 4096)]
for pk, bs in cases:
    t0 = time.time(); c, its = run(pk, bs)
    print(f"{pk:7s} block {bs:8d}: cut {c:.4f} delta {(c-mu)/mu:.4f} cg_iters {sum(its)} {its[:12]} ({time.time()-t0:.0f}s)", flush=True)
