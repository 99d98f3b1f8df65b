"""Seeded synthetic inputs for the IRLS s-t min-cut hot path.

This module is shared by the CPU oracle tests and the CUDA path. It holds none
of the method's arithmetic (no reweighting, no Laplacian, no CG, no sweep): it
only draws graphs and capacities with numpy's PCG64 ``default_rng(seed)`` in a
fixed draw order, following SURVEY.md §8(d) and the configs of BASELINE.json.

The paper's datasets (UF sparse matrix road graphs, UWO segmentation grids;
PAPER.md L342) are not available, so these stand in for them.

Conventions
-----------
* Stencil graphs: node id ``u = x + nx*(y + ny*z)``; ``cx[u]`` is the capacity
  of edge (u, u+1) (0 at x = nx-1), ``cy[u]`` of (u, u+nx) (0 at y = ny-1),
  ``cz[u]`` of (u, u+nx*ny) (0 at z = nz-1).  ``cs[u]``/``ct[u]`` are the
  terminal capacities to the virtual source s = N and sink t = N+1.
* CSR graphs: symmetric, over all n nodes including s and t, int64 row_ptr,
  int32 col, float64 w.
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "config1", "config2", "config3", "config4", "config5_factors",
    "blob_grid", "uniform_grid", "road_graph", "stencil_to_csr",
    "tiny_graphs", "random_small_graph", "zero_nlink_grid",
]


def _stencil(nx, ny, nz, cx, cy, cz, cs, ct):
    return dict(kind="stencil", nx=int(nx), ny=int(ny), nz=int(nz),
                cx=np.ascontiguousarray(cx, dtype=np.float64).ravel(),
                cy=np.ascontiguousarray(cy, dtype=np.float64).ravel(),
                cz=np.ascontiguousarray(cz, dtype=np.float64).ravel(),
                cs=np.ascontiguousarray(cs, dtype=np.float64).ravel(),
                ct=np.ascontiguousarray(ct, dtype=np.float64).ravel())


def uniform_grid(nx=32, ny=32, seed=0, lo=0.1, hi=1.0, tlo=0.0, thi=2.0):
    """Config-1 recipe (BASELINE.json configs[0]): 2-D 4-neighbour grid.

    Draw order: cx U[lo,hi) (ny rows x (nx-1)), cy U[lo,hi) ((ny-1) rows x nx),
    cs U[tlo,thi) (N), ct U[tlo,thi) (N).
    """
    rng = np.random.default_rng(seed)
    N = nx * ny
    cx = np.zeros((ny, nx)); cy = np.zeros((ny, nx))
    cx[:, : nx - 1] = rng.uniform(lo, hi, (ny, nx - 1))
    cy[: ny - 1, :] = rng.uniform(lo, hi, (ny - 1, nx))
    cs = rng.uniform(tlo, thi, N)
    ct = rng.uniform(tlo, thi, N)
    return _stencil(nx, ny, 1, cx, cy, np.zeros(N), cs, ct)


def config1():
    """BASELINE configs[0]: 32x32, n-links U[0.1,1.0), t-links U[0,2), seed 0."""
    return uniform_grid(32, 32, seed=0)


def blob_grid(nx, ny, nz, seed, n_blobs=20, sigma=(5.0, 20.0), lam=2.0,
              noise=0.05, beta_sigma=0.1, amplitude=1.0):
    """GraphCut-style 3-D 6-neighbour grid (configs 2, 4).

    Draw order: for each blob, centre mu = uniform([0,0,0],[nx,ny,nz]) in
    (x,y,z) order then sigma = uniform(*sigma); then noise
    normal(0, noise, (nz,ny,nx)).  I = sum_b A*exp(-|p-mu_b|^2/(2 sigma_b^2))
    + noise (evaluated separably per blob).  n-link c = exp(-dI^2/(2*0.1^2))
    per +axis edge; cs = lam*max(0, I-0.5), ct = lam*max(0, 0.5-I).
    """
    rng = np.random.default_rng(seed)
    blobs = []
    for _ in range(n_blobs):
        mu = rng.uniform([0.0, 0.0, 0.0], [nx, ny, nz])
        sg = rng.uniform(sigma[0], sigma[1])
        blobs.append((mu, sg))
    I = rng.normal(0.0, noise, (nz, ny, nx))
    xs = np.arange(nx, dtype=np.float64)
    ys = np.arange(ny, dtype=np.float64)
    zs = np.arange(nz, dtype=np.float64)
    for mu, sg in blobs:
        inv = 1.0 / (2.0 * sg * sg)
        ex = amplitude * np.exp(-((xs - mu[0]) ** 2) * inv)
        ey = np.exp(-((ys - mu[1]) ** 2) * inv)
        ez = np.exp(-((zs - mu[2]) ** 2) * inv)
        # I += ez[:,None,None]*ey[None,:,None]*ex[None,None,:], plane by plane
        eyx = ey[:, None] * ex[None, :]
        for z in range(nz):
            I[z] += ez[z] * eyx
    denom = 2.0 * beta_sigma * beta_sigma
    cx = np.zeros((nz, ny, nx)); cy = np.zeros((nz, ny, nx)); cz = np.zeros((nz, ny, nx))
    cx[:, :, : nx - 1] = np.exp(-((I[:, :, 1:] - I[:, :, :-1]) ** 2) / denom)
    cy[:, : ny - 1, :] = np.exp(-((I[:, 1:, :] - I[:, :-1, :]) ** 2) / denom)
    cz[: nz - 1, :, :] = np.exp(-((I[1:, :, :] - I[:-1, :, :]) ** 2) / denom)
    cs = lam * np.maximum(0.0, I - 0.5)
    ct = lam * np.maximum(0.0, 0.5 - I)
    return _stencil(nx, ny, nz, cx, cy, cz, cs, ct)


def config2():
    """BASELINE configs[1]: 128^3 blob grid, seed 1."""
    return blob_grid(128, 128, 128, seed=1)


def config4():
    """BASELINE configs[3]: 512x512x256 blob grid, sigma U[20,80], seed 3."""
    return blob_grid(512, 512, 256, seed=3, sigma=(20.0, 80.0))


def config5_factors(n, n_problems=10, seed=4):
    """BASELINE configs[4] (A19): per problem, fresh U[0.99,1.01] factors for
    cs (n draws) then ct (n draws); applied cumulatively by the caller."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n_problems):
        fs = rng.uniform(0.99, 1.01, n)
        ft = rng.uniform(0.99, 1.01, n)
        out.append((fs, ft))
    return out


def zero_nlink_grid(nx, ny, nz, seed, lo=0.0, hi=2.0):
    """A grid whose n-links are all zero: every pixel is an independent
    two-edge path s-u-t (SURVEY §8(c) pin (iii))."""
    rng = np.random.default_rng(seed)
    N = nx * ny * nz
    cs = rng.uniform(lo, hi, N)
    ct = rng.uniform(lo, hi, N)
    z = np.zeros(N)
    return _stencil(nx, ny, nz, z, z.copy(), z.copy(), cs, ct)


# ----------------------------------------------------------------------------
# CSR graphs
# ----------------------------------------------------------------------------

def _csr_from_edges(n, u, v, w):
    """Symmetric CSR (both directions) from an undirected edge list with no
    duplicate pairs; columns ascending within each row."""
    u = np.asarray(u, dtype=np.int64); v = np.asarray(v, dtype=np.int64)
    w = np.asarray(w, dtype=np.float64)
    rows = np.concatenate([u, v]); cols = np.concatenate([v, u]); vals = np.concatenate([w, w])
    order = np.lexsort((cols, rows))
    rows = rows[order]; cols = cols[order]; vals = vals[order]
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(row_ptr, rows + 1, 1)
    row_ptr = np.cumsum(row_ptr)
    return row_ptr, cols.astype(np.int32), vals


def stencil_to_csr(g):
    """Express a stencil graph as a CSR graph with s = N, t = N+1.  Only edges
    with positive capacity are emitted."""
    nx, ny, nz = g["nx"], g["ny"], g["nz"]
    N = nx * ny * nz
    ids = np.arange(N, dtype=np.int64)
    x = ids % nx; y = (ids // nx) % ny; z = ids // (nx * ny)
    us, vs, ws = [], [], []
    for c, ok, off in ((g["cx"], x < nx - 1, 1), (g["cy"], y < ny - 1, nx),
                       (g["cz"], z < nz - 1, nx * ny)):
        m = ok & (c > 0)
        us.append(ids[m]); vs.append(ids[m] + off); ws.append(c[m])
    m = g["cs"] > 0
    us.append(ids[m]); vs.append(np.full(int(m.sum()), N, dtype=np.int64)); ws.append(g["cs"][m])
    m = g["ct"] > 0
    us.append(ids[m]); vs.append(np.full(int(m.sum()), N + 1, dtype=np.int64)); ws.append(g["ct"][m])
    row_ptr, col, w = _csr_from_edges(N + 2, np.concatenate(us), np.concatenate(vs), np.concatenate(ws))
    return dict(kind="csr", n=N + 2, row_ptr=row_ptr, col=col, w=w, s=N, t=N + 1)


def road_graph(side=4900, seed=2, p_delete=0.3, knn=1000, knn_weight=10.0, jitter=0.3):
    """Road-network-like planar graph (BASELINE configs[2]).

    Draw order: jitter uniform(-j, j, (side^2, 2)); deletion uniforms
    random(m_grid) over horizontal edges row-major then vertical edges
    row-major (delete if < p_delete); lognormal(0,1) per surviving edge in the
    same order.  Keep the largest connected component (relabelled in
    ascending original id).  s / t = LCC nodes nearest (0, (side-1)/2) and
    (side-1, (side-1)/2) in jittered coordinates (ties by id); each is joined
    to its `knn` nearest LCC nodes (Euclidean on jittered coordinates, ties by
    id, excluding itself) with weight `knn_weight`, merged by summation with
    existing edges.
    """
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import connected_components

    rng = np.random.default_rng(seed)
    N = side * side
    jit = rng.uniform(-jitter, jitter, (N, 2))
    # horizontal then vertical edges, row-major
    yy, xx = np.meshgrid(np.arange(side, dtype=np.int64), np.arange(side - 1, dtype=np.int64), indexing="ij")
    hu = (yy * side + xx).ravel(); hv = hu + 1
    yy, xx = np.meshgrid(np.arange(side - 1, dtype=np.int64), np.arange(side, dtype=np.int64), indexing="ij")
    vu = (yy * side + xx).ravel(); vv = vu + side
    del yy, xx
    eu = np.concatenate([hu, vu]); ev = np.concatenate([hv, vv])
    del hu, hv, vu, vv
    keep = rng.random(eu.shape[0]) >= p_delete
    eu = eu[keep]; ev = ev[keep]
    ew = rng.lognormal(0.0, 1.0, eu.shape[0])
    A = coo_matrix((np.ones(eu.shape[0], dtype=np.int8), (eu, ev)), shape=(N, N))
    ncomp, lab = connected_components(A, directed=False)
    del A
    big = np.argmax(np.bincount(lab))
    in_lcc = lab == big
    new_id = np.full(N, -1, dtype=np.int64)
    lcc_nodes = np.nonzero(in_lcc)[0]
    new_id[lcc_nodes] = np.arange(lcc_nodes.shape[0])
    m = in_lcc[eu]  # both endpoints share a component
    eu = new_id[eu[m]]; ev = new_id[ev[m]]; ew = ew[m]
    n = lcc_nodes.shape[0]
    px = (lcc_nodes % side).astype(np.float64) + jit[lcc_nodes, 0]
    py = (lcc_nodes // side).astype(np.float64) + jit[lcc_nodes, 1]
    mid = (side - 1) / 2.0

    def nearest(qx, qy):
        d2 = (px - qx) ** 2 + (py - qy) ** 2
        return int(np.lexsort((np.arange(n), d2))[0])

    s = nearest(0.0, mid); t = nearest(float(side - 1), mid)
    extra_u, extra_v = [], []
    for term in (s, t):
        d2 = (px - px[term]) ** 2 + (py - py[term]) ** 2
        d2[term] = np.inf
        cand = np.argpartition(d2, knn + 64)[: knn + 64] if n > knn + 64 else np.arange(n)
        order = np.lexsort((cand, d2[cand]))
        nbrs = cand[order[:knn]]
        nbrs = nbrs[np.isfinite(d2[nbrs])]
        extra_u.append(np.full(nbrs.shape[0], term, dtype=np.int64)); extra_v.append(nbrs.astype(np.int64))
    eu = np.concatenate([eu] + extra_u); ev = np.concatenate([ev] + extra_v)
    ew = np.concatenate([ew] + [np.full(a.shape[0], knn_weight) for a in extra_u])
    # merge duplicates (a kNN edge on top of a grid edge) by summation
    a = np.minimum(eu, ev); b = np.maximum(eu, ev)
    key = a * n + b
    order = np.argsort(key, kind="stable")
    key = key[order]; ew = ew[order]
    uniq, start = np.unique(key, return_index=True)
    wsum = np.add.reduceat(ew, start)
    row_ptr, col, w = _csr_from_edges(n, uniq // n, uniq % n, wsum)
    return dict(kind="csr", n=int(n), row_ptr=row_ptr, col=col, w=w, s=int(s), t=int(t))


def config3():
    """BASELINE configs[2]: 4900x4900 jittered road-like grid, seed 2."""
    return road_graph(4900, seed=2)


# ----------------------------------------------------------------------------
# Tiny graphs for pins (SPEC worked examples, brute force)
# ----------------------------------------------------------------------------

def _csr_edges(n, edges, s, t):
    u = [e[0] for e in edges]; v = [e[1] for e in edges]; w = [e[2] for e in edges]
    row_ptr, col, ww = _csr_from_edges(n, u, v, w)
    return dict(kind="csr", n=n, row_ptr=row_ptr, col=col, w=ww, s=s, t=t)


def tiny_graphs():
    """SPEC.md worked examples as CSR graphs.
    Node ids: listed per graph."""
    return {
        # path s - a - t, c(s,a)=2, c(a,t)=1 ; ids s=0, a=1, t=2
        "path": _csr_edges(3, [(0, 1, 2.0), (1, 2, 1.0)], 0, 2),
        # triangle s,a,t with (s,a,1), (a,t,1), (s,t,0.5); ids s=0,a=1,t=2
        "triangle": _csr_edges(3, [(0, 1, 1.0), (1, 2, 1.0), (0, 2, 0.5)], 0, 2),
        # 4-cycle s-a-t-b-s unit weights; ids s=0, a=1, t=2, b=3
        "cycle4": _csr_edges(4, [(0, 1, 1.0), (1, 2, 1.0), (2, 3, 1.0), (3, 0, 1.0)], 0, 2),
        # path s-a-b-t unit weights; ids s=0, a=1, b=2, t=3
        "path4": _csr_edges(4, [(0, 1, 1.0), (1, 2, 1.0), (2, 3, 1.0)], 0, 3),
        # symmetric path s-a-t with equal weights
        "path_sym": _csr_edges(3, [(0, 1, 1.5), (1, 2, 1.5)], 0, 2),
    }


def random_small_graph(n, m_extra, seed, wlo=0.1, whi=2.0):
    """A connected random graph on n nodes (s = 0, t = n-1): a random spanning
    tree plus m_extra extra distinct edges, weights U[wlo, whi)."""
    rng = np.random.default_rng(seed)
    perm = rng.permutation(n)
    edges = {}
    for i in range(1, n):
        j = int(rng.integers(0, i))
        a, b = int(perm[i]), int(perm[j])
        edges[(min(a, b), max(a, b))] = None
    tries = 0
    while len(edges) < n - 1 + m_extra and tries < 100 * (m_extra + 1):
        a, b = (int(v) for v in rng.integers(0, n, 2))
        tries += 1
        if a != b:
            edges[(min(a, b), max(a, b))] = None
    keys = sorted(edges)
    w = rng.uniform(wlo, whi, len(keys))
    return _csr_edges(n, [(a, b, float(c)) for (a, b), c in zip(keys, w)], 0, n - 1)
