"""Independent test-side constructions (no oracle, no CUDA code).

Dense incidence-matrix forms of the paper's operators (Eq. 1, Eq. 8, Eq. 7) and
brute-force cut enumeration, used to pin the oracle.
"""
from __future__ import annotations

import itertools

import numpy as np


def edge_list(spec):
    """Undirected edge list (u, v, c) over original ids, u < v, from a
    synthetic spec (stencil: s = N, t = N+1)."""
    if spec["kind"] == "csr":
        rp, col, w = spec["row_ptr"], spec["col"], spec["w"]
        out = {}
        for u in range(spec["n"]):
            for e in range(rp[u], rp[u + 1]):
                v = int(col[e])
                if u < v:
                    out[(u, v)] = out.get((u, v), 0.0) + float(w[e])
        return spec["n"], spec["s"], spec["t"], [(u, v, c) for (u, v), c in sorted(out.items()) if c > 0]
    nx, ny, nz = spec["nx"], spec["ny"], spec["nz"]
    N = nx * ny * nz
    E = []
    for u in range(N):
        x, y, z = u % nx, (u // nx) % ny, u // (nx * ny)
        if x < nx - 1 and spec["cx"][u] > 0: E.append((u, u + 1, float(spec["cx"][u])))
        if y < ny - 1 and spec["cy"][u] > 0: E.append((u, u + nx, float(spec["cy"][u])))
        if z < nz - 1 and spec["cz"][u] > 0: E.append((u, u + nx * ny, float(spec["cz"][u])))
        if spec["cs"][u] > 0: E.append((u, N, float(spec["cs"][u])))
        if spec["ct"][u] > 0: E.append((u, N + 1, float(spec["ct"][u])))
    return N + 2, N, N + 1, E


def incidence(n, E):
    """B (m x n, arbitrary orientation) and the capacity vector c (Eq. 1)."""
    B = np.zeros((len(E), n))
    c = np.zeros(len(E))
    for i, (u, v, w) in enumerate(E):
        B[i, u] = 1.0; B[i, v] = -1.0; c[i] = w
    return B, c


def dense_irls_system(n, s, t, E, x=None, eps=1e-6):
    """Eq. 4 + Eq. 8 + Eq. 7 in matrix form: W = C when x is None,
    else w = sqrt((CBx)^2 + eps^2); L = B^T C W^-1 C B; reduced system
    (Z^T L Z) v = -Z^T L e_s.  Returns (Lred, b, keep) with keep the
    non-terminal ids in ascending order."""
    B, c = incidence(n, E)
    if x is None:
        w = c.copy()
    else:
        w = np.sqrt((c * (B @ x)) ** 2 + eps ** 2)
    L = B.T @ np.diag(c * c / w) @ B
    keep = np.array([i for i in range(n) if i not in (s, t)], dtype=np.int64)
    Lr = L[np.ix_(keep, keep)]
    b = -L[keep, s]
    return Lr, b, keep


def cut_value(E, side):
    return sum(c for u, v, c in E if side[u] != side[v])


def brute_force_mincut(n, s, t, E):
    """Minimum over all 2^(n-2) s-t cuts."""
    others = [i for i in range(n) if i not in (s, t)]
    best, best_side = None, None
    for bits in itertools.product((0, 1), repeat=len(others)):
        side = np.zeros(n, dtype=np.uint8)
        side[s] = 1
        for i, b in zip(others, bits):
            side[i] = b
        val = cut_value(E, side)
        if best is None or val < best:
            best, best_side = val, side
    return best, best_side


def prefix_sweep_bruteforce(n, s, t, E, x_full):
    """Sweep cut by definition: evaluate the cut of every prefix of the order
    (x desc, id asc) over non-terminals, s first, t last; first minimum."""
    others = [i for i in range(n) if i not in (s, t)]
    order = sorted(others, key=lambda i: (-x_full[i], i))
    best, best_k = None, None
    side = np.zeros(n, dtype=np.uint8); side[s] = 1
    for k in range(len(order) + 1):
        if k > 0:
            side[order[k - 1]] = 1
        val = cut_value(E, side)
        if best is None or val < best:
            best, best_k = val, k
    return best, best_k, order
