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


# --------------------------------------------------------------------------
# Textbook Jacobi-PCG in numpy (no oracle import), written from SURVEY §8(c)
# O5 / DESIGN A9, A13 ("preconditioned conjugate gradient", P:L242
# warm start, "relative residual", "50 PCG iterations at
# maximum") and the Chronopoulos-Gear form of A31.  Dense matrices, numpy
# dot products (a different summation order from the contract's C3 tree),
# used to pin the oracle's stopping rule at loose tolerances.
# --------------------------------------------------------------------------

def np_jacobi_pcg(A, b, x0, rtol, cap, precond_norm=True, variant="hs"):
    """Solve A v = b by CG preconditioned with M = diag(A), from x0.

    Stopping (A9/A13): before each iteration, stop if
    ||res|| <= rtol * ref or k == cap, where res = M^-1 r and ref = ||M^-1 b||
    (preconditioned norm) or res = r and ref = ||b|| (unpreconditioned).
    b = 0 returns v = 0 with 0 iterations.  Returns (x, k, res/ref)."""
    Minv = 1.0 / np.diag(A)
    x = np.array(x0, dtype=np.float64)
    ref = np.linalg.norm(Minv * b) if precond_norm else np.linalg.norm(b)
    if ref == 0.0:
        return np.zeros_like(b), 0, 0.0
    r = b - A @ x
    z = Minv * r

    def resid(r, z):
        return np.linalg.norm(z if precond_norm else r)

    res = resid(r, z)
    k = 0
    if variant == "hs":
        p = z.copy()
        rho = r @ z
        while True:
            if res <= rtol * ref or k == cap:
                break
            q = A @ p
            alpha = rho / (p @ q)
            x = x + alpha * p
            r = r - alpha * q
            z = Minv * r
            rho_new = r @ z
            res = resid(r, z)
            p = z + (rho_new / rho) * p
            rho = rho_new
            k += 1
    else:  # Chronopoulos-Gear: carries w = A z and s = A p, one reduction per iteration
        rho = r @ z
        w = A @ z
        alpha = rho / (z @ w)
        beta = 0.0
        p = np.zeros_like(b)
        s = np.zeros_like(b)
        while True:
            if res <= rtol * ref or k == cap:
                break
            p = z + beta * p
            s = w + beta * s
            x = x + alpha * p
            r = r - alpha * s
            z = Minv * r
            w = A @ z
            gamma, delta = r @ z, z @ w
            res = resid(r, z)
            k += 1
            beta = gamma / rho
            alpha = gamma / (delta - beta * gamma / alpha)
            rho = gamma
    return x, k, (res / ref)


def full_potentials(n, s, t, keep, v):
    """The full voltage vector of Eq. 5: x_s = 1, x_t = 0, x[keep] = v."""
    x = np.zeros(n)
    x[s] = 1.0
    x[keep] = v
    return x


# --------------------------------------------------------------------------
# The same PCG under the written arithmetic contract (SURVEY §8(c) C1-C3,
# O1-O5, O5'), re-implemented in numpy from that text (no oracle import):
# elementwise IEEE operations (numpy never contracts to FMA), per-node sums
# over ascending neighbour ids, and the C3 reduction tree.  Finite-precision
# CG at rtol 1e-3 is chaotic in the summation order (a textbook numpy PCG
# flips a few iteration counts and drifts by 1e-4), so bitwise agreement
# with the oracle needs the contract's order; this is that order, written
# independently.
# --------------------------------------------------------------------------

def np_c3_sum(v):
    """C3: 4096-element chunks; "thread" t of 256 sums the
    elements base + 2t + 512j + e (j = 0..7, e = 0, 1) sequentially from +0.0;
    warp lanes combine by offsets 16, 8, 4, 2, 1 (lane i += lane i+off); the 8
    warp sums by offsets 4, 2, 1; the chunk partials of 8 fixed groups
    [floor(gK/8), floor((g+1)K/8)) are each reduced as a fresh list by the same
    procedure until one value remains; the 8 group sums by offsets 4, 2, 1.
    Elements past the end contribute +0.0."""
    v = np.asarray(v, dtype=np.float64)

    def chunks(a):
        K = max((a.shape[0] + 4095) // 4096, 0)
        pad = np.zeros(K * 4096)
        pad[: a.shape[0]] = a
        blk = pad.reshape(K, 8, 256, 2)                # [chunk, j, t, e] -> index 512j + 2t + e
        acc = np.zeros((K, 256))
        for j in range(8):
            for e in range(2):
                acc = acc + blk[:, j, :, e]
        lanes = acc.reshape(K, 8, 32).copy()
        for off in (16, 8, 4, 2, 1):
            lanes[:, :, :off] = lanes[:, :, :off] + lanes[:, :, off:2 * off]
        w = lanes[:, :, 0].copy()
        for off in (4, 2, 1):
            w[:, :off] = w[:, :off] + w[:, off:2 * off]
        return w[:, 0]

    def reduce_list(a):
        if a.shape[0] == 0:
            return 0.0
        while a.shape[0] > 1:
            a = chunks(a)
        return float(a[0])

    part = chunks(v) if v.shape[0] else np.zeros(0)
    K = part.shape[0]
    g = np.array([reduce_list(part[gi * K // 8:(gi + 1) * K // 8]) for gi in range(8)])
    for off in (4, 2, 1):
        g[:off] = g[:off] + g[off:2 * off]
    return float(g[0])


class ContractSystem:
    """Reduced system of Eq. 7 on the non-terminal nodes (ascending original
    id), stored as padded ascending neighbour lists: nbr[u, j] (−1 = none),
    cap[u, j]; terminal capacities cs, ct."""

    def __init__(self, spec):
        n, s, t, E = edge_list(spec)
        keep = [i for i in range(n) if i not in (s, t)]
        rid = {o: i for i, o in enumerate(keep)}
        nb = [dict() for _ in keep]
        cs = np.zeros(len(keep)); ct = np.zeros(len(keep))
        for u, v, c in E:
            if u not in rid and v not in rid:
                continue                                # direct s-t edge: a constant (A5)
            if u in rid and v in rid:
                nb[rid[u]][rid[v]] = nb[rid[u]].get(rid[v], 0.0) + c
                nb[rid[v]][rid[u]] = nb[rid[v]].get(rid[u], 0.0) + c
            else:
                a, term = (u, v) if u in rid else (v, u)
                if term == s:
                    cs[rid[a]] += c
                elif term == t:
                    ct[rid[a]] += c
        m = max([len(d) for d in nb] + [1])
        self.n = len(keep)
        self.nbr = -np.ones((self.n, m), dtype=np.int64)
        self.cap = np.zeros((self.n, m))
        for u, d in enumerate(nb):
            for j, v in enumerate(sorted(d)):
                self.nbr[u, j] = v
                self.cap[u, j] = d[v]
        self.cs, self.ct = cs, ct
        self.keep = np.array(keep, dtype=np.int64)

    @staticmethod
    def _g(c, d, eps2):
        a = c * d
        return (c * c) / np.sqrt(a * a + eps2)          # Eq. 4 + Eq. 8 (O3, A2)

    def assemble(self, x=None, eps=1e-6):
        """O1/O3/O4: per-edge g, D = ((sum_asc g) + gs) + gt, Dinv, b = gs."""
        eps2 = eps * eps
        valid = self.nbr >= 0
        if x is None:
            g = self.cap.copy(); gs = self.cs.copy(); gt = self.ct.copy()
        else:
            xv = x[np.where(valid, self.nbr, 0)]
            g = np.where(valid, self._g(self.cap, x[:, None] - xv, eps2), 0.0)
            gs = self._g(self.cs, 1.0 - x, eps2)
            gt = self._g(self.ct, x, eps2)
        acc = np.zeros(self.n)
        for j in range(self.nbr.shape[1]):
            acc = acc + g[:, j]
        D = (acc + gs) + gt
        return g, D, 1.0 / D, gs

    def matvec(self, g, D, p):
        """O2: acc = sum_asc g_uv p_v from +0.0; q = D p - acc."""
        acc = np.zeros(self.n)
        valid = self.nbr >= 0
        for j in range(self.nbr.shape[1]):
            acc = acc + np.where(valid[:, j], g[:, j] * p[np.where(valid[:, j], self.nbr[:, j], 0)], 0.0)
        return D * p - acc


def contract_pcg(sysm, g, D, Dinv, b, x0, rtol, cap, precond_norm=True, variant="hs", mutate=None):
    """O5 (Hestenes-Stiefel) / O5' (Chronopoulos-Gear, A31) under C1-C3.
    Returns (x, k, converged, rel_res); raises on breakdown.

    ``mutate`` injects one plausible mistake (HS only; for the test that the
    pin discriminates): "ref_b" (ref = ||b|| under the preconditioned norm),
    "test_after" (no test before the first iteration), "res_squared"
    (||res||^2 compared with rtol*ref), "cold" (x0 ignored)."""
    C3 = np_c3_sum
    x = np.zeros_like(b) if mutate == "cold" else np.array(x0, dtype=np.float64)
    r = b - sysm.matvec(g, D, x)
    z = r * Dinv
    rho = C3(r * z)
    mb = b * Dinv
    ref = float(np.sqrt(C3(mb * mb) if precond_norm and mutate != "ref_b" else C3(b * b)))
    if ref == 0.0:
        return np.zeros_like(b), 0, 1, 0.0

    def resid(r, z):
        v = float(np.sqrt(C3(z * z) if precond_norm else C3(r * r)))
        return v * v if mutate == "res_squared" else v

    res = resid(r, z)
    k = 0
    stop = lambda: res <= rtol * ref or k == cap
    if variant == "hs":
        p = z.copy()
        while (mutate == "test_after" and k == 0) or not stop():
            q = sysm.matvec(g, D, p)
            pi = C3(p * q)
            if not (pi > 0.0) or np.isinf(pi):
                raise FloatingPointError("breakdown")
            alpha = rho / pi
            x = x + alpha * p
            r = r - alpha * q
            z = r * Dinv
            rho1 = C3(r * z)
            res = resid(r, z)
            beta = rho1 / rho
            p = z + beta * p
            rho = rho1
            k += 1
    else:
        alpha = beta = 0.0
        if not stop():
            w = sysm.matvec(g, D, z)
            delta = C3(z * w)
            alpha = rho / delta
        p = np.zeros_like(b); s = np.zeros_like(b)
        while not stop():
            p = z.copy() if k == 0 else z + beta * p
            s = w.copy() if k == 0 else w + beta * s
            x = x + alpha * p
            r = r - alpha * s
            z = r * Dinv
            w = sysm.matvec(g, D, z)
            gamma = C3(r * z); delta = C3(z * w)
            res = float(np.sqrt(C3(z * z) if precond_norm else C3(r * r)))
            k += 1
            beta = gamma / rho
            t = beta * gamma
            t = t / alpha
            den = delta - t
            rho = gamma
            if not stop():
                alpha = gamma / den
    return x, k, int(res <= rtol * ref), res / ref


def contract_irls(sysm, T, eps, rtol, cap, precond_norm=True, warm=True, variant="hs"):
    """O6 (Algorithm 1): x^(0) with W = C from 0, then T
    reweighted solves, warm-started from x^(l-1) or cold."""
    g, D, Dinv, b = sysm.assemble(None, eps)
    x, k, conv, rr = contract_pcg(sysm, g, D, Dinv, b, np.zeros(sysm.n), rtol, cap, precond_norm, variant)
    xs, ks, rrs = [x], [k], [rr]
    for _ in range(T):
        g, D, Dinv, b = sysm.assemble(x, eps)
        x0 = x if warm else np.zeros(sysm.n)
        x, k, conv, rr = contract_pcg(sysm, g, D, Dinv, b, x0, rtol, cap, precond_norm, variant)
        xs.append(x); ks.append(k); rrs.append(rr)
    return np.array(xs), ks, rrs
