"""Probe for SURVEY §8(f) NEXT #2 (block-Jacobi with exact block solves):
PCG iteration counts on a reweighted IRLS system (the oracle's x^(1) of a
blob grid, numpy/scipy, NOT the contract arithmetic) with point Jacobi vs
x-line block Jacobi (tridiagonal blocks solved exactly by LU — the paper's
"block Jacobi with LU blocks" with one block per grid line), at the paper's
rtol 1e-3 and a tight 1e-6, warm (x0 = x^(1)) and cold.

usage: python tools/precond_probe.py [nx]      (grid nx x nx x nx/2)
"""
import sys

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spl

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import oracle  # noqa: E402
from synthetic import generators as gen  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 64
ny, nz = nx, nx // 2
spec = gen.blob_grid(nx, ny, nz, seed=1, sigma=(5.0 * nx / 128, 20.0 * nx / 128))
S = oracle.Solver(oracle.Graph(spec), T=3)
S.init()
S.step()
x = S.x()
N = x.size
ids = np.arange(N)
xx, yy, zz = ids % nx, (ids // nx) % ny, ids // (nx * ny)
eps2 = 1e-12


def rw(c, d):
    return np.where(c > 0, c * c / np.sqrt((c * d) ** 2 + eps2), 0.0)


gx = np.where(xx < nx - 1, rw(spec["cx"], x - np.roll(x, -1)), 0.0)
gy = np.where(yy < ny - 1, rw(spec["cy"], x - np.roll(x, -nx)), 0.0)
gz = np.where(zz < nz - 1, rw(spec["cz"], x - np.roll(x, -nx * ny)), 0.0)
gs, gt = rw(spec["cs"], 1.0 - x), rw(spec["ct"], x)
D = (gx + np.roll(gx, 1) * (xx > 0) + gy + np.roll(gy, nx) * (yy > 0) + gz + np.roll(gz, nx * ny) * (zz > 0)
     + gs + gt)
A = (sp.diags(D) - sp.diags(gx[:-1], 1) - sp.diags(gx[:-1], -1) - sp.diags(gy[:-nx], nx) - sp.diags(gy[:-nx], -nx)
     - sp.diags(gz[:-nx * ny], nx * ny) - sp.diags(gz[:-nx * ny], -nx * ny)).tocsr()
b = gs
lu = spl.splu((sp.diags(D) - sp.diags(gx[:-1], 1) - sp.diags(gx[:-1], -1)).tocsc())


def pcg(Minv, x0, rtol, cap=5000):
    r = b - A @ x0
    z = Minv(r)
    p = z.copy()
    rho = r @ z
    ref = np.linalg.norm(Minv(b))
    xk = x0.copy()
    for k in range(cap):
        if np.linalg.norm(z) <= rtol * ref:
            return k
        q = A @ p
        al = rho / (p @ q)
        xk += al * p
        r -= al * q
        z = Minv(r)
        rn = r @ z
        p = z + rn / rho * p
        rho = rn
    return cap


for rtol in (1e-3, 1e-6):
    for name, M in (("point Jacobi", lambda r: r / D), ("x-line Jacobi", lu.solve)):
        print(f"n={N} rtol={rtol:g} {name:14s} warm {pcg(M, x.copy(), rtol):5d}  cold {pcg(M, np.zeros(N), rtol):5d}")
