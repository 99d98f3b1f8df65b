"""Size of the two-level coarse graph G_c on the BASELINE configs:
solve on the GPU, then (numpy, approximate reduction order) K-means with
initial centres 0.1/0.9, gamma0 = c0 + 0.05, gamma1 = c1 - 0.05, and the
S0/S1/Sc split; reports |Sc|, coarse n-links and connected components of the
coarse graph.  A sizing probe for the max-flow design, not a parity tool.

usage: python tools/coarse_stats.py [--configs 2,3,4]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import scipy.sparse as sp  # noqa: E402
from scipy.sparse.csgraph import connected_components  # noqa: E402

from paper_1501_03105_b200 import build, irls as I  # noqa: E402
from synthetic import generators as gen  # noqa: E402


def kmeans(x):
    c0, c1 = 0.1, 0.9
    for r in range(100):
        a1 = np.abs(x - c1) < np.abs(x - c0)
        n1 = int(a1.sum()); n0 = x.size - n1
        d0 = x[~a1].sum() / n0 if n0 else c0
        d1 = x[a1].sum() / n1 if n1 else c1
        if d0 == c0 and d1 == c1:
            return c0, c1, r + 1
        c0, c1 = d0, d1
    return c0, c1, 100


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,3,4")
    args = ap.parse_args()
    build.build()
    for cid in [int(c) for c in args.configs.split(",")]:
        spec = {2: gen.config2, 3: gen.config3, 4: gen.config4}[cid]()
        m = I.MinCut.from_spec(spec, I.options(T=50))
        m.irls_solve(I.IRLS_FROM_SCRATCH, T=50, reports=False)
        xf = m.irls_get_potentials()
        _, _, k, cut = m.irls_sweep_cut(side=False)
        m.close()
        if spec["kind"] == "stencil":
            N = spec["nx"] * spec["ny"] * spec["nz"]
            x = np.concatenate([xf[:N], [1.0, 0.0]])
        else:
            x = xf
        t0 = time.perf_counter()
        c0, c1, rounds = kmeans(x)
        g0, g1 = c0 + 0.05, c1 - 0.05
        cls = np.where(x <= g0, 0, np.where(x >= g1, 1, 2))
        sc = cls == 2
        nc = int(sc.sum())
        res = {"config": cid, "c0": c0, "c1": c1, "rounds": rounds, "gamma0": g0, "gamma1": g1,
               "n": int(x.size), "n0": int((cls == 0).sum()), "n1": int((cls == 1).sum()), "nc": nc,
               "sweep_cut": cut, "x_lt_0": int((x < 0).sum()), "x_exact0": int((x == 0).sum()),
               "hist": np.histogram(x, bins=20, range=(-0.0, 1.0))[0].tolist()}
        if spec["kind"] == "stencil":
            nx, ny, nz = spec["nx"], spec["ny"], spec["nz"]
            ids = np.arange(N).reshape(nz, ny, nx)
            us, vs = [], []
            for cap, sl_u, sl_v in ((spec["cx"].reshape(nz, ny, nx), (slice(None), slice(None), slice(0, -1)),
                                     (slice(None), slice(None), slice(1, None))),
                                    (spec["cy"].reshape(nz, ny, nx), (slice(None), slice(0, -1), slice(None)),
                                     (slice(None), slice(1, None), slice(None))),
                                    (spec["cz"].reshape(nz, ny, nx), (slice(0, -1), slice(None), slice(None)),
                                     (slice(1, None), slice(None), slice(None)))):
                u = ids[sl_u].ravel(); v = ids[sl_v].ravel(); c = cap[sl_u].ravel()
                keep = sc[u] & sc[v] & (c > 0)
                us.append(u[keep]); vs.append(v[keep])
            u = np.concatenate(us); v = np.concatenate(vs)
        else:
            rp, col = spec["row_ptr"], spec["col"]
            rows = np.repeat(np.arange(spec["n"]), np.diff(rp))
            keep = sc[rows] & sc[col] & (rows < col)
            u, v = rows[keep], col[keep]
        res["coarse_nlinks"] = int(u.size)
        if nc:
            cid_map = np.cumsum(sc) - 1
            A = sp.coo_matrix((np.ones(u.size), (cid_map[u], cid_map[v])), shape=(nc, nc)).tocsr()
            ncomp, lab = connected_components(A, directed=False)
            sizes = np.bincount(lab)
            res.update({"components": int(ncomp), "largest_component": int(sizes.max()),
                        "components_ge_1000": int((sizes >= 1000).sum())})
        res["probe_s"] = time.perf_counter() - t0
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
