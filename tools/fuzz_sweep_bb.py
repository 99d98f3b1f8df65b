"""Randomised check of the branch-and-bound sweep (sweep_bb.cu) at sizes where
it runs (n~ >= 2^20): random grid shapes and CSR graphs, potentials of several
structures (solved, rounded to a few digits, tied levels, i.i.d., solved plus
noise), each swept without the order (branch and bound, or its fallback) and
compared with the oracle's full sort on the same potentials: k, the cut
value's bits and side[].  usage: python tools/fuzz_sweep_bb.py [cases] [seed]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1501_03105_b200 import build, irls as I  # noqa: E402
from synthetic import generators as gen  # noqa: E402

build.build()
cases = int(sys.argv[1]) if len(sys.argv) > 1 else 20
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 3)
fails = bb_runs = 0
for case in range(cases):
    nx = int(rng.choice([64, 96, 128, 192, 256, 512]))
    ny = int(rng.choice([32, 64, 96, 128]))
    nz = max(1, (1 << 20) // (nx * ny) + int(rng.integers(0, 48)))
    g = gen.blob_grid(nx, ny, nz, seed=int(rng.integers(1 << 30)), n_blobs=int(rng.integers(2, 30)))
    spec = gen.stencil_to_csr(g) if rng.random() < 0.25 else g
    m = I.MinCut.from_spec(spec, I.options(T=3))
    S = oracle.Solver(oracle.Graph(spec), T=3)
    m.irls_solve(I.IRLS_FROM_SCRATCH, T=3, reports=False)
    xs = m.irls_get_potentials()
    kind = rng.choice(["solved", "round", "levels", "iid", "noisy"])
    if kind == "round":
        x = np.round(xs, int(rng.integers(1, 5)))
    elif kind == "levels":
        L = int(rng.integers(2, 9))
        x = np.linspace(0.0, 1.0, L)[rng.integers(0, L, m.n)]
    elif kind == "iid":
        x = rng.random(m.n)
    elif kind == "noisy":
        x = xs + rng.normal(0.0, 1e-3, m.n)
    else:
        x = xs
    m.irls_set_potentials(x)
    side, _, k, cut = m.irls_sweep_cut(side=True)
    sorted_nodes = m.irls_get_stats()["sweep_sorted"]
    bb_runs += sorted_nodes < m.n
    sw = S.sweep(x)
    ok = k == sw.k and float(cut).hex() == float(sw.cut_value).hex() and np.array_equal(side, sw.side)
    fails += not ok
    print(f"case {case}: {spec['kind'] if 'kind' in spec else 'grid'} {nx}x{ny}x{nz} n={m.n} {kind:6s} "
          f"k={k} sorted={sorted_nodes} {'ok' if ok else 'MISMATCH oracle k=%d' % sw.k}", flush=True)
    m.close()
print(f"{cases} cases ({bb_runs} by branch and bound), {fails} failures")
sys.exit(1 if fails else 0)
