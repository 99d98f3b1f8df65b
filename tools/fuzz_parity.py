"""Randomised parity sweep: random grid shapes / CSR graphs, random options
(PCG form, norm, warm/cold, rtol, cap, loop mode, trace, fixed-point exit,
block-Jacobi block size where compatible),
single rank and virtual groups — every case compared with the oracle
bitwise (reports, x^(T), sweep).  usage: python tools/fuzz_parity.py [cases] [seed]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1501_03105_b200 import build, irls as I  # noqa: E402
from synthetic import generators as gen  # noqa: E402

build.build()
cases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
fails = 0
for case in range(cases):
    kind = rng.choice(["grid", "grid", "csr"])
    if kind == "grid":
        nx, ny, nz = int(rng.integers(1, 70)), int(rng.integers(1, 40)), int(rng.integers(1, 12))
        if nx * ny * nz < 2:
            nx = 2
        spec = gen.blob_grid(nx, ny, nz, seed=int(rng.integers(1 << 30)), n_blobs=int(rng.integers(1, 6)),
                             sigma=(1.0, 6.0))
        desc = f"grid {nx}x{ny}x{nz}"
    else:
        n = int(rng.integers(10, 3000))
        spec = gen.random_small_graph(n, int(rng.integers(n, 3 * n)), seed=int(rng.integers(1 << 30)))
        desc = f"csr n={n}"
    T = int(rng.integers(0, 8))
    o = dict(T=T, cg_variant=int(rng.integers(0, 2)), cg_norm=int(rng.integers(0, 2)),
             warm_start=int(rng.integers(0, 2)), cg_rtol=float(rng.choice([1e-3, 1e-6, 1e-10])),
             cg_max_iter=int(rng.choice([5, 50, 500])), loop_mode=int(rng.integers(0, 2)),
             record_trace=int(rng.integers(0, 2)), fixed_point_exit=int(rng.integers(0, 2)))
    if o["cg_variant"] == 0 and not o["record_trace"] and rng.integers(0, 2):
        o["block_size"] = int(rng.choice([1, 3, 16, 64, 200]))
    try:
        m = I.MinCut.from_spec(spec, I.options(**o))
        reps, tot = m.irls_solve(I.IRLS_FROM_SCRATCH)
        S = oracle.Solver(oracle.Graph(spec), T=T, cg_norm=o["cg_norm"], warm_start=bool(o["warm_start"]),
                          cg_rtol=o["cg_rtol"], cg_max_iter=o["cg_max_iter"], cg_variant=o["cg_variant"],
                          block_size=o.get("block_size", 0))
        _, oreps = S.run(record=False)
        ok = [r["cg_iters"] for r in reps] == [r["cg_iters"] for r in oreps]
        ok = ok and [r["rel_res"] for r in reps] == [r["rel_res"] for r in oreps]
        ok = ok and np.array_equal(m.irls_get_potentials().view(np.uint64), S.x().view(np.uint64))
        side, order, k, cut = m.irls_sweep_cut(order=True)
        sw = S.sweep()
        ok = ok and k == sw.k and cut == sw.cut_value and np.array_equal(side, sw.side)
        ok = ok and np.array_equal(order.astype(np.int64), sw.order)
        m.close()
    except Exception as e:  # noqa: BLE001
        ok = False
        desc += f" EXC {e}"
    if not ok:
        fails += 1
        print(f"FAIL case {case}: {desc} {o}", flush=True)
# virtual groups: chunk-aligned slabs (64 x 64 planes) and CSR strips
vcases = max(cases // 10, 1)
for case in range(vcases):
    world = int(rng.choice([2, 4, 8]))
    if rng.integers(0, 3) > 0:
        nz = int(rng.integers(world, 28))
        spec = gen.blob_grid(64, 64, nz, seed=int(rng.integers(1 << 30)), sigma=(2.0, 8.0))
        desc = f"vgroup W={world} grid 64x64x{nz}"
    else:
        world = min(world, 4)
        spec = gen.road_graph(int(rng.integers(190, 260)), seed=int(rng.integers(1 << 20)), knn=60)
        desc = f"vgroup W={world} road n={spec['n']}"
    T = int(rng.integers(1, 8))
    o = dict(T=T, cg_variant=int(rng.integers(0, 2)), p2p=int(rng.integers(0, 2)),
             record_trace=int(rng.integers(0, 2)), warm_start=int(rng.integers(0, 2)),
             fixed_point_exit=int(rng.integers(0, 2)))
    if o["cg_variant"] == 0 and not o["p2p"] and not o["record_trace"] and rng.integers(0, 2):
        o["block_size"] = int(rng.choice([8, 64]))
    try:
        g = I.VGroup(spec, world, I.options(**o))
    except I.IrlsError:
        continue  # an unaligned partition is refused by design
    try:
        reps, tot = g.irls_vgroup_solve(I.IRLS_FROM_SCRATCH)
        S = oracle.Solver(oracle.Graph(spec), T=T, warm_start=bool(o["warm_start"]), cg_variant=o["cg_variant"],
                          block_size=o.get("block_size", 0))
        _, oreps = S.run(record=False)
        ok = [r["cg_iters"] for r in reps] == [r["cg_iters"] for r in oreps]
        ok = ok and np.array_equal(g.irls_vgroup_get_potentials().view(np.uint64), S.x().view(np.uint64))
        side, order, k, cut = g.irls_vgroup_sweep_cut(order=True)
        sw = S.sweep()
        ok = ok and k == sw.k and cut == sw.cut_value
        g.close()
    except Exception as e:  # noqa: BLE001
        ok = False
        desc += f" EXC {e}"
    if not ok:
        fails += 1
        print(f"FAIL vcase {case}: {desc} {o}", flush=True)
print(f"{cases} + {vcases} virtual-group cases, {fails} failures", flush=True)
