"""Command line: IRLS s-t min cut of a BASELINE config or a graph file.

    python -m paper_1501_03105_b200 --config 2 --rounding both --trace trace.csv
    python -m paper_1501_03105_b200 --graph g.npz --lambda2 --exact
    python -m paper_1501_03105_b200 --config 4 --virtual-ranks 8 --p2p

A graph file is an .npz with either a grid (kind="stencil": nx, ny, nz, cx,
cy, cz, cs, ct) or a CSR graph over all nodes incl. s and t (kind="csr": n,
row_ptr, col, w, s, t), as synthetic/generators.py builds them.  The trace
is the per-step report (SPEC's IrlsTrace: step, CG iterations, converged,
residuals, S_eps, flow value, x range, ms) as CSV.  Every step runs in the
CUDA library; this module only parses arguments and prints.
"""
from __future__ import annotations

import argparse
import csv
import json
import os
import sys
import time

import numpy as np

from . import build, irls as I


def load_graph(args):
    if args.graph:
        z = np.load(args.graph, allow_pickle=False)
        spec = {k: z[k] for k in z.files}
        spec["kind"] = str(spec["kind"])
        for k in ("nx", "ny", "nz", "n", "s", "t"):
            if k in spec:
                spec[k] = int(spec[k])
        return spec, args.graph
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if root not in sys.path:
        sys.path.insert(0, root)
    from synthetic import generators as gen
    make = {1: gen.config1, 2: gen.config2, 3: gen.config3, 4: gen.config4}[args.config]
    return make(), f"BASELINE config {args.config}"


def main(argv=None):
    ap = argparse.ArgumentParser(prog="python -m paper_1501_03105_b200", description=__doc__.split("\n\n")[0])
    src = ap.add_mutually_exclusive_group(required=True)
    src.add_argument("--config", type=int, choices=[1, 2, 3, 4],
                     help="BASELINE configs 1-4 (config 5 is a warm-started sequence: tools/bench_configs.py)")
    src.add_argument("--graph", help=".npz graph file")
    ap.add_argument("--T", type=int, default=50)
    ap.add_argument("--eps", type=float, default=1e-6)
    ap.add_argument("--rtol", type=float, default=None, help="CG relative tolerance (default 1e-3; config 1: 1e-10)")
    ap.add_argument("--cap", type=int, default=None, help="CG iteration cap (default 50; config 1: 100000)")
    ap.add_argument("--norm", choices=["preconditioned", "unpreconditioned"], default=None)
    ap.add_argument("--cold", action="store_true", help="cold-start every CG solve")
    ap.add_argument("--fixed-point-exit", action="store_true")
    ap.add_argument("--cg-variant", choices=["hs", "cg"], default="hs",
                    help="Hestenes-Stiefel PCG (default) or Chronopoulos-Gear (one reduction per iteration)")
    ap.add_argument("--rounding", choices=["sweep", "two_level", "both"], default="sweep")
    ap.add_argument("--lambda2", action="store_true", help="Cheeger-type lambda_2 (P:L207-226)")
    ap.add_argument("--exact", action="store_true", help="exact min cut mu* and delta (Eq. 13)")
    ap.add_argument("--trace", help="write the per-step report as CSV")
    ap.add_argument("--side", help="write the source-side indicator (uint8, one per node) as .npy")
    ap.add_argument("--virtual-ranks", type=int, default=0,
                    help="run the W-rank data path (z-slabs / id strips) as a virtual group on this GPU")
    ap.add_argument("--p2p", action="store_true", help="virtual ranks: peer-memory collectives")
    args = ap.parse_args(argv)

    build.build()
    spec, what = load_graph(args)
    c1 = args.config == 1
    rtol = args.rtol if args.rtol is not None else (1e-10 if c1 else 1e-3)
    cap = args.cap if args.cap is not None else (100000 if c1 else 50)
    norm = args.norm or ("unpreconditioned" if c1 else "preconditioned")
    opts = I.options(T=args.T, eps=args.eps, cg_rtol=rtol, cg_max_iter=cap,
                     cg_norm=I.IRLS_NORM_UNPRECONDITIONED if norm == "unpreconditioned" else I.IRLS_NORM_PRECONDITIONED,
                     warm_start=0 if args.cold else 1, fixed_point_exit=1 if args.fixed_point_exit else 0,
                     record_trace=1 if args.trace else 0,
                     cg_variant=I.IRLS_CG_CG if args.cg_variant == "cg" else I.IRLS_CG_HS)
    if args.virtual_ranks:
        unsupported = [f for f, on in (("--lambda2", args.lambda2), ("--exact", args.exact), ("--trace", args.trace))
                       if on]
        if unsupported:
            ap.error(f"--virtual-ranks does not support {', '.join(unsupported)}")
        opts.p2p = 1 if args.p2p else 0
        t0 = time.perf_counter()
        g = I.VGroup(spec, args.virtual_ranks, opts)
        out = {"graph": what, "virtual_ranks": args.virtual_ranks, "p2p": bool(args.p2p),
               "create_s": time.perf_counter() - t0}
        t0 = time.perf_counter()
        reps, iters = g.irls_vgroup_solve(I.IRLS_FROM_SCRATCH)
        out.update({"solve_s": time.perf_counter() - t0, "cg_iters": iters})
        side = None
        if args.rounding in ("sweep", "both"):
            side, _, k, cut = g.irls_vgroup_sweep_cut()
            out["sweep"] = {"cut": cut, "k": k}
        if args.rounding in ("two_level", "both"):
            side2, rep = g.irls_vgroup_two_level_cut()
            out["two_level"] = {"cut": rep["cut_value"], "coarse_nodes": rep["nc"]}
            side = side if side is not None else side2
        if args.side:
            np.save(args.side, side)
        g.close()
        print(json.dumps(out, indent=1))
        return
    t0 = time.perf_counter()
    m = I.MinCut.from_spec(spec, opts)
    st = m.irls_get_stats()
    out = {"graph": what, "nodes": st["n_nonterminal"], "n_links": st["n_links"],
           "create_s": time.perf_counter() - t0}
    t0 = time.perf_counter()
    reps, iters = m.irls_solve(I.IRLS_FROM_SCRATCH, T=args.T)
    out.update({"solve_s": time.perf_counter() - t0, "cg_iters": iters})
    side = None
    if args.rounding in ("sweep", "both"):
        t0 = time.perf_counter()
        side, _, k, cut = m.irls_sweep_cut()
        out["sweep"] = {"cut": cut, "k": k, "s": time.perf_counter() - t0}
    if args.rounding in ("two_level", "both"):
        side2, rep = m.irls_two_level_cut()
        out["two_level"] = {"cut": rep["cut_value"], "coarse_nodes": rep["nc"], "ms_gpu": rep["ms_gpu"],
                            "ms_maxflow": rep["ms_maxflow"]}
        if args.rounding == "two_level" or rep["cut_value"] < out["sweep"]["cut"]:
            side = side2
    if args.lambda2:
        out["lambda2"] = m.irls_lambda2()["lambda2"]
    if args.exact:
        _, ex = m.irls_exact_min_cut(side=False)
        mu = ex["cut_value"]
        out["mu_star"] = mu
        for key in ("sweep", "two_level"):
            if key in out and mu > 0:
                out[key]["delta"] = (out[key]["cut"] - mu) / mu
    if args.trace:
        with open(args.trace, "w", newline="") as f:
            w = csv.writer(f)
            cols = ["cg_iters", "converged", "rel_res", "true_rel_res", "S_eps", "flow_value", "x_min", "x_max", "ms"]
            w.writerow(["step"] + cols)
            for i, r in enumerate(reps):
                w.writerow([i] + [r[c] for c in cols])
    if args.side and side is not None:
        np.save(args.side, side)
    m.close()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
