"""Table 4 analogue: cut quality of the sweep cut and of the
two-level rounding, delta = (mu - mu*) / mu* (Eq. 13), with mu* the exact
minimum cut of the whole graph (irls_exact_min_cut: the same host max-flow
with no contraction), plus the two-level phase times (Table 2's "two-level"
column) on the BASELINE configs, one GPU.

usage: python tools/quality.py [--configs 1,2,3,4] [--no-exact 4]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1501_03105_b200 import build, irls as I  # noqa: E402
from synthetic import generators as gen  # noqa: E402


def timed(fn):
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    out = fn()
    e1.record(s)
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4")
    ap.add_argument("--no-exact", default="")
    ap.add_argument("--out", default="gpurun_out/quality.json")
    args = ap.parse_args()
    build.build()
    skip = {int(c) for c in args.no_exact.split(",") if c}
    out = []
    for cid in [int(c) for c in args.configs.split(",")]:
        if cid == 1:
            spec, opts = gen.config1(), I.options(T=50, cg_rtol=1e-10, cg_max_iter=100000, cg_norm=1)
        else:
            spec, opts = {2: gen.config2, 3: gen.config3, 4: gen.config4}[cid](), I.options(T=50)
        m = I.MinCut.from_spec(spec, opts, I.comm_desc(1, 0, 0, None, torch.cuda.current_stream().cuda_stream))
        (_, iters), solve_ms = timed(lambda: m.irls_solve(I.IRLS_FROM_SCRATCH, T=50, reports=False))
        (_, _, k, sweep), sweep_ms = timed(lambda: m.irls_sweep_cut(side=False))
        t0 = time.perf_counter()
        _, tl = m.irls_two_level_cut(side=False)
        tl_wall = (time.perf_counter() - t0) * 1e3
        res = {"config": cid, "nodes": m.n, "cg_iters": iters, "solve_ms": solve_ms, "sweep_ms": sweep_ms,
               "sweep_cut": sweep, "two_level": tl, "two_level_wall_ms": tl_wall}
        if cid not in skip:
            t0 = time.perf_counter()
            _, ex = m.irls_exact_min_cut(side=False)
            res["exact"] = {"mu_star": ex["cut_value"], "certified": ex["certified"], "ms_maxflow": ex["ms_maxflow"],
                            "wall_ms": (time.perf_counter() - t0) * 1e3}
            mu = ex["cut_value"]
            res["delta_sweep"] = (sweep - mu) / mu
            res["delta_two_level"] = (tl["cut_value"] - mu) / mu
        m.close()
        print(json.dumps(res), flush=True)
        out.append(res)
        os.makedirs(os.path.dirname(args.out), exist_ok=True)
        json.dump(out, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
