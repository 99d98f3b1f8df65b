"""Sensitivity of the IRLS policy (SURVEY §8(d) config-2 sensitivity runs;
VERDICT r1 item 9; Fig. 1) on one GPU.

Part A — config 2 (128^3 blobs) under several CG policies: the bench's
(rtol 1e-3 preconditioned norm, cap 50), cap 300 (§5.2's cap), the
UNPRECONDITIONED norm, and tighter tolerances.  Per policy: total CG
iterations, iterations per step, the solve at which IRLS freezes (first warm
step with 0 iterations: x^(l) = x^(l-1), and every later step repeats it),
time-to-cut, and the cut quality delta = (mu - mu*)/mu* (Eq. 13) of the
sweep and of the two-level rounding, mu* from profiles/r01_quality.json.

Part B — config 5's warm-started sequence (A19: 10 cumulative t-link
rescalings) vs cold starts, under the same policies: the paper's Fig. 1
claim (warm starts save PCG iterations) is only testable where the sequence
does not freeze; at rtol 1e-3 it freezes after one iteration (A9: ||M^-1 b||
grows like c^2/eps, so a +-1% t-link change never trips the test).

usage: python tools/sensitivity.py [--out gpurun_out/sensitivity.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1501_03105_b200 import build, irls as I  # noqa: E402
from synthetic import generators as gen  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
POLICIES = [  # (name, rtol, cap, norm)
    ("paper: rtol 1e-3, cap 50, precond (bench)", 1e-3, 50, 0),
    ("rtol 1e-3, cap 300, precond", 1e-3, 300, 0),
    ("rtol 1e-3, cap 50, UNprecond", 1e-3, 50, 1),
    ("rtol 1e-3, cap 300, UNprecond", 1e-3, 300, 1),
    ("rtol 1e-6, cap 300, precond", 1e-6, 300, 0),
    ("rtol 1e-8, cap 1000, precond", 1e-8, 1000, 0),
]


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
    ap.add_argument("--out", default="gpurun_out/sensitivity.json")
    a = ap.parse_args()
    build.build()
    mu = {c["config"]: c["exact"]["mu_star"] for c in json.load(open(os.path.join(ROOT, "profiles", "r01_quality.json")))
          if "exact" in c}[2]
    spec = gen.config2()
    stream = torch.cuda.current_stream().cuda_stream
    comm = I.comm_desc(1, 0, 0, None, stream)
    out = {"config2": [], "config5": []}
    for name, rtol, cap, norm in POLICIES:
        opts = I.options(T=50, cg_rtol=rtol, cg_max_iter=cap, cg_norm=norm)
        m = I.MinCut.from_spec(spec, opts, comm)
        m.irls_solve(I.IRLS_FROM_SCRATCH, T=50, reports=False)  # graph build
        (reps, tot), ms = timed(lambda: m.irls_solve(I.IRLS_FROM_SCRATCH, T=50))
        (_, _, k, cut), ms2 = timed(lambda: m.irls_sweep_cut(side=False))
        _, tl = m.irls_two_level_cut(side=False)
        its = [r["cg_iters"] for r in reps]
        freeze = next((i for i in range(1, len(its)) if its[i] == 0), None)
        r = {"policy": name, "rtol": rtol, "cap": cap, "norm": "unpreconditioned" if norm else "preconditioned",
             "cg_iters": tot, "per_step": its[:16], "freezes_at_solve": freeze, "time_to_cut_ms": ms + ms2,
             "sweep_cut": cut, "delta_sweep": (cut - mu) / mu, "two_level_cut": tl["cut_value"],
             "delta_two_level": (tl["cut_value"] - mu) / mu, "x_min": reps[-1]["x_min"] if "x_min" in reps[-1] else None}
        print(json.dumps(r), flush=True)
        out["config2"].append(r)
        # config 5: warm sequence (IRLS_CONTINUE) vs cold (FROM_SCRATCH) per problem
        mc = I.MinCut.from_spec(spec, opts, comm)
        cs, ct = spec["cs"].copy(), spec["ct"].copy()
        warm_it = cold_it = 0
        warm_ms = cold_ms = 0.0
        per = []
        for fs, ft in gen.config5_factors(cs.shape[0], n_problems=10, seed=4):
            cs, ct = cs * fs, ct * ft
            m.irls_set_terminal_weights(cs, ct)
            (_, tw), t1 = timed(lambda: m.irls_solve(I.IRLS_CONTINUE, T=50, reports=False))
            mc.irls_set_terminal_weights(cs, ct)
            (_, tc), t2 = timed(lambda: mc.irls_solve(I.IRLS_FROM_SCRATCH, T=50, reports=False))
            warm_it += tw
            cold_it += tc
            warm_ms += t1
            cold_ms += t2
            per.append((tw, tc))
        _, _, kw, cw = m.irls_sweep_cut(side=False)
        _, _, kc, cc = mc.irls_sweep_cut(side=False)
        r5 = {"policy": name, "warm_cg_iters": warm_it, "cold_cg_iters": cold_it, "warm_ms": warm_ms,
              "cold_ms": cold_ms, "per_problem_warm_cold": per, "warm_cut": cw, "cold_cut": cc}
        print(json.dumps(r5), flush=True)
        out["config5"].append(r5)
        m.close()
        mc.close()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
