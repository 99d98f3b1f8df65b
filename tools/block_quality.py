"""Block-Jacobi preconditioning (A32; P:L235-242,
P:L365) at the paper's policy (rtol 1e-3 preconditioned, cap 50, T = 50,
warm): per block size B (0 = point Jacobi), total CG iterations, time-to-cut
(irls_solve + sweep, CUDA events), per-kernel times of the factor / apply /
reduce and the K3 SpMV (launch list from irls_time_kernel is not used: the
solve graph is timed whole), and the cut quality delta = (mu - mu*) / mu*
(Eq. 13) of the sweep and of the two-level rounding, mu* from
profiles/r01_quality.json (irls_exact_min_cut, certified exact max-flow).

usage: python tools/block_quality.py [--config 3] [--blocks 0,16,64,256] [--out gpurun_out/blocks.json]
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


def timed(fn, reps=1):
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(reps):
        out = fn()
    e1.record(s)
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--blocks", default="0,16,64,256")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default="gpurun_out/blocks.json")
    a = ap.parse_args()
    build.build()
    spec = {2: gen.config2, 3: gen.config3, 4: gen.config4}[a.config]()
    mu = {c["config"]: c["exact"]["mu_star"] for c in json.load(open(os.path.join(ROOT, "profiles", "r01_quality.json")))
          if "exact" in c}.get(a.config)
    stream = torch.cuda.current_stream().cuda_stream
    out = []
    for B in [int(b) for b in a.blocks.split(",")]:
        m = I.MinCut.from_spec(spec, I.options(T=50, block_size=B), I.comm_desc(1, 0, 0, None, stream))
        m.irls_solve(I.IRLS_FROM_SCRATCH, T=50, reports=False)  # warm-up (graph build)

        def step():
            reps, tot = m.irls_solve(I.IRLS_FROM_SCRATCH, T=50)
            _, _, k, cut = m.irls_sweep_cut(side=False)
            return reps, tot, cut
        (reps, tot, cut), ms = timed(step, a.reps)
        _, tl = m.irls_two_level_cut(side=False)
        n_links = m.irls_get_stats()["n_links"]
        r = {"block_size": B, "cg_iters": tot, "per_step": [x["cg_iters"] for x in reps][:12],
             "time_to_cut_ms": ms, "gedge_s": n_links * tot / (ms * 1e-3) / 1e9,
             "sweep_cut": cut, "two_level_cut": tl["cut_value"], "two_level_nc": tl["nc"],
             "two_level_ms": tl["ms_total"]}
        if mu:
            r["mu_star"] = mu
            r["delta_sweep"] = (cut - mu) / mu
            r["delta_two_level"] = (tl["cut_value"] - mu) / mu
        print(json.dumps(r), flush=True)
        out.append(r)
        m.close()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
