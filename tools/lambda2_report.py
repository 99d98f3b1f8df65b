"""The Cheeger-type diagnostic on the BASELINE
configs: lambda_2 by one cold Jacobi-PCG solve of the (1, -1) system, its CG
iterations and device time, and Theorem 4's sandwich phi^2/2 <= lambda_2 <=
2 phi with phi = mu* / C (mu* from profiles/r01_quality.json).
usage: python tools/lambda2_report.py [--configs 1,2,3,4] [--rtol 1e-8]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1501_03105_b200 import build, irls as I  # noqa: E402
from synthetic import generators as gen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="1,2,3,4")
ap.add_argument("--rtol", type=float, default=1e-8)
ap.add_argument("--cap", type=int, default=20000)
ap.add_argument("--out", default="gpurun_out/lambda2.json")
args = ap.parse_args()
build.build()
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
mu = {}
try:
    for e in json.load(open(os.path.join(root, "profiles", "r01_quality.json"))):
        mu[e["config"]] = e["exact"]["mu_star"]
except Exception:
    pass
out = []
for cfg in [int(c) for c in args.configs.split(",")]:
    spec = {1: gen.config1, 2: gen.config2, 3: gen.config3, 4: gen.config4}[cfg]()
    m = I.MinCut.from_spec(spec, I.options(T=1))
    t0 = time.perf_counter()
    r = m.irls_lambda2(cg_rtol=args.rtol, cg_max_iter=args.cap, cg_norm=I.IRLS_NORM_UNPRECONDITIONED)
    wall = time.perf_counter() - t0
    e = {"config": cfg, "lambda2": r["lambda2"], "xLx": r["xLx"], "C": r["C"], "cg_iters": r["cg_iters"],
         "converged": r["converged"], "rel_res": r["rel_res"], "ms_solve": r["ms"], "wall_s": wall,
         "rtol": args.rtol}
    if cfg in mu:
        phi = mu[cfg] / r["C"]
        e.update({"mu_star": mu[cfg], "phi": phi, "cheeger_lower": phi * phi / 2, "cheeger_upper": 2 * phi,
                  "sandwich_holds": bool(phi * phi / 2 <= r["lambda2"] <= 2 * phi)})
    print(json.dumps(e), flush=True)
    out.append(e)
    m.close()
os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
json.dump(out, open(args.out, "w"), indent=1)
