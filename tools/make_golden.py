"""Write the oracle's full-size trajectories as golden digests (tests/golden/).

Imports only oracle/ (the float64 CPU oracle, test infrastructure) and
synthetic/ (seeded inputs): no value here comes from the CUDA path.  The GPU
suite (tests/test_gpu_fullsize.py) compares the library against these files,
so the driver's `-m gpu` run checks BASELINE's full sizes without paying the
oracle's minutes of host time.

Per solve l the file holds every report field (floats as exact hex strings)
and the SHA-256 of x^(l) as little-endian float64 bytes; per sweep k, the cut
value (hex), and the SHA-256 of side[] (uint8) and of order[] (int32).

Policy (DESIGN A9/A10, the bench's): eps 1e-6, T = 50, rtol 1e-3,
preconditioned norm, cap 50, warm start.

usage: python tools/make_golden.py config4 config5 config3 [--threads N]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from synthetic import generators as gen  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
POLICY = dict(eps=1e-6, T=50, cg_rtol=1e-3, cg_max_iter=50, cg_norm=0, warm_start=True)


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def rep_json(r: dict) -> dict:
    return {k: (v.hex() if isinstance(v, float) else int(v)) for k, v in r.items()}


def sweep_json(S) -> dict:
    sw = S.sweep()
    return dict(k=int(sw.k), cut_value=float(sw.cut_value).hex(), side_sha256=sha(sw.side.astype(np.uint8)),
                order_sha256=sha(sw.order.astype(np.int32)))


def trajectory(spec, name, note):
    t0 = time.perf_counter()
    S = oracle.Solver(oracle.Graph(spec), **POLICY)
    solves = []
    for l in range(POLICY["T"] + 1):
        r = S.init() if l == 0 else S.step()
        solves.append(dict(l=l, report=rep_json(r), x_sha256=sha(S.x())))
        print(f"{name}: solve {l} cg_iters {r['cg_iters']} ({time.perf_counter() - t0:.0f} s)", flush=True)
    out = dict(config=name, note=note, policy=POLICY, n=int(S.n), solves=solves, sweep=sweep_json(S),
               total_cg_iters=sum(s["report"]["cg_iters"] for s in solves),
               oracle_seconds=round(time.perf_counter() - t0, 1), oracle_threads=oracle.set_num_threads(0))
    return out


def config5():
    """A19: config 2, then 10 problems with cumulative U[0.99,1.01] factors on
    cs and ct; each continues from the previous x^(T) (IRLS_CONTINUE)."""
    t0 = time.perf_counter()
    spec = gen.config2()
    S = oracle.Solver(oracle.Graph(spec), **POLICY)
    base = [rep_json(S.init())] + [rep_json(S.step()) for _ in range(POLICY["T"])]
    problems = [dict(problem=0, reports=base, x_sha256=sha(S.x()), sweep=sweep_json(S))]
    cs, ct = spec["cs"].copy(), spec["ct"].copy()
    for i, (fs, ft) in enumerate(gen.config5_factors(cs.shape[0], n_problems=10, seed=4), start=1):
        cs, ct = cs * fs, ct * ft
        S.set_terminal_weights(cs, ct)
        reps = [rep_json(S.step()) for _ in range(POLICY["T"])]
        problems.append(dict(problem=i, reports=reps, x_sha256=sha(S.x()), sweep=sweep_json(S)))
        print(f"config5: problem {i} cg_iters {sum(r['cg_iters'] for r in reps)} "
              f"({time.perf_counter() - t0:.0f} s)", flush=True)
    return dict(config="config5", note="BASELINE configs[4]: config 2 + 10 cumulative terminal-weight problems "
                "(A19), each IRLS_CONTINUE with T = 50 from the previous x^(T)", policy=POLICY,
                n=int(S.n), problems=problems, oracle_seconds=round(time.perf_counter() - t0, 1),
                oracle_threads=oracle.set_num_threads(0))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+", choices=["config2", "config3", "config4", "config5"])
    ap.add_argument("--threads", type=int, default=0)
    a = ap.parse_args()
    oracle.set_num_threads(a.threads)
    for c in a.configs:
        if c == "config5":
            out = config5()
        else:
            spec = getattr(gen, c)()
            out = trajectory(spec, c, {"config2": "BASELINE configs[1]: 128^3 blob grid, seed 1",
                                       "config3": "BASELINE configs[2]: 4900^2 road-like CSR, seed 2",
                                       "config4": "BASELINE configs[3]: 512x512x256 blob grid, seed 3"}[c])
        path = os.path.join(GOLD, f"{c}_trajectory.json")
        with open(path, "w") as f:
            json.dump(out, f, indent=1)
            f.write("\n")
        print("wrote", path, flush=True)


if __name__ == "__main__":
    main()
