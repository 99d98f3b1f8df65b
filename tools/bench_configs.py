"""Measure every BASELINE config on one GPU (time-to-cut, CG iterations,
GEdge/s, per-kernel times) and write a JSON summary.

usage: python tools/bench_configs.py [--configs 1,2,3,4,5] [--out gpurun_out/configs.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
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


def run_config(cid, reps=3):
    t0 = time.perf_counter()
    if cid == 1:
        spec, opts = gen.config1(), I.options(T=50, cg_rtol=1e-10, cg_max_iter=100000, cg_norm=1)
    elif cid in (2, 5):
        spec, opts = gen.config2(), I.options(T=50)
    elif cid == 3:
        spec, opts = gen.config3(), I.options(T=50)
    else:
        spec, opts = gen.config4(), I.options(T=50)
    t_gen = time.perf_counter() - t0
    stream = torch.cuda.current_stream().cuda_stream
    comm = I.comm_desc(1, 0, 0, None, stream)
    t0 = time.perf_counter()
    m = I.MinCut.from_spec(spec, opts, comm)
    torch.cuda.synchronize()
    t_create = time.perf_counter() - t0
    st = m.irls_get_stats()
    res = {"config": cid, "kind": spec["kind"], "nodes": st["n_nonterminal"], "n_links": st["n_links"],
           "gen_s": t_gen, "create_s": t_create}
    if cid == 5:
        # warm-started sequence vs cold starts (A19)
        cs, ct = spec["cs"].copy(), spec["ct"].copy()
        m.irls_solve(I.IRLS_FROM_SCRATCH, T=50, reports=False)
        warm_iters, warm_ms, cold_iters, cold_ms = 0, 0.0, 0, 0.0
        mc = I.MinCut.from_spec(spec, opts, comm)
        for fs, ft in gen.config5_factors(cs.shape[0], n_problems=10, seed=4):
            cs, ct = cs * fs, ct * ft
            m.irls_set_terminal_weights(cs, ct)
            (r, tot), ms = timed(lambda: m.irls_solve(I.IRLS_CONTINUE, T=50, reports=False))
            warm_iters += tot
            warm_ms += ms
            mc.irls_set_terminal_weights(cs, ct)
            (r, tot), ms = timed(lambda: mc.irls_solve(I.IRLS_FROM_SCRATCH, T=50, reports=False))
            cold_iters += tot
            cold_ms += ms
        _, _, k, cut = m.irls_sweep_cut(side=False)
        # the same warm sequence with the exact fixed-point exit
        mf = I.MinCut.from_spec(spec, I.options(T=50, fixed_point_exit=1), comm)
        mf.irls_solve(I.IRLS_FROM_SCRATCH, T=50, reports=False)
        cs, ct = spec["cs"].copy(), spec["ct"].copy()
        fp_iters, fp_ms = 0, 0.0
        for fs, ft in gen.config5_factors(cs.shape[0], n_problems=10, seed=4):
            cs, ct = cs * fs, ct * ft
            mf.irls_set_terminal_weights(cs, ct)
            (r, tot), ms = timed(lambda: mf.irls_solve(I.IRLS_CONTINUE, T=50, reports=False))
            fp_iters += tot
            fp_ms += ms
        _, _, kf, cutf = mf.irls_sweep_cut(side=False)
        mf.close()
        res.update({"warm_total_cg_iters": warm_iters, "warm_ms": warm_ms, "cold_total_cg_iters": cold_iters,
                    "cold_ms": cold_ms, "final_k": k, "final_cut": cut,
                    "warm_fixed_point_exit_ms": fp_ms, "warm_fixed_point_exit_iters": fp_iters,
                    "fixed_point_exit_same_cut": bool(kf == k and cutf == cut)})
        mc.close()
        m.close()
        return res
    m.irls_solve(I.IRLS_FROM_SCRATCH, T=50, reports=False)  # warm-up (graph build)
    m.irls_sweep_cut(side=False)
    times, sweeps = [], []
    for _ in range(reps):
        (reps_, tot), ms = timed(lambda: m.irls_solve(I.IRLS_FROM_SCRATCH, T=50))
        (_, _, k, cut), ms2 = timed(lambda: m.irls_sweep_cut(side=False))
        times.append(ms)
        sweeps.append(ms2)
    ms, ms2 = float(np.median(times)), float(np.median(sweeps))
    res.update({"cg_iters": tot, "per_step_iters": [r["cg_iters"] for r in reps_], "solve_ms": ms,
                "sweep_ms": ms2, "time_to_cut_ms": ms + ms2, "k": k, "cut": cut,
                "GEdge_s_whole": st["n_links"] * tot / ((ms + ms2) * 1e-3) / 1e9})
    n = st["n_local"]
    kt = {}
    for name, w, b in (("K3", 0, None), ("K5", 1, 40), ("K1", 2, None)):
        t = m.irls_time_kernel(w, 10)
        kt[name] = {"ms": t}
        if b:
            kt[name]["GBps_alg"] = b * n / (t * 1e-3) / 1e9
    if spec["kind"] == "stencil":
        kt["K3"]["GBps_alg"] = 80 * n / (kt["K3"]["ms"] * 1e-3) / 1e9
        kt["K1"]["GBps_alg_104"] = 104 * n / (kt["K1"]["ms"] * 1e-3) / 1e9
    else:
        # CSR: K3 reads z,p_old,x,D + (g 8 B + col 4 B) per stored entry; writes p,q,x
        ent = 2 * st["n_links"]
        k3b = 56 * n + 12 * ent
        kt["K3"]["GBps_alg"] = k3b / (kt["K3"]["ms"] * 1e-3) / 1e9
        kt["K3"]["alg_bytes"] = k3b
    res["kernels"] = kt
    m.close()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--out", default="gpurun_out/configs.json")
    args = ap.parse_args()
    build.build()
    out = []
    for c in [int(x) for x in args.configs.split(",")]:
        r = run_config(c)
        print(json.dumps(r), flush=True)
        out.append(r)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(out, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
