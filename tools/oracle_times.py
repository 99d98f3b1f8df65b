"""Time-to-cut of the float64 CPU oracle (single thread, as it stands) on the
BASELINE configs, on this host — the "oracle timed beside it" of SURVEY §8(d).
usage: python tools/oracle_times.py [--configs 1,2,3,4]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from synthetic import generators as gen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="1,2,3,4")
ap.add_argument("--out", default="gpurun_out/oracle_times.json")
args = ap.parse_args()
oracle.build()
res = []
for cid in [int(c) for c in args.configs.split(",")]:
    spec = {1: gen.config1, 2: gen.config2, 3: gen.config3, 4: gen.config4}[cid]()
    kw = dict(cg_rtol=1e-10, cg_max_iter=100000, cg_norm=1) if cid == 1 else {}
    G = oracle.Graph(spec)
    S = oracle.Solver(G, T=50, **kw)
    t0 = time.perf_counter()
    _, reps = S.run(record=False)
    t1 = time.perf_counter()
    sw = S.sweep()
    t2 = time.perf_counter()
    iters = sum(r["cg_iters"] for r in reps)
    r = {"config": cid, "nodes": G.n, "n_links": G.nnz // 2, "cg_iters": iters, "solve_s": t1 - t0,
         "sweep_s": t2 - t1, "time_to_cut_s": t2 - t0, "GEdge_s": G.nnz // 2 * iters / (t2 - t0) / 1e9,
         "cut": sw.cut_value, "threads": 1, "host_cores": os.cpu_count()}
    print(json.dumps(r), flush=True)
    res.append(r)
    del S, G
os.makedirs(os.path.dirname(args.out), exist_ok=True)
json.dump(res, open(args.out, "w"), indent=1)
