"""Per-kernel timing on a solved state (CUDA events via irls_time_kernel)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="config4")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--solves", type=int, default=2)
args = ap.parse_args()
from paper_1501_03105_b200 import build, irls as I  # noqa: E402
from synthetic import generators as gen  # noqa: E402

build.build()
spec = getattr(gen, args.config)()
m = I.MinCut.from_spec(spec, I.options(T=50))
st = m.irls_get_stats()
n = st["n_local"]
csr = spec["kind"] == "csr"
import torch  # noqa: E402
for i in range(args.solves):
    torch.cuda.synchronize()
    t = time.perf_counter()
    reps, tot = m.irls_solve(I.IRLS_FROM_SCRATCH, T=50, reports=True)
    t1 = time.perf_counter()
    m.irls_sweep_cut(side=False)
    t2 = time.perf_counter()
    print(f"solve {1e3 * (t1 - t):.1f} ms sweep {1e3 * (t2 - t1):.1f} ms cg_iters={tot}")
ent = 2 * st["n_links"]
for name, w, b in (("K3 pspmv", 0, 80), ("K5 axpy", 1, 40), ("K1 assemble", 2, 104)):
    ms = m.irls_time_kernel(w, args.reps)
    if csr:  # K3 56 B/node + 12 B/entry; K1 56 B/node + 20 B/entry
        by = {0: 56 * n + 12 * ent, 1: 40 * n, 2: 56 * n + 20 * ent}[w]
        print(f"{name:12s} {ms:.4f} ms  {by / ms / 1e6:.0f} GB/s (algorithmic {by / 1e9:.3f} GB)")
    else:
        print(f"{name:12s} {ms:.4f} ms  {b * n / ms / 1e6:.0f} GB/s (algorithmic {b} B/node)")
