"""One IRLS solve + sweep cut on a config, for ncu launch lists / captures.

usage: python tools/profile_step.py [--config config4] [--T 50] [--loop-mode 1] [--cg-variant cg] [--block-size B]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="config4")
ap.add_argument("--T", type=int, default=50)
ap.add_argument("--solves", type=int, default=1)
ap.add_argument("--loop-mode", type=int, default=0)
ap.add_argument("--cg-variant", default="hs", choices=["hs", "cg"])
ap.add_argument("--block-size", type=int, default=0)
args = ap.parse_args()

from paper_1501_03105_b200 import build, irls as I  # noqa: E402
from synthetic import generators as gen  # noqa: E402

build.build()
spec = getattr(gen, args.config)()
m = I.MinCut.from_spec(spec, I.options(T=args.T, loop_mode=args.loop_mode, block_size=args.block_size,
                                      cg_variant=I.IRLS_CG_CG if args.cg_variant == "cg" else I.IRLS_CG_HS))
for _ in range(args.solves):
    t = time.perf_counter()
    reps, tot = m.irls_solve(I.IRLS_FROM_SCRATCH, T=args.T)
    side, order, k, cut = m.irls_sweep_cut(side=False)
    print(f"solve+sweep {1e3 * (time.perf_counter() - t):.1f} ms cg_iters={tot} k={k} cut={cut!r}",
          [r["cg_iters"] for r in reps])
m.close()
