"""Per-solve device times (CUDA events around each graph launch, from the
step reports) next to the kernel-only estimate, to expose launch/graph
overhead per solve.  usage: python tools/step_times.py [--config config4]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="config4")
args = ap.parse_args()
from paper_1501_03105_b200 import build, irls as I  # noqa: E402
from synthetic import generators as gen  # noqa: E402

build.build()
spec = getattr(gen, args.config)()
m = I.MinCut.from_spec(spec, I.options(T=50))
for _ in range(2):
    reps, tot = m.irls_solve(I.IRLS_FROM_SCRATCH, T=50)
k3 = m.irls_time_kernel(I.KERNEL_PSPMV, 10)
k5 = m.irls_time_kernel(I.KERNEL_AXPY, 10)
k1 = m.irls_time_kernel(I.KERNEL_ASSEMBLE, 10)
print(f"K3 {k3:.4f} K5 {k5:.4f} K1 {k1:.4f} ms")
tot_ms = sum(r["ms"] for r in reps)
est = sum(k1 + r["cg_iters"] * (k3 + k5) for r in reps[1:])
print(f"sum of per-solve ms {tot_ms:.2f}; kernel estimate (steps 1..50) {est:.2f}; init solve {reps[0]['ms']:.2f} ms "
      f"({reps[0]['cg_iters']} iters)")
for i, r in enumerate(reps[:14]):
    print(i, r["cg_iters"], f"{r['ms']:.3f} ms", f"est {k1 + r['cg_iters'] * (k3 + k5):.3f}")
