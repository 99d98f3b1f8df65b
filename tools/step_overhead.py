"""Where the time of a zero-iteration IRLS step goes (config 4 after the
fixed point): one irls_step (its own graph: K1 -> WHILE(0) -> finish ->
report), K1 alone (irls_time_kernel), and the per-step time inside the
multi-step graph (report timestamps; ms_assemble = previous report -> end of
the assembly).  usage: python tools/step_overhead.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1501_03105_b200 import build, irls as I  # noqa: E402
from synthetic import generators as gen  # noqa: E402

build.build()
spec = gen.config4()
for lm in (0, 1):
    m = I.MinCut.from_spec(spec, I.options(T=50, loop_mode=lm))
    reps, _ = m.irls_solve(I.IRLS_FROM_SCRATCH, T=50)
    reps, _ = m.irls_solve(I.IRLS_FROM_SCRATCH, T=50)
    zero = [r["ms"] for r in reps[1:] if r["cg_iters"] == 0]
    if lm == 0:
        za = [r["ms_assemble"] for r in reps[1:] if r["cg_iters"] == 0]
        one = [(r["ms"], r["ms_assemble"]) for r in reps[1:] if r["cg_iters"] == 1]
        print(f"graph: zero-iteration steps: previous end -> assembly end {sum(za) / max(len(za), 1):.3f} ms, "
              f"-> report {sum(zero) / max(len(zero), 1):.3f} ms; one-iteration steps (ms, ms_assemble): {one[:3]}",
              flush=True)
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    n = 10
    for _ in range(n):
        r = m.irls_step()
    e1.record(s)
    torch.cuda.synchronize()
    k1 = m.irls_time_kernel(I.KERNEL_ASSEMBLE, 10)
    print(f"loop_mode {lm}: zero-iteration steps in irls_solve {sum(zero) / max(len(zero), 1):.3f} ms "
          f"({len(zero)} steps); irls_step {e0.elapsed_time(e1) / n:.3f} ms (host-timed incl. report copy); "
          f"K1 alone {k1:.3f} ms", flush=True)
    m.close()
