"""Time the GPU sweep cut (O7) on a BASELINE config after a full
irls_solve: CUDA events around irls_sweep_cut (host round trip for the digit
histograms included), median of --reps.

usage: python tools/sweep_time.py [--config 4] [--reps 7]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1501_03105_b200 import build, irls as I  # noqa: E402
from synthetic import generators as gen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--reps", type=int, default=7)
    a = ap.parse_args()
    build.build()
    spec = {2: gen.config2, 3: gen.config3, 4: gen.config4}[a.config]()
    stream = torch.cuda.current_stream()
    m = I.MinCut.from_spec(spec, I.options(T=50), I.comm_desc(1, 0, 0, None, stream.cuda_stream))
    m.irls_solve(I.IRLS_FROM_SCRATCH, T=50, reports=False)
    m.irls_sweep_cut(side=False)
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        _, _, k, cut = m.irls_sweep_cut(side=False)
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(json.dumps({"config": a.config, "sweep_ms_median": statistics.median(ts), "sweep_ms": ts, "k": k,
                      "cut": cut, "launches": m.irls_get_stats()["launches"],
                      "sorted": m.irls_get_stats()["sweep_sorted"]}))


if __name__ == "__main__":
    main()
