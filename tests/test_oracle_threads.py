"""The oracle's OpenMP loops ("OpenMP over C3 chunks") do not
change a bit: 1 thread and many threads give identical x^(l), reports, sweep,
two-level and lambda_2 outputs (CPU only)."""
import os

import numpy as np
import pytest

import oracle
from synthetic import generators as gen


def _run(spec, threads, variant=0):
    oracle.set_num_threads(threads)
    S = oracle.Solver(oracle.Graph(spec), T=6, cg_variant=variant)
    xs, reps = S.run()
    sw = S.sweep()
    tl = S.two_level()
    lam = S.lambda2(rtol=1e-6, max_iter=500)
    return xs, reps, sw, tl, lam


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("kind", ["stencil", "csr"])
def test_thread_count_is_bitwise_invisible(kind, variant):
    spec = gen.blob_grid(64, 48, 12, seed=9, sigma=(3.0, 9.0))   # 36,864 nodes = 9 chunks (ragged groups)
    if kind == "csr":
        spec = gen.stencil_to_csr(spec)
    many = max(4, os.cpu_count() or 4)
    try:
        a = _run(spec, 1, variant)
        b = _run(spec, many, variant)
    finally:
        oracle.set_num_threads(os.cpu_count() or 1)
    assert np.array_equal(a[0].view(np.uint64), b[0].view(np.uint64))
    assert a[1] == b[1]
    assert a[2].k == b[2].k and a[2].cut_value == b[2].cut_value and np.array_equal(a[2].order, b[2].order)
    assert a[3].cut_value == b[3].cut_value and np.array_equal(a[3].side, b[3].side)
    assert a[4] == b[4]
