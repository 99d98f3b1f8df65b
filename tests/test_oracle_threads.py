"""The oracle's OpenMP loops ("OpenMP over C3 chunks") do not
change a bit: 1 thread and many threads give identical x^(l), reports, sweep
and lambda_2 outputs, with point and block Jacobi (CPU only).  The graph is
large enough (18 chunks, 73,728 nodes) for every parallel loop to run
threaded."""
import os

import numpy as np
import pytest

import oracle
from synthetic import generators as gen


def _run(spec, threads, variant=0, block_size=0):
    oracle.set_num_threads(threads)
    S = oracle.Solver(oracle.Graph(spec), T=6, cg_variant=variant, block_size=block_size)
    xs, reps = S.run()
    sw = S.sweep()
    lam = S.lambda2(rtol=1e-6, max_iter=40)
    return xs, reps, sw, lam


@pytest.mark.parametrize("variant,block_size", [(0, 0), (1, 0), (0, 64)])
@pytest.mark.parametrize("kind", ["stencil", "csr"])
def test_thread_count_is_bitwise_invisible(kind, variant, block_size):
    spec = gen.blob_grid(64, 96, 12, seed=9, sigma=(3.0, 9.0))   # 73,728 nodes = 18 chunks (ragged groups)
    if kind == "csr":
        spec = gen.stencil_to_csr(spec)
    many = max(4, os.cpu_count() or 4)
    try:
        a = _run(spec, 1, variant, block_size)
        b = _run(spec, many, variant, block_size)
    finally:
        oracle.set_num_threads(os.cpu_count() or 1)
    assert np.array_equal(a[0].view(np.uint64), b[0].view(np.uint64))
    assert a[1] == b[1]
    assert a[2].k == b[2].k and a[2].cut_value == b[2].cut_value and np.array_equal(a[2].order, b[2].order)
    assert a[3] == b[3]
