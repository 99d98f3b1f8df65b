"""The branch-and-bound sweep (sweep_bb.cu; DESIGN.md §6 sweep row): when the
caller does not ask for the order, graphs with n~ >= 2^20 find k (the first
minimiser of the exact prefix sequence P_i, A15), the cut value and side[]
from bucket sums and a sort of the candidate buckets only.  Against the
oracle's full sort (orc_sweep on the same potentials) and the library's own
full path (IRLS_SWEEP_FULL=1): k, cut value and side[] bitwise, on
  - solved potentials (config 2 after a short solve: the pruning case),
  - potentials with massive ties (a handful of distinct values; ties are
    ordered by ascending id, A14), all-equal potentials (one key),
  - i.i.d. uniform potentials (no structure: the bound prunes little and the
    path may fall back to the full sort — still the same result),
  - minimum at position 0 or n (the empty set / all non-terminals),
  - a CSR graph over 2^20 nodes (SELL sweep kernels),
and NaN potentials fail with IRLS_ERR_BAD_POTENTIAL on this path too."""
import os

import numpy as np
import pytest

import oracle
from synthetic import generators as gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def irls():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1501_03105_b200 import build, irls as I
    build.build()
    return I


@pytest.fixture(scope="module")
def shared(irls):
    spec = gen.blob_grid(128, 128, 64, seed=11)
    return spec, oracle.Solver(oracle.Graph(spec), T=4)


@pytest.fixture
def grid(irls, shared):
    """A 128x128x64 blob grid (n~ = 2^20): a fresh GPU context per test (a
    sweep whose bound prunes too little makes the context skip the attempt
    for its next sweeps) and an oracle solver over the same graph (the oracle
    only sweeps given potentials)."""
    spec, S = shared
    m = irls.MinCut.from_spec(spec, irls.options(T=4))
    yield spec, m, S
    m.close()


def _full(m):
    os.environ["IRLS_SWEEP_FULL"] = "1"
    try:
        side, _, k, cut = m.irls_sweep_cut(side=True)
        assert m.irls_get_stats()["sweep_sorted"] == m.n
        return side, k, cut
    finally:
        os.environ.pop("IRLS_SWEEP_FULL", None)


def _check(m, S, x, expect_bb=True):
    m.irls_set_potentials(x)
    side, _, k, cut = m.irls_sweep_cut(side=True)
    sorted_nodes = m.irls_get_stats()["sweep_sorted"]
    if expect_bb:
        assert sorted_nodes < m.n // 4, sorted_nodes
    sw = S.sweep(x)
    assert k == sw.k, (k, sw.k)
    assert float(cut).hex() == float(sw.cut_value).hex(), (cut, sw.cut_value)
    assert np.array_equal(side, sw.side)
    fs, fk, fc = _full(m)
    assert fk == k and float(fc).hex() == float(cut).hex() and np.array_equal(fs, side)
    # order=True always takes the full sort and agrees
    _, order, k2, c2 = m.irls_sweep_cut(side=False, order=True)
    assert k2 == k and c2 == cut and np.array_equal(order.astype(np.int64), sw.order)
    return sorted_nodes


def test_solved_potentials(irls, grid):
    spec, m, S = grid
    assert m.n >= 1 << 20
    m.irls_solve(irls.IRLS_FROM_SCRATCH, T=4, reports=False)
    x = m.irls_get_potentials()
    _check(m, S, x)


@pytest.mark.parametrize("levels", [1, 2, 5])
def test_ties(irls, grid, levels):
    spec, m, S = grid
    rng = np.random.default_rng(levels)
    vals = np.linspace(0.0, 1.0, levels)
    x = vals[rng.integers(0, levels, m.n)]
    _check(m, S, x, expect_bb=False)


def test_ties_on_solved(irls, grid):
    """Solved potentials rounded to 3 digits: long runs of equal keys inside
    the candidate buckets (ties leave in ascending id)."""
    spec, m, S = grid
    m.irls_solve(irls.IRLS_FROM_SCRATCH, T=4, reports=False)
    x = np.round(m.irls_get_potentials(), 3)
    assert len(np.unique(x)) < 1100
    _check(m, S, x, expect_bb=True)


def test_skip_after_failed_pruning(irls, grid):
    """When the bound prunes too little (here: a limit of 1000 candidate
    nodes), the sweep falls back to the full sort and the next 8 sweeps skip
    the attempt; then it tries again."""
    spec, m, S = grid
    m.irls_solve(irls.IRLS_FROM_SCRATCH, T=4, reports=False)
    xs = m.irls_get_potentials()
    os.environ["IRLS_SWEEP_BB_MAX"] = "1000"
    try:
        k0 = m.irls_sweep_cut(side=False)[2]
    finally:
        os.environ.pop("IRLS_SWEEP_BB_MAX", None)
    assert m.irls_get_stats()["sweep_sorted"] == m.n
    for i in range(9):
        k = m.irls_sweep_cut(side=False)[2]
        if i < 8:
            assert m.irls_get_stats()["sweep_sorted"] == m.n
    assert 0 < m.irls_get_stats()["sweep_sorted"] < m.n // 4
    assert k == k0 == S.sweep(xs).k


def test_uniform_random(irls, grid):
    spec, m, S = grid
    x = np.random.default_rng(5).random(m.n)
    _check(m, S, x, expect_bb=False)


@pytest.mark.parametrize("val", [0.0, 1.0])
def test_extreme_ends(irls, grid, val):
    """x = 1 everywhere except a few nodes: with huge source-side weights the
    first minimum can sit at position 0 or n."""
    spec, m, S = grid
    x = np.full(m.n, val)
    x[::4099] = 1.0 - val
    _check(m, S, x, expect_bb=False)


def test_nan(irls, grid):
    spec, m, S = grid
    x = np.zeros(m.n)
    x[12345] = np.nan
    m.irls_set_potentials(x)
    with pytest.raises(irls.IrlsError) as e:
        m.irls_sweep_cut(side=False)
    assert irls.STATUS_NAMES[e.value.code] == "IRLS_ERR_BAD_POTENTIAL"
    # the context stays usable
    _check(m, S, np.linspace(0.0, 1.0, m.n)[::-1].copy(), expect_bb=False)


def test_csr_over_2e20(irls):
    g = gen.blob_grid(128, 96, 96, seed=3)  # 1.18M nodes, as a CSR graph
    spec = gen.stencil_to_csr(g)
    m = irls.MinCut.from_spec(spec, irls.options(T=3))
    S = oracle.Solver(oracle.Graph(spec), T=3)
    assert m.n >= 1 << 20
    m.irls_solve(irls.IRLS_FROM_SCRATCH, T=3, reports=False)
    _check(m, S, m.irls_get_potentials())
    m.close()
