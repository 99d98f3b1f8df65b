"""Degenerate and edge inputs through the C ABI against the oracle: no
non-terminal at all (only s, t and a direct edge), a single non-terminal,
b = 0 (no source links: v = 0), s and t disconnected (A8: allowed,
cut = c_st), a graph whose every n-link is absent (c = 0, A6), and a grid
with one plane / one row."""
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


def both(I, spec, T=5, **kw):
    m = I.MinCut.from_spec(spec, I.options(T=T, **kw))
    reps, tot = m.irls_solve(I.IRLS_FROM_SCRATCH, T=T)
    S = oracle.Solver(oracle.Graph(spec), T=T, **{k: v for k, v in kw.items() if k in ("cg_rtol", "cg_max_iter")})
    _, oreps = S.run(record=False)
    for a, b in zip(reps, oreps):
        assert (a["cg_iters"], a["converged"], a["rel_res"]) == (b["cg_iters"], b["converged"], b["rel_res"])
    assert np.array_equal(m.irls_get_potentials(), S.x())
    side, _, k, cut = m.irls_sweep_cut()
    sw = S.sweep()
    assert (k, cut) == (sw.k, sw.cut_value) and np.array_equal(side, sw.side)
    tside, tl = m.irls_two_level_cut()
    otl = S.two_level()
    assert tl["cut_value"] == otl.cut_value and np.array_equal(tside, otl.side)
    return m, S


def test_no_nonterminals(irls):
    """Only s - t (direct edge c_st = 3): every cut is {s}, value 3; lambda_2
    of a single edge is 1."""
    spec = gen._csr_edges(2, [(0, 1, 3.0)], 0, 1)
    m, S = both(irls, spec)
    r = m.irls_lambda2()
    assert r["lambda2"] == 1.0 and r["lambda2"] == S.lambda2()[0]


def test_single_nonterminal(irls):
    spec = gen._csr_edges(3, [(0, 1, 2.0), (1, 2, 1.0), (0, 2, 0.25)], 0, 2)
    both(irls, spec, T=10, cg_rtol=1e-12, cg_max_iter=100)


def test_zero_rhs(irls):
    """No source links: b = 0, so every solve returns v = 0 and the
    sweep keeps S = {s}."""
    spec = gen.uniform_grid(8, 6, seed=3)
    spec["cs"] = np.zeros_like(spec["cs"])
    m, S = both(irls, spec)
    assert not m.irls_get_potentials().any()


def test_disconnected_terminals(irls):
    """s and t in different components (each touches a terminal edge): the
    cut is c_st = 0 (A8)."""
    spec = gen._csr_edges(6, [(0, 1, 1.0), (1, 2, 2.0), (3, 4, 1.5), (4, 5, 1.0)], 0, 5)
    m, S = both(irls, spec, T=5, cg_rtol=1e-12, cg_max_iter=100)
    _, _, _, cut = m.irls_sweep_cut(side=False)
    assert cut == 0.0


def test_all_nlinks_absent(irls):
    """Every n-link c = 0 (A6): independent two-edge paths per node."""
    spec = gen.zero_nlink_grid(16, 12, 3, seed=2)
    both(irls, spec, T=8)


@pytest.mark.parametrize("dims", [(64, 1, 1), (1, 64, 1), (2, 2, 64), (512, 1, 1)])
def test_thin_grids(irls, dims):
    spec = gen.blob_grid(*dims, seed=9, sigma=(1.0, 3.0))
    both(irls, spec, T=6)


def test_csr_terminal_update_singular(irls):
    """A8 at irls_set_terminal_weights on a CSR graph: removing the last
    terminal edge of a component is rejected (IRLS_ERR_SINGULAR), as the
    oracle's nonsingularity check rejects that graph."""
    spec = gen._csr_edges(6, [(0, 1, 1.0), (1, 2, 2.0), (3, 4, 1.5), (4, 5, 1.0)], 0, 5)
    m = irls.MinCut.from_spec(spec, irls.options(T=3))
    m.irls_solve(irls.IRLS_FROM_SCRATCH, T=3)
    cs, ct = oracle.Graph(spec).terminals()
    bad_cs, bad_ct = cs.copy(), ct.copy()
    bad_cs[0] = 0.0  # node 1 (reduced 0) loses its s-link: component {1, 2} keeps no anchor
    with pytest.raises(irls.IrlsError) as e:
        m.irls_set_terminal_weights(bad_cs, bad_ct)
    assert e.value.code == 5
    m.irls_set_terminal_weights(cs * 2.0, ct * 3.0)  # still anchored: accepted


def test_stencil_terminal_update_singular_leaves_context_intact(irls):
    """A8 at irls_set_terminal_weights on a grid: a rejected
    update (IRLS_ERR_SINGULAR) must not reach the device.  The next
    IRLS_CONTINUE solve runs on the previous weights, bitwise as the oracle
    continuing without the update."""
    spec = gen.zero_nlink_grid(8, 8, 1, seed=4)   # every pixel its own component (pin (iii))
    T = 3
    m = irls.MinCut.from_spec(spec, irls.options(T=T))
    m.irls_solve(irls.IRLS_FROM_SCRATCH, T=T)
    S = oracle.Solver(oracle.Graph(spec), T=T)
    S.run(record=False)
    bad_cs, bad_ct = spec["cs"].copy(), spec["ct"].copy()
    bad_cs[5] = 0.0
    bad_ct[5] = 0.0                                  # pixel 5 loses both terminal edges: singular
    with pytest.raises(irls.IrlsError) as e:
        m.irls_set_terminal_weights(bad_cs, bad_ct)
    assert e.value.code == 5
    m.irls_solve(irls.IRLS_CONTINUE, T=T)
    for _ in range(T):
        S.step()
    assert np.array_equal(m.irls_get_potentials(), S.x())
    side, _, k, cut = m.irls_sweep_cut()
    sw = S.sweep()
    assert k == sw.k and cut == sw.cut_value and np.array_equal(side, sw.side)
    m.close()


def test_solve_T_must_match_options(irls):
    """irls_solve runs irls_options.T steps; the binding sizes the report
    buffer from the context and refuses a different T (a smaller one used
    to size the host buffer too small)."""
    spec = gen.blob_grid(16, 12, 4, seed=3)
    m = irls.MinCut.from_spec(spec, irls.options(T=5))
    with pytest.raises(ValueError):
        m.irls_solve(irls.IRLS_FROM_SCRATCH, T=4)
    reps, _ = m.irls_solve(irls.IRLS_FROM_SCRATCH)
    assert len(reps) == 6
    m.close()
