"""Pins of the oracle's Chronopoulos-Gear PCG (O5', A31; SURVEY §8(f) NEXT
#3), CPU only.  Its iterates equal Hestenes-Stiefel's in exact arithmetic,
so everything that pins O5 pins it too, independently of O5's code: SPEC's
worked example, dense library solves of the paper's systems, the IRLS
closed forms, the exact power-of-two scaling, a diagonal system (Jacobi is
exact: one iteration) and b = 0.  Against O5 itself only the Krylov
equivalence is checked (same iteration counts, x within rounding)."""
import json
import os

import mpmath
import numpy as np
import pytest

import oracle
from synthetic import generators as gen
from tests import helpers as H

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
TINY = gen.tiny_graphs()


def solver(spec, **kw):
    return oracle.Solver(oracle.Graph(spec), cg_variant=1, **kw)


def test_spec_path4():
    S = solver(TINY["path4"], cg_rtol=1e-14, cg_max_iter=100)
    S.init()
    np.testing.assert_allclose(S.x(), GOLD["pcg_path4"]["v"], rtol=1e-14)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_init_solve_matches_dense(seed):
    spec = gen.random_small_graph(60, 90, seed=seed)
    n, s, t, E = H.edge_list(spec)
    Lr, b, keep = H.dense_irls_system(n, s, t, E)
    v = np.linalg.solve(Lr, b)
    S = solver(spec, cg_rtol=1e-14, cg_max_iter=10000)
    S.init()
    np.testing.assert_allclose(S.x(), v, rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("seed", [3, 4])
def test_reweighted_step_matches_dense(seed):
    spec = gen.random_small_graph(40, 70, seed=seed)
    n, s, t, E = H.edge_list(spec)
    S = solver(spec, cg_rtol=1e-14, cg_max_iter=10000, eps=1e-4)
    S.init()
    x_prev = np.zeros(n); x_prev[s] = 1.0
    x_prev[np.array([i for i in range(n) if i not in (s, t)])] = S.x()
    Lr, b, keep = H.dense_irls_system(n, s, t, E, x=x_prev, eps=1e-4)
    v = np.linalg.solve(Lr, b)
    S.step()
    np.testing.assert_allclose(S.x(), v, rtol=1e-8, atol=1e-11)


def test_irls_path_T10_closed_form():
    S = solver(TINY["path"], T=10, cg_rtol=1e-14, cg_max_iter=100)
    xs, _ = S.run()
    mpmath.mp.dps = 50
    c1, c2, eps = mpmath.mpf(2), mpmath.mpf(1), mpmath.mpf("1e-6")
    x = c1 / (c1 + c2)
    for l in range(11):
        assert float(xs[l, 0]) == pytest.approx(float(x), rel=1e-13), l
        g1 = c1 ** 2 / mpmath.sqrt(c1 ** 2 * (1 - x) ** 2 + eps ** 2)
        g2 = c2 ** 2 / mpmath.sqrt(c2 ** 2 * x ** 2 + eps ** 2)
        x = g1 / (g1 + g2)


def test_diagonal_system_one_iteration():
    """No n-links: L~ is diagonal, Jacobi is exact, every solve converges in
    one iteration to the per-pixel two-edge closed form."""
    spec = gen.zero_nlink_grid(13, 7, 5, seed=11, lo=0.05, hi=2.0)
    S = solver(spec, T=4, cg_rtol=1e-12, cg_max_iter=50)
    xs, reps = S.run()
    c1, c2 = spec["cs"], spec["ct"]
    np.testing.assert_allclose(xs[0], c1 / (c1 + c2), rtol=1e-13, atol=1e-15)
    assert reps[0]["cg_iters"] == 1


def test_zero_rhs():
    spec = gen.uniform_grid(5, 4, seed=1)
    spec["cs"][:] = 0.0
    S = solver(spec, T=1, cg_rtol=1e-10, cg_max_iter=100)
    xs, reps = S.run()
    assert (xs == 0.0).all() and reps[0]["cg_iters"] == 0


def test_scaling_metamorphic_bitwise():
    """(c, eps) -> (2c, 2eps): every recurrence scalar and vector scales by
    an exact power of two (z, p, x, alpha, beta unchanged), so x^(l) and the
    iteration counts are bitwise unchanged."""
    spec = gen.blob_grid(10, 9, 7, seed=5, sigma=(2.0, 5.0))
    spec2 = dict(spec)
    for k in ("cx", "cy", "cz", "cs", "ct"):
        spec2[k] = spec[k] * 2.0
    x1, r1 = solver(spec, T=6, eps=1e-6).run()
    x2, r2 = solver(spec2, T=6, eps=2e-6).run()
    assert np.array_equal(x1, x2)
    assert [r["cg_iters"] for r in r1] == [r["cg_iters"] for r in r2]


@pytest.mark.parametrize("spec", [gen.blob_grid(12, 10, 8, seed=7, sigma=(2.0, 5.0)),
                                  gen.road_graph(60, seed=3, knn=30)])
def test_krylov_equivalence_with_hs(spec):
    """Same Krylov iterates as O5 in exact arithmetic: at a tight tolerance
    the init solve takes the same number of iterations and lands on the same
    x up to rounding."""
    a = oracle.Solver(oracle.Graph(spec), T=0, cg_rtol=1e-9, cg_max_iter=100000, cg_variant=0)
    b = oracle.Solver(oracle.Graph(spec), T=0, cg_rtol=1e-9, cg_max_iter=100000, cg_variant=1)
    ra, rb = a.init(), b.init()
    assert abs(ra["cg_iters"] - rb["cg_iters"]) <= 1
    np.testing.assert_allclose(b.x(), a.x(), rtol=1e-7, atol=1e-9)


def test_irls_invariants_paper_policy():
    """The paper's policy (rtol 1e-3, cap 50): box and Prop. 3 within the
    tolerance, S_eps monotone under a tight tolerance."""
    spec = gen.uniform_grid(12, 10, seed=21)
    xs, reps = solver(spec, T=15, cg_rtol=1e-11, cg_max_iter=100000).run()
    for r in reps:
        assert r["x_min"] >= -1e-10 and r["x_max"] <= 1 + 1e-10
        assert r["flow_value"] == pytest.approx(r["current_s"], rel=1e-8)
    Se = [r["S_eps"] for r in reps]
    assert all(a <= b * (1 + 1e-9) for a, b in zip(Se[1:], Se[:-1]))
