"""Pins of the oracle's Cheeger-type diagnostic lambda_2 (P:L207-226,
Theorem 4; the constrained-WLS characterisation P:L543-551; SURVEY §8(f)
NEXT #4) against things other than itself: SPEC's worked examples
(S:L494-495), the finite generalized eigenvalues of the pencil (L, D) from a
dense scipy eigensolve (Eq. spectral), the Cheeger sandwich
phi^2/2 <= lambda_2 <= 2 phi with phi from brute-force min cuts, and scale
invariance."""
import numpy as np
import pytest
import scipy.linalg

import oracle
from synthetic import generators as gen
from tests import helpers as H


def solver(spec, **kw):
    return oracle.Solver(oracle.Graph(spec), **kw)


def dense_pencil_lambda2(n, s, t, E):
    """lambda_2 of L x = lambda D x, D = diag(d), d_s = d_t = C = 2 sum c
    (P:L211-219): the finite eigenvalues of the rank-2 pencil are 0 and
    lambda_2; eliminate the non-terminals (Schur complement) and solve the
    2x2 pencil exactly."""
    L = np.zeros((n, n))
    for u, v, c in E:
        L[u, u] += c; L[v, v] += c; L[u, v] -= c; L[v, u] -= c
    C = 2.0 * sum(c for _, _, c in E)
    keep = [s, t]
    rest = [i for i in range(n) if i not in keep]
    A = L[np.ix_(keep, keep)]
    if rest:
        A = A - L[np.ix_(keep, rest)] @ np.linalg.solve(L[np.ix_(rest, rest)], L[np.ix_(rest, keep)])
    w = scipy.linalg.eigvals(A, C * np.eye(2))
    w = np.sort(np.real(w))
    return w[1], C


def test_spec_unit_path():
    """unit path s-a-t -> lambda_2 = 0.25, C = 4, x_a = 0."""
    spec = gen._csr_edges(3, [(0, 1, 1.0), (1, 2, 1.0)], 0, 2)
    lam, xLx, C, it, x = solver(spec).lambda2(want_x=True)
    assert lam == 0.25 and C == 4.0 and xLx == 2.0 and x.tolist() == [0.0]


def test_spec_single_edge():
    """a single edge s-t of weight c -> C = 2c, x^T L x = 4c, lambda_2 = 1."""
    spec = gen._csr_edges(2, [(0, 1, 3.0)], 0, 1)
    lam, xLx, C, it = solver(spec).lambda2()
    assert (lam, xLx, C, it) == (1.0, 12.0, 6.0, 0)


def test_spec_single_edge_via_path_limit():
    """a single edge s-t -> lambda_2 = 1.  Here as the direct s-t
    constant c_st (A5) next to a non-terminal hanging off s: x_a = 1, so
    x^T L x = 4 c_st and C = 2 (c_st + c_sa); with c_sa -> small, lambda_2 -> 1."""
    spec = gen._csr_edges(3, [(0, 2, 3.0), (0, 1, 1e-9)], 0, 2)
    S = solver(spec)
    lam, xLx, C, _ = S.lambda2()
    assert xLx == pytest.approx(12.0, rel=1e-15)
    assert lam == pytest.approx(12.0 / (4.0 * (3.0 + 1e-9)), rel=1e-15)


@pytest.mark.parametrize("seed", range(6))
def test_matches_dense_pencil_eigenvalue(seed):
    spec = gen.random_small_graph(10 + 3 * seed, 12 + 4 * seed, seed=900 + seed)
    n, s, t, E = H.edge_list(spec)
    ref, Cref = dense_pencil_lambda2(n, s, t, E)
    lam, xLx, C, it = solver(spec).lambda2(rtol=1e-14, max_iter=10000)
    assert C == pytest.approx(Cref, rel=1e-14)
    assert lam == pytest.approx(ref, rel=1e-9)


@pytest.mark.parametrize("seed", range(6))
def test_cheeger_sandwich(seed):
    """Theorem 4: phi^2 / 2 <= lambda_2 <= 2 phi, phi = mu* / C (every s-t cut
    has min vol = C)."""
    spec = gen.random_small_graph(12, 14 + 2 * seed, seed=950 + seed, wlo=0.05, whi=3.0)
    n, s, t, E = H.edge_list(spec)
    mu, _ = H.brute_force_mincut(n, s, t, E)
    lam, _, C, _ = solver(spec).lambda2(rtol=1e-14, max_iter=10000)
    phi = mu / C
    assert phi ** 2 / 2 <= lam * (1 + 1e-12)
    assert lam <= 2 * phi * (1 + 1e-12)


def test_scale_invariance_and_state_restored():
    spec = gen.blob_grid(12, 10, 4, seed=4, sigma=(2.0, 4.0))
    S = solver(spec, T=3)
    S.run(record=False)
    x_before = S.x().copy()
    lam, _, _, _ = S.lambda2(rtol=1e-12, max_iter=10000)
    assert np.array_equal(S.x(), x_before)
    spec2 = dict(spec)
    for k in ("cx", "cy", "cz", "cs", "ct"):
        spec2[k] = spec[k] * 4.0
    lam2, _, _, _ = solver(spec2).lambda2(rtol=1e-12, max_iter=10000)
    assert lam2 == pytest.approx(lam, rel=1e-12)
    assert -1.0 <= S.lambda2(rtol=1e-12, max_iter=10000, want_x=True)[4].min()
