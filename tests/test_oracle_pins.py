"""Pins of the CPU oracle against things other than itself (CPU only).

Every test cites what fixes the expected value: a SPEC worked example
(tests/golden/spec_examples.json), a closed form of the method, a dense
library solve of the paper's matrix-form equations, brute-force enumeration,
networkx, or an invariant the paper proves.
"""
import json
import math
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
    G = oracle.Graph(spec)
    return oracle.Solver(G, **kw)


# --------------------------------------------------------------------------
# SPEC worked examples
# --------------------------------------------------------------------------

def test_assemble_path_init():
    S = solver(TINY["path"], cg_rtol=1e-14, cg_max_iter=100)
    a = S.assemble()
    gold = GOLD["assemble_path_init"]
    assert a["D"].tolist() == gold["D"] and a["gs"].tolist() == gold["b"]
    S.init()
    assert S.x()[0] == pytest.approx(gold["v"][0], rel=1e-15)


def test_assemble_cycle4_init():
    S = solver(TINY["cycle4"], cg_rtol=1e-14, cg_max_iter=100)
    a = S.assemble()
    gold = GOLD["assemble_cycle4_init"]
    assert a["D"].tolist() == gold["D"] and a["gs"].tolist() == gold["b"]
    S.init()
    np.testing.assert_allclose(S.x(), gold["v"], rtol=1e-15)
    x = S.x()
    assert x[0] == x[1]  # automorphism a <-> b


def test_pcg_path4():
    S = solver(TINY["path4"], cg_rtol=1e-14, cg_max_iter=100)
    S.init()
    np.testing.assert_allclose(S.x(), GOLD["pcg_path4"]["v"], rtol=1e-14)


def test_flow_value_and_S_eps_path_init():
    S = solver(TINY["path"], cg_rtol=1e-14, cg_max_iter=100)
    rep = S.init()
    assert rep["flow_value"] == pytest.approx(GOLD["flow_value_path_init"]["value"], rel=1e-14)
    assert rep["current_s"] == pytest.approx(GOLD["flow_value_path_init"]["value"], rel=1e-14)
    assert rep["S_eps"] == pytest.approx(GOLD["S_eps_path_init"]["value"], abs=GOLD["S_eps_path_init"]["abs_tol"])


def test_reweight_path_erratum():
    """S:L261 corrected: x_a = 2/3 gives w = (sqrt(4/9+eps^2), sqrt(4/9+eps^2))
    so g = (6, 1.5) and the next iterate is x_a = 0.8."""
    gold = GOLD["reweight_path_x23"]
    S = solver(TINY["path"], cg_rtol=1e-14, cg_max_iter=100)
    a = S.assemble(np.array([2.0 / 3.0]))
    assert a["gs"][0] == pytest.approx(gold["g"][0], rel=gold["rel_tol"])
    assert a["gt"][0] == pytest.approx(gold["g"][1], rel=gold["rel_tol"])
    S.init()
    S.step()
    assert S.x()[0] == pytest.approx(gold["x_next"], rel=1e-11)


def test_zero_gradient_edge_gives_eps():
    """an edge whose endpoints have equal x has w = eps exactly, so
    its conductance is c^2/eps."""
    spec = gen._csr_edges(4, [(0, 1, 1.0), (1, 2, 3.0), (2, 3, 1.0)], 0, 3)
    S = solver(spec, eps=1e-3)
    a = S.assemble(np.array([0.25, 0.25]))
    assert a["g"][0] == 9.0 / 1e-3 and a["g"][1] == 9.0 / 1e-3


def test_irls_path_T10_closed_form():
    """S:L279 and the two-edge closed form x' = g1/(g1+g2),
    evaluated at 50 digits with mpmath."""
    S = solver(TINY["path"], T=10, cg_rtol=1e-14, cg_max_iter=100)
    xs, reps = S.run()
    mpmath.mp.dps = 50
    c1, c2, eps = mpmath.mpf(2), mpmath.mpf(1), mpmath.mpf("1e-6")
    x = c1 / (c1 + c2)
    for l in range(11):
        assert float(xs[l, 0]) == pytest.approx(float(x), rel=1e-13), l
        g1 = c1 ** 2 / mpmath.sqrt(c1 ** 2 * (1 - x) ** 2 + eps ** 2)
        g2 = c2 ** 2 / mpmath.sqrt(c2 ** 2 * x ** 2 + eps ** 2)
        x = g1 / (g1 + g2)
    assert xs[10, 0] > GOLD["irls_path_T10"]["x10_min"]
    assert xs[10, 0] == pytest.approx(GOLD["irls_path_T10"]["x10_closed_form"], abs=1e-9)


def test_irls_symmetric_fixed_point():
    S = solver(TINY["path_sym"], T=5, cg_rtol=1e-14, cg_max_iter=100)
    xs, _ = S.run()
    assert (xs[:, 0] == GOLD["irls_symmetric"]["x"]).all()


def test_T0_returns_init():
    S = solver(gen.uniform_grid(6, 5, seed=3), T=0, cg_rtol=1e-12, cg_max_iter=1000)
    xs, reps = S.run()
    S2 = solver(gen.uniform_grid(6, 5, seed=3), T=0, cg_rtol=1e-12, cg_max_iter=1000)
    S2.init()
    assert xs.shape[0] == 1 and np.array_equal(xs[0], S2.x())


def test_sweep_and_cut_examples():
    S = solver(TINY["path"])
    sw = S.sweep(np.array([0.9]))
    gold = GOLD["sweep_path_x09"]
    assert sw.side.tolist() == gold["side"] and sw.cut_value == gold["value"]
    St = solver(TINY["triangle"])
    assert St.cut_value(np.array(GOLD["cut_triangle_s"]["side"], np.uint8)) == GOLD["cut_triangle_s"]["value"]
    assert S.cut_value(np.array(GOLD["cut_path_sa"]["side"], np.uint8)) == GOLD["cut_path_sa"]["value"]
    assert S.maxflow()[0] == GOLD["maxflow_path"]["value"]
    assert St.maxflow()[0] == GOLD["maxflow_triangle"]["value"]
    # triangle: direct s-t edge is the additive constant c_st (A5)
    sw = St.sweep(np.array([0.5]))
    assert sw.cut_value == 1.5


# --------------------------------------------------------------------------
# Closed forms at scale: zero n-links => independent two-edge paths
# --------------------------------------------------------------------------

def test_zero_nlink_grid_matches_two_edge_closed_form():
    spec = gen.zero_nlink_grid(13, 7, 5, seed=11, lo=0.05, hi=2.0)
    S = solver(spec, T=8, cg_rtol=1e-14, cg_max_iter=50, eps=1e-6)
    xs, reps = S.run()
    c1, c2 = spec["cs"], spec["ct"]
    x = c1 / (c1 + c2)
    eps = 1e-6
    for l in range(9):
        np.testing.assert_allclose(xs[l], x, rtol=1e-13, atol=1e-15)
        g1 = c1 ** 2 / np.sqrt(c1 ** 2 * (1 - x) ** 2 + eps ** 2)
        g2 = c2 ** 2 / np.sqrt(c2 ** 2 * x ** 2 + eps ** 2)
        x = g1 / (g1 + g2)


# --------------------------------------------------------------------------
# Dense library solves of the matrix-form equations
# --------------------------------------------------------------------------

@pytest.mark.parametrize("seed", [0, 1, 2])
def test_init_solve_matches_dense(seed):
    spec = gen.random_small_graph(60, 90, seed=seed)
    n, s, t, E = H.edge_list(spec)
    Lr, b, keep = H.dense_irls_system(n, s, t, E)
    v = np.linalg.solve(Lr, b)
    S = solver(spec, cg_rtol=1e-14, cg_max_iter=10000)
    S.init()
    np.testing.assert_allclose(S.x(), v, rtol=1e-9, atol=1e-12)
    assert (v >= -1e-12).all() and (v <= 1 + 1e-12).all()  # Prop. 2 box


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


def test_flow_value_is_effective_conductance():
    """Prop. 3: for the W = C system, x^T L x is the s-t effective conductance
    1/R_eff with R_eff = (e_s-e_t)^T L^+ (e_s-e_t) (dense pseudo-inverse)."""
    spec = gen.random_small_graph(30, 50, seed=7)
    n, s, t, E = H.edge_list(spec)
    B, c = H.incidence(n, E)
    Lfull = B.T @ np.diag(c) @ B
    chi = np.zeros(n); chi[s] = 1; chi[t] = -1
    reff = chi @ np.linalg.pinv(Lfull) @ chi
    S = solver(spec, cg_rtol=1e-14, cg_max_iter=10000)
    rep = S.init()
    assert rep["flow_value"] == pytest.approx(1.0 / reff, rel=1e-9)
    assert rep["current_s"] == pytest.approx(1.0 / reff, rel=1e-9)


# --------------------------------------------------------------------------
# Brute force / max-flow
# --------------------------------------------------------------------------

@pytest.mark.parametrize("seed", range(6))
def test_bruteforce_mincut_and_sweep(seed):
    spec = gen.random_small_graph(12 + seed % 4, 10 + 2 * seed, seed=100 + seed)
    n, s, t, E = H.edge_list(spec)
    mu, side_bf = H.brute_force_mincut(n, s, t, E)
    S = solver(spec, T=20, cg_rtol=1e-10, cg_max_iter=1000)
    flow, side_ek = S.maxflow()
    assert flow == pytest.approx(mu, rel=1e-12)
    assert H.cut_value(E, side_ek) == pytest.approx(mu, rel=1e-12)
    S.run(record=False)
    xfull = np.zeros(n); xfull[s] = 1.0
    xfull[S.graph.orig] = S.x()
    sw = S.sweep()
    best, best_k, order = H.prefix_sweep_bruteforce(n, s, t, E, xfull)
    assert sw.k == best_k
    assert sw.order.tolist() == order
    assert sw.cut_value == pytest.approx(best, rel=1e-12)
    assert sw.cut_value >= mu * (1 - 1e-12)
    assert H.cut_value(E, sw.side) == pytest.approx(sw.cut_value, rel=1e-12)
    # fixed-point prefix value agrees with the cut value
    assert sw.pk * 2.0 ** (-sw.F) == pytest.approx(sw.cut_value, rel=1e-12)


def test_edmonds_karp_matches_networkx_config1():
    nx = pytest.importorskip("networkx")
    spec = gen.config1()
    n, s, t, E = H.edge_list(spec)
    Gx = nx.Graph()
    for u, v, c in E:
        Gx.add_edge(u, v, capacity=c)
    val, _ = nx.minimum_cut(Gx, s, t)
    S = solver(spec)
    flow, side = S.maxflow()
    assert flow == pytest.approx(val, rel=1e-10)
    assert S.cut_value(side) == pytest.approx(val, rel=1e-10)


def test_sweep_of_optimal_indicator_returns_optimum():
    """sweeping an exact optimal indicator yields a min cut."""
    spec = gen.uniform_grid(9, 8, seed=5)
    S = solver(spec)
    mu, side = S.maxflow()
    x = side[S.graph.orig].astype(np.float64)
    sw = S.sweep(x)
    assert sw.cut_value == pytest.approx(mu, rel=1e-12)


def test_sweep_ties_and_signed_zero():
    """A14: total order (x desc, id asc); -0.0 == +0.0; NaN rejected."""
    spec = gen.uniform_grid(5, 4, seed=9)
    S = solver(spec)
    x = np.zeros(20); x[[3, 7, 11]] = 0.5; x[[1, 2]] = -0.0; x[5] = 1.0
    sw = S.sweep(x)
    expect = [5, 3, 7, 11] + [i for i in range(20) if i not in (5, 3, 7, 11)]
    assert sw.order.tolist() == expect
    x[4] = np.nan
    with pytest.raises(oracle.OracleError) as ei:
        S.sweep(x)
    assert ei.value.code == 7


# --------------------------------------------------------------------------
# Invariants
# --------------------------------------------------------------------------

def test_invariants_tight_tolerance():
    spec = gen.uniform_grid(12, 10, seed=21)
    S = solver(spec, T=15, cg_rtol=1e-11, cg_max_iter=100000)
    xs, reps = S.run()
    rtol = 1e-11
    for l, r in enumerate(reps):
        assert r["x_min"] >= -10 * rtol and r["x_max"] <= 1 + 10 * rtol      # Prop. 2
        assert r["flow_value"] == pytest.approx(r["current_s"], rel=1e-8)     # Prop. 3
        assert r["converged"] == 1
    Se = [r["S_eps"] for r in reps]
    for a, b in zip(Se[1:], Se[:-1]):   # descent of S_eps (A4; Beck)
        assert a <= b * (1 + 1e-9)


def test_scaling_metamorphic_bitwise():
    """(c, eps) -> (2c, 2eps) leaves every x^(l) bitwise unchanged (powers of
    two scale exactly; Eq. 4 and Eq. 8 are homogeneous)."""
    spec = gen.blob_grid(10, 9, 7, seed=5, sigma=(2.0, 5.0))
    spec2 = dict(spec)
    for k in ("cx", "cy", "cz", "cs", "ct"):
        spec2[k] = spec[k] * 2.0
    S1 = solver(spec, T=6, eps=1e-6)
    S2 = solver(spec2, T=6, eps=2e-6)
    x1, r1 = S1.run(); x2, r2 = S2.run()
    assert np.array_equal(x1, x2)
    assert [r["cg_iters"] for r in r1] == [r["cg_iters"] for r in r2]
    assert all(b["S_eps"] == 2 * a["S_eps"] for a, b in zip(r1, r2))


def test_source_sink_swap():
    spec = gen.uniform_grid(7, 6, seed=13)
    sw_spec = dict(spec); sw_spec["cs"], sw_spec["ct"] = spec["ct"], spec["cs"]
    S1 = solver(spec, T=5, cg_rtol=1e-12, cg_max_iter=10000)
    S2 = solver(sw_spec, T=5, cg_rtol=1e-12, cg_max_iter=10000)
    x1, _ = S1.run(); x2, _ = S2.run()
    np.testing.assert_allclose(x2, 1 - x1, atol=1e-9)


def test_warm_start_not_worse_in_total():
    """Fig. 1, qualitative: warm starts need no more PCG
    iterations in total than cold starts."""
    spec = gen.blob_grid(16, 16, 8, seed=1, sigma=(3.0, 8.0))
    Sw = solver(spec, T=20, cg_rtol=1e-3, cg_max_iter=300)
    Sc = solver(spec, T=20, cg_rtol=1e-3, cg_max_iter=300, warm_start=False)
    _, rw = Sw.run(record=False); _, rc = Sc.run(record=False)
    assert sum(r["cg_iters"] for r in rw) <= sum(r["cg_iters"] for r in rc)


# --------------------------------------------------------------------------
# Validation / status codes
# --------------------------------------------------------------------------

def test_status_codes():
    with pytest.raises(oracle.OracleError) as e:
        oracle.Graph(gen._csr_edges(3, [(0, 1, 1.0), (1, 2, 1.0)], 1, 1))
    assert e.value.code == 2
    with pytest.raises(oracle.OracleError) as e:
        oracle.Graph(gen._csr_edges(3, [(0, 1, -1.0), (1, 2, 1.0)], 0, 2))
    assert e.value.code == 3
    with pytest.raises(oracle.OracleError) as e:
        oracle.Graph(gen._csr_edges(3, [(0, 1, np.nan), (1, 2, 1.0)], 0, 2))
    assert e.value.code == 3
    bad = gen._csr_edges(3, [(0, 1, 1.0), (1, 2, 1.0)], 0, 2)
    bad["w"] = bad["w"].copy(); bad["w"][0] = 5.0
    with pytest.raises(oracle.OracleError) as e:
        oracle.Graph(bad)
    assert e.value.code == 4
    # component {3,4} has no terminal edge -> singular (Prop. 1, A8)
    G = oracle.Graph(gen._csr_edges(5, [(0, 1, 1.0), (1, 2, 1.0), (3, 4, 1.0)], 0, 2))
    assert G.check_nonsingular() == 5
    assert oracle.Graph(TINY["path"]).check_nonsingular() == 0


def test_duplicate_edges_merge_by_sum():
    rp = np.array([0, 2, 5, 6], dtype=np.int64)
    col = np.array([1, 1, 0, 0, 2, 1], dtype=np.int32)
    w = np.array([1.0, 1.0, 1.0, 1.0, 1.0, 1.0])
    dup = dict(kind="csr", n=3, row_ptr=rp, col=col, w=w, s=0, t=2)
    S1 = solver(dup, cg_rtol=1e-14, cg_max_iter=10)
    S1.init()
    assert S1.x()[0] == pytest.approx(2.0 / 3.0, rel=1e-15)


# --------------------------------------------------------------------------
# C3 reduction and fixed-point sweep arithmetic
# --------------------------------------------------------------------------

@pytest.mark.parametrize("n", [0, 1, 2, 511, 4095, 4096, 4097, 8 * 4096 + 3, 100003])
def test_c3_exact_on_integers(n):
    rng = np.random.default_rng(n)
    v = rng.integers(-1000, 1000, n).astype(np.float64)
    assert oracle.c3_sum(v) == float(v.sum(dtype=np.int64)) if n else oracle.c3_sum(v) == 0.0


@pytest.mark.parametrize("n", [3, 4097, 70001])
def test_c3_error_bound(n):
    rng = np.random.default_rng(n + 1)
    v = rng.standard_normal(n)
    exact = math.fsum(v)
    bound = 64 * np.finfo(float).eps * np.abs(v).sum()
    assert abs(oracle.c3_sum(v) - exact) <= bound
    gs = oracle.c3_group_sums(v)
    t4 = [gs[i] + gs[i + 4] for i in range(4)]
    t2 = [t4[0] + t4[2], t4[1] + t4[3]]
    assert oracle.c3_sum(v) == t2[0] + t2[1]


def test_c3_tree_order_hand_derived():
    """Tiny inputs where the order is visible: thread 0 sums elements 0,1
    sequentially, thread 1 holds element 2, lanes combine at offset 1."""
    assert oracle.c3_sum(np.array([1.0, 1e16, -1e16])) == 0.0      # (1 + 1e16) + (-1e16)
    assert oracle.c3_sum(np.array([1e16, -1e16, 1.0])) == 1.0      # (1e16 - 1e16) + 1
    # element 512 is thread 0's third element: ((v0 + v1) + v512)
    v = np.zeros(600); v[0] = 1.0; v[1] = 1e16; v[512] = -1e16
    assert oracle.c3_sum(v) == 0.0
    # element 2 (thread 1) joins thread 0 at the last shuffle step
    v = np.zeros(600); v[0] = 1e16; v[2] = 1.0; v[512] = -1e16
    assert oracle.c3_sum(v) == 1.0


def test_fixed_point_F_and_exactness():
    spec = gen.uniform_grid(6, 6, seed=2)
    S = solver(spec)
    sw = S.sweep(np.linspace(1, 0, 36))
    cmax = max(spec["cx"].max(), spec["cy"].max(), spec["cs"].max(), spec["ct"].max())
    e = math.frexp(cmax)[1]
    cnt = int((spec["cx"] > 0).sum() + (spec["cy"] > 0).sum() + (spec["cs"] > 0).sum() + (spec["ct"] > 0).sum())
    assert sw.F == 124 - e - cnt.bit_length()
    n, s, t, E = H.edge_list(spec)
    assert sw.pk * 2.0 ** (-sw.F) == pytest.approx(H.cut_value(E, sw.side), rel=1e-14)
