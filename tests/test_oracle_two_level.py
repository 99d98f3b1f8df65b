"""Pins of the oracle's two-level rounding
against things other than itself (CPU only): SPEC worked examples of
cluster_voltages / coarsen / two_level_round, scikit-learn's
Lloyd K-means, the paper's Proposition on constructed
potentials, exhaustive enumeration of coarse cuts (cut-value preservation
under lifting), brute-force and networkx minimum cuts.
"""
import itertools

import numpy as np
import pytest

import oracle
from synthetic import generators as gen
from tests import helpers as H

TINY = gen.tiny_graphs()


def solver(spec, **kw):
    return oracle.Solver(oracle.Graph(spec), **kw)


def line_graph(n_mid, seed=0):
    """s - u_1 - ... - u_k - t with random weights: n_mid non-terminals."""
    rng = np.random.default_rng(seed)
    n = n_mid + 2
    edges = [(i, i + 1, float(rng.uniform(0.5, 2.0))) for i in range(n - 1)]
    return gen._csr_edges(n, edges, 0, n - 1)


# --------------------------------------------------------------------------
# K-means (A25)
# --------------------------------------------------------------------------

def test_kmeans_spec_polarized():
    """S:L363 voltages {0,0,0,1,1} -> centres (0,1), gamma = (0.05, 0.95).
    Terminals contribute x_s = 1, x_t = 0, so the non-terminals are {0,0,1}."""
    S = solver(line_graph(3))
    (c0, c1, g0, g1), r = S.kmeans2(np.array([0.0, 0.0, 1.0]))
    assert (c0, c1) == (0.0, 1.0)
    assert g0 == pytest.approx(0.05, abs=1e-16) and g1 == pytest.approx(0.95, abs=1e-16)
    assert r <= 2  # S:L395 fully separated bimodal input converges in <= 2 rounds


def test_kmeans_spec_hand_round():
    """S:L364 {0.0, 0.1, 0.8, 0.9} -> (0.05, 0.85): here the multiset is
    {x_t=0, 0.1, 0.8, x_s=1} (terminals included, A25); one hand Lloyd round
    from (0.1, 0.9) assigns {0, 0.1} | {0.8, 1} -> (0.05, 0.9), then stable."""
    S = solver(line_graph(2))
    (c0, c1, g0, g1), r = S.kmeans2(np.array([0.1, 0.8]))
    assert c0 == pytest.approx(0.05, rel=1e-15) and c1 == pytest.approx(0.9, rel=1e-15)
    assert g0 == pytest.approx(0.10, rel=1e-15) and g1 == pytest.approx(0.85, rel=1e-15)
    assert r == 2


def test_crossing_thresholds_fall_back_to_centres():
    """A26': centres less than 0.1 apart make c0 + 0.05 >= c1 - 0.05;
    the thresholds fall back to (c0, c1).  Hand example: 200 nodes at 0.48 and
    200 at 0.52 plus x_t = 0, x_s = 1.  Lloyd from (0.1, 0.9): midpoint 0.5
    splits {0.48 x200, 0} | {0.52 x200, 1}, giving c0 = 96/201, c1 = 105/201
    (0.0448 apart), after which the assignment is stable."""
    n_mid = 400
    spec = line_graph(n_mid, seed=3)
    x = np.where(np.arange(n_mid) % 2 == 0, 0.48, 0.52)
    S = solver(spec)
    (c0, c1, g0, g1), r = S.kmeans2(x)
    assert c0 == pytest.approx(96.0 / 201.0, rel=1e-14) and c1 == pytest.approx(105.0 / 201.0, rel=1e-14)
    assert (g0, g1) == (c0, c1)
    tl = S.two_level(x)
    assert (tl.gamma0, tl.gamma1) == (c0, c1)
    # 0.48 > c0 and 0.52 < c1: no node is contracted, G_c = G and the rounding is
    # the exact minimum cut of the path: its lightest edge
    assert tl.nc == n_mid and tl.n0 == 0 and tl.n1 == 0
    n, s_id, t_id, E = H.edge_list(spec)
    w_min = min(c for _, _, c in E)
    assert tl.cut_value == pytest.approx(w_min, rel=1e-15)
    assert H.cut_value(E, tl.side) == pytest.approx(w_min, rel=1e-15)


@pytest.mark.parametrize("seed", range(5))
def test_kmeans_matches_sklearn_lloyd(seed):
    """Lloyd's fixed point from the same initial centres equals scikit-learn's
    KMeans(init=[[0.1],[0.9]], n_init=1, algorithm='lloyd')."""
    sk = pytest.importorskip("sklearn.cluster")
    rng = np.random.default_rng(seed)
    m = 500 + 137 * seed
    x = np.concatenate([rng.beta(0.6, 4.0, m // 2), rng.beta(4.0, 0.6, m - m // 2)])
    rng.shuffle(x)
    S = solver(line_graph(m, seed))
    (c0, c1, _, _), _ = S.kmeans2(x)
    km = sk.KMeans(n_clusters=2, init=np.array([[0.1], [0.9]]), n_init=1, algorithm="lloyd", tol=0.0,
                   max_iter=100).fit(np.concatenate([x, [1.0, 0.0]])[:, None])
    ref = sorted(km.cluster_centers_.ravel())
    assert c0 == pytest.approx(ref[0], rel=1e-12) and c1 == pytest.approx(ref[1], rel=1e-12)
    # and it is a Lloyd fixed point by definition (exact sums via fsum)
    full = np.concatenate([x, [1.0, 0.0]])
    a1 = np.abs(full - c1) < np.abs(full - c0)
    assert c0 == pytest.approx(np.mean(full[~a1]), rel=1e-13)
    assert c1 == pytest.approx(np.mean(full[a1]), rel=1e-13)


# --------------------------------------------------------------------------
# Coarsening (A27)
# --------------------------------------------------------------------------

def _coarse_cut(co, src_bits):
    """Cut value of a coarse labelling (1 = source side) from the fixed-point
    coarse graph: s_c-t_c edge + s-links of sink nodes + t-links of source
    nodes + n-links across."""
    v = co.qst
    for u in range(co.nc):
        v += co.qt[u] if src_bits[u] else co.qs[u]
        for e in range(co.ptr[u], co.ptr[u + 1]):
            w = int(co.col[e])
            if w > u and src_bits[u] != src_bits[w]:
                v += co.cap[e]
    return v


@pytest.mark.parametrize("seed", range(4))
def test_coarse_cut_preserved_under_lifting(seed):
    """for EVERY coarse labelling, its cut value on G_c equals the cut
    value (by definition over the edge list) of the lifted labelling
    on G.  Exhaustive over 2^|Sc| labellings, |Sc| <= 10."""
    spec = gen.random_small_graph(16, 18, seed=300 + seed)
    n, s, t, E = H.edge_list(spec)
    S = solver(spec)
    rng = np.random.default_rng(seed)
    x = rng.choice([0.0, 0.02, 0.5, 0.97, 1.0], size=S.n, p=[0.3, 0.1, 0.3, 0.1, 0.2])
    x[x == 0.5] = rng.uniform(0.2, 0.8, int((x == 0.5).sum()))
    co = S.coarsen(x, 0.1, 0.9)
    assert co.nc == int((x > 0.1).sum() - (x >= 0.9).sum())
    assert 1 <= co.nc <= 10
    scale = 2.0 ** (-co.F)
    orig = S.graph.orig
    for bits in itertools.product((0, 1), repeat=co.nc):
        side = np.zeros(n, dtype=np.uint8)
        side[s] = 1
        for u in range(S.n):
            side[orig[u]] = 1 if co.cls[u] == 1 else (bits[co.cid[u]] if co.cls[u] == 2 else 0)
        assert _coarse_cut(co, bits) * scale == pytest.approx(H.cut_value(E, side), rel=1e-13)


def test_coarsen_spec_polarized_and_identity():
    """a fully polarised x matching a cut S gives Sc empty and
    G_c = {s_c, t_c} with one edge of weight cut(S); a path s-a-t with x_a
    between the thresholds gives G_c isomorphic to the original."""
    spec = gen.uniform_grid(6, 5, seed=2)
    n, s, t, E = H.edge_list(spec)
    S = solver(spec)
    _, side = S.maxflow()
    x = side[S.graph.orig].astype(np.float64)
    co = S.coarsen(x, 0.05, 0.95)
    assert co.nc == 0
    assert co.qst * 2.0 ** (-co.F) == pytest.approx(H.cut_value(E, side), rel=1e-13)
    P = solver(TINY["path"])
    co = P.coarsen(np.array([0.5]), 0.05, 0.95)
    assert co.nc == 1 and co.qst == 0
    assert co.qs[0] * 2.0 ** (-co.F) == 2.0 and co.qt[0] * 2.0 ** (-co.F) == 1.0


# --------------------------------------------------------------------------
# Exact coarse max-flow (A28)
# --------------------------------------------------------------------------

@pytest.mark.parametrize("seed", range(4))
def test_maxflow_coarse_is_minimal_min_cut(seed):
    """The coarse solve returns the minimum cut value (brute force over all
    coarse labellings) and the MINIMAL minimum-cut source side: the
    intersection of every optimal source set."""
    spec = gen.random_small_graph(14, 16, seed=400 + seed)
    S = solver(spec)
    rng = np.random.default_rng(seed)
    x = rng.uniform(0.0, 1.0, S.n)
    co = S.coarsen(x, 0.08, 0.92)
    flow, src = oracle.maxflow_coarse(co.nc, co.ptr, co.col, co.cap, co.qs, co.qt, co.qst)
    vals = {bits: _coarse_cut(co, bits) for bits in itertools.product((0, 1), repeat=co.nc)}
    best = min(vals.values())
    assert flow == best
    inter = np.ones(co.nc, dtype=np.uint8)
    for bits, v in vals.items():
        if v == best:
            inter &= np.array(bits, dtype=np.uint8)
    assert src.tolist() == inter.tolist()
    assert _coarse_cut(co, tuple(src.tolist())) == best


def test_maxflow_coarse_equal_cut_ties():
    """Unit 4-cycle s-a-t-b (several optima): the minimal source side
    is {s}, value 2."""
    S = solver(TINY["cycle4"])
    co = S.coarsen(np.array([0.5, 0.5]), 0.1, 0.9)
    flow, src = oracle.maxflow_coarse(co.nc, co.ptr, co.col, co.cap, co.qs, co.qt, co.qst)
    assert flow * 2.0 ** (-co.F) == 2.0 and src.tolist() == [0, 0]


# --------------------------------------------------------------------------
# Two-level end to end
# --------------------------------------------------------------------------

@pytest.mark.parametrize("seed", range(5))
def test_proposition_constructed_potentials(seed):
    """P:L283-286 (Proposition): if S1 lies in the source side and S0 in the
    sink side of some min cut, the min cut of G_c induces a min cut of G.  x
    is built from a brute-force optimum (polarised near its sides, random
    middle nodes) and coarsened at thresholds (0.1, 0.9); the lifted coarse
    optimum must equal the brute-force minimum.  With the K-means thresholds
    two_level() must do the same whenever the hypothesis holds for them."""
    spec = gen.random_small_graph(15, 20, seed=500 + seed)
    n, s, t, E = H.edge_list(spec)
    mu, side_bf = H.brute_force_mincut(n, s, t, E)
    S = solver(spec)
    rng = np.random.default_rng(seed)
    opt = side_bf[S.graph.orig].astype(bool)
    x = np.where(opt, rng.uniform(0.97, 1.0, S.n), rng.uniform(0.0, 0.03, S.n))
    mid = rng.random(S.n) < 0.4
    x[mid] = rng.uniform(0.3, 0.7, int(mid.sum()))
    co = S.coarsen(x, 0.1, 0.9)
    assert co.nc == int(mid.sum())
    flow, src = oracle.maxflow_coarse(co.nc, co.ptr, co.col, co.cap, co.qs, co.qt, co.qst)
    side = np.zeros(n, dtype=np.uint8)
    side[s] = 1
    for u in range(S.n):
        side[S.graph.orig[u]] = 1 if co.cls[u] == 1 else (src[co.cid[u]] if co.cls[u] == 2 else 0)
    assert H.cut_value(E, side) == pytest.approx(mu, rel=1e-12)
    assert flow * 2.0 ** (-co.F) == pytest.approx(mu, rel=1e-12)
    r = S.two_level(x)
    s1 = x >= r.gamma1
    s0 = (x <= r.gamma0)
    s1 &= ~s0
    if not (s1 & ~opt).any() and not (s0 & opt).any():
        assert r.cut_value == pytest.approx(mu, rel=1e-12)
    assert H.cut_value(E, r.side) == pytest.approx(r.cut_value, rel=1e-12)
    assert r.cut_value >= mu * (1 - 1e-12)


def test_polarized_correct_x_gives_optimum():
    """a fully polarised correct x returns the optimal cut (delta = 0)."""
    spec = gen.uniform_grid(10, 9, seed=7)
    S = solver(spec)
    mu, side = S.maxflow()
    r = S.two_level(side[S.graph.orig].astype(np.float64))
    assert r.nc == 0 and r.cut_value == pytest.approx(mu, rel=1e-12)
    assert (r.c0, r.c1) == (0.0, 1.0)


@pytest.mark.parametrize("seed", range(4))
def test_two_level_after_irls_bounds(seed):
    """On IRLS potentials: mu* <= two-level <= sweep (Table 4's
    dominance as a regression expectation), and the reported value is the
    cut of the returned set by definition."""
    spec = gen.random_small_graph(16, 22, seed=600 + seed)
    n, s, t, E = H.edge_list(spec)
    mu, _ = H.brute_force_mincut(n, s, t, E)
    S = solver(spec, T=10)
    S.run(record=False)
    r = S.two_level()
    sw = S.sweep()
    assert r.cut_value >= mu * (1 - 1e-12)
    assert r.cut_value <= sw.cut_value * (1 + 1e-12)
    assert H.cut_value(E, r.side) == pytest.approx(r.cut_value, rel=1e-12)
    assert r.side[s] == 1 and r.side[t] == 0


def test_two_level_config1_matches_networkx():
    """Config 1 (32x32): after IRLS at the config's tolerance, two-level
    finds the exact minimum (networkx minimum_cut) while the sweep does not."""
    nx = pytest.importorskip("networkx")
    spec = gen.config1()
    n, s, t, E = H.edge_list(spec)
    Gx = nx.Graph()
    for u, v, c in E:
        Gx.add_edge(u, v, capacity=c)
    mu, _ = nx.minimum_cut(Gx, s, t)
    S = solver(spec, T=10, cg_rtol=1e-10, cg_max_iter=100000, cg_norm=1)
    S.run(record=False)
    r = S.two_level()
    assert r.cut_value == pytest.approx(mu, rel=1e-12)
    assert S.sweep().cut_value > mu * (1 + 1e-6)
