"""GPU parity of the two-level rounding:
the CUDA path (K-means, classification, coarse graph on the GPU; exact
max-flow on the host; lift and C3 cut on the GPU) through the C ABI against
the oracle, both started from their OWN bitwise-equal IRLS runs.

Bar: bitwise equality of the centres, thresholds and round count, the
S0/S1/Sc classes, the whole fixed-point coarse graph, the max-flow value, the
returned set and the cut value (integer work bit-exact; float work under the
arithmetic contract).  Full size: config 2 (K-means and coarse graph against
the oracle at 2.1M nodes; the max-flow certified by strong duality)."""
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


def _bitwise(a, b):
    return np.array_equal(np.asarray(a, dtype=np.float64).view(np.uint64),
                          np.asarray(b, dtype=np.float64).view(np.uint64))


def solve_both(I, spec, T, **kw):
    opts = I.options(T=T, **{k: v for k, v in kw.items()})
    m = I.MinCut.from_spec(spec, opts)
    m.irls_solve(I.IRLS_FROM_SCRATCH, T=T, reports=False)
    okw = {"cg_rtol": kw.get("cg_rtol", 1e-3), "cg_max_iter": kw.get("cg_max_iter", 50),
           "cg_norm": kw.get("cg_norm", 0)}
    S = oracle.Solver(oracle.Graph(spec), T=T, **okw)
    S.run(record=False)
    assert _bitwise(m.irls_get_potentials(), S.x())
    return m, S


def compare_coarse(m, S, rep):
    """The GPU coarse graph equals the oracle's, entry by entry."""
    co = S.coarsen(S.x(), rep["gamma0"], rep["gamma1"])
    assert rep["F"] == co.F
    assert rep["nc"] == co.nc and rep["coarse_nlinks"] * 2 == len(co.col)
    g = m.irls_two_level_get_coarse(co.nc, len(co.col))
    assert np.array_equal(g["cls"], co.cls)
    assert np.array_equal(g["ptr"].astype(np.int64), co.ptr)
    assert np.array_equal(g["col"].astype(np.int64), co.col)
    scale = 2.0 ** co.F
    assert [int(np.rint(np.ldexp(c, co.F))) for c in g["cap"]] == co.cap
    assert g["qs"] == co.qs and g["qt"] == co.qt and g["qst"] == co.qst
    return co


def check_two_level(I, m, S, coarse=True):
    side, rep = m.irls_two_level_cut()
    r = S.two_level()
    assert (rep["c0"], rep["c1"], rep["gamma0"], rep["gamma1"]) == (r.c0, r.c1, r.gamma0, r.gamma1)
    assert rep["kmeans_rounds"] == r.rounds
    assert (rep["n0"], rep["n1"], rep["nc"]) == (r.n0, r.n1, r.nc)
    assert rep["certified"] == 1
    assert rep["coarse_flow"] == np.ldexp(float(r.flow), -r.F)
    assert np.array_equal(side, r.side)
    assert rep["cut_value"] == r.cut_value
    if coarse:
        compare_coarse(m, S, rep)
    return side, rep, r


@pytest.mark.parametrize("name", ["path", "cycle4", "path4", "triangle"])
def test_tiny_graphs(irls, name):
    m, S = solve_both(irls, gen.tiny_graphs()[name], T=10, cg_rtol=1e-12, cg_max_iter=100)
    check_two_level(irls, m, S)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_random_graphs(irls, seed):
    spec = gen.random_small_graph(300 + 50 * seed, 500, seed=800 + seed)
    m, S = solve_both(irls, spec, T=8)
    check_two_level(irls, m, S)


def test_config1_exact(irls):
    """Config 1 at its own tolerance: two-level is exact (networkx-pinned in
    the oracle tests) and bitwise equal to the oracle."""
    m, S = solve_both(irls, gen.config1(), T=50, cg_rtol=1e-10, cg_max_iter=100000, cg_norm=1)
    side, rep, r = check_two_level(irls, m, S)
    flow, _ = S.maxflow()
    assert rep["cut_value"] == pytest.approx(flow, rel=1e-12)


@pytest.mark.parametrize("shape", [(48, 40, 24), (33, 17, 9)])
def test_blob_grids_ragged(irls, shape):
    """Config-2 recipe on grids whose chunk counts are ragged (stencil)."""
    nx, ny, nz = shape
    spec = gen.blob_grid(nx, ny, nz, seed=1, sigma=(3.0, 9.0))
    m, S = solve_both(irls, spec, T=12)
    side, rep, r = check_two_level(irls, m, S)
    sw = S.sweep()
    assert rep["cut_value"] <= sw.cut_value  # Table 4's dominance on this instance


def test_road_like_csr(irls):
    spec = gen.road_graph(side=60, seed=2, knn=40)
    m, S = solve_both(irls, spec, T=10)
    check_two_level(irls, m, S)


def test_stencil_equals_csr(irls):
    """The same grid through both layouts gives the same two-level result."""
    spec = gen.blob_grid(20, 18, 6, seed=3, sigma=(2.0, 6.0))
    a = irls.MinCut.from_spec(spec, irls.options(T=8))
    b = irls.MinCut.from_spec(gen.stencil_to_csr(spec), irls.options(T=8))
    a.irls_solve(irls.IRLS_FROM_SCRATCH, T=8, reports=False)
    b.irls_solve(irls.IRLS_FROM_SCRATCH, T=8, reports=False)
    sa, ra = a.irls_two_level_cut()
    sb, rb = b.irls_two_level_cut()
    assert ra["cut_value"] == rb["cut_value"] and np.array_equal(sa, sb)


def test_vgroup_equals_one_rank(irls):
    """The multi-GPU path (gather to rank 0) gives the one-rank result."""
    spec = gen.blob_grid(64, 64, 16, seed=5, sigma=(3.0, 8.0))  # group-aligned slabs for W = 2, 4, 8
    m = irls.MinCut.from_spec(spec, irls.options(T=10))
    m.irls_solve(irls.IRLS_FROM_SCRATCH, T=10, reports=False)
    s1, r1 = m.irls_two_level_cut()
    for W in (2, 4, 8):
        g = irls.VGroup(spec, W, irls.options(T=10))
        g.irls_vgroup_solve(irls.IRLS_FROM_SCRATCH, T=10)
        sw, rw = g.irls_vgroup_two_level_cut()
        assert np.array_equal(sw, s1) and rw["cut_value"] == r1["cut_value"]
        assert rw["nc"] == r1["nc"] and rw["c0"] == r1["c0"] and rw["c1"] == r1["c1"]


def test_crossing_thresholds(irls):
    """A26': centres < 0.1 apart -> thresholds (c0, c1), bitwise as
    the oracle (K-means, classes, coarse graph, set, cut)."""
    spec = gen.random_small_graph(600, 900, seed=77)
    m = irls.MinCut.from_spec(spec, irls.options(T=2))
    S = oracle.Solver(oracle.Graph(spec), T=2)
    rng = np.random.default_rng(5)
    x = np.where(rng.random(m.n) < 0.5, 0.48, 0.52) + rng.uniform(-0.004, 0.004, m.n)
    m.irls_set_potentials(x)
    S.set_x(x)
    side, rep, r = check_two_level(irls, m, S)
    assert (rep["gamma0"], rep["gamma1"]) == (rep["c0"], rep["c1"])


def test_errors_and_repeat(irls):
    spec = gen.blob_grid(16, 16, 4, seed=2, sigma=(2.0, 5.0))
    m = irls.MinCut.from_spec(spec, irls.options(T=4))
    with pytest.raises(irls.IrlsError) as e:
        m.irls_two_level_cut()
    assert e.value.code == 8  # IRLS_ERR_STATE before a solve
    m.irls_solve(irls.IRLS_FROM_SCRATCH, T=4, reports=False)
    s1, r1 = m.irls_two_level_cut()
    s2, r2 = m.irls_two_level_cut()  # buffers reused
    assert np.array_equal(s1, s2) and r1["cut_value"] == r2["cut_value"]
    x = m.irls_get_potentials()
    x[7] = np.nan
    m.irls_set_potentials(x)
    with pytest.raises(irls.IrlsError) as e:
        m.irls_two_level_cut()
    assert e.value.code == 7  # IRLS_ERR_BAD_POTENTIAL


@pytest.mark.slow
def test_config2_full_size(irls):
    """Config 2 (128^3, 2.1M nodes) in the bench configuration: the oracle's
    own IRLS run, K-means and coarse graph equal the GPU's bitwise; the
    208k-node coarse max-flow is certified by strong duality, and the cut of
    the returned set on G equals the coarse flow value."""
    spec = gen.config2()
    m, S = solve_both(irls, spec, T=50)
    side, rep = m.irls_two_level_cut()
    (c0, c1, g0, g1), rounds = S.kmeans2()
    assert (rep["c0"], rep["c1"], rep["gamma0"], rep["gamma1"], rep["kmeans_rounds"]) == (c0, c1, g0, g1, rounds)
    compare_coarse(m, S, rep)
    assert rep["certified"] == 1
    assert rep["cut_value"] == pytest.approx(rep["coarse_flow"], rel=1e-12)
    assert S.cut_value(side) == pytest.approx(rep["cut_value"], rel=1e-12)
    _, _, _, sweep_cut = m.irls_sweep_cut(side=False)
    assert rep["cut_value"] <= sweep_cut


def test_exact_min_cut_on_a_communicator(irls):
    """mu* (no contraction) on a multi-rank context (1-rank NCCL
    communicator: gather, rank-0 max-flow, broadcast) equals the plain call,
    before any solve."""
    import torch
    spec = gen.blob_grid(30, 24, 4, seed=6, sigma=(2.0, 6.0))
    m = irls.MinCut.from_spec(spec, irls.options(T=4))
    s1, r1 = m.irls_exact_min_cut()
    comm = irls.comm_desc(1, 0, 0, irls.irls_nccl_unique_id(), torch.cuda.current_stream().cuda_stream)
    g = irls.MinCut.from_spec(spec, irls.options(T=4), comm)
    s2, r2 = g.irls_exact_min_cut()
    assert r1["cut_value"] == r2["cut_value"] and np.array_equal(s1, s2)
    g.close()
    m.close()
