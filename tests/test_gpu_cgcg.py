"""Chronopoulos-Gear PCG on the GPU (irls_options.cg_variant = IRLS_CG_CG;
SURVEY §8(f) NEXT #3; O5' / A31): one kernel and one C3 reduction per
iteration.  Bar: BITWISE equality with the oracle's O5' (every x^(l), every
iteration count and residual), on stencil and CSR paths, graph and host
loops, warm / cold / sequences, and on W virtual ranks (slabs and strips,
NCCL-copy or peer-memory collectives) and a 1-rank NCCL communicator."""
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


def lockstep(I, spec, T, *, eps=1e-6, rtol=1e-3, max_iter=50, norm=0, warm=True, loop_mode=0, record=False):
    opts = I.options(eps=eps, T=T, cg_rtol=rtol, cg_max_iter=max_iter, cg_norm=norm, warm_start=int(warm),
                     loop_mode=loop_mode, record_trace=int(record), cg_variant=I.IRLS_CG_CG)
    m = I.MinCut.from_spec(spec, opts)
    S = oracle.Solver(oracle.Graph(spec), eps=eps, T=T, cg_rtol=rtol, cg_max_iter=max_iter, cg_norm=norm,
                      warm_start=warm, cg_variant=1)
    for l in range(T + 1):
        rg = m.irls_init() if l == 0 else m.irls_step()
        ro = S.init() if l == 0 else S.step()
        assert rg["cg_iters"] == ro["cg_iters"], (l, rg["cg_iters"], ro["cg_iters"])
        assert rg["rel_res"] == ro["rel_res"], l
        assert np.array_equal(m.irls_get_potentials().view(np.uint64), S.x().view(np.uint64)), l
        if record:
            for k in ("S_eps", "flow_value", "true_rel_res", "x_min", "x_max"):
                assert rg[k] == ro[k], (l, k)
    return m, S


def check_sweep(m, S):
    side, order, k, cut = m.irls_sweep_cut(side=True, order=True)
    sw = S.sweep()
    assert k == sw.k and cut == sw.cut_value
    assert np.array_equal(side, sw.side) and np.array_equal(order.astype(np.int64), sw.order)


@pytest.mark.parametrize("shape", [(16, 12, 9), (33, 17, 8), (64, 64, 3), (70, 1, 1), (31, 29, 1)])
def test_blob_grids(irls, shape):
    nx, ny, nz = shape
    spec = gen.blob_grid(nx, ny, nz, seed=nx + ny, sigma=(2.0, 6.0))
    m, S = lockstep(irls, spec, T=8, record=True)
    check_sweep(m, S)


@pytest.mark.parametrize("loop_mode", [0, 1])
def test_graph_and_host_loops_cold(irls, loop_mode):
    spec = gen.blob_grid(48, 40, 6, seed=3, sigma=(3.0, 8.0))
    m, S = lockstep(irls, spec, T=6, warm=False, loop_mode=loop_mode)
    check_sweep(m, S)


def test_unpreconditioned_tight(irls):
    spec = gen.uniform_grid(20, 18, seed=4)
    lockstep(irls, spec, T=5, rtol=1e-10, max_iter=100000, norm=1)


@pytest.mark.parametrize("name", ["road", "random"])
def test_csr(irls, name):
    spec = gen.road_graph(90, seed=5, knn=40) if name == "road" else gen.random_small_graph(300, 500, seed=8)
    m, S = lockstep(irls, spec, T=8, record=True)
    check_sweep(m, S)


def test_solve_sequence_and_zero_rhs(irls):
    """irls_solve (multi-step graph), a terminal-weight sequence, and b = 0."""
    spec = gen.blob_grid(64, 32, 8, seed=6, sigma=(3.0, 8.0))
    T = 12
    m = irls.MinCut.from_spec(spec, irls.options(T=T, cg_variant=irls.IRLS_CG_CG))
    S = oracle.Solver(oracle.Graph(spec), T=T, cg_variant=1)
    reps, tot = m.irls_solve(irls.IRLS_FROM_SCRATCH, T=T)
    _, oreps = S.run(record=False)
    assert [r["cg_iters"] for r in reps] == [r["cg_iters"] for r in oreps]
    assert np.array_equal(m.irls_get_potentials(), S.x())
    cs, ct = spec["cs"].copy(), spec["ct"].copy()
    for fs, ft in gen.config5_factors(cs.shape[0], n_problems=2, seed=4):
        cs, ct = cs * fs, ct * ft
        m.irls_set_terminal_weights(cs, ct)
        S.set_terminal_weights(cs, ct)
        m.irls_solve(irls.IRLS_CONTINUE, T=T)
        for _ in range(T):
            S.step()
        assert np.array_equal(m.irls_get_potentials(), S.x())
    z = gen.uniform_grid(9, 7, seed=1)
    z["cs"][:] = 0.0
    mz = irls.MinCut.from_spec(z, irls.options(T=2, cg_variant=irls.IRLS_CG_CG))
    reps, tot = mz.irls_solve(irls.IRLS_FROM_SCRATCH, T=2)
    assert tot == 0 and (mz.irls_get_potentials() == 0.0).all()


def test_fixed_point_exit(irls):
    spec = gen.blob_grid(64, 64, 16, seed=9, sigma=(3.0, 8.0))
    T = 40
    a = irls.MinCut.from_spec(spec, irls.options(T=T, cg_variant=irls.IRLS_CG_CG))
    b = irls.MinCut.from_spec(spec, irls.options(T=T, cg_variant=irls.IRLS_CG_CG, fixed_point_exit=1))
    ra, ta = a.irls_solve(irls.IRLS_FROM_SCRATCH, T=T)
    rb, tb = b.irls_solve(irls.IRLS_FROM_SCRATCH, T=T)
    assert ta == tb and np.array_equal(a.irls_get_potentials(), b.irls_get_potentials())
    assert [r["rel_res"] for r in ra] == [r["rel_res"] for r in rb]


@pytest.mark.parametrize("p2p", [0, 1])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_vgroup_slabs(irls, world, p2p):
    spec = gen.blob_grid(64, 64, 20, seed=5, sigma=(3.0, 10.0))
    T = 12
    S = oracle.Solver(oracle.Graph(spec), T=T, cg_variant=1)
    _, oreps = S.run(record=False)
    g = irls.VGroup(spec, world, irls.options(T=T, record_trace=1, cg_variant=irls.IRLS_CG_CG, p2p=p2p))
    reps, tot = g.irls_vgroup_solve(irls.IRLS_FROM_SCRATCH, T=T)
    assert [r["cg_iters"] for r in reps] == [r["cg_iters"] for r in oreps]
    assert [r["rel_res"] for r in reps] == [r["rel_res"] for r in oreps]
    assert np.array_equal(g.irls_vgroup_get_potentials(), S.x())
    side, order, k, cut = g.irls_vgroup_sweep_cut(order=True)
    sw = S.sweep()
    assert k == sw.k and cut == sw.cut_value
    g.close()


@pytest.mark.parametrize("p2p", [0, 1])
@pytest.mark.parametrize("world", [2, 4])
def test_vgroup_csr_strips(irls, world, p2p):
    spec = gen.road_graph(200, seed=2, knn=60)
    T = 10
    S = oracle.Solver(oracle.Graph(spec), T=T, cg_variant=1)
    _, oreps = S.run(record=False)
    g = irls.VGroup(spec, world, irls.options(T=T, cg_variant=irls.IRLS_CG_CG, p2p=p2p))
    reps, tot = g.irls_vgroup_solve(irls.IRLS_FROM_SCRATCH, T=T)
    assert [r["cg_iters"] for r in reps] == [r["cg_iters"] for r in oreps]
    assert np.array_equal(g.irls_vgroup_get_potentials(), S.x())
    g.close()


@pytest.mark.parametrize("p2p", [0, 1])
@pytest.mark.parametrize("loop_mode", [1, 2])
def test_nccl_one_rank(irls, loop_mode, p2p):
    import torch
    spec = gen.blob_grid(64, 64, 16, seed=3, sigma=(3.0, 8.0))
    T = 10
    S = oracle.Solver(oracle.Graph(spec), T=T, cg_variant=1)
    S.run(record=False)
    comm = irls.comm_desc(1, 0, 0, irls.irls_nccl_unique_id(), torch.cuda.current_stream().cuda_stream)
    g = irls.MinCut.from_spec(spec, irls.options(T=T, loop_mode=loop_mode, cg_variant=irls.IRLS_CG_CG, p2p=p2p),
                              comm)
    g.irls_solve(irls.IRLS_FROM_SCRATCH, T=T)
    assert np.array_equal(g.irls_get_potentials(), S.x())
    g.close()


@pytest.mark.slow
def test_config2_full_size(irls):
    """BASELINE config 2 (128^3) with CG-CG: every step's iteration count and
    x^(50) bitwise equal to the oracle's O5'; the sweep cut too."""
    spec = gen.config2()
    S = oracle.Solver(oracle.Graph(spec), T=50, cg_variant=1)
    _, oreps = S.run(record=False)
    m = irls.MinCut.from_spec(spec, irls.options(T=50, cg_variant=irls.IRLS_CG_CG))
    reps, tot = m.irls_solve(irls.IRLS_FROM_SCRATCH, T=50)
    assert [r["cg_iters"] for r in reps] == [r["cg_iters"] for r in oreps]
    assert np.array_equal(m.irls_get_potentials(), S.x())
    check_sweep(m, S)


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("norm", [0, 1])
@pytest.mark.parametrize("warm", [True, False])
@pytest.mark.parametrize("kind", ["grid", "csr"])
def test_option_matrix(irls, variant, norm, warm, kind):
    """Every combination of PCG form, residual norm, warm/cold start and
    graph kind against the oracle, bitwise (reports and x^(T))."""
    spec = (gen.blob_grid(40, 28, 5, seed=13, sigma=(2.0, 6.0)) if kind == "grid"
            else gen.random_small_graph(2500, 4000, seed=17))
    T = 6
    opts = irls.options(T=T, cg_norm=norm, warm_start=int(warm), cg_variant=variant, cg_rtol=1e-4, cg_max_iter=80)
    m = irls.MinCut.from_spec(spec, opts)
    reps, tot = m.irls_solve(irls.IRLS_FROM_SCRATCH, T=T)
    S = oracle.Solver(oracle.Graph(spec), T=T, cg_norm=norm, warm_start=warm, cg_variant=variant, cg_rtol=1e-4,
                      cg_max_iter=80)
    _, oreps = S.run(record=False)
    assert [r["cg_iters"] for r in reps] == [r["cg_iters"] for r in oreps]
    assert [r["rel_res"] for r in reps] == [r["rel_res"] for r in oreps]
    assert np.array_equal(m.irls_get_potentials(), S.x())
