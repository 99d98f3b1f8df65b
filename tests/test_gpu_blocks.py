"""GPU parity of the block-Jacobi preconditioner (A32; SURVEY §8(f) NEXT #2;
P:L235-242 "block Jacobi" with exact "LU" blocks) through the C ABI
against the oracle: every x^(l), every CG iteration count, converged flag and
relative residual, and the sweep — bitwise — for BFS blocks of several sizes
on random graphs, ragged blob grids (stencil and CSR), a road-like graph, in
graph and host-loop mode, warm and cold, both norms, with the fixed-point
exit, on virtual ranks (blocks never cross a C3 group, so W = 1/2/4/8 give
the same bits), and the option's error cases."""
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


def _bits(a):
    return np.asarray(a, dtype=np.float64).view(np.uint64)


def lockstep(I, spec, T, B, *, rtol=1e-3, cap=50, norm=0, warm=True, loop_mode=0):
    m = I.MinCut.from_spec(spec, I.options(T=T, cg_rtol=rtol, cg_max_iter=cap, cg_norm=norm, warm_start=int(warm),
                                           loop_mode=loop_mode, block_size=B))
    S = oracle.Solver(oracle.Graph(spec), T=T, cg_rtol=rtol, cg_max_iter=cap, cg_norm=norm, warm_start=warm,
                      block_size=B)
    for l in range(T + 1):
        rg = m.irls_init() if l == 0 else m.irls_step()
        ro = S.init() if l == 0 else S.step()
        assert rg["cg_iters"] == ro["cg_iters"], (l, rg["cg_iters"], ro["cg_iters"])
        assert np.array_equal(_bits(m.irls_get_potentials()), _bits(S.x())), f"x^({l})"
        assert rg["converged"] == ro["converged"] and rg["rel_res"] == ro["rel_res"] and rg["ref"] == ro["ref"], l
    return m, S


def check_sweep(m, S):
    side, order, k, cut = m.irls_sweep_cut(side=True, order=True)
    sw = S.sweep()
    assert k == sw.k and cut == sw.cut_value
    assert np.array_equal(side, sw.side) and np.array_equal(order.astype(np.int64), sw.order)


@pytest.mark.parametrize("B", [1, 16, 64, 256])
@pytest.mark.parametrize("seed", [0, 1])
def test_random_graphs(irls, seed, B):
    spec = gen.random_small_graph(3000 + 900 * seed, 5000, seed=500 + seed)
    m, S = lockstep(irls, spec, T=8, B=B)
    check_sweep(m, S)


@pytest.mark.parametrize("B", [8, 64, 200])
@pytest.mark.parametrize("shape", [(48, 40, 24), (33, 17, 9), (512, 6, 3)])
def test_blob_grids_stencil(irls, shape, B):
    spec = gen.blob_grid(*shape, seed=1, sigma=(3.0, 9.0))
    m, S = lockstep(irls, spec, T=6, B=B)
    check_sweep(m, S)


@pytest.mark.parametrize("B", [32, 128])
def test_stencil_equals_csr(irls, B):
    """The same grid as a stencil and as CSR: identical adjacency order, hence
    identical blocks and bits (C2)."""
    spec = gen.blob_grid(40, 36, 10, seed=4, sigma=(3.0, 8.0))
    a, _ = lockstep(irls, spec, T=5, B=B)
    b, _ = lockstep(irls, gen.stencil_to_csr(spec), T=5, B=B)
    assert np.array_equal(_bits(a.irls_get_potentials()), _bits(b.irls_get_potentials()))


def test_road_like(irls):
    spec = gen.road_graph(200, seed=2, knn=100)
    m, S = lockstep(irls, spec, T=10, B=64)
    check_sweep(m, S)


@pytest.mark.parametrize("loop_mode", [0, 1])
@pytest.mark.parametrize("norm,warm", [(0, True), (1, True), (0, False)])
def test_modes(irls, norm, warm, loop_mode):
    spec = gen.blob_grid(40, 30, 12, seed=6, sigma=(3.0, 8.0))
    lockstep(irls, spec, T=6, B=48, norm=norm, warm=warm, loop_mode=loop_mode)


def test_solve_graph_and_fixed_point_exit(irls):
    """irls_solve (the multi-step graph) and the fixed-point exit give the
    oracle's x^(T), counts and sweep."""
    spec = gen.blob_grid(64, 40, 16, seed=2, sigma=(3.0, 9.0))
    T = 20
    S = oracle.Solver(oracle.Graph(spec), T=T, block_size=64)
    xs, oreps = S.run()
    for fpx in (0, 1):
        m = irls.MinCut.from_spec(spec, irls.options(T=T, block_size=64, fixed_point_exit=fpx))
        reps, total = m.irls_solve(irls.IRLS_FROM_SCRATCH, T=T)
        assert [r["cg_iters"] for r in reps] == [r["cg_iters"] for r in oreps]
        assert np.array_equal(_bits(m.irls_get_potentials()), _bits(xs[-1]))
        check_sweep(m, S)
        m.close()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_virtual_ranks(irls, world):
    """Blocks live inside C3 groups, so every world size computes the same
    blocks and bits (slabs and CSR strips)."""
    for spec in (gen.blob_grid(64, 64, 16, seed=3, sigma=(3.0, 9.0)),
                 gen.stencil_to_csr(gen.blob_grid(64, 64, 16, seed=3, sigma=(3.0, 9.0)))):
        T = 6
        S = oracle.Solver(oracle.Graph(spec), T=T, block_size=64)
        xs, oreps = S.run()
        g = irls.VGroup(spec, world, irls.options(T=T, block_size=64))
        reps, total = g.irls_vgroup_solve(irls.IRLS_FROM_SCRATCH)
        assert [r["cg_iters"] for r in reps] == [r["cg_iters"] for r in oreps]
        assert np.array_equal(_bits(g.irls_vgroup_get_potentials()), _bits(xs[-1]))
        g.close()


def test_terminal_weight_sequence(irls):
    spec = gen.blob_grid(24, 24, 12, seed=1, sigma=(3.0, 8.0))
    T = 8
    m = irls.MinCut.from_spec(spec, irls.options(T=T, block_size=64))
    S = oracle.Solver(oracle.Graph(spec), T=T, block_size=64)
    m.irls_solve(irls.IRLS_FROM_SCRATCH, T=T)
    S.run(record=False)
    cs, ct = spec["cs"].copy(), spec["ct"].copy()
    for fs, ft in gen.config5_factors(cs.shape[0], n_problems=2, seed=4):
        cs, ct = cs * fs, ct * ft
        m.irls_set_terminal_weights(cs, ct)
        S.set_terminal_weights(cs, ct)
        _, tot = m.irls_solve(irls.IRLS_CONTINUE, T=T)
        assert tot == sum(S.step()["cg_iters"] for _ in range(T))
        assert np.array_equal(_bits(m.irls_get_potentials()), _bits(S.x()))


def test_lambda2_stays_point_jacobi(irls):
    """A30: lambda_2's solve uses point Jacobi whatever the context's
    preconditioner."""
    spec = gen.blob_grid(32, 30, 8, seed=2, sigma=(3.0, 8.0))
    a = irls.MinCut.from_spec(spec, irls.options(T=3, block_size=64))
    b = irls.MinCut.from_spec(spec, irls.options(T=3))
    ra, rb = a.irls_lambda2(cg_rtol=1e-8), b.irls_lambda2(cg_rtol=1e-8)
    assert ra["lambda2"] == rb["lambda2"] and ra["cg_iters"] == rb["cg_iters"]
    S = oracle.Solver(oracle.Graph(spec), T=3, block_size=64)
    lam, xlx, C, it = S.lambda2(rtol=1e-8, norm=1)
    assert ra["lambda2"] == lam and ra["cg_iters"] == it


@pytest.mark.parametrize("kw", [dict(block_size=-1), dict(block_size=257), dict(block_size=8, cg_variant=1),
                                dict(block_size=8, record_trace=1)])
def test_invalid_options(irls, kw):
    spec = gen.blob_grid(16, 16, 4, seed=2, sigma=(2.0, 5.0))
    with pytest.raises(irls.IrlsError) as e:
        irls.MinCut.from_spec(spec, irls.options(T=2, **kw))
    assert e.value.code == 1
