"""The multi-GPU z-slab data path, executed on one GPU as a virtual group
(irls_vgroup_*): W ranks' kernels, ghost planes, per-rank C3 group sums,
slot-exact allreduce, ghost p updates, finalize kernels and the rank-0 sweep.
Only NCCL is replaced (by device copies).  The bar is bitwise equality with
one rank and with the oracle: the contract makes the result independent of W.
p2p=1 runs the peer-memory collectives instead (group owners store their
slot sums into every rank's buffer + arrival counters the finalize kernels
wait on; K5 stores z's boundary planes into the neighbours' ghost planes):
the same bits again.
"""
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


def single(I, spec, opts, T):
    m = I.MinCut.from_spec(spec, opts)
    reps, tot = m.irls_solve(I.IRLS_FROM_SCRATCH, T=T)
    sw = m.irls_sweep_cut(order=True)
    return m, reps, tot, sw


@pytest.mark.parametrize("p2p", [0, 1])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_vgroup_equals_single_and_oracle(irls, world, p2p):
    # 64x64x20: one chunk per plane, uneven slabs (2 or 3 planes per group)
    spec = gen.blob_grid(64, 64, 20, seed=5, sigma=(3.0, 10.0))
    T = 20
    opts = irls.options(T=T, record_trace=1)
    m, reps1, tot1, sw1 = single(irls, spec, opts, T)
    g = irls.VGroup(spec, world, irls.options(T=T, record_trace=1, p2p=p2p))
    reps, tot = g.irls_vgroup_solve(irls.IRLS_FROM_SCRATCH, T=T)
    assert tot == tot1
    for a, b in zip(reps, reps1):
        for k in ("cg_iters", "converged", "rel_res", "S_eps", "flow_value", "current_s", "true_rel_res",
                  "x_min", "x_max"):
            assert a[k] == b[k], k
    x = g.irls_vgroup_get_potentials()
    assert np.array_equal(x, m.irls_get_potentials())
    S = oracle.Solver(oracle.Graph(spec), T=T)
    S.run(record=False)
    assert np.array_equal(x, S.x())
    side, order, k, cut = g.irls_vgroup_sweep_cut(order=True)
    assert k == sw1[2] and cut == sw1[3]
    assert np.array_equal(side, sw1[0]) and np.array_equal(order, sw1[1])
    g.close()


@pytest.mark.parametrize("p2p", [0, 1])
@pytest.mark.parametrize("world", [2, 8])
def test_vgroup_cold_and_sequence(irls, world, p2p):
    spec = gen.blob_grid(64, 64, 16, seed=2, sigma=(3.0, 8.0))
    T = 8
    for warm in (0, 1):
        opts = irls.options(T=T, warm_start=warm)
        m = irls.MinCut.from_spec(spec, opts)
        g = irls.VGroup(spec, world, irls.options(T=T, warm_start=warm, p2p=p2p))
        _, t1 = m.irls_solve(irls.IRLS_FROM_SCRATCH, T=T)
        _, t2 = g.irls_vgroup_solve(irls.IRLS_FROM_SCRATCH, T=T)
        assert t1 == t2
        cs, ct = spec["cs"].copy(), spec["ct"].copy()
        for fs, ft in gen.config5_factors(cs.shape[0], n_problems=2, seed=4):
            cs, ct = cs * fs, ct * ft
            m.irls_set_terminal_weights(cs, ct)
            g.irls_vgroup_set_terminal_weights(cs, ct)
            _, t1 = m.irls_solve(irls.IRLS_CONTINUE, T=T)
            _, t2 = g.irls_vgroup_solve(irls.IRLS_CONTINUE, T=T)
            assert t1 == t2
            assert np.array_equal(g.irls_vgroup_get_potentials(), m.irls_get_potentials())
        g.close()


@pytest.mark.parametrize("p2p", [0, 1])
@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("nz", [16, 32])
def test_vgroup_fused_rows_of_512(irls, world, p2p, nz):
    """512-wide rows (fused reweight kernel incl. the ghost -z slot), one
    chunk per plane, 16 or 32 planes (slabs of 8 planes or more run the
    z-cluster K1): bitwise equal to one rank."""
    spec = gen.blob_grid(512, 8, nz, seed=8, sigma=(3.0, 8.0))
    T = 10
    m, reps1, tot1, sw1 = single(irls, spec, irls.options(T=T), T)
    g = irls.VGroup(spec, world, irls.options(T=T, p2p=p2p))
    reps, tot = g.irls_vgroup_solve(irls.IRLS_FROM_SCRATCH, T=T)
    assert [r["cg_iters"] for r in reps] == [r["cg_iters"] for r in reps1]
    assert np.array_equal(g.irls_vgroup_get_potentials(), m.irls_get_potentials())
    g.close()


@pytest.mark.slow
@pytest.mark.parametrize("p2p", [0, 1])
def test_vgroup_config2_world8(irls, p2p):
    """BASELINE config 2 (128^3), 8 virtual ranks of 16 planes each."""
    spec = gen.config2()
    opts = irls.options(T=50)
    m, reps1, tot1, sw1 = single(irls, spec, opts, 50)
    g = irls.VGroup(spec, 8, irls.options(T=50, p2p=p2p))
    reps, tot = g.irls_vgroup_solve(irls.IRLS_FROM_SCRATCH, T=50)
    assert [r["cg_iters"] for r in reps] == [r["cg_iters"] for r in reps1]
    assert np.array_equal(g.irls_vgroup_get_potentials(), m.irls_get_potentials())
    side, _, k, cut = g.irls_vgroup_sweep_cut()
    assert k == sw1[2] and cut == sw1[3] and np.array_equal(side, sw1[0])
    g.close()


def test_vgroup_rejects_unaligned(irls):
    spec = gen.blob_grid(40, 36, 29, seed=1)  # group boundaries fall inside planes
    with pytest.raises(irls.IrlsError):
        irls.VGroup(spec, 2)


@pytest.mark.parametrize("p2p", [0, 1])
@pytest.mark.parametrize("loop_mode", [1, 2])
def test_nccl_one_rank_communicator(irls, loop_mode, p2p):
    """The NCCL code path on one GPU: world_size 1 with an NCCL id runs the
    multi-rank host loop, ncclAllReduce of the slots, the finalize kernels,
    the gather and the ncclBroadcast of the sweep / two-level results over a
    1-rank communicator.  Bitwise equal to the plain single-GPU path."""
    import torch
    spec = gen.blob_grid(64, 64, 16, seed=3, sigma=(3.0, 8.0))
    T = 12
    m, reps1, tot1, sw1 = single(irls, spec, irls.options(T=T, record_trace=1), T)
    comm = irls.comm_desc(1, 0, 0, irls.irls_nccl_unique_id(), torch.cuda.current_stream().cuda_stream)
    g = irls.MinCut.from_spec(spec, irls.options(T=T, record_trace=1, loop_mode=loop_mode, p2p=p2p), comm)
    reps, tot = g.irls_solve(irls.IRLS_FROM_SCRATCH, T=T)
    assert tot == tot1
    for a, b in zip(reps, reps1):
        for k in ("cg_iters", "rel_res", "S_eps", "flow_value", "x_min", "x_max"):
            assert a[k] == b[k], k
    assert np.array_equal(g.irls_get_potentials(), m.irls_get_potentials())
    side, order, k, cut = g.irls_sweep_cut(order=True)
    assert k == sw1[2] and cut == sw1[3] and np.array_equal(side, sw1[0])
    s2, r2 = g.irls_two_level_cut()
    s1, r1 = m.irls_two_level_cut()
    assert np.array_equal(s1, s2) and r1["cut_value"] == r2["cut_value"]
    g.close()
    # the same through a 1-rank communicator on a CSR graph (id strips, W = 1)
    spec = gen.road_graph(120, seed=2, knn=50)
    m, reps1, tot1, sw1 = single(irls, spec, irls.options(T=T), T)
    comm = irls.comm_desc(1, 0, 0, irls.irls_nccl_unique_id(), torch.cuda.current_stream().cuda_stream)  # one id per comm
    g = irls.MinCut.from_spec(spec, irls.options(T=T, loop_mode=loop_mode, p2p=p2p), comm)
    _, tot = g.irls_solve(irls.IRLS_FROM_SCRATCH, T=T)
    assert tot == tot1 and np.array_equal(g.irls_get_potentials(), m.irls_get_potentials())
    side, _, k, cut = g.irls_sweep_cut()
    assert k == sw1[2] and cut == sw1[3] and np.array_equal(side, sw1[0])
    g.close()


@pytest.mark.parametrize("p2p", [0, 1])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_vgroup_csr_strips(irls, world, p2p):
    """CSR id strips (SURVEY §8(e), config 3's partition): every rank's rows
    with a ghost block refreshed by the halo (packed send lists), per-rank C3
    groups, slot allreduce, ghost p update, gather and the rank-0 sweep and
    two-level rounding: bitwise equal to one rank and to the oracle."""
    spec = gen.road_graph(200, seed=2, knn=60)  # 39,469 non-terminals: 9.6 chunks, ragged strips
    T = 12
    m, reps1, tot1, sw1 = single(irls, spec, irls.options(T=T, record_trace=1), T)
    g = irls.VGroup(spec, world, irls.options(T=T, record_trace=1, p2p=p2p))
    reps, tot = g.irls_vgroup_solve(irls.IRLS_FROM_SCRATCH, T=T)
    assert tot == tot1
    for a, b in zip(reps, reps1):
        for k in ("cg_iters", "converged", "rel_res", "S_eps", "flow_value", "true_rel_res", "x_min", "x_max"):
            assert a[k] == b[k], k
    x = g.irls_vgroup_get_potentials()
    assert np.array_equal(x, m.irls_get_potentials())
    S = oracle.Solver(oracle.Graph(spec), T=T)
    S.run(record=False)
    assert np.array_equal(x, S.x())
    side, order, k, cut = g.irls_vgroup_sweep_cut(order=True)
    assert k == sw1[2] and cut == sw1[3] and np.array_equal(side, sw1[0])
    s2, r2 = g.irls_vgroup_two_level_cut()
    s1, r1 = m.irls_two_level_cut()
    assert np.array_equal(s1, s2) and r1["cut_value"] == r2["cut_value"]
    # a config-5 style sequence on the strips (terminal weights of every strip)
    cs, ct = S.graph.terminals()
    for fs, ft in gen.config5_factors(cs.shape[0], n_problems=2, seed=4):
        cs, ct = cs * fs, ct * ft
        m.irls_set_terminal_weights(cs, ct)
        g.irls_vgroup_set_terminal_weights(cs, ct)
        _, t1 = m.irls_solve(irls.IRLS_CONTINUE, T=T)
        _, t2 = g.irls_vgroup_solve(irls.IRLS_CONTINUE, T=T)
        assert t1 == t2
        assert np.array_equal(g.irls_vgroup_get_potentials(), m.irls_get_potentials())
    g.close()


@pytest.mark.slow
@pytest.mark.parametrize("p2p", [0, 1])
def test_vgroup_config3_world8(irls, p2p):
    """BASELINE config 3 (road-like CSR, 23.7M nodes) as 8 id strips: every
    step's iteration count, x^(50) and the sweep equal one rank bitwise
    (p2p: the strips' z halo as peer stores + pushed group sums)."""
    spec = gen.config3()
    m, reps1, tot1, sw1 = single(irls, spec, irls.options(T=50), 50)
    g = irls.VGroup(spec, 8, irls.options(T=50, p2p=p2p))
    reps, tot = g.irls_vgroup_solve(irls.IRLS_FROM_SCRATCH, T=50)
    assert [r["cg_iters"] for r in reps] == [r["cg_iters"] for r in reps1]
    assert np.array_equal(g.irls_vgroup_get_potentials(), m.irls_get_potentials())
    side, _, k, cut = g.irls_vgroup_sweep_cut()
    assert k == sw1[2] and cut == sw1[3] and np.array_equal(side, sw1[0])
    g.close()


def test_vgroup_csr_rejects_too_few_chunks(irls):
    spec = gen.road_graph(60, seed=2, knn=40)  # < 8 chunks
    with pytest.raises(irls.IrlsError):
        irls.VGroup(spec, 2)


@pytest.mark.parametrize("p2p", [0, 1])
@pytest.mark.parametrize("world", [2, 4])
def test_vgroup_fixed_point_exit(irls, world, p2p):
    """fixed_point_exit on W ranks (host loop): a frozen step skips its
    assembly on every rank and its START finalize with it (no producer ran,
    so with p2p there is nothing to wait for); reports and x^(T) equal one
    rank with the same option and one rank without it."""
    spec = gen.blob_grid(64, 64, 16, seed=9, sigma=(3.0, 8.0))
    T = 40
    m, reps1, tot1, _ = single(irls, spec, irls.options(T=T), T)
    mf, repsf, totf, _ = single(irls, spec, irls.options(T=T, fixed_point_exit=1), T)
    assert totf == tot1
    assert any(r["cg_iters"] == 0 for r in reps1[1:]), "case must reach a fixed point"
    g = irls.VGroup(spec, world, irls.options(T=T, fixed_point_exit=1, p2p=p2p))
    reps, tot = g.irls_vgroup_solve(irls.IRLS_FROM_SCRATCH, T=T)
    assert tot == tot1
    assert [r["cg_iters"] for r in reps] == [r["cg_iters"] for r in reps1]
    assert [r["rel_res"] for r in reps] == [r["rel_res"] for r in repsf]
    assert np.array_equal(g.irls_vgroup_get_potentials(), m.irls_get_potentials())
    g.close()


def test_vgroup_p2p_rejects_bad_flag(irls):
    spec = gen.blob_grid(64, 64, 16, seed=9)
    with pytest.raises(irls.IrlsError):
        irls.VGroup(spec, 2, irls.options(p2p=2))


def test_halo_timing_entry(irls):
    """irls_time_kernel(KERNEL_HALO) (bench's NVLink line at N > 1): runs on
    an NCCL context (here a 1-rank communicator: no peers, an empty exchange)
    without changing the state; refused on a plain single-GPU context."""
    import torch
    spec = gen.blob_grid(64, 64, 16, seed=3, sigma=(3.0, 8.0))
    comm = irls.comm_desc(1, 0, 0, irls.irls_nccl_unique_id(), torch.cuda.current_stream().cuda_stream)
    g = irls.MinCut.from_spec(spec, irls.options(T=4, loop_mode=1), comm)
    g.irls_solve(irls.IRLS_FROM_SCRATCH, T=4)
    x0 = g.irls_get_potentials()
    assert g.irls_time_kernel(irls.KERNEL_HALO, 5) >= 0.0
    assert np.array_equal(g.irls_get_potentials(), x0)
    g.close()
    m = irls.MinCut.from_spec(spec, irls.options(T=4))
    m.irls_solve(irls.IRLS_FROM_SCRATCH, T=4)
    with pytest.raises(irls.IrlsError):
        m.irls_time_kernel(irls.KERNEL_HALO, 5)
    m.close()
