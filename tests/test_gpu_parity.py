"""GPU parity: the CUDA path through the C ABI vs the float64 CPU oracle.

Under the arithmetic contract (C1 no FMA, C2 ascending
neighbour order, C3 fixed reduction tree) both sides perform the same IEEE
operations in the same order, so the bar here is BITWISE equality of every
potential x^(l), every CG iteration count, and the sweep outputs (side, order,
k, cut value).  The north_star tolerances (1e-8 relative 2-norm per IRLS
iteration, 1e-12 relative cut value, identical sets) are implied and also
asserted explicitly via `rel2`.
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


def rel2(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def lockstep(I, spec, T, *, eps=1e-6, rtol=1e-3, max_iter=50, norm=0, warm=True, loop_mode=0, record=False):
    """Run GPU irls_init / irls_step and the oracle side by side; compare x^(l)
    and the iteration counts after every step."""
    opts = I.options(eps=eps, T=T, cg_rtol=rtol, cg_max_iter=max_iter, cg_norm=norm, warm_start=int(warm),
                     loop_mode=loop_mode, record_trace=int(record))
    m = I.MinCut.from_spec(spec, opts)
    G = oracle.Graph(spec)
    S = oracle.Solver(G, eps=eps, T=T, cg_rtol=rtol, cg_max_iter=max_iter, cg_norm=norm, warm_start=warm)
    for l in range(T + 1):
        rg = m.irls_init() if l == 0 else m.irls_step()
        ro = S.init() if l == 0 else S.step()
        xg, xo = m.irls_get_potentials(), S.x()
        assert rg["cg_iters"] == ro["cg_iters"], (l, rg["cg_iters"], ro["cg_iters"])
        assert rel2(xg, xo) <= 1e-8, l
        assert np.array_equal(xg.view(np.uint64), xo.view(np.uint64)), f"x^({l}) not bitwise equal"
        assert rg["converged"] == ro["converged"]
        assert rg["rel_res"] == ro["rel_res"]
        if record:
            for k in ("S_eps", "flow_value", "current_s", "true_rel_res", "x_min", "x_max"):
                assert rg[k] == ro[k], (l, k, rg[k], ro[k])
    return m, S


def check_sweep(m, S):
    side, order, k, cut = m.irls_sweep_cut(side=True, order=True)
    sw = S.sweep()
    assert k == sw.k
    assert np.array_equal(side, sw.side)
    assert np.array_equal(order.astype(np.int64), sw.order)
    assert cut == sw.cut_value
    assert abs(cut - sw.cut_value) <= 1e-12 * abs(sw.cut_value)
    return side, k, cut


# --------------------------------------------------------------------------
# SPEC examples and tiny graphs (CSR path)
# --------------------------------------------------------------------------

@pytest.mark.parametrize("name", ["path", "cycle4", "path4", "triangle", "path_sym"])
def test_tiny_graphs(irls, name):
    spec = gen.tiny_graphs()[name]
    m, S = lockstep(irls, spec, T=10, rtol=1e-12, max_iter=100)
    check_sweep(m, S)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_random_small_graphs(irls, seed):
    spec = gen.random_small_graph(300, 500, seed=seed)
    m, S = lockstep(irls, spec, T=8, rtol=1e-8, max_iter=2000, record=True)
    check_sweep(m, S)


# --------------------------------------------------------------------------
# config 1 (BASELINE configs[0]) — stencil, CSR, both norms, full trajectory
# --------------------------------------------------------------------------

def test_config1_stencil_full_trajectory(irls):
    m, S = lockstep(irls, gen.config1(), T=50, rtol=1e-10, max_iter=100000, norm=1)
    side, k, cut = check_sweep(m, S)
    mu, _ = S.maxflow()
    assert cut >= mu * (1 - 1e-12)


def test_config1_csr_equals_stencil(irls):
    spec = gen.config1()
    csr = gen.stencil_to_csr(spec)
    opts = irls.options(T=12, cg_rtol=1e-10, cg_max_iter=100000, cg_norm=1)
    a = irls.MinCut.from_spec(spec, opts)
    b = irls.MinCut.from_spec(csr, opts)
    ra, ta = a.irls_solve(irls.IRLS_FROM_SCRATCH, T=12)
    rb, tb = b.irls_solve(irls.IRLS_FROM_SCRATCH, T=12)
    assert ta == tb
    assert np.array_equal(a.irls_get_potentials(), b.irls_get_potentials())
    sa = a.irls_sweep_cut(order=True)
    sb = b.irls_sweep_cut(order=True)
    assert sa[2] == sb[2] and sa[3] == sb[3]
    assert np.array_equal(sa[0], sb[0]) and np.array_equal(sa[1], sb[1])


def test_config1_preconditioned_norm(irls):
    m, S = lockstep(irls, gen.config1(), T=50, rtol=1e-3, max_iter=50, norm=0, record=True)
    check_sweep(m, S)


# --------------------------------------------------------------------------
# config-2 recipe at reduced size (ragged chunks), paper tolerance
# --------------------------------------------------------------------------

@pytest.mark.parametrize("loop_mode", [0, 1])
def test_blob_grid_ragged(irls, loop_mode):
    spec = gen.blob_grid(40, 36, 29, seed=1, sigma=(3.0, 9.0))
    m, S = lockstep(irls, spec, T=50, loop_mode=loop_mode)
    check_sweep(m, S)


@pytest.mark.parametrize("dims", [(64, 64, 20), (128, 64, 9), (128, 32, 6)])
def test_blob_grid_chunk_planes(irls, dims):
    """Planes that are whole C3 chunks (the geometry of configs 2, 4, 5)."""
    spec = gen.blob_grid(*dims, seed=3, sigma=(3.0, 10.0))
    m, S = lockstep(irls, spec, T=30, record=True)
    check_sweep(m, S)
    m2, S2 = lockstep(irls, spec, T=6, warm=False)


@pytest.mark.parametrize("dims", [(512, 12, 6), (512, 7, 3), (1024, 5, 4), (1536, 3, 4), (512, 16, 5), (512, 8, 37),
                                  (512, 24, 1),
                                  # whole chunks per plane, planes a multiple of 8: the z-cluster K1
                                  (512, 8, 16), (512, 16, 24), (1024, 8, 8)])
def test_fused_reweight_rows_of_512(irls, dims):
    """nx a multiple of 512 (config 4's rows): the single-pass fused reweight
    kernel (-y conductance from the thread's own earlier row, -x by shuffle,
    -z recomputed), with ragged chunks, whole-chunk planes and single planes;
    warm and cold, graph and host loop, trace diagnostics."""
    spec = gen.blob_grid(*dims, seed=6, sigma=(3.0, 9.0))
    m, S = lockstep(irls, spec, T=20, record=True)
    check_sweep(m, S)
    lockstep(irls, spec, T=5, warm=False, loop_mode=1)


def test_blob_grid_cold_start(irls):
    spec = gen.blob_grid(24, 20, 18, seed=7, sigma=(2.0, 6.0))
    m, S = lockstep(irls, spec, T=12, warm=False, record=True)
    check_sweep(m, S)


def test_solve_equals_lockstep_and_reports(irls):
    spec = gen.blob_grid(32, 32, 16, seed=2, sigma=(3.0, 8.0))
    opts = irls.options(T=20)
    m = irls.MinCut.from_spec(spec, opts)
    reps, total = m.irls_solve(irls.IRLS_FROM_SCRATCH, T=20)
    S = oracle.Solver(oracle.Graph(spec), T=20)
    xs, oreps = S.run()
    assert [r["cg_iters"] for r in reps] == [r["cg_iters"] for r in oreps]
    assert total == sum(r["cg_iters"] for r in oreps)
    assert np.array_equal(m.irls_get_potentials(), xs[-1])
    st = m.irls_get_stats()
    assert st["cg_iters"] == total and st["launches"] >= 2 * total


# --------------------------------------------------------------------------
# road-like CSR (config-3 recipe at reduced size)
# --------------------------------------------------------------------------

def test_road_graph_csr(irls):
    spec = gen.road_graph(160, seed=2, knn=60)
    m, S = lockstep(irls, spec, T=50)
    check_sweep(m, S)


# --------------------------------------------------------------------------
# closed form at scale: zero n-links (independent two-edge paths)
# --------------------------------------------------------------------------

def test_zero_nlink_closed_form(irls):
    spec = gen.zero_nlink_grid(96, 80, 33, seed=3, lo=0.05, hi=2.0)
    m = irls.MinCut.from_spec(spec, irls.options(T=4, cg_rtol=1e-14, cg_max_iter=20))
    c1, c2 = spec["cs"], spec["ct"]
    x = c1 / (c1 + c2)
    eps = 1e-6
    for l in range(5):
        m.irls_init() if l == 0 else m.irls_step()
        np.testing.assert_allclose(m.irls_get_potentials(), x, rtol=1e-13, atol=1e-15)
        g1 = c1 ** 2 / np.sqrt(c1 ** 2 * (1 - x) ** 2 + eps ** 2)
        g2 = c2 ** 2 / np.sqrt(c2 ** 2 * x ** 2 + eps ** 2)
        x = g1 / (g1 + g2)


# --------------------------------------------------------------------------
# warm-started sequence (config-5 recipe at reduced size)
# --------------------------------------------------------------------------

def test_terminal_weight_sequence(irls):
    spec = gen.blob_grid(24, 24, 12, seed=1, sigma=(3.0, 8.0))
    T = 10
    opts = irls.options(T=T)
    m = irls.MinCut.from_spec(spec, opts)
    S = oracle.Solver(oracle.Graph(spec), T=T)
    m.irls_solve(irls.IRLS_FROM_SCRATCH, T=T)
    S.run(record=False)
    cs, ct = spec["cs"].copy(), spec["ct"].copy()
    for fs, ft in gen.config5_factors(cs.shape[0], n_problems=3, seed=4):
        cs, ct = cs * fs, ct * ft
        m.irls_set_terminal_weights(cs, ct)
        S.set_terminal_weights(cs, ct)
        reps, tot = m.irls_solve(irls.IRLS_CONTINUE, T=T)
        otot = 0
        for _ in range(T):
            otot += S.step()["cg_iters"]
        assert tot == otot
        assert np.array_equal(m.irls_get_potentials(), S.x())
        check_sweep(m, S)


# --------------------------------------------------------------------------
# sweep edge cases on given potentials (both sides get the same synthetic x)
# --------------------------------------------------------------------------

def test_sweep_ties_signed_zero_out_of_box(irls):
    spec = gen.uniform_grid(37, 29, seed=4)
    n = 37 * 29
    rng = np.random.default_rng(0)
    x = rng.choice([0.0, -0.0, 0.25, 0.5, 1.0, 1.0000001, -3e-5], size=n)
    m = irls.MinCut.from_spec(spec, irls.options(T=1))
    m.irls_set_potentials(x)
    S = oracle.Solver(oracle.Graph(spec), T=1)
    S.set_x(x)
    check_sweep(m, S)
    x[5] = np.nan
    m.irls_set_potentials(x)
    with pytest.raises(irls.IrlsError) as e:
        m.irls_sweep_cut()
    assert e.value.code == 7


def test_sweep_all_equal_and_large(irls):
    spec = gen.uniform_grid(64, 48, seed=5)
    m = irls.MinCut.from_spec(spec, irls.options(T=1))
    S = oracle.Solver(oracle.Graph(spec), T=1)
    for x in (np.zeros(64 * 48), np.full(64 * 48, 0.5), np.linspace(1.0, 0.0, 64 * 48) ** 3):
        m.irls_set_potentials(x)
        S.set_x(x)
        check_sweep(m, S)


# --------------------------------------------------------------------------
# validation codes agree with the oracle
# --------------------------------------------------------------------------

def test_error_codes(irls):
    cases = [gen._csr_edges(3, [(0, 1, -1.0), (1, 2, 1.0)], 0, 2),
             gen._csr_edges(5, [(0, 1, 1.0), (1, 2, 1.0), (3, 4, 1.0)], 0, 2)]
    bad = gen._csr_edges(3, [(0, 1, 1.0), (1, 2, 1.0)], 0, 2)
    bad["w"] = bad["w"].copy(); bad["w"][0] = 5.0
    cases.append(bad)
    for spec in cases:
        try:
            code_o = oracle.Graph(spec).check_nonsingular()
        except oracle.OracleError as e:
            code_o = e.code
        with pytest.raises(irls.IrlsError) as e:
            irls.MinCut.from_spec(spec)
        assert e.value.code == code_o
    st = gen.uniform_grid(5, 5, seed=1)
    st["cx"] = st["cx"].copy(); st["cx"][3] = np.inf
    with pytest.raises(irls.IrlsError) as e:
        irls.MinCut.from_spec(st)
    assert e.value.code == 3
    st = gen.zero_nlink_grid(4, 4, 1, seed=1)
    st["cs"] = st["cs"].copy(); st["ct"] = st["ct"].copy(); st["cs"][2] = 0.0; st["ct"][2] = 0.0
    with pytest.raises(irls.IrlsError) as e:
        irls.MinCut.from_spec(st)
    assert e.value.code == 5


def test_time_kernel_restores_state(irls):
    spec = gen.blob_grid(32, 32, 32, seed=1, sigma=(3.0, 8.0))
    m = irls.MinCut.from_spec(spec, irls.options(T=3))
    m.irls_solve(irls.IRLS_FROM_SCRATCH, T=3)
    x0 = m.irls_get_potentials()
    for w in (0, 1, 2):
        assert m.irls_time_kernel(w, 3) > 0
    assert np.array_equal(x0, m.irls_get_potentials())
    r = m.irls_step()
    S = oracle.Solver(oracle.Graph(spec), T=4)
    S.run(record=False)
    assert np.array_equal(m.irls_get_potentials(), S.x())


# --------------------------------------------------------------------------
# fixed_point_exit: skipped repeats of a frozen step give the same bits
# --------------------------------------------------------------------------

@pytest.mark.parametrize("kind", ["stencil_fused", "stencil_pair", "stencil_odd", "csr"])
@pytest.mark.parametrize("loop_mode", [0, 1])
def test_fixed_point_exit_bitwise(irls, kind, loop_mode):
    """A warm reweight step with 0 CG iterations leaves x unchanged, so every
    later step repeats it; with fixed_point_exit the library skips them on
    the device.  x^(T), every report and the sweep equal the oracle that
    runs all T steps."""
    spec = {"stencil_fused": lambda: gen.blob_grid(512, 8, 6, seed=4, sigma=(3.0, 8.0)),
            "stencil_pair": lambda: gen.blob_grid(64, 40, 12, seed=4, sigma=(3.0, 8.0)),
            "stencil_odd": lambda: gen.blob_grid(33, 17, 9, seed=4, sigma=(3.0, 8.0)),
            "csr": lambda: gen.road_graph(80, seed=2, knn=50)}[kind]()
    T = 30
    m = irls.MinCut.from_spec(spec, irls.options(T=T, fixed_point_exit=1, loop_mode=loop_mode, record_trace=1))
    reps, tot = m.irls_solve(irls.IRLS_FROM_SCRATCH, T=T)
    S = oracle.Solver(oracle.Graph(spec), T=T)
    _, oreps = S.run(record=False)
    assert [r["cg_iters"] for r in reps] == [r["cg_iters"] for r in oreps]
    assert any(r["cg_iters"] == 0 for r in oreps[1:]), "test case never freezes"
    for a, b in zip(reps, oreps):
        for k in ("rel_res", "S_eps", "flow_value", "x_min", "x_max"):
            assert a[k] == b[k], k
    assert np.array_equal(m.irls_get_potentials().view(np.uint64), S.x().view(np.uint64))
    check_sweep(m, S)
    # the kernel timer still times real work after a frozen solve
    assert m.irls_time_kernel(irls.KERNEL_ASSEMBLE, 2) > 0.0


def test_fixed_point_exit_sequence(irls):
    """Config-5 style sequence: every IRLS_CONTINUE after new terminal weights
    runs its first step; results equal the default (every step executed)."""
    spec = gen.blob_grid(64, 64, 16, seed=2, sigma=(3.0, 8.0))
    a = irls.MinCut.from_spec(spec, irls.options(T=10, fixed_point_exit=1))
    b = irls.MinCut.from_spec(spec, irls.options(T=10))
    ra, _ = a.irls_solve(irls.IRLS_FROM_SCRATCH, T=10)
    rb, _ = b.irls_solve(irls.IRLS_FROM_SCRATCH, T=10)
    cs, ct = spec["cs"].copy(), spec["ct"].copy()
    for fs, ft in gen.config5_factors(cs.shape[0], n_problems=3, seed=4):
        cs, ct = cs * fs, ct * ft
        for m in (a, b):
            m.irls_set_terminal_weights(cs, ct)
        ra, ta = a.irls_solve(irls.IRLS_CONTINUE, T=10)
        rb, tb = b.irls_solve(irls.IRLS_CONTINUE, T=10)
        assert [r["cg_iters"] for r in ra] == [r["cg_iters"] for r in rb]
        assert np.array_equal(a.irls_get_potentials(), b.irls_get_potentials())


def test_torch_owned_device_memory(irls):
    """device_alloc / device_free (irls_comm_desc): every array of the context
    is a torch tensor; results bitwise equal to the library pool; everything
    is returned at destroy."""
    import torch
    spec = gen.blob_grid(64, 40, 12, seed=4, sigma=(3.0, 8.0))
    a = irls.MinCut.from_spec(spec, irls.options(T=8))
    ra, ta = a.irls_solve(irls.IRLS_FROM_SCRATCH, T=8)
    sa = a.irls_sweep_cut()
    mem = irls.TorchDeviceMemory(0)
    comm = irls.comm_desc(1, 0, 0, None, torch.cuda.current_stream().cuda_stream, memory=mem)
    b = irls.MinCut.from_spec(spec, irls.options(T=8), comm)
    held = mem.bytes_held
    assert held > 0
    rb, tb = b.irls_solve(irls.IRLS_FROM_SCRATCH, T=8)
    sb = b.irls_sweep_cut()
    tl_b = b.irls_two_level_cut()
    lam_b = b.irls_lambda2(cg_rtol=1e-8, cg_max_iter=10000)
    assert mem.bytes_held > held  # sweep / two-level buffers came from torch too
    assert ta == tb and np.array_equal(a.irls_get_potentials(), b.irls_get_potentials())
    assert sa[2:] == sb[2:] and np.array_equal(sa[0], sb[0])
    assert tl_b[1]["cut_value"] == a.irls_two_level_cut()[1]["cut_value"]
    assert lam_b["lambda2"] == a.irls_lambda2(cg_rtol=1e-8, cg_max_iter=10000)["lambda2"]
    b.close()
    torch.cuda.synchronize()
    assert mem.bytes_held == 0 and not mem.tensors
