"""The GPU preparation of a CSR graph at create (csr_prep.cu: validation,
duplicate merge in CSR order (A7), exact symmetry, terminal split, c_st
(A5), F, Prop. 1 / A8, SELL-64) against the host preparation
(IRLS_HOST_CSR_PREP=1) and the oracle: the same error code for every bad
input, and — on graphs with unsorted rows, repeated entries (summed in CSR
order, so the merged capacities are order-sensitive), zero weights, a direct
s-t edge and terminal rows — bitwise the same potentials, iteration counts
and sweep."""
import os

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


def _create(I, spec, host, T=6):
    if host:
        os.environ["IRLS_HOST_CSR_PREP"] = "1"
    try:
        return I.MinCut.from_spec(spec, I.options(T=T))
    finally:
        os.environ.pop("IRLS_HOST_CSR_PREP", None)


def _messy(seed, n=3000, m=6000):
    """Symmetric CSR with shuffled rows, duplicate (u, v) entries split into
    parts (summed in CSR order), zero-weight edges, and an s-t edge."""
    rng = np.random.default_rng(seed)
    spec = gen.random_small_graph(n, m, seed=seed)
    rp, col, w = spec["row_ptr"], spec["col"], spec["w"]
    rows = []
    for u in range(n):
        ent = [(int(v), float(x)) for v, x in zip(col[rp[u]:rp[u + 1]], w[rp[u]:rp[u + 1]])]
        rows.append(ent)
    # split some undirected edges into two parts, the same split on both sides
    parts = {}
    for u in range(n):
        for v, x in rows[u]:
            if u < v and rng.random() < 0.2:
                a = float(rng.uniform(0.1, 0.9)) * x
                parts[(u, v)] = (a, x - a)
    new = [[] for _ in range(n)]
    for u in range(n):
        for v, x in rows[u]:
            key = (min(u, v), max(u, v))
            if key in parts:
                a, b = parts[key]
                new[u].append((v, a)); new[u].append((v, b))
            else:
                new[u].append((v, x))
    for u, v in ((5, 17), (17, 5)):
        new[u].append((v, 0.0))                                     # zero-weight edge
    s, t = spec["s"], spec["t"]
    new[s].append((t, 0.75)); new[t].append((s, 0.75))              # direct s-t edge (A5)
    row_ptr = [0]; cc = []; ww = []
    for u in range(n):
        ent = new[u]
        order = rng.permutation(len(ent))
        for i in order:
            cc.append(ent[i][0]); ww.append(ent[i][1])
        row_ptr.append(len(cc))
    return dict(kind="csr", n=n, row_ptr=np.array(row_ptr, np.int64), col=np.array(cc, np.int32),
                w=np.array(ww, np.float64), s=s, t=t)


@pytest.mark.parametrize("seed", [0, 1])
def test_gpu_prep_equals_host_prep_and_oracle(irls, seed):
    spec = _messy(seed)
    T = 6
    a = _create(irls, spec, host=False, T=T)
    b = _create(irls, spec, host=True, T=T)
    ra, ta = a.irls_solve(irls.IRLS_FROM_SCRATCH, T=T)
    rb, tb = b.irls_solve(irls.IRLS_FROM_SCRATCH, T=T)
    S = oracle.Solver(oracle.Graph(spec), T=T)
    xs, oreps = S.run()
    assert [r["cg_iters"] for r in ra] == [r["cg_iters"] for r in rb] == [r["cg_iters"] for r in oreps]
    xa, xb = a.irls_get_potentials(), b.irls_get_potentials()
    assert np.array_equal(xa.view(np.uint64), xb.view(np.uint64))
    assert np.array_equal(xa.view(np.uint64), xs[-1].view(np.uint64))
    sa, oa, ka, ca = a.irls_sweep_cut(order=True)
    sb, ob, kb, cb = b.irls_sweep_cut(order=True)
    sw = S.sweep()
    assert ka == kb == sw.k and ca == cb == sw.cut_value
    assert np.array_equal(sa, sb) and np.array_equal(oa, ob)
    assert a.irls_get_stats()["n_links"] == b.irls_get_stats()["n_links"]
    # the kept components drive set_terminal_weights' A8 check identically
    cs, ct = oracle.Graph(spec).terminals()
    a.irls_set_terminal_weights(cs * 1.5, ct * 0.5)
    b.irls_set_terminal_weights(cs * 1.5, ct * 0.5)


def test_road_like_equal(irls):
    spec = gen.road_graph(150, seed=2, knn=80)
    a = _create(irls, spec, host=False)
    b = _create(irls, spec, host=True)
    a.irls_solve(irls.IRLS_FROM_SCRATCH, T=6)
    b.irls_solve(irls.IRLS_FROM_SCRATCH, T=6)
    assert np.array_equal(a.irls_get_potentials(), b.irls_get_potentials())


def _bad_cases():
    good = gen._csr_edges(4, [(0, 1, 1.0), (1, 2, 2.0), (2, 3, 1.0)], 0, 3)
    out = []
    for name, mut in (("negative", lambda w, c: w.__setitem__(1, -1.0)),
                      ("nan", lambda w, c: w.__setitem__(2, np.nan)),
                      ("inf", lambda w, c: w.__setitem__(0, np.inf)),
                      ("col_oob", lambda w, c: c.__setitem__(1, 9)),
                      ("col_negative", lambda w, c: c.__setitem__(3, -2))):
        spec = dict(good)
        spec["w"] = good["w"].copy(); spec["col"] = good["col"].copy()
        mut(spec["w"], spec["col"])
        out.append((name, spec))
    # asymmetric weight
    spec = dict(good); spec["w"] = good["w"].copy(); spec["w"][1] = 1.5
    out.append(("asymmetric", spec))
    # self loop
    out.append(("self_loop", gen._csr_edges(4, [(0, 1, 1.0), (1, 2, 2.0), (2, 3, 1.0)], 0, 3)))
    rp, col = out[-1][1]["row_ptr"], out[-1][1]["col"].copy()
    col[rp[1]] = 1
    out[-1][1]["col"] = col
    # singular: a component without a terminal edge (A8)
    out.append(("singular", gen._csr_edges(6, [(0, 1, 1.0), (1, 2, 1.0), (3, 4, 1.0)], 0, 2)))
    return out


@pytest.mark.parametrize("name,spec", _bad_cases(), ids=[c[0] for c in _bad_cases()])
def test_error_codes_match_host_and_oracle(irls, name, spec):
    codes = []
    for host in (False, True):
        with pytest.raises(irls.IrlsError) as e:
            _create(irls, spec, host=host)
        codes.append(e.value.code)
    try:
        code_o = oracle.Graph(spec).check_nonsingular()
    except oracle.OracleError as e:
        code_o = e.code
    assert codes[0] == codes[1] == code_o, (name, codes, code_o)
