"""The library's exact coarse max-flow (Boykov-Kolmogorov on the host,
maxflow.cu) against the oracle's Edmonds-Karp on the same fixed-point coarse
graphs (CPU only; the second level of two-level rounding).  Both
must return the same flow value and the same minimal min-cut source side
(bit-exact integers, A28)."""
import numpy as np
import pytest

import oracle
from synthetic import generators as gen


@pytest.fixture(scope="module")
def L():
    from paper_1501_03105_b200 import build, irls
    build.build()
    return irls


def coarse_of(spec, x, g0, g1):
    S = oracle.Solver(oracle.Graph(spec))
    return S.coarsen(x, g0, g1)


def check(L, co):
    f_o, src_o = oracle.maxflow_coarse(co.nc, co.ptr, co.col, co.cap, co.qs, co.qt, co.qst)
    f_l, src_l, cert = L.irls_coarse_maxflow(co.nc, co.ptr.astype(np.int32), co.col.astype(np.int32), co.cap,
                                             co.qs, co.qt)
    assert cert == 1
    assert f_l + co.qst == f_o
    assert src_l.tolist() == src_o.tolist()


@pytest.mark.parametrize("seed", range(8))
def test_bk_matches_oracle_random_graphs(L, seed):
    spec = gen.random_small_graph(60 + 10 * seed, 90 + 15 * seed, seed=700 + seed)
    rng = np.random.default_rng(seed)
    n = spec["n"] - 2
    x = rng.uniform(0.0, 1.0, n)
    check(L, coarse_of(spec, x, 0.15, 0.85))


@pytest.mark.parametrize("shape", [(24, 20, 1), (9, 8, 7), (40, 3, 2)])
def test_bk_matches_oracle_whole_grid(L, shape):
    """No coarsening (every node in Sc): the exact min cut of a blob grid."""
    nx, ny, nz = shape
    spec = gen.blob_grid(nx, ny, nz, seed=11, n_blobs=4, sigma=(2.0, 5.0))
    x = np.full(nx * ny * nz, 0.5)
    co = coarse_of(spec, x, 0.1, 0.9)
    assert co.nc == nx * ny * nz
    check(L, co)


def test_bk_ties_and_zero_graph(L):
    """Unit 4-cycle (several optima): minimal source side is empty; a graph
    with no Sc nodes gives flow 0."""
    spec = gen.tiny_graphs()["cycle4"]
    co = coarse_of(spec, np.array([0.5, 0.5]), 0.1, 0.9)
    check(L, co)
    f, src, cert = L.irls_coarse_maxflow(0, np.zeros(1, np.int32), [], [], [], [])
    assert f == 0 and cert == 1


def test_bk_rejects_asymmetric(L):
    with pytest.raises(L.IrlsError):
        L.irls_coarse_maxflow(2, np.array([0, 1, 1], np.int32), np.array([1], np.int32), [5], [1, 0], [0, 1])


def test_bk_components_in_parallel(L):
    """Many components solved on host threads (the path large coarse graphs
    take; enabled here for a small graph through IRLS_MAXFLOW_PAR_MIN, read
    once per process — set by conftest for the whole session): the same flow
    and minimal source side as the oracle's Edmonds-Karp."""
    import numpy as np
    parts, off = [], 0
    for k in range(8):
        sp = gen.blob_grid(40, 25, 2, seed=100 + k, n_blobs=3, sigma=(2.0, 6.0))
        parts.append((sp, off))
        off += 40 * 25 * 2
    # one block-diagonal coarse graph: every node in Sc, components = the grids
    cos = []
    for sp, o in parts:
        co = coarse_of(sp, np.full(40 * 25 * 2, 0.5), 0.1, 0.9)
        cos.append((co, o))
    nc = off
    ptr = [0]
    col, cap, qs, qt = [], [], [], []
    for co, o in cos:
        for u in range(co.nc):
            for e in range(co.ptr[u], co.ptr[u + 1]):
                col.append(int(co.col[e]) + o)
                cap.append(co.cap[e])
            ptr.append(len(col))
        qs += co.qs
        qt += co.qt
    f_l, src_l, cert = L.irls_coarse_maxflow(nc, np.array(ptr, np.int32), np.array(col, np.int32), cap, qs, qt)
    f_o, src_o = oracle.maxflow_coarse(nc, np.array(ptr), np.array(col), cap, qs, qt, 0)
    assert cert == 1 and f_l == f_o and src_l.tolist() == src_o.tolist()
