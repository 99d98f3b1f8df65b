"""Pins of the oracle's block-Jacobi preconditioner (A32; SURVEY §8(f)
NEXT #2; "block Jacobi" with exact "LU" blocks) against
things other than itself (CPU only): the partition's defining properties, a
dense LDL^T written out in Python loops (bitwise: the envelope factorisation
must equal the dense algorithm), numpy.linalg.solve of every block, the dense
solve of the whole system, and the one-block limit (M = L~: one iteration)."""
import os

import numpy as np
import pytest

import oracle
from synthetic import generators as gen
from tests import helpers as H


def solver(spec, **kw):
    return oracle.Solver(oracle.Graph(spec), **kw)


def groups(n):
    K = (n + 4095) // 4096
    return [(min(n, 4096 * (g * K // 8)), min(n, 4096 * ((g + 1) * K // 8))) for g in range(8)]


def adjacency(spec):
    sysm = H.ContractSystem(spec)
    nbr = [[int(v) for v in row if v >= 0] for row in sysm.nbr]
    return sysm, nbr


CASES = [("random", gen.random_small_graph(300, 500, seed=41)),
         ("blob", gen.blob_grid(20, 18, 7, seed=3, sigma=(2.0, 5.0))),
         ("road", gen.road_graph(45, seed=2, knn=25)),
         ("ragged", gen.blob_grid(64, 40, 6, seed=8, sigma=(3.0, 9.0)))]   # 15,360 nodes: 4 chunks, 8 groups


@pytest.mark.parametrize("B", [1, 7, 64])
@pytest.mark.parametrize("name,spec", CASES, ids=[c[0] for c in CASES])
def test_partition_definition(name, spec, B):
    """Every node in exactly one block; blocks <= B nodes, inside one C3
    group, each connected through its BFS parents; a block is a BFS of the
    group's unassigned nodes from its lowest-id free root (no block could
    have grown: it is full or it has no free in-group neighbour left)."""
    S = solver(spec, block_size=B)
    bptr, bnode, bfirst, boff = S.blocks()
    sysm, nbr = adjacency(spec)
    n = sysm.n
    assert sorted(bnode.tolist()) == list(range(n))
    gl = groups(n)
    gid = np.zeros(n, dtype=np.int64)
    for g, (lo, hi) in enumerate(gl):
        gid[lo:hi] = g
    blk = np.zeros(n, dtype=np.int64)
    for b in range(len(bptr) - 1):
        blk[bnode[bptr[b]:bptr[b + 1]]] = b
    seen_before = set()
    for b in range(len(bptr) - 1):
        nodes = bnode[bptr[b]:bptr[b + 1]].tolist()
        assert 1 <= len(nodes) <= B
        assert len({int(gid[u]) for u in nodes}) == 1
        # root: the lowest id not in an earlier block of its group
        g = int(gid[nodes[0]])
        free = [u for u in range(*gl[g]) if u not in seen_before]
        assert nodes[0] == min(free)
        # BFS discovery order: each later node is a neighbour of an earlier one, and
        # its first in-block neighbour (by position) is where it was discovered
        pos = {u: i for i, u in enumerate(nodes)}
        for i, u in enumerate(nodes[1:], start=1):
            earlier = [pos[w] for w in nbr[u] if w in pos and pos[w] < i]
            assert earlier, "not connected to an earlier node of its block"
            assert bfirst[bptr[b] + i] == min(earlier)
        # maximal: a non-full block has no free in-group neighbour
        if len(nodes) < B:
            for u in nodes:
                for w in nbr[u]:
                    if gid[w] == g and w not in seen_before:
                        assert w in pos
        seen_before.update(nodes)


def dense_ldlt(A):
    """LDL^T of a dense SPD matrix by rows (Crout), every sum over k ascending,
    products ((L_ik * L_jk) * d_k) — written from A32's definition."""
    m = A.shape[0]
    L = np.zeros((m, m))
    d = np.zeros(m)
    for i in range(m):
        for j in range(i):
            acc = A[i, j]
            for k in range(j):
                acc = acc - (L[i, k] * L[j, k]) * d[k]
            L[i, j] = acc / d[j]
        acc = A[i, i]
        for k in range(i):
            acc = acc - (L[i, k] * L[i, k]) * d[k]
        d[i] = acc
    return L, d


def block_matrices(S, spec, x=None, eps=1e-6):
    """The blocks A_B of L~ (init, or reweighted at x), assembled in numpy
    (tests/helpers.ContractSystem, Eq. 4/7/8), with the oracle's partition."""
    sysm = H.ContractSystem(spec)
    g, D, _, b = sysm.assemble(x, eps)
    bptr, bnode, bfirst, boff = S.blocks()
    out = []
    for i in range(len(bptr) - 1):
        nodes = bnode[bptr[i]:bptr[i + 1]]
        pos = {int(u): k for k, u in enumerate(nodes)}
        A = np.diag(D[nodes])
        for k, u in enumerate(nodes):
            for j, v in enumerate(sysm.nbr[u]):
                if v >= 0 and int(v) in pos:
                    A[k, pos[int(v)]] = -g[u, j]
        out.append((nodes, bptr[i], A))
    return out, bfirst, boff


def dense_system(spec, x=None, eps=1e-6):
    n, s, t, E = H.edge_list(spec)
    keep = np.array([i for i in range(n) if i not in (s, t)], dtype=np.int64)
    xf = None if x is None else H.full_potentials(n, s, t, keep, x)
    Lr, b, _ = H.dense_irls_system(n, s, t, E, x=xf, eps=eps)
    return Lr, b


@pytest.mark.parametrize("name,spec", CASES[:3], ids=[c[0] for c in CASES[:3]])
def test_factor_equals_dense_ldlt_bitwise(name, spec):
    """The envelope factorisation equals the dense algorithm bit for bit (the
    dense matrix's entries taken from the oracle's own assembly, so only the
    factorisation is compared); and L D L^T = A_B to rounding against the
    numpy-assembled block."""
    B = 24
    S = solver(spec, block_size=B, T=1)
    xs, _ = S.run()
    x = xs[0]
    a = S.assemble(x)
    z, env, Dd = S.precond(np.ones(S.n), x=x)
    blocks, bfirst, boff = block_matrices(S, spec, x=x)
    sysm = H.ContractSystem(spec)
    g_of, e = {}, 0
    for u in range(sysm.n):          # the oracle's g per adjacency entry, ascending neighbours
        for v in sysm.nbr[u]:
            if v >= 0:
                g_of[(u, int(v))] = a["g"][e]
                e += 1
    for nodes, p0, Ai in blocks[:40]:
        m = len(nodes)
        A = np.diag(a["D"][nodes])
        for i, u in enumerate(nodes):
            for j, v in enumerate(nodes):
                if (int(u), int(v)) in g_of:
                    A[i, j] = -g_of[(int(u), int(v))]
        L, d = dense_ldlt(A)
        assert np.array_equal(d, Dd[p0:p0 + m])
        for i in range(m):
            f = bfirst[p0 + i]
            assert np.array_equal(env[boff[p0 + i]:boff[p0 + i + 1]], L[i, f:i]), (i, f)
            assert np.all(L[i, :f] == 0.0)
        U = L + np.eye(m)                                  # unit lower factor
        np.testing.assert_allclose(U @ np.diag(d) @ U.T, Ai, rtol=1e-11, atol=1e-11 * np.abs(Ai).max())


@pytest.mark.parametrize("B", [5, 64, 300])
@pytest.mark.parametrize("name,spec", CASES, ids=[c[0] for c in CASES])
def test_apply_equals_block_solves(name, spec, B):
    """z = M^-1 r equals numpy.linalg.solve of every block (init and a
    reweighted system), within the block's condition number x rounding."""
    S = solver(spec, block_size=B, T=1)
    xs, _ = S.run()
    rng = np.random.default_rng(5)
    for x in (None, xs[1]):
        r = rng.standard_normal(S.n)
        z, _, _ = S.precond(r, x=x)
        blocks, _, _ = block_matrices(S, spec, x=x)
        for nodes, _, A in blocks:
            zb = np.linalg.solve(A, r[nodes])
            bound = 1e-14 * len(nodes) * np.linalg.cond(A) * np.linalg.norm(zb) + 1e-300
            assert np.linalg.norm(z[nodes] - zb) <= bound


@pytest.mark.parametrize("name,spec", CASES[:3], ids=[c[0] for c in CASES[:3]])
def test_block_pcg_converges_to_dense_solve(name, spec):
    """O5 with the block M at tight tolerance solves L~ v = b (dense solve),
    init and one reweighted step."""
    S = solver(spec, block_size=64, T=1, cg_rtol=1e-13, cg_max_iter=20000)
    S.init()
    Lr, b = dense_system(spec)
    np.testing.assert_allclose(S.x(), np.linalg.solve(Lr, b), rtol=1e-8, atol=1e-11)
    x0 = S.x()
    S.step()
    Lr, b = dense_system(spec, x=x0)
    np.testing.assert_allclose(S.x(), np.linalg.solve(Lr, b), rtol=1e-7, atol=1e-10)


def test_one_block_is_a_direct_solve():
    """n <= 4096 and B >= n on a connected graph: one block, M = L~, so the
    first PCG iteration lands on the solution (the second test stops it)."""
    spec = gen.random_small_graph(400, 600, seed=12)
    S = solver(spec, block_size=4096, T=3, cg_rtol=1e-6, cg_max_iter=100)
    bptr, _, _, _ = S.blocks()
    assert len(bptr) == 2
    xs, reps = S.run()
    assert [r["cg_iters"] for r in reps] == [1, 1, 1, 1]
    assert all(r["true_rel_res"] < 1e-7 for r in reps)


def test_unit_blocks_match_point_jacobi():
    """B = 1: M = diag(L~) up to rounding (r / D instead of r * (1/D)): the
    same solution at tight tolerance, the same iteration counts at the
    paper's tolerance up to rounding flips."""
    spec = CASES[1][1]
    a = solver(spec, block_size=1, T=5, cg_rtol=1e-12, cg_max_iter=10000)
    b = solver(spec, block_size=0, T=5, cg_rtol=1e-12, cg_max_iter=10000)
    xa, _ = a.run(); xb, _ = b.run()
    np.testing.assert_allclose(xa, xb, rtol=1e-9, atol=1e-12)


def test_block_options_rejected_with_cgcg():
    with pytest.raises(MemoryError):
        solver(CASES[0][1], block_size=8, cg_variant=1)


def test_blocks_cut_quality_not_worse_on_road():
    """The reason for NEXT #2: at the paper's policy the
    block preconditioner carries information further per iteration; on a
    small road graph its sweep cut is no worse than point Jacobi's."""
    spec = gen.road_graph(120, seed=2, knn=60)
    cuts = {}
    for B in (0, 256):
        S = solver(spec, block_size=B, T=50)
        S.run(record=False)
        cuts[B] = S.sweep().cut_value
    assert cuts[256] <= cuts[0] * (1 + 1e-12)
