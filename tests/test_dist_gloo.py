"""Multi-rank host logic of the z-slab path, world_size 2 over gloo on CPU.

The CUDA/NCCL data path needs GPUs; what is checked here is everything the
ranks must agree on, using the library's own host plan functions:
  - irls_plan_stencil: slabs tile the grid, start/end on plane boundaries and
    own whole C3 groups;
  - irls_halo_plan: exchanging the planned planes fills each ghost plane with
    exactly the neighbour's boundary plane (the library's NCCL halo sends and
    receives these offsets);
  - slot-exact allreduce (C3 step 8): each rank contributes only the group
    sums it owns, the cross-rank SUM is exact, and irls_combine_slots gives
    the single-process C3 result bitwise;
  - gather to rank 0 of the slabs reproduces the global vector.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        import oracle
        from paper_1501_03105_b200 import irls as I

        out = {}
        # ---- slab plans of the BASELINE grids and a small test grid
        for dims in ((512, 512, 256), (128, 128, 128), (16, 16, 64)):
            z0, z1, g0, g1 = I.irls_plan_stencil(*dims, world, rank)
            plans = [None] * world
            dist.all_gather_object(plans, (z0, z1, g0, g1))
            out[dims] = plans

        # ---- CSR id strips (config 3's n~, a ragged one, exactly 8 chunks)
        for nr in (23734786, 39469, 8 * 4096):
            strip = I.irls_plan_csr(nr, world, rank)
            plans = [None] * world
            dist.all_gather_object(plans, strip)
            out[("csr", nr)] = plans
            # slot-exact allreduce over the strip's own C3 groups
            v = np.random.default_rng(nr % 1000).standard_normal(nr)
            gs = oracle.c3_group_sums(v)
            mine = np.zeros(8)
            mine[strip[2]:strip[3]] = gs[strip[2]:strip[3]]
            t = torch.from_numpy(mine.copy())
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            out[("csr_sum", nr)] = I.irls_combine_slots(t.numpy()) == oracle.c3_sum(v)

        # ---- halo exchange with the library's plan
        nx, ny, nz = 16, 16, 64
        N, P = nx * ny * nz, nx * ny
        glob = np.random.default_rng(7).standard_normal(N)
        h = I.irls_halo_plan(nx, ny, nz, world, rank)
        lo = h["first_plane"] * P
        n_own = h["n_own"]
        local = np.full(n_own + 2 * P, np.nan)
        base = P  # local index 0 of the owned range
        local[base:base + n_own] = glob[lo:lo + n_own]
        reqs = []
        bufs = {}
        for side in ("lo", "hi"):
            peer = h["peer_" + side]
            if peer < 0:
                continue
            send = torch.from_numpy(local[base + h["send_" + side]: base + h["send_" + side] + h["count"]].copy())
            bufs[side] = torch.empty(h["count"], dtype=torch.float64)
            reqs.append(dist.isend(send, peer))
            reqs.append(dist.irecv(bufs[side], peer))
        for r in reqs:
            r.wait()
        for side, b in bufs.items():
            off = base + h["recv_" + side]
            local[off:off + h["count"]] = b.numpy()
        ok_lo = h["peer_lo"] < 0 or np.array_equal(local[base - P:base], glob[lo - P:lo])
        ok_hi = h["peer_hi"] < 0 or np.array_equal(local[base + n_own:base + n_own + P],
                                                   glob[lo + n_own:lo + n_own + P])
        out["halo"] = (ok_lo, ok_hi)

        # ---- slot-exact allreduce of C3 group sums
        v = np.random.default_rng(11).standard_normal(N) * 1e3
        gs = oracle.c3_group_sums(v)
        z0, z1, g0, g1 = I.irls_plan_stencil(nx, ny, nz, world, rank)
        mine = np.zeros(8)
        mine[g0:g1] = gs[g0:g1]
        t = torch.from_numpy(mine.copy())
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        out["slots_exact"] = np.array_equal(t.numpy(), gs)
        out["combined"] = I.irls_combine_slots(t.numpy()) == oracle.c3_sum(v)

        # ---- CSR id strips: the library's halo plan (irls_csr_halo_plan, the
        # lists irls_mincut_create_csr builds) drives a real exchange over gloo
        # in the layout the library uses (owned rows, then the ghost block);
        # every ghost slot must receive its node's value, and the strips
        # gathered to rank 0 must rebuild the vector
        from synthetic import generators as gen
        spec = gen.road_graph(300, seed=2, knn=100)   # ~88k non-terminals: 22 chunks
        n, sid, tid = spec["n"], spec["s"], spec["t"]
        keep = np.array([u for u in range(n) if u not in (sid, tid)], dtype=np.int64)
        red = -np.ones(n, dtype=np.int64)
        red[keep] = np.arange(keep.shape[0])
        rp, cl, ww = spec["row_ptr"], spec["col"], spec["w"]
        aptr, aidx = [0], []
        for u in keep:
            nb = sorted({int(red[v]) for v, c in zip(cl[rp[u]:rp[u + 1]], ww[rp[u]:rp[u + 1]])
                         if red[v] >= 0 and c > 0})
            aidx.extend(nb)
            aptr.append(len(aidx))
        aptr = np.array(aptr, dtype=np.int64)
        aidx = np.array(aidx, dtype=np.int32)
        nr = keep.shape[0]
        gv = np.random.default_rng(3).standard_normal(nr)
        hp = I.irls_csr_halo_plan(aptr, aidx, world, rank)
        clo, chi = hp["lo"], hp["hi"]
        loc = np.concatenate([gv[clo:chi], np.full(hp["ghosts"].shape[0], np.nan)])
        reqs, rbufs = [], {}
        for peer in range(world):
            if peer == rank:
                continue
            a, b = hp["send_off"][peer], hp["send_off"][peer + 1]
            if b > a:
                reqs.append(dist.isend(torch.from_numpy(loc[hp["send_idx"][a:b]].copy()), peer))
            a, b = hp["recv_off"][peer], hp["recv_off"][peer + 1]
            if b > a:
                rbufs[peer] = torch.empty(b - a, dtype=torch.float64)
                reqs.append(dist.irecv(rbufs[peer], peer))
        for r in reqs:
            r.wait()
        for peer, buf in rbufs.items():
            a = hp["recv_off"][peer]
            loc[chi - clo + a: chi - clo + a + buf.shape[0]] = buf.numpy()
        ghost_ok = np.array_equal(loc[chi - clo:], gv[hp["ghosts"]])
        # every neighbour of an owned row is owned or a ghost (the SpMV's columns)
        need = {int(v) for r in range(clo, chi) for v in aidx[aptr[r]:aptr[r + 1]] if not clo <= v < chi}
        out["csr_halo"] = (ghost_ok, need == set(hp["ghosts"].tolist()), hp["ghosts"].shape[0] > 0)
        if rank == 0:
            full = np.empty(nr)
            full[clo:chi] = loc[:chi - clo]
            for r in range(1, world):
                pr = I.irls_plan_csr(nr, world, r)
                buf = torch.empty(pr[1] - pr[0], dtype=torch.float64)
                dist.recv(buf, r)
                full[pr[0]:pr[1]] = buf.numpy()
            out["csr_gather"] = np.array_equal(full, gv)
        else:
            dist.send(torch.from_numpy(loc[:chi - clo].copy()), 0)

        # ---- gather of the slabs to rank 0
        mine = torch.from_numpy(glob[lo:lo + n_own].copy())
        if rank == 0:
            full = np.empty(N)
            full[lo:lo + n_own] = glob[lo:lo + n_own]
            for r in range(1, world):
                hr = I.irls_halo_plan(nx, ny, nz, world, r)
                buf = torch.empty(hr["n_own"], dtype=torch.float64)
                dist.recv(buf, r)
                full[hr["first_plane"] * P: hr["first_plane"] * P + hr["n_own"]] = buf.numpy()
            out["gather"] = np.array_equal(full, glob)
        else:
            dist.send(mine, 0)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_csr_halo_exchange_and_gather(results):
    for rank in (0, 1):
        ghost_ok, cover_ok, nonempty = results[rank]["csr_halo"]
        assert ghost_ok and cover_ok and nonempty, rank
    assert results[0]["csr_gather"]


@pytest.fixture(scope="module")
def results():
    from paper_1501_03105_b200 import build
    build.build()
    import oracle
    oracle.build()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_slab_plans_tile_the_grid(results):
    for dims in ((512, 512, 256), (128, 128, 128), (16, 16, 64)):
        plans = results[0][dims]
        assert plans == results[1][dims]
        assert plans[0][0] == 0 and plans[-1][1] == dims[2]
        assert plans[0][1] == plans[1][0]
        assert [p[2:] for p in plans] == [(0, 4), (4, 8)]


def test_csr_strips(results):
    """Id strips tile [0, n~), start on chunk (4096) boundaries, own the C3
    groups [4r, 4r + 4), and the slot allreduce over them is the one-process
    C3 sum bitwise."""
    for nr in (23734786, 39469, 8 * 4096):
        plans = results[0][("csr", nr)]
        assert plans == results[1][("csr", nr)]
        assert plans[0][0] == 0 and plans[-1][1] == nr and plans[0][1] == plans[1][0]
        assert all(p[0] % 4096 == 0 for p in plans)
        assert [p[2:] for p in plans] == [(0, 4), (4, 8)]
        for r in (0, 1):
            assert results[r][("csr_sum", nr)]


def test_halo_plan_exchange(results):
    for r in (0, 1):
        assert results[r]["halo"] == (True, True)


def test_slot_exact_allreduce(results):
    for r in (0, 1):
        assert results[r]["slots_exact"] and results[r]["combined"]


def test_gather_to_root(results):
    assert results[0]["gather"]
