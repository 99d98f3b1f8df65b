#!/usr/bin/env python
"""Benchmark of the IRLS s-t min-cut hot path (BASELINE.json metric).

One "step" = one whole pass of the hot path over the workload: irls_solve
(x^(0) + T=50 reweight/assemble/PCG steps, eps=1e-6, PCG rtol 1e-3 in the
preconditioned norm, cap 50, warm start) followed by the GPU sweep cut.
Workload (N=1): BASELINE configs[3], the 512x512x256 blob grid (67.1M
non-terminals, 200.8M n-links) — the largest config and the one the scaling
target is quoted on.  With torchrun (N>1) it is z-slab partitioned (strong
scaling: total work fixed).

value  = CG edge-visits per second of the whole job = |E~| * (CG iterations
         per solve) * K / (device time of K steps, max over ranks), inputs
         resident in HBM (uploaded by create, untimed);
e2e    = the same metric through the C ABI with pinned HOST buffers: create
         (H2D of the capacities) + solve + sweep (D2H of the cut side) +
         destroy inside the timed region;
roofline = the dominant kernel (K3: fused p-update + SpMV + p.q), timed with
         CUDA events on the library's stream;
cpu_baseline = the float64 CPU oracle (OpenMP, every host core) on the whole
         workload graph: x^(0) + 3 IRLS steps + the sweep.

`--impl reference` times the oracle (the reference arm of this tier).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "CG edge-visits/s (GEdge/s) of the IRLS min-cut hot path (solve + sweep cut)"
UNIT = "GEdge/s"
K3_BYTES_PER_NODE = 80   # read z,p_old,x,gx,gy,gz,D (56) + write p,q,x (24)
K5_BYTES_PER_NODE = 40   # read r,q,Dinv (24) + write r,z (16)
K1_BYTES_PER_NODE = 104  # read x,cx,cy,cz,cs,ct (48) + write gx,gy,gz,D,Dinv,r,z (56)


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def workload(name):
    from synthetic import generators as gen
    if name == "config4":
        return gen.config4(), "config4: 512x512x256 6-neighbour blob grid (BASELINE configs[3]), seed 3"
    if name == "config3":
        return gen.config3(), "config3: 4900^2 road-like CSR graph, 30% edges deleted, LCC (BASELINE configs[2]), seed 2"
    if name == "config2":
        return gen.config2(), "config2: 128^3 6-neighbour blob grid (BASELINE configs[1]), seed 1"
    if name == "config1":
        return gen.config1(), "config1: 32x32 4-neighbour grid (BASELINE configs[0]), seed 0"
    raise SystemExit(f"unknown config {name}")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for s in self.samples for n, v in zip(names, s[3:]) if v.strip().lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# oracle (cpu_baseline and the reference arm)
# ---------------------------------------------------------------------------

def oracle_sample(spec, planes=None, T=3, sweep=True):
    """The float64 oracle (OpenMP over C3 chunks and node loops, every host
    core; bitwise thread-invariant) on the workload: the whole graph
    (planes=None) or its first `planes` z-planes, init + T IRLS steps (cap 50,
    rtol 1e-3) + the sweep.  Returns (GEdge/s, seconds, threads, description)."""
    import oracle
    threads = oracle.set_num_threads(os.cpu_count() or 1)
    if spec["kind"] == "csr":
        sub, what = spec, "the whole workload"
        if planes is not None:  # a bounded instance of the config-3 recipe
            from synthetic import generators as gen
            sub, what = gen.road_graph(1000, seed=2, knn=200), "the config-3 recipe at 1000^2"
    elif planes is None:
        sub, what = spec, "the whole workload"
    else:
        n = spec["nx"] * spec["ny"] * planes
        sub = dict(spec)
        sub["nz"] = planes
        for k in ("cx", "cy", "cz", "cs", "ct"):
            sub[k] = np.ascontiguousarray(spec[k][:n])
        what = f"z-planes 0..{planes - 1} of the workload"
    t0 = time.perf_counter()
    G = oracle.Graph(sub)
    S = oracle.Solver(G, T=T)
    links = G.nnz // 2
    t1 = time.perf_counter()
    _, reps = S.run(record=False)
    if sweep:
        S.sweep()
    dt = time.perf_counter() - t1
    iters = sum(r["cg_iters"] for r in reps)
    desc = (f"oracle (plain C, OpenMP, {threads} threads) on {what} ({G.n} nodes, {links} n-links): "
            f"init + {T} IRLS steps{' + sweep' if sweep else ''}, {iters} CG iterations in {dt:.1f} s "
            f"(graph build {t1 - t0:.1f} s untimed)")
    return links * iters / dt / 1e9, dt, threads, desc


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    spec, wdesc = workload(args.config)
    import oracle
    oracle.build()
    for _ in range(args.warmup if args.warmup < 1 else 1):
        oracle_sample(spec, planes=args.ref_planes, T=args.ref_T)
    vals, times = [], []
    desc, cores = "", 1
    for _ in range(args.steps):
        v, dt, cores, desc = oracle_sample(spec, planes=args.ref_planes, T=args.ref_T)
        vals.append(v)
        times.append(dt)
    val = statistics.median(vals)
    line = {"metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(times), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wdesc, "sample": desc}, "impl": "reference",
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# the GPU arm
# ---------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--config", default="config4")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--e2e-serial", action="store_true", help="e2e: one step after the other (no create/solve overlap)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-planes", type=int, default=16,
                    help="reference arm: z-planes of the workload per step (bounded so K steps end in minutes)")
    ap.add_argument("--ref-T", type=int, default=3)
    ap.add_argument("--cpu-T", type=int, default=3, help="cpu_baseline: IRLS steps after x^(0) on the whole graph")
    ap.add_argument("--loop-mode", type=int, default=0,
                    help="0: CUDA graphs with device-side loops (NCCL / peer stores captured on N > 1); 1: host loop")
    ap.add_argument("--no-two-level", action="store_true")
    ap.add_argument("--no-fixed-point-exit", action="store_true")
    ap.add_argument("--cg-variant", default="hs", choices=["hs", "cg"],
                    help="PCG form: Hestenes-Stiefel (default) or Chronopoulos-Gear (one reduction per iteration)")
    ap.add_argument("--p2p", type=int, default=1, choices=[0, 1],
                    help="N>1: per-iteration collectives over peer memory (irls_options.p2p: slot sums and the z "
                         "halo stored by the kernels that produce them; falls back to NCCL if the peer mapping "
                         "fails at create) or, 0, NCCL")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_1501_03105_b200 import build, irls as I
    if rank == 0:
        build.build()
    if world > 1:
        dist.barrier()

    spec, wdesc = workload(args.config)
    T = 50
    cgv = I.IRLS_CG_CG if args.cg_variant == "cg" else I.IRLS_CG_HS
    opts = I.options(T=T, loop_mode=args.loop_mode, p2p=args.p2p, cg_variant=cgv)
    stream = torch.cuda.current_stream()
    uid = None
    if world > 1:
        obj = [I.irls_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    # device memory: torch's caching allocator owns every array of the contexts
    mem = I.TorchDeviceMemory(local)
    comm = I.comm_desc(world, rank, local, uid, stream.cuda_stream, memory=mem)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def fresh_comm():
        """A new NCCL id for every communicator (an id serves one create)."""
        if world == 1:
            return comm
        obj = [I.irls_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return I.comm_desc(world, rank, local, obj[0], stream.cuda_stream, memory=mem)

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident value -------------------------------------------
    m, p2p_note = None, None
    try:
        m = I.MinCut.from_spec(spec, opts, comm)
        ok = 1
    except I.IrlsError as e:
        if world == 1 or not args.p2p:
            raise
        ok, p2p_note = 0, f"p2p create failed ({e}); NCCL collectives used"
    if world > 1 and args.p2p:
        t = torch.tensor([ok], dtype=torch.int32, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        if int(t.item()) == 0:  # every rank falls back together (collective create)
            if m is not None:
                m.close()
            args.p2p = 0
            p2p_note = p2p_note or "a peer's p2p create failed; NCCL collectives used"
            opts = I.options(T=T, loop_mode=args.loop_mode, p2p=0, cg_variant=cgv)
            m = I.MinCut.from_spec(spec, opts, fresh_comm())
    st = m.irls_get_stats()
    n_links = st["n_links"]
    for _ in range(args.warmup):
        m.irls_solve(I.IRLS_FROM_SCRATCH, T=T, reports=False)
        m.irls_sweep_cut(side=False)
    barrier()
    iters_per_step, launches = [], 0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            _, tot = m.irls_solve(I.IRLS_FROM_SCRATCH, T=T, reports=False)
            launches += m.irls_get_stats()["launches"]
            _, _, k, cut = m.irls_sweep_cut(side=False)
            launches += m.irls_get_stats()["launches"]
            iters_per_step.append(tot)
        ev1.record(stream)
        barrier()
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    total_iters = sum(iters_per_step)
    value = n_links * total_iters / (ms * 1e-3) / 1e9
    clocks = clk.summary()

    # ---- the same steps with fixed_point_exit (an exact shortcut, reported
    # beside the headline, which executes every one of the T + 1 solves): a
    # warm reweight step that stops before its first CG iteration leaves x
    # unchanged, so the remaining steps repeat it bit for bit; the library
    # skips them on the device.  Same x^(T), same reports, same cut.
    fpx = None
    if not args.no_fixed_point_exit:
        m.close()
        m = I.MinCut.from_spec(spec, I.options(T=T, loop_mode=args.loop_mode, fixed_point_exit=1, p2p=args.p2p,
                                               cg_variant=cgv), fresh_comm())
        for _ in range(args.warmup):
            m.irls_solve(I.IRLS_FROM_SCRATCH, T=T, reports=False)
            m.irls_sweep_cut(side=False)
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        fit, frep = 0, None
        for _ in range(args.steps):
            frep, tot = m.irls_solve(I.IRLS_FROM_SCRATCH, T=T, reports=True)
            _, _, fk, fcut = m.irls_sweep_cut(side=False)
            fit += tot
        f1.record(stream)
        barrier()
        fms = max_over_ranks(f0.elapsed_time(f1))
        first0 = next((i for i, r in enumerate(frep) if i > 0 and r["cg_iters"] == 0), T)
        fpx = {"value": n_links * fit / (fms * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": fms / args.steps,
               "cg_iters_per_step": fit // args.steps, "solves_executed": min(first0 + 1, T + 1),
               "solves_total": T + 1, "same_cut": bool(fcut == cut and fk == k),
               "what": "irls_options.fixed_point_exit = 1: steps after the first warm reweight step with 0 CG "
                       "iterations are skipped on the device (bitwise the same x^(T) and reports); "
                       "not the headline"}

    # ---- dominant kernel roofline (CUDA events on the library stream) ------
    peaks = measured_peaks()
    peak = peaks.get("hbm_gbs", 6650.0)
    n_own = st["n_local"]
    t_k3 = m.irls_time_kernel(I.KERNEL_PSPMV, 20)
    t_k5 = m.irls_time_kernel(I.KERNEL_AXPY, 20)
    t_k1 = m.irls_time_kernel(I.KERNEL_ASSEMBLE, 10)
    csr = spec["kind"] == "csr"
    # algorithmic bytes per launch; CSR: K3 56 B/node + 12 B per
    # stored entry, K1 56 B/node + 20 B per entry (this rank's rows)
    ent = 2 * n_links * n_own / max(st["n_nonterminal"], 1)
    k3_bytes = (56 * n_own + 12 * ent) if csr else K3_BYTES_PER_NODE * n_own
    k1_bytes = (56 * n_own + 20 * ent) if csr else K1_BYTES_PER_NODE * n_own
    ach = k3_bytes / (t_k3 * 1e-3) / 1e9
    traffic = None
    try:  # per-launch DRAM bytes of K3 from the committed ncu --set full capture (same config)
        tj = json.load(open(os.path.join(ROOT, "profiles", "r02_k3_traffic.json")))
        if args.config == "config4" and world == 1:
            traffic = tj["traffic_GB_per_launch"] / (t_k3 * 1e-3)
    except Exception:
        pass
    kernels = {
        "K3_pspmv": {"ms": t_k3, "GBps": ach, "bytes_per_launch": k3_bytes},
        "K5_axpy_jacobi": {"ms": t_k5, "GBps": K5_BYTES_PER_NODE * n_own / (t_k5 * 1e-3) / 1e9,
                           "bytes_per_node": K5_BYTES_PER_NODE},
        "K1_reweight_assemble": {"ms": t_k1, "GBps": k1_bytes / (t_k1 * 1e-3) / 1e9,
                                 "bytes_per_node": K1_BYTES_PER_NODE},
    }
    cg_iter_ms = t_k3 + t_k5
    roof_name = "K3 fused p-update + SpMV + p.q " + ("(SELL-64 CSR)" if csr else "(stencil)")
    roof_bytes, roof_ms = k3_bytes, t_k3
    if cgv == I.IRLS_CG_CG:  # the single kernel of a Chronopoulos-Gear iteration
        t_cg = m.irls_time_kernel(I.KERNEL_CGCG, 20)
        cg_bytes = (96 * n_own + 12 * ent) if csr else 120 * n_own
        kernels["CGCG_iteration"] = {"ms": t_cg, "GBps": cg_bytes / (t_cg * 1e-3) / 1e9, "bytes_per_launch": cg_bytes}
        cg_iter_ms = t_cg
        roof_name, roof_bytes, roof_ms = "Chronopoulos-Gear iteration (one kernel)", cg_bytes, t_cg
        ach = roof_bytes / (roof_ms * 1e-3) / 1e9
        traffic = None
    # ---- N > 1: the z halo against the NVLink roofline (the bytes each rank
    # sends per CG iteration over the measured 770 GB/s per-direction peer
    # bandwidth of B200_PROFILING.md; 900 GB/s nominal)
    nvlink = None
    if world > 1:
        t_halo = max_over_ranks(m.irls_time_kernel(I.KERNEL_HALO, 20))
        if not csr:
            h = I.irls_halo_plan(spec["nx"], spec["ny"], spec["nz"], world, rank)
            sent = max_over_ranks(8.0 * h["count"] * ((h["peer_lo"] >= 0) + (h["peer_hi"] >= 0)))
            nv_ach = sent / (t_halo * 1e-3) / 1e9
            nvlink = {"bound": "nvlink", "achieved": nv_ach, "peak": 770.0, "unit": "GB/s", "frac": nv_ach / 770.0,
                      "bytes_per_cg_iter_per_rank": sent, "halo_ms": t_halo,
                      "peak_source": "B200_PROFILING.md measured peer copy per direction (900 nominal)",
                      "what": "one z halo (a plane to each neighbour, ncclSend/Recv), max over ranks"}
        else:
            nvlink = {"halo_ms": t_halo, "achieved": None,
                      "what": "CSR strips: halo time only (send-list bytes not exported)"}
    # two-level rounding of the same x^(T), once,
    # outside the timed step: device phases + the host max-flow, timed apart
    two_level = None
    if not args.no_two_level:
        _, tl = m.irls_two_level_cut(side=False)
        two_level = {k: tl[k] for k in ("cut_value", "c0", "c1", "gamma0", "gamma1", "kmeans_rounds", "n0", "n1",
                                        "nc", "coarse_nlinks", "certified", "ms_gpu", "ms_copy", "ms_maxflow",
                                        "ms_total")}
        two_level["sweep_cut_value"] = cut
        two_level["what"] = ("two-level rounding of x^(T): K-means + coarsening + lift + cut on the GPU (ms_gpu), "
                             "coarse graph D2H/H2D (ms_copy), exact max-flow on G_c on the host (ms_maxflow)")
    m.close()

    # ---- e2e through the C ABI with pinned host buffers ---------------------
    pinned = {}
    arrays = ("row_ptr", "col", "w") if csr else ("cx", "cy", "cz", "cs", "ct")
    for name in arrays:
        a = np.ascontiguousarray(spec[name])
        t = torch.empty(a.shape[0], dtype=getattr(torch, str(a.dtype)), pin_memory=True)
        t.numpy()[:] = a
        pinned[name] = t.numpy()
    n_total = spec["n"] if csr else spec["nx"] * spec["ny"] * spec["nz"] + 2
    side_host = torch.empty(n_total, dtype=torch.uint8, pin_memory=True).numpy()
    h2d = sum(a.nbytes for a in pinned.values())
    d2h = side_host.shape[0] if rank == 0 else 0
    import ctypes as C

    phase_ms = {"create": 0.0, "solve": 0.0, "sweep_d2h": 0.0, "destroy": 0.0}

    def e2e_step(record=False):
        comm = fresh_comm()  # a fresh NCCL id per communicator (part of the user's create path)
        t0 = time.perf_counter()
        if csr:
            mm = I.MinCut.irls_mincut_create_csr(spec["n"], pinned["row_ptr"], pinned["col"], pinned["w"], spec["s"],
                                                 spec["t"], opts, comm)
        else:
            mm = I.MinCut.irls_mincut_create_stencil(spec["nx"], spec["ny"], spec["nz"], pinned["cx"], pinned["cy"],
                                                     pinned["cz"], pinned["cs"], pinned["ct"], opts, comm)
        t1 = time.perf_counter()
        _, tot = mm.irls_solve(I.IRLS_FROM_SCRATCH, T=T, reports=False)
        t2 = time.perf_counter()
        kk, cc = C.c_int64(), C.c_double()
        rc = I.lib().irls_sweep_cut(mm.h, side_host.ctypes.data_as(C.c_void_p) if rank == 0 else None, None,
                                    C.byref(kk), C.byref(cc))
        if rc:
            raise I.IrlsError(rc, "irls_sweep_cut")
        t3 = time.perf_counter()
        mm.close()
        t4 = time.perf_counter()
        if record:  # host clock around each (blocking) call: where the end-to-end time goes
            for key, dt in (("create", t1 - t0), ("solve", t2 - t1), ("sweep_d2h", t3 - t2), ("destroy", t4 - t3)):
                phase_ms[key] += 1e3 * dt / args.e2e_steps
        return tot

    e2e_step()  # warm-up (first-touch of the allocator's blocks for the sweep buffers)
    e2e_iters = 0
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    step_ms = []
    for _ in range(args.e2e_steps):
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        e2e_iters += e2e_step(record=True)
        s1.record(stream)
        s1.synchronize()
        step_ms.append(s0.elapsed_time(s1))
    e1.record(stream)
    barrier()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1))
    e2e_value = n_links * e2e_iters / (e2e_ms * 1e-3) / 1e9
    e2e_serial = {"value": e2e_value, "ms_per_step": e2e_ms / args.e2e_steps, "step_ms": step_ms,
                  "phase_ms_host_clock": phase_ms}

    # pipelined (one rank): two contexts on two streams, step i+1's create (the
    # H2D of its inputs from pinned memory, validation) runs on a host thread
    # while step i solves and sweeps; every step still copies its inputs in and
    # its side[] out inside the timed region
    e2e_mode = "serial"
    p_phase = None
    if world == 1 and not args.e2e_serial:
        from concurrent.futures import ThreadPoolExecutor
        pstreams = [torch.cuda.Stream(), torch.cuda.Stream()]
        pcomms = [I.comm_desc(1, 0, local, None, ps.cuda_stream, memory=mem) for ps in pstreams]

        p_times = []

        def p_create(cm):
            t0c = time.perf_counter()
            mm = p_create0(cm)
            p_times.append(("create", 1e3 * (time.perf_counter() - t0c)))
            return mm

        def p_create0(cm):
            if csr:
                return I.MinCut.irls_mincut_create_csr(spec["n"], pinned["row_ptr"], pinned["col"], pinned["w"],
                                                       spec["s"], spec["t"], opts, cm)
            return I.MinCut.irls_mincut_create_stencil(spec["nx"], spec["ny"], spec["nz"], pinned["cx"], pinned["cy"],
                                                       pinned["cz"], pinned["cs"], pinned["ct"], opts, cm)

        def p_run(mm):
            t0r = time.perf_counter()
            _, tot = mm.irls_solve(I.IRLS_FROM_SCRATCH, T=T, reports=False)
            p_times.append(("solve", 1e3 * (time.perf_counter() - t0r)))
            kk, cc = C.c_int64(), C.c_double()
            rc = I.lib().irls_sweep_cut(mm.h, side_host.ctypes.data_as(C.c_void_p), None, C.byref(kk), C.byref(cc))
            if rc:
                raise I.IrlsError(rc, "irls_sweep_cut")
            t1r = time.perf_counter()
            p_times.append(("sweep_d2h", 1e3 * (t1r - t0r) - p_times[-1][1]))
            mm.close()
            p_times.append(("destroy", 1e3 * (time.perf_counter() - t1r)))
            return tot

        with ThreadPoolExecutor(1) as ex:
            # warm-up: two overlapped steps, so the allocator holds two contexts' blocks
            fut = ex.submit(p_create, pcomms[0])
            for i in range(2):
                mm = fut.result()
                if i == 0:
                    fut = ex.submit(p_create, pcomms[1])
                p_run(mm)
            barrier()
            p_times.clear()
            p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            p0.record(stream)
            piters = 0
            fut = ex.submit(p_create, pcomms[0])
            for i in range(args.e2e_steps):
                mm = fut.result()
                if i + 1 < args.e2e_steps:
                    fut = ex.submit(p_create, pcomms[(i + 1) % 2])
                piters += p_run(mm)
            torch.cuda.synchronize()
            p1.record(stream)
            p1.synchronize()
        e2e_ms = p0.elapsed_time(p1)
        e2e_value = n_links * piters / (e2e_ms * 1e-3) / 1e9
        step_ms = None
        e2e_mode = "pipelined"
        p_phase = {k: statistics.mean([v for kk, v in p_times if kk == k])
                   for k in ("create", "solve", "sweep_d2h", "destroy") if any(kk == k for kk, _ in p_times)}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---- cpu baseline (rank 0, N=1 only) -----------------------------------
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        v, dt, threads, desc = oracle_sample(spec, planes=None, T=args.cpu_T)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": desc}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wdesc, "nodes": int(st["n_nonterminal"]), "n_links": int(n_links),
                   "T": T, "eps": 1e-6, "cg_rtol": 1e-3, "cg_max_iter": 50, "cg_norm": "preconditioned",
                   "cg_iters_per_step": iters_per_step[-1], "time_to_cut_ms": ms / args.steps,
                   "l2": "inputs (8.6 GB working set) larger than the 126 MB L2; no flush",
                   "parallelism": f"z-slab x{world}", "cut_value": cut, "k": k,
                   "cg_iter_ms_kernels": cg_iter_ms, "loop_mode": "host" if args.loop_mode == 1 else "graph",
                   "collectives": "none (1 rank)" if world == 1 else ("peer memory" if args.p2p else "nccl"),
                   "collectives_note": p2p_note,
                   "cg_variant": "Chronopoulos-Gear" if args.cg_variant == "cg" else "Hestenes-Stiefel"},
        "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                     "traffic": traffic, "traffic_note": "ncu dram__bytes_read+write per K3 launch "
                     "(profiles/r02_k3_traffic.json) over the live K3 duration, GB/s; algorithmic bytes per launch "
                     f"= {roof_bytes / 1e9:.3f} GB", "kernel": roof_name,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)" if "hbm_gbs" in peaks
                     else "fallback 6650 GB/s (B200_PROFILING.md)",
                     "frac_of_nominal_8TBps": ach / 8000.0, "kernels": kernels},
        "cpu_baseline": cpu,
        "nvlink": nvlink,
        "two_level": two_level,
        "fixed_point_exit": fpx,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_ms / args.e2e_steps, "mode": e2e_mode,
                "pipelined_phase_ms_host_clock": p_phase,
                "what": "per step: create from pinned host arrays (H2D of the inputs) + solve + sweep (side[] to "
                        "host) + destroy; pipelined = step i+1's create on a second stream/context while step i "
                        "solves (one rank), device-timed over all steps",
                "serial": e2e_serial},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
