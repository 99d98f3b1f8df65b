"""Thin ctypes binding of include/irls_mincut.h (argument marshalling only).

Every function keeps the C name; every step of the hot path runs in
libirls_mincut.so.  There is no CPU fallback: if the library is missing the
import of ``lib()`` raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libirls_mincut.so")

IRLS_OK = 0
STATUS_NAMES = {0: "IRLS_OK", 1: "IRLS_ERR_INVALID_ARGUMENT", 2: "IRLS_ERR_SOURCE_EQUALS_SINK",
                3: "IRLS_ERR_BAD_CAPACITY", 4: "IRLS_ERR_NOT_SYMMETRIC", 5: "IRLS_ERR_SINGULAR",
                6: "IRLS_ERR_CG_BREAKDOWN", 7: "IRLS_ERR_BAD_POTENTIAL", 8: "IRLS_ERR_STATE",
                9: "IRLS_ERR_CUDA", 10: "IRLS_ERR_NCCL", 11: "IRLS_ERR_OOM"}
IRLS_FROM_SCRATCH, IRLS_CONTINUE = 0, 1
IRLS_NORM_PRECONDITIONED, IRLS_NORM_UNPRECONDITIONED = 0, 1
IRLS_LOOP_GRAPH, IRLS_LOOP_HOST, IRLS_LOOP_GRAPH_NCCL = 0, 1, 2
IRLS_CG_HS, IRLS_CG_CG = 0, 1
KERNEL_PSPMV, KERNEL_AXPY, KERNEL_ASSEMBLE, KERNEL_HALO, KERNEL_CGCG = 0, 1, 2, 3, 4


class irls_options(C.Structure):
    _fields_ = [("eps", C.c_double), ("T", C.c_int32), ("cg_rtol", C.c_double), ("cg_max_iter", C.c_int32),
                ("cg_norm", C.c_int32), ("warm_start", C.c_int32), ("record_trace", C.c_int32),
                ("loop_mode", C.c_int32), ("fixed_point_exit", C.c_int32), ("p2p", C.c_int32),
                ("cg_variant", C.c_int32), ("block_size", C.c_int32)]


DEVICE_ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
DEVICE_FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p)


class irls_comm_desc(C.Structure):
    _fields_ = [("world_size", C.c_int32), ("rank", C.c_int32), ("device", C.c_int32),
                ("nccl_unique_id", C.c_void_p), ("cuda_stream", C.c_void_p),
                ("device_alloc", DEVICE_ALLOC_FN), ("device_free", DEVICE_FREE_FN), ("alloc_user", C.c_void_p)]


class TorchDeviceMemory:
    """device_alloc / device_free backed by torch's caching allocator: every
    array of a context is a torch uint8 tensor held here until it is freed
    (argument marshalling only; the library owns the layout)."""

    def __init__(self, device=0):
        import torch
        self._torch = torch
        self.device = device
        self.tensors = {}
        self.alloc = DEVICE_ALLOC_FN(self._alloc)
        self.free = DEVICE_FREE_FN(self._free)

    def _alloc(self, nbytes, stream, user):
        try:
            t = self._torch.empty(int(nbytes), dtype=self._torch.uint8, device=f"cuda:{self.device}")
        except Exception:
            return None
        self.tensors[t.data_ptr()] = t
        return t.data_ptr()

    def _free(self, ptr, stream, user):
        self.tensors.pop(ptr, None)

    @property
    def bytes_held(self):
        return sum(t.numel() for t in self.tensors.values())


class irls_step_report(C.Structure):
    _fields_ = [("cg_iters", C.c_int32), ("converged", C.c_int32), ("status", C.c_int32), ("reserved", C.c_int32),
                ("rel_res", C.c_double), ("true_rel_res", C.c_double), ("S_eps", C.c_double),
                ("flow_value", C.c_double), ("current_s", C.c_double), ("x_min", C.c_double),
                ("x_max", C.c_double), ("ref", C.c_double), ("ms", C.c_float), ("ms_assemble", C.c_float)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if not k.startswith("reserved")}


class irls_halo(C.Structure):
    _fields_ = [("count", C.c_int64), ("n_own", C.c_int64), ("send_lo", C.c_int64), ("recv_lo", C.c_int64),
                ("send_hi", C.c_int64), ("recv_hi", C.c_int64), ("peer_lo", C.c_int32), ("peer_hi", C.c_int32),
                ("first_plane", C.c_int32), ("reserved", C.c_int32)]


class irls_two_level_report(C.Structure):
    _fields_ = [("c0", C.c_double), ("c1", C.c_double), ("gamma0", C.c_double), ("gamma1", C.c_double),
                ("kmeans_rounds", C.c_int32), ("certified", C.c_int32), ("n0", C.c_int64), ("n1", C.c_int64),
                ("nc", C.c_int64), ("coarse_nlinks", C.c_int64), ("augmentations", C.c_int64), ("F", C.c_int32),
                ("pad", C.c_int32), ("coarse_flow", C.c_double), ("cut_value", C.c_double), ("ms_gpu", C.c_float),
                ("ms_copy", C.c_float), ("ms_maxflow", C.c_float), ("ms_total", C.c_float)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "pad"}


class irls_lambda2_report(C.Structure):
    _fields_ = [("lambda2", C.c_double), ("xLx", C.c_double), ("C", C.c_double), ("rel_res", C.c_double),
                ("cg_iters", C.c_int32), ("converged", C.c_int32), ("ms", C.c_float), ("launches", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class irls_stats(C.Structure):
    _fields_ = [("launches", C.c_int64), ("cg_iters", C.c_int64), ("n_nonterminal", C.c_int64),
                ("n_links", C.c_int64), ("n_local", C.c_int64),
                ("sweep_sorted", C.c_int64)]


_lib = None

# exported symbols of include/irls_mincut.h
SYMBOLS = ["irls_options_default", "irls_nccl_unique_id", "irls_mincut_create_stencil", "irls_mincut_create_csr",
           "irls_init", "irls_step", "irls_solve", "irls_sweep_cut", "irls_get_side", "irls_set_terminal_weights",
           "irls_get_potentials", "irls_set_potentials", "irls_get_stats", "irls_time_kernel",
           "irls_mincut_destroy", "irls_status_string", "irls_last_error", "irls_plan_stencil",
           "irls_halo_plan", "irls_combine_slots", "irls_vgroup_create_stencil", "irls_vgroup_solve",
           "irls_vgroup_sweep_cut", "irls_vgroup_get_potentials", "irls_vgroup_set_terminal_weights",
           "irls_vgroup_destroy", "irls_two_level_cut", "irls_two_level_get_coarse", "irls_coarse_maxflow",
           "irls_vgroup_two_level_cut", "irls_exact_min_cut", "irls_lambda2", "irls_vgroup_create_csr", "irls_vgroup_last_error", "irls_plan_csr", "irls_csr_halo_plan"]


def lib():
    """Load libirls_mincut.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run paper_1501_03105_b200.build.build() "
                               "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        L.irls_options_default.argtypes = [C.POINTER(irls_options)]
        L.irls_nccl_unique_id.argtypes = [C.c_char_p]
        L.irls_mincut_create_stencil.argtypes = [C.POINTER(P), C.POINTER(irls_comm_desc), C.c_int32, C.c_int32,
                                                 C.c_int32, P, P, P, P, P, C.POINTER(irls_options)]
        L.irls_mincut_create_csr.argtypes = [C.POINTER(P), C.POINTER(irls_comm_desc), C.c_int64, P, P, P,
                                             C.c_int64, C.c_int64, C.POINTER(irls_options)]
        L.irls_init.argtypes = [P, C.POINTER(irls_step_report)]
        L.irls_step.argtypes = [P, C.POINTER(irls_step_report)]
        L.irls_solve.argtypes = [P, C.c_int32, P, C.POINTER(C.c_int64)]
        L.irls_sweep_cut.argtypes = [P, P, P, C.POINTER(C.c_int64), C.POINTER(C.c_double)]
        L.irls_get_side.argtypes = [P, P]
        L.irls_set_terminal_weights.argtypes = [P, P, P]
        L.irls_get_potentials.argtypes = [P, P]
        L.irls_set_potentials.argtypes = [P, P]
        L.irls_get_stats.argtypes = [P, C.POINTER(irls_stats)]
        L.irls_time_kernel.argtypes = [P, C.c_int32, C.c_int32, C.POINTER(C.c_float)]
        L.irls_mincut_destroy.argtypes = [P]
        L.irls_mincut_destroy.restype = None
        L.irls_status_string.argtypes = [C.c_int]
        L.irls_status_string.restype = C.c_char_p
        L.irls_last_error.argtypes = [P]
        L.irls_last_error.restype = C.c_char_p
        L.irls_plan_stencil.argtypes = [C.c_int32] * 5 + [C.POINTER(C.c_int32)] * 4
        L.irls_halo_plan.argtypes = [C.c_int32] * 5 + [C.POINTER(irls_halo)]
        L.irls_vgroup_create_stencil.argtypes = [C.POINTER(P), C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                                 C.c_int32, P, P, P, P, P, C.POINTER(irls_options)]
        L.irls_vgroup_create_csr.argtypes = [C.POINTER(P), C.c_int32, C.c_int32, C.c_int64, P, P, P, C.c_int64,
                                             C.c_int64, C.POINTER(irls_options)]
        L.irls_plan_csr.argtypes = [C.c_int64, C.c_int32, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                    C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        L.irls_vgroup_last_error.argtypes = [P]
        L.irls_vgroup_last_error.restype = C.c_char_p
        L.irls_vgroup_solve.argtypes = [P, C.c_int32, P, C.POINTER(C.c_int64)]
        L.irls_vgroup_sweep_cut.argtypes = [P, P, P, C.POINTER(C.c_int64), C.POINTER(C.c_double)]
        L.irls_vgroup_get_potentials.argtypes = [P, P]
        L.irls_vgroup_set_terminal_weights.argtypes = [P, P, P]
        L.irls_vgroup_destroy.argtypes = [P]
        L.irls_two_level_cut.argtypes = [P, P, C.POINTER(irls_two_level_report)]
        L.irls_lambda2.argtypes = [P, C.c_double, C.c_int32, C.c_int32, P, C.POINTER(irls_lambda2_report)]
        L.irls_exact_min_cut.argtypes = [P, P, C.POINTER(irls_two_level_report)]
        L.irls_vgroup_two_level_cut.argtypes = [P, P, C.POINTER(irls_two_level_report)]
        L.irls_two_level_get_coarse.argtypes = [P] * 8
        L.irls_coarse_maxflow.argtypes = [C.c_int32, P, P, P, P, P, P, P, C.POINTER(C.c_int32)]
        L.irls_vgroup_destroy.restype = None
        L.irls_combine_slots.argtypes = [P]
        L.irls_combine_slots.restype = C.c_double
        _lib = L
    return _lib


class IrlsError(RuntimeError):
    def __init__(self, code, where, detail=""):
        super().__init__(f"{where}: {STATUS_NAMES.get(code, code)} {detail}")
        self.code = code


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _f64_n(a, n, what):
    """A host float64 array of exactly n entries (the C side reads n)."""
    a = _f64(a)
    if a.ndim != 1 or a.shape[0] != n:
        raise ValueError(f"{what}: expected {n} float64 values, got shape {a.shape}")
    return a


def options(**kw) -> irls_options:
    o = irls_options()
    lib().irls_options_default(C.byref(o))
    for k, v in kw.items():
        if not hasattr(o, k):
            raise TypeError(f"unknown option {k}")
        setattr(o, k, v)
    return o


def comm_desc(world_size=1, rank=0, device=0, unique_id: bytes | None = None, stream=None,
              memory: "TorchDeviceMemory | None" = None):
    """irls_comm_desc; memory: a TorchDeviceMemory to make torch own the
    context's device arrays (it must outlive the context)."""
    d = irls_comm_desc()
    d.world_size, d.rank, d.device = world_size, rank, device
    d._uid = C.create_string_buffer(unique_id, 128) if unique_id is not None else None
    d.nccl_unique_id = C.cast(d._uid, C.c_void_p) if d._uid is not None else None
    d.cuda_stream = stream
    if memory is not None:
        d.device_alloc, d.device_free = memory.alloc, memory.free
        d._memory = memory
    return d


# ---------------------------------------------------------------------------
# functions with the C names
# ---------------------------------------------------------------------------

def irls_nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    rc = lib().irls_nccl_unique_id(buf)
    if rc:
        raise IrlsError(rc, "irls_nccl_unique_id")
    return buf.raw


def irls_plan_stencil(nx, ny, nz, world, rank):
    out = [C.c_int32() for _ in range(4)]
    rc = lib().irls_plan_stencil(nx, ny, nz, world, rank, *[C.byref(o) for o in out])
    if rc:
        raise IrlsError(rc, "irls_plan_stencil")
    return tuple(o.value for o in out)  # z0, z1, g0, g1


def irls_halo_plan(nx, ny, nz, world, rank) -> dict:
    h = irls_halo()
    rc = lib().irls_halo_plan(nx, ny, nz, world, rank, C.byref(h))
    if rc:
        raise IrlsError(rc, "irls_halo_plan")
    return {k: getattr(h, k) for k, _ in h._fields_ if k != "reserved"}


def irls_csr_halo_plan(aptr, aidx, world, rank) -> dict:
    """Host-only halo plan of id strip `rank` over the reduced adjacency."""
    aptr = np.ascontiguousarray(aptr, dtype=np.int64)
    aidx = np.ascontiguousarray(aidx, dtype=np.int32) if len(aidx) else np.zeros(1, np.int32)
    nr = aptr.shape[0] - 1
    lo_hi = np.zeros(2, np.int64); ro = np.zeros(world + 1, np.int64); so = np.zeros(world + 1, np.int64)
    f = lib().irls_csr_halo_plan
    f.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                  C.c_void_p, C.c_int64, C.c_void_p, C.c_int64]
    rc = f(nr, _ptr(aptr), _ptr(aidx), world, rank, _ptr(lo_hi), _ptr(ro), _ptr(so), None, 0, None, 0)
    if rc:
        raise IrlsError(rc, "irls_csr_halo_plan")
    gh = np.zeros(max(int(ro[-1]), 1), np.int32); sd = np.zeros(max(int(so[-1]), 1), np.int32)
    rc = f(nr, _ptr(aptr), _ptr(aidx), world, rank, _ptr(lo_hi), _ptr(ro), _ptr(so), _ptr(gh), gh.shape[0],
           _ptr(sd), sd.shape[0])
    if rc:
        raise IrlsError(rc, "irls_csr_halo_plan")
    return dict(lo=int(lo_hi[0]), hi=int(lo_hi[1]), recv_off=ro, send_off=so, ghosts=gh[: ro[-1]],
                send_idx=sd[: so[-1]])


def irls_plan_csr(nr, world, rank):
    """Host-only: (lo, hi, g0, g1) of rank's id strip."""
    lo, hi, g0, g1 = C.c_int64(), C.c_int64(), C.c_int32(), C.c_int32()
    rc = lib().irls_plan_csr(nr, world, rank, C.byref(lo), C.byref(hi), C.byref(g0), C.byref(g1))
    if rc:
        raise IrlsError(rc, "irls_plan_csr")
    return lo.value, hi.value, g0.value, g1.value


def irls_combine_slots(slots) -> float:
    s = _f64(slots)
    assert s.shape == (8,)
    return lib().irls_combine_slots(_ptr(s))


def words_to_ints(w) -> list:
    """128-bit two's complement (lo, hi) uint64 pairs -> Python ints."""
    w = np.asarray(w, dtype=np.uint64).reshape(-1, 2)
    out = []
    for lo, hi in w:
        v = int(lo) + (int(hi) << 64)
        out.append(v - (1 << 128) if v >= 1 << 127 else v)
    return out


def ints_to_words(vals) -> np.ndarray:
    w = np.zeros(2 * max(len(vals), 1), dtype=np.uint64)
    for i, v in enumerate(vals):
        v &= (1 << 128) - 1
        w[2 * i] = v & ((1 << 64) - 1)
        w[2 * i + 1] = v >> 64
    return w


def irls_coarse_maxflow(nc, ptr, col, cap, qs, qt):
    """The library's exact coarse max-flow (host): (flow int, src uint8[nc], certified)."""
    p = np.ascontiguousarray(ptr, dtype=np.int32)
    c = np.ascontiguousarray(col, dtype=np.int32) if len(col) else np.zeros(1, np.int32)
    src = np.zeros(max(nc, 1), dtype=np.uint8)
    fl = np.zeros(2, dtype=np.uint64)
    cert = C.c_int32()
    cw, sw, tw = ints_to_words(list(cap)), ints_to_words(list(qs)), ints_to_words(list(qt))
    rc = lib().irls_coarse_maxflow(nc, _ptr(p), _ptr(c), _ptr(cw), _ptr(sw), _ptr(tw), _ptr(src), _ptr(fl),
                                   C.byref(cert))
    if rc:
        raise IrlsError(rc, "irls_coarse_maxflow")
    return words_to_ints(fl)[0], src[:nc], cert.value


class MinCut:
    """One context (one rank) of the IRLS min-cut library."""

    def __init__(self, h, n, n_total, T=None):
        self.h = h
        self.n = n
        self.n_total = n_total
        self.T = T  # irls_options.T of the context: irls_solve runs T steps

    # -- creation ----------------------------------------------------------
    @classmethod
    def irls_mincut_create_stencil(cls, nx, ny, nz, cx, cy, cz, cs, ct, opts: irls_options | None = None,
                                   comm: irls_comm_desc | None = None):
        arrs = [_f64(a) for a in (cx, cy, cz, cs, ct)]
        N = nx * ny * nz
        if any(a.shape[0] != N for a in arrs):
            raise ValueError("capacity arrays must have nx*ny*nz entries")
        opts = opts or options()
        h = C.c_void_p()
        rc = lib().irls_mincut_create_stencil(C.byref(h), C.byref(comm) if comm else None, nx, ny, nz,
                                              *[_ptr(a) for a in arrs], C.byref(opts))
        if rc:
            raise IrlsError(rc, "irls_mincut_create_stencil")
        m = cls(h, N, N + 2, opts.T)
        m._comm = comm  # keeps a caller allocator's callbacks alive
        return m

    @classmethod
    def irls_mincut_create_csr(cls, n, row_ptr, col, w, s, t, opts: irls_options | None = None,
                               comm: irls_comm_desc | None = None):
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        cl = np.ascontiguousarray(col, dtype=np.int32)
        ww = _f64(w)
        opts = opts or options()
        h = C.c_void_p()
        rc = lib().irls_mincut_create_csr(C.byref(h), C.byref(comm) if comm else None, n, _ptr(rp), _ptr(cl),
                                          _ptr(ww), s, t, C.byref(opts))
        if rc:
            raise IrlsError(rc, "irls_mincut_create_csr")
        m = cls(h, n - 2, n, opts.T)
        m._comm = comm
        return m

    @classmethod
    def from_spec(cls, spec, opts=None, comm=None):
        """Create from a synthetic.generators dict."""
        if spec["kind"] == "stencil":
            return cls.irls_mincut_create_stencil(spec["nx"], spec["ny"], spec["nz"], spec["cx"], spec["cy"],
                                                  spec["cz"], spec["cs"], spec["ct"], opts, comm)
        return cls.irls_mincut_create_csr(spec["n"], spec["row_ptr"], spec["col"], spec["w"], spec["s"],
                                          spec["t"], opts, comm)

    def _check(self, rc, where):
        if rc:
            detail = lib().irls_last_error(self.h) if self.h else b""
            raise IrlsError(rc, where, detail.decode(errors="replace") if detail else "")

    # -- solves ------------------------------------------------------------
    def irls_init(self) -> dict:
        r = irls_step_report()
        self._check(lib().irls_init(self.h, C.byref(r)), "irls_init")
        return r.as_dict()

    def irls_step(self) -> dict:
        r = irls_step_report()
        self._check(lib().irls_step(self.h, C.byref(r)), "irls_step")
        return r.as_dict()

    def irls_solve(self, mode=IRLS_FROM_SCRATCH, T=None, reports=True):
        """irls_solve runs the context's irls_options.T steps; `T`, if given,
        must equal it (it only documents the caller's expectation)."""
        if T is not None and self.T is not None and T != self.T:
            raise ValueError(f"irls_solve runs the context's T = {self.T} steps (irls_options.T), not {T}")
        T = self.T if self.T is not None else T
        nrep = (T + 1 if mode == IRLS_FROM_SCRATCH else T) if T is not None else None
        buf = (irls_step_report * max(nrep, 1))() if (reports and nrep is not None) else None
        total = C.c_int64()
        self._check(lib().irls_solve(self.h, mode, C.cast(buf, C.c_void_p) if buf is not None else None,
                                     C.byref(total)), "irls_solve")
        return ([r.as_dict() for r in buf[:nrep]] if buf is not None else None), total.value

    def irls_sweep_cut(self, side=True, order=False):
        s = np.zeros(self.n_total, dtype=np.uint8) if side else None
        o = np.zeros(max(self.n, 1), dtype=np.int32) if order else None
        k = C.c_int64()
        cut = C.c_double()
        self._check(lib().irls_sweep_cut(self.h, _ptr(s), _ptr(o), C.byref(k), C.byref(cut)), "irls_sweep_cut")
        return s, (o[: self.n] if o is not None else None), k.value, cut.value

    def irls_two_level_cut(self, side=True):
        """Two-level rounding: (side or None, report dict)."""
        sd = np.zeros(self.n_total, dtype=np.uint8) if side else None
        r = irls_two_level_report()
        self._check(lib().irls_two_level_cut(self.h, _ptr(sd), C.byref(r)), "irls_two_level_cut")
        return sd, r.as_dict()

    def irls_lambda2(self, cg_rtol=1e-12, cg_max_iter=100000, cg_norm=IRLS_NORM_UNPRECONDITIONED, want_x=False):
        """Cheeger-type diagnostic (A30): report dict (+ the solution v)."""
        x = np.zeros(max(self.n, 1)) if want_x else None
        r = irls_lambda2_report()
        self._check(lib().irls_lambda2(self.h, cg_rtol, cg_max_iter, cg_norm, _ptr(x), C.byref(r)), "irls_lambda2")
        return (r.as_dict(), x[: self.n]) if want_x else r.as_dict()

    def irls_exact_min_cut(self, side=True):
        """mu* of the whole graph (no contraction): (side or None, report dict)."""
        sd = np.zeros(self.n_total, dtype=np.uint8) if side else None
        r = irls_two_level_report()
        self._check(lib().irls_exact_min_cut(self.h, _ptr(sd), C.byref(r)), "irls_exact_min_cut")
        return sd, r.as_dict()

    def irls_two_level_get_coarse(self, nc, entries):
        cls = np.zeros(max(self.n, 1), dtype=np.int8)
        ptr = np.zeros(nc + 1, dtype=np.int32)
        col = np.zeros(max(entries, 1), dtype=np.int32)
        cap = np.zeros(max(entries, 1))
        qs = np.zeros(2 * max(nc, 1), dtype=np.uint64)
        qt = np.zeros(2 * max(nc, 1), dtype=np.uint64)
        qst = np.zeros(2, dtype=np.uint64)
        self._check(lib().irls_two_level_get_coarse(self.h, _ptr(cls), _ptr(ptr), _ptr(col), _ptr(cap), _ptr(qs),
                                                    _ptr(qt), _ptr(qst)), "irls_two_level_get_coarse")
        return dict(cls=cls[: self.n], ptr=ptr, col=col[:entries], cap=cap[:entries], qs=words_to_ints(qs[: 2 * nc]),
                    qt=words_to_ints(qt[: 2 * nc]), qst=words_to_ints(qst)[0])

    def irls_get_side(self):
        s = np.zeros(self.n_total, dtype=np.uint8)
        self._check(lib().irls_get_side(self.h, _ptr(s)), "irls_get_side")
        return s

    def irls_set_terminal_weights(self, cs, ct):
        a, b = _f64_n(cs, self.n, "cs"), _f64_n(ct, self.n, "ct")
        self._check(lib().irls_set_terminal_weights(self.h, _ptr(a), _ptr(b)), "irls_set_terminal_weights")

    def irls_get_potentials(self):
        x = np.zeros(max(self.n, 1))
        self._check(lib().irls_get_potentials(self.h, _ptr(x)), "irls_get_potentials")
        return x[: self.n]

    def irls_set_potentials(self, x):
        a = _f64_n(x, self.n, "x")
        self._check(lib().irls_set_potentials(self.h, _ptr(a)), "irls_set_potentials")

    def irls_get_stats(self) -> dict:
        s = irls_stats()
        self._check(lib().irls_get_stats(self.h, C.byref(s)), "irls_get_stats")
        return {k: getattr(s, k) for k, _ in s._fields_}

    def irls_time_kernel(self, which, reps=10) -> float:
        ms = C.c_float()
        self._check(lib().irls_time_kernel(self.h, which, reps, C.byref(ms)), "irls_time_kernel")
        return ms.value

    def irls_mincut_destroy(self):
        if self.h:
            lib().irls_mincut_destroy(self.h)
            self.h = None

    close = irls_mincut_destroy

    def __del__(self):
        try:
            self.irls_mincut_destroy()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.irls_mincut_destroy()


class VGroup:
    """W ranks of the multi-GPU path (z-slabs of a grid, id strips of a CSR
    graph) on one device (irls_vgroup_*)."""

    def __init__(self, spec, world, opts: irls_options | None = None, device=0):
        self.opts = opts or options()
        self.h = C.c_void_p()
        if spec["kind"] == "stencil":
            arrs = [_f64(spec[k]) for k in ("cx", "cy", "cz", "cs", "ct")]
            self.n = spec["nx"] * spec["ny"] * spec["nz"]
            self.n_total = self.n + 2
            rc = lib().irls_vgroup_create_stencil(C.byref(self.h), world, device, spec["nx"], spec["ny"], spec["nz"],
                                                  *[_ptr(a) for a in arrs], C.byref(self.opts))
        else:
            rp = np.ascontiguousarray(spec["row_ptr"], dtype=np.int64)
            cl = np.ascontiguousarray(spec["col"], dtype=np.int32)
            ww = _f64(spec["w"])
            self.n = spec["n"] - 2
            self.n_total = spec["n"]
            rc = lib().irls_vgroup_create_csr(C.byref(self.h), world, device, spec["n"], _ptr(rp), _ptr(cl), _ptr(ww),
                                              spec["s"], spec["t"], C.byref(self.opts))
        if rc:
            self.h = None
            raise IrlsError(rc, "irls_vgroup_create")

    def irls_vgroup_solve(self, mode=IRLS_FROM_SCRATCH, T=None):
        if T is not None and T != self.opts.T:
            raise ValueError(f"irls_vgroup_solve runs the group's T = {self.opts.T} steps (irls_options.T), not {T}")
        T = self.opts.T
        nrep = T + 1 if mode == IRLS_FROM_SCRATCH else T
        buf = (irls_step_report * max(nrep, 1))() if nrep is not None else None
        total = C.c_int64()
        rc = lib().irls_vgroup_solve(self.h, mode, C.cast(buf, C.c_void_p) if buf is not None else None,
                                     C.byref(total))
        if rc:
            raise IrlsError(rc, "irls_vgroup_solve", lib().irls_vgroup_last_error(self.h).decode(errors="replace"))
        return ([r.as_dict() for r in buf[:nrep]] if buf is not None else None), total.value

    def irls_vgroup_sweep_cut(self, order=False):
        side = np.zeros(self.n_total, dtype=np.uint8)
        o = np.zeros(max(self.n, 1), dtype=np.int32) if order else None
        k, cut = C.c_int64(), C.c_double()
        rc = lib().irls_vgroup_sweep_cut(self.h, _ptr(side), _ptr(o), C.byref(k), C.byref(cut))
        if rc:
            raise IrlsError(rc, "irls_vgroup_sweep_cut")
        return side, o, k.value, cut.value

    def irls_vgroup_two_level_cut(self):
        side = np.zeros(self.n_total, dtype=np.uint8)
        r = irls_two_level_report()
        rc = lib().irls_vgroup_two_level_cut(self.h, _ptr(side), C.byref(r))
        if rc:
            raise IrlsError(rc, "irls_vgroup_two_level_cut")
        return side, r.as_dict()

    def irls_vgroup_get_potentials(self):
        x = np.zeros(self.n)
        rc = lib().irls_vgroup_get_potentials(self.h, _ptr(x))
        if rc:
            raise IrlsError(rc, "irls_vgroup_get_potentials")
        return x

    def irls_vgroup_set_terminal_weights(self, cs, ct):
        a, b = _f64_n(cs, self.n, "cs"), _f64_n(ct, self.n, "ct")
        rc = lib().irls_vgroup_set_terminal_weights(self.h, _ptr(a), _ptr(b))
        if rc:
            raise IrlsError(rc, "irls_vgroup_set_terminal_weights")

    def close(self):
        if self.h:
            lib().irls_vgroup_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
