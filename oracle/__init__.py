"""ctypes binding of the float64 CPU oracle (oracle/irls_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` leg; never by the product path
(paper_1501_03105_b200), which shares no code with it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "irls_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile the oracle (plain C, gcc) next to its source."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


class Options(C.Structure):
    _fields_ = [("eps", C.c_double), ("T", C.c_int32), ("cg_rtol", C.c_double),
                ("cg_max_iter", C.c_int32), ("cg_norm", C.c_int32), ("warm_start", C.c_int32)]


class Report(C.Structure):
    _fields_ = [("cg_iters", C.c_int32), ("converged", C.c_int32), ("rel_res", C.c_double),
                ("true_rel_res", C.c_double), ("S_eps", C.c_double), ("flow_value", C.c_double),
                ("current_s", C.c_double), ("x_min", C.c_double), ("x_max", C.c_double),
                ("ref", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        P = C.c_void_p
        dp = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
        i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
        i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
        u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
        u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
        L.orc_graph_from_stencil.argtypes = [C.POINTER(P), C.c_int64, C.c_int64, C.c_int64, dp, dp, dp, dp, dp]
        L.orc_graph_from_csr.argtypes = [C.POINTER(P), C.c_int64, i64p, i32p, dp, C.c_int64, C.c_int64]
        L.orc_graph_free.argtypes = [P]
        for f in ("orc_graph_n", "orc_graph_n_total", "orc_graph_nnz"):
            getattr(L, f).argtypes = [P]; getattr(L, f).restype = C.c_int64
        L.orc_graph_c_st.argtypes = [P]; L.orc_graph_c_st.restype = C.c_double
        L.orc_graph_orig_ids.argtypes = [P, i64p]
        L.orc_graph_terminals.argtypes = [P, dp, dp]
        L.orc_check_nonsingular.argtypes = [P]
        L.orc_c3_sum.argtypes = [dp, C.c_int64]; L.orc_c3_sum.restype = C.c_double
        L.orc_c3_group_sums.argtypes = [dp, C.c_int64, dp]
        L.orc_state_new.argtypes = [P, C.POINTER(Options)]; L.orc_state_new.restype = P
        L.orc_state_free.argtypes = [P]
        L.orc_init.argtypes = [P, C.POINTER(Report)]
        L.orc_step.argtypes = [P, C.POINTER(Report)]
        L.orc_get_x.argtypes = [P, dp]
        L.orc_set_x.argtypes = [P, dp]
        L.orc_set_terminal_weights.argtypes = [P, dp, dp]
        L.orc_assemble_export.argtypes = [P, P, dp, dp, dp, dp, dp]
        L.orc_irls_run.argtypes = [P, P, P]
        L.orc_sweep.argtypes = [P, dp, u8p, P, C.POINTER(C.c_int64), C.POINTER(C.c_double),
                                C.POINTER(C.c_int32), u64p]
        L.orc_cut_value.argtypes = [P, u8p]; L.orc_cut_value.restype = C.c_double
        L.orc_maxflow_ek.argtypes = [P, C.POINTER(C.c_double), u8p]
        _lib = L
    return _lib


STATUS = {0: "OK", 1: "INVALID_ARGUMENT", 2: "SOURCE_EQUALS_SINK", 3: "BAD_CAPACITY",
          4: "NOT_SYMMETRIC", 5: "SINGULAR", 6: "CG_BREAKDOWN", 7: "BAD_POTENTIAL",
          8: "STATE", 11: "OOM"}


class OracleError(RuntimeError):
    def __init__(self, code, where=""):
        super().__init__(f"{where}: oracle status {code} ({STATUS.get(code, '?')})")
        self.code = code


def _check(rc, where):
    if rc != 0:
        raise OracleError(rc, where)


def c3_sum(v) -> float:
    v = np.ascontiguousarray(v, dtype=np.float64)
    return lib().orc_c3_sum(v, v.shape[0])


def c3_group_sums(v) -> np.ndarray:
    v = np.ascontiguousarray(v, dtype=np.float64)
    out = np.zeros(8)
    lib().orc_c3_group_sums(v, v.shape[0], out)
    return out


class Graph:
    """Oracle graph built from a synthetic.generators dict (stencil or csr)."""

    def __init__(self, spec):
        L = lib()
        h = C.c_void_p()
        if spec["kind"] == "stencil":
            f = lambda k: np.ascontiguousarray(spec[k], dtype=np.float64)
            rc = L.orc_graph_from_stencil(C.byref(h), spec["nx"], spec["ny"], spec["nz"],
                                          f("cx"), f("cy"), f("cz"), f("cs"), f("ct"))
        else:
            rc = L.orc_graph_from_csr(C.byref(h), spec["n"],
                                      np.ascontiguousarray(spec["row_ptr"], dtype=np.int64),
                                      np.ascontiguousarray(spec["col"], dtype=np.int32),
                                      np.ascontiguousarray(spec["w"], dtype=np.float64),
                                      spec["s"], spec["t"])
        _check(rc, "graph")
        self.h = h
        self.n = L.orc_graph_n(h)
        self.n_total = L.orc_graph_n_total(h)
        self.nnz = L.orc_graph_nnz(h)
        self.c_st = L.orc_graph_c_st(h)
        self.orig = np.zeros(self.n, dtype=np.int64)
        L.orc_graph_orig_ids(h, self.orig)

    def check_nonsingular(self) -> int:
        return lib().orc_check_nonsingular(self.h)

    def terminals(self):
        cs = np.zeros(self.n); ct = np.zeros(self.n)
        lib().orc_graph_terminals(self.h, cs, ct)
        return cs, ct

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_graph_free(self.h)
            self.h = None


@dataclass
class SweepResult:
    side: np.ndarray
    order: np.ndarray
    k: int
    cut_value: float
    F: int
    pk: int


class Solver:
    """IRLS state over a Graph (Algorithm 1)."""

    def __init__(self, graph: Graph, eps=1e-6, T=50, cg_rtol=1e-3, cg_max_iter=50,
                 cg_norm=0, warm_start=True):
        self.graph = graph
        self.opts = Options(eps, T, cg_rtol, cg_max_iter, cg_norm, int(bool(warm_start)))
        self.h = lib().orc_state_new(graph.h, C.byref(self.opts))
        if not self.h:
            raise MemoryError("orc_state_new")
        self.n = graph.n

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_state_free(self.h)
            self.h = None

    def init(self) -> dict:
        r = Report(); _check(lib().orc_init(self.h, C.byref(r)), "init"); return r.as_dict()

    def step(self) -> dict:
        r = Report(); _check(lib().orc_step(self.h, C.byref(r)), "step"); return r.as_dict()

    def x(self) -> np.ndarray:
        out = np.zeros(self.n); lib().orc_get_x(self.h, out); return out

    def set_x(self, x):
        lib().orc_set_x(self.h, np.ascontiguousarray(x, dtype=np.float64))

    def set_terminal_weights(self, cs, ct):
        _check(lib().orc_set_terminal_weights(self.h, np.ascontiguousarray(cs, dtype=np.float64),
                                              np.ascontiguousarray(ct, dtype=np.float64)), "set_tw")

    def assemble(self, x=None):
        n = self.n
        g = np.zeros(max(self.graph.nnz, 1)); gs = np.zeros(n); gt = np.zeros(n)
        D = np.zeros(n); Dinv = np.zeros(n)
        xp = None
        if x is not None:
            x = np.ascontiguousarray(x, dtype=np.float64); xp = x.ctypes.data_as(C.c_void_p)
        lib().orc_assemble_export(self.h, xp, g, gs, gt, D, Dinv)
        return dict(g=g[: self.graph.nnz], gs=gs, gt=gt, D=D, Dinv=Dinv)

    def run(self, record=True):
        """init + T steps; returns (xs[(T+1), n] or None, reports)."""
        T = self.opts.T
        xs = np.zeros((T + 1, self.n)) if record else None
        reps = (Report * (T + 1))()
        _check(lib().orc_irls_run(self.h, xs.ctypes.data_as(C.c_void_p) if record else None,
                                  C.cast(reps, C.c_void_p)), "run")
        return xs, [r.as_dict() for r in reps]

    def sweep(self, x=None) -> SweepResult:
        x = self.x() if x is None else np.ascontiguousarray(x, dtype=np.float64)
        side = np.zeros(self.graph.n_total, dtype=np.uint8)
        order = np.zeros(max(self.n, 1), dtype=np.int64)
        k = C.c_int64(); cut = C.c_double(); F = C.c_int32(); pk = np.zeros(2, dtype=np.uint64)
        _check(lib().orc_sweep(self.h, x, side, order.ctypes.data_as(C.c_void_p), C.byref(k),
                               C.byref(cut), C.byref(F), pk), "sweep")
        pkv = int(pk[0]) + (int(pk[1]) << 64)
        if pkv >= 1 << 127:
            pkv -= 1 << 128
        return SweepResult(side, order[: self.n], k.value, cut.value, F.value, pkv)

    def cut_value(self, side) -> float:
        return lib().orc_cut_value(self.h, np.ascontiguousarray(side, dtype=np.uint8))

    def maxflow(self):
        side = np.zeros(self.graph.n_total, dtype=np.uint8)
        flow = C.c_double()
        _check(lib().orc_maxflow_ek(self.h, C.byref(flow), side), "maxflow")
        return flow.value, side
