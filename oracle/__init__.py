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

CFLAGS = ["-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile the oracle (plain C, gcc) next to its source."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


class Options(C.Structure):
    _fields_ = [("eps", C.c_double), ("T", C.c_int32), ("cg_rtol", C.c_double),
                ("cg_max_iter", C.c_int32), ("cg_norm", C.c_int32), ("warm_start", C.c_int32),
                ("cg_variant", C.c_int32), ("block_size", C.c_int32)]


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
        L.orc_set_num_threads.argtypes = [C.c_int]; L.orc_set_num_threads.restype = C.c_int
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
        L.orc_block_count.argtypes = [P]; L.orc_block_count.restype = C.c_int64
        L.orc_block_env_size.argtypes = [P]; L.orc_block_env_size.restype = C.c_int64
        L.orc_block_export.argtypes = [P, i64p, i64p, i64p, i64p]
        L.orc_precond_export.argtypes = [P, P, dp, dp, dp, dp]
        L.orc_sweep.argtypes = [P, dp, u8p, P, C.POINTER(C.c_int64), C.POINTER(C.c_double),
                                C.POINTER(C.c_int32), u64p]
        L.orc_cut_value.argtypes = [P, u8p]; L.orc_cut_value.restype = C.c_double
        L.orc_maxflow_ek.argtypes = [P, C.POINTER(C.c_double), u8p]
        i8p = np.ctypeslib.ndpointer(np.int8, flags="C_CONTIGUOUS")
        L.orc_lambda2.argtypes = [P, C.c_double, C.c_int32, C.c_int32, dp, C.POINTER(C.c_int32), P]
        L.orc_kmeans2.argtypes = [P, dp, dp, C.POINTER(C.c_int32)]
        L.orc_coarsen.argtypes = [P, dp, C.c_double, C.c_double, i8p, i64p, C.POINTER(C.c_int64), i64p, i64p,
                                  u64p, u64p, u64p, u64p, C.POINTER(C.c_int32)]
        L.orc_maxflow_coarse.argtypes = [C.c_int64, i64p, i64p, u64p, u64p, u64p, u64p, u8p, u64p]
        L.orc_two_level.argtypes = [P, dp, u8p, C.POINTER(C.c_double), dp, i64p, u64p, C.POINTER(C.c_int32)]
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


def set_num_threads(n: int = 0) -> int:
    """OpenMP threads of the oracle (0: keep); returns the count in effect.
    Results do not depend on it (tests/test_oracle_threads.py)."""
    return lib().orc_set_num_threads(int(n))


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


def q_to_int(words) -> int:
    """128-bit two's complement (lo, hi) words -> Python int."""
    v = int(words[0]) + (int(words[1]) << 64)
    return v - (1 << 128) if v >= 1 << 127 else v


def q_array(words) -> list:
    w = np.asarray(words, dtype=np.uint64).reshape(-1, 2)
    return [q_to_int(r) for r in w]


@dataclass
class Coarse:
    cls: np.ndarray      # per reduced node: 0 = S0, 1 = S1, 2 = Sc
    cid: np.ndarray      # coarse id (Sc) or -1
    nc: int
    ptr: np.ndarray      # [nc+1]
    col: np.ndarray      # coarse ids, ascending per row
    cap: list            # fixed-point integers per entry
    qs: list             # s_c-link per coarse node
    qt: list             # t_c-link per coarse node
    qst: int             # s_c-t_c edge
    F: int


@dataclass
class TwoLevelResult:
    side: np.ndarray
    cut_value: float
    c0: float
    c1: float
    gamma0: float
    gamma1: float
    rounds: int
    n0: int
    n1: int
    nc: int
    coarse_entries: int
    flow: int
    F: int


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
                 cg_norm=0, warm_start=True, cg_variant=0, block_size=0):
        self.graph = graph
        self.opts = Options(eps, T, cg_rtol, cg_max_iter, cg_norm, int(bool(warm_start)), int(cg_variant),
                            int(block_size))
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

    def blocks(self):
        """A32 partition: (bptr[nblk+1], bnode[n], bfirst[n], boff[n+1])."""
        L = lib()
        nb, n = L.orc_block_count(self.h), self.n
        bptr = np.zeros(nb + 1, dtype=np.int64); bnode = np.zeros(max(n, 1), dtype=np.int64)
        bfirst = np.zeros(max(n, 1), dtype=np.int64); boff = np.zeros(n + 1, dtype=np.int64)
        L.orc_block_export(self.h, bptr, bnode, bfirst, boff)
        return bptr, bnode[:n], bfirst[:n], boff

    def precond(self, r, x=None):
        """Assemble at x (None: W = C), factor, and return (z = M^-1 r, L envelope, pivots)."""
        L = lib()
        n = self.n
        r = np.ascontiguousarray(r, dtype=np.float64)
        z = np.zeros(max(n, 1)); env = np.zeros(max(L.orc_block_env_size(self.h), 1)); Dd = np.zeros(max(n, 1))
        xp = None
        if x is not None:
            x = np.ascontiguousarray(x, dtype=np.float64); xp = x.ctypes.data_as(C.c_void_p)
        L.orc_precond_export(self.h, xp, r, z, env, Dd)
        return z[:n], env, Dd[:n]

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
        pkv = q_to_int(pk)
        return SweepResult(side, order[: self.n], k.value, cut.value, F.value, pkv)

    def cut_value(self, side) -> float:
        return lib().orc_cut_value(self.h, np.ascontiguousarray(side, dtype=np.uint8))

    def kmeans2(self, x=None):
        """A25: (c0, c1, gamma0, gamma1), rounds."""
        x = self.x() if x is None else np.ascontiguousarray(x, dtype=np.float64)
        out = np.zeros(4); r = C.c_int32()
        _check(lib().orc_kmeans2(self.h, x, out, C.byref(r)), "kmeans2")
        return tuple(float(v) for v in out), r.value

    def coarsen(self, x, gamma0, gamma1) -> Coarse:
        x = np.ascontiguousarray(x, dtype=np.float64)
        n, nnz = self.n, max(self.graph.nnz, 1)
        cls = np.zeros(max(n, 1), dtype=np.int8); cid = np.zeros(max(n, 1), dtype=np.int64)
        ptr = np.zeros(n + 1, dtype=np.int64); col = np.zeros(nnz, dtype=np.int64)
        cap = np.zeros(2 * nnz, dtype=np.uint64); qs = np.zeros(2 * max(n, 1), dtype=np.uint64)
        qt = np.zeros(2 * max(n, 1), dtype=np.uint64); qst = np.zeros(2, dtype=np.uint64)
        nc = C.c_int64(); F = C.c_int32()
        _check(lib().orc_coarsen(self.h, x, gamma0, gamma1, cls, cid, C.byref(nc), ptr, col, cap, qs, qt, qst,
                                 C.byref(F)), "coarsen")
        nc = nc.value
        m = int(ptr[nc])
        return Coarse(cls[:n], cid[:n], nc, ptr[: nc + 1].copy(), col[:m].copy(), q_array(cap[: 2 * m]),
                      q_array(qs[: 2 * nc]), q_array(qt[: 2 * nc]), q_to_int(qst), F.value)

    def two_level(self, x=None) -> TwoLevelResult:
        x = self.x() if x is None else np.ascontiguousarray(x, dtype=np.float64)
        side = np.zeros(self.graph.n_total, dtype=np.uint8)
        cut = C.c_double(); d = np.zeros(4); ii = np.zeros(5, dtype=np.int64)
        fl = np.zeros(2, dtype=np.uint64); F = C.c_int32()
        _check(lib().orc_two_level(self.h, x, side, C.byref(cut), d, ii, fl, C.byref(F)), "two_level")
        return TwoLevelResult(side, cut.value, *[float(v) for v in d], *[int(v) for v in ii], q_to_int(fl), F.value)

    def lambda2(self, rtol=1e-12, max_iter=100000, norm=1, want_x=False):
        """A30: (lambda_2, x^T L x, C, cg_iters[, v])."""
        out = np.zeros(3); it = C.c_int32()
        xo = np.zeros(max(self.n, 1)) if want_x else None
        _check(lib().orc_lambda2(self.h, rtol, max_iter, norm, out, C.byref(it),
                                 xo.ctypes.data_as(C.c_void_p) if want_x else None), "lambda2")
        res = (float(out[0]), float(out[1]), float(out[2]), it.value)
        return res + (xo[: self.n],) if want_x else res

    def maxflow(self):
        side = np.zeros(self.graph.n_total, dtype=np.uint8)
        flow = C.c_double()
        _check(lib().orc_maxflow_ek(self.h, C.byref(flow), side), "maxflow")
        return flow.value, side


def maxflow_coarse(nc, ptr, col, cap, qs, qt, qst):
    """Exact max-flow on a fixed-point coarse graph (A28): (flow, src[nc])."""
    def words(vals):
        w = np.zeros(2 * max(len(vals), 1), dtype=np.uint64)
        for i, v in enumerate(vals):
            v &= (1 << 128) - 1
            w[2 * i] = v & ((1 << 64) - 1); w[2 * i + 1] = v >> 64
        return w
    src = np.zeros(max(nc, 1), dtype=np.uint8); fl = np.zeros(2, dtype=np.uint64)
    _check(lib().orc_maxflow_coarse(nc, np.ascontiguousarray(ptr, dtype=np.int64),
                                    np.ascontiguousarray(col, dtype=np.int64) if len(col) else np.zeros(1, np.int64),
                                    words(cap), words(qs), words(qt), words([qst]), src, fl), "maxflow_coarse")
    return q_to_int(fl), src[:nc]
