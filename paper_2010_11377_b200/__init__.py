"""B200-native solve phase for the coupled s-stage IRK systems of arXiv 2010.11377.

Host mirror of the reference's (irkprec) C++ solver interface for the hot path,
over the C ABI of ``include/irkdev.h`` (``lib/libirkdev.so``):

==========================  =====================================================
this module                 reference (``/root/reference/proj``)
==========================  =====================================================
``make_radau_iia``          ``make_radau_iia`` (butcher.hpp:31-34)
``make_lobatto_iiic``       ``make_lobatto_iiic`` (butcher.hpp:36-40)
``ldu_factorize``           ``ldu_factorize`` (butcher.hpp:49-58)
``precond_coeff``           ``precond_coeff`` (butcher.hpp:77)
``custom_coeff``            ``custom_coeff`` (butcher.hpp:81)
``amg_setup``               ``amg_setup`` (amg.hpp:52)
``BlockPreconditioner``     ``BlockPreconditioner`` (stage.hpp:54-95)
``StageOperator``           ``StageOperator`` (stage.hpp:16-42)
``irk_step``                ``irk_step`` (irk.hpp:36-39)
``integrate``               ``integrate`` (irk.hpp:49-59)
``GmresConfig``             ``GmresConfig`` (gmres.hpp:17-21) + ``restart``
``SolveReport``             ``SolveReport`` (gmres.hpp:23-38)
==========================  =====================================================

Errors follow the reference: ``ValueError`` for ``std::invalid_argument``,
``SingularError``, ``NumericalError``; GMRES non-convergence is reported in
``SolveReport.converged``, never raised.  Every solve-phase operation runs on
the GPU; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np

from . import _abi
from ._abi import CudaError, IoError, NumericalError, SingularError, Unsupported, check

__all__ = [
    "CsrMatrix", "Scheme", "CoeffKind", "CoeffStructure", "ButcherTable", "PrecondCoeff",
    "AmgParams", "AmgHierarchy", "GmresConfig", "SolveReport", "IrkStepResult",
    "LinearParabolicSystem", "ProblemSetup", "BlockPreconditioner", "StageOperator",
    "make_radau_iia", "make_lobatto_iiic", "make_table", "ldu_factorize", "precond_coeff",
    "custom_coeff", "read_coeff_file", "make_coeff", "amg_setup", "amg_setup_device", "make_heat_setup", "make_double_glazing_setup", "irk_step",
    "integrate", "SingularError", "NumericalError", "CudaError", "Unsupported",
    "IoError",
]


@dataclass
class CsrMatrix:
    """CSR with int32 indices and fp64 values (csr.hpp:15-32)."""
    row_ptr: np.ndarray
    col_idx: np.ndarray
    vals: np.ndarray
    n_cols: int

    @property
    def n_rows(self) -> int:
        return len(self.row_ptr) - 1

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def view(self) -> _abi.irk_csr:
        self.row_ptr = np.ascontiguousarray(self.row_ptr, dtype=np.int32)
        self.col_idx = np.ascontiguousarray(self.col_idx, dtype=np.int32)
        self.vals = np.ascontiguousarray(self.vals, dtype=np.float64)
        return _abi.csr_view(self.row_ptr, self.col_idx, self.vals, self.n_cols)

    @classmethod
    def from_view(cls, v: _abi.irk_csr) -> "CsrMatrix":
        rp, ci, vals, nc = _abi.csr_arrays(v)
        return cls(rp, ci, vals, nc)

    def matvec(self, x: np.ndarray) -> np.ndarray:
        """Host convenience product (tests/diagnostics only)."""
        rows = np.repeat(np.arange(self.n_rows), np.diff(self.row_ptr))
        return np.bincount(rows, weights=self.vals * x[self.col_idx], minlength=self.n_rows)


class Scheme(IntEnum):
    RadauIIA = 0
    LobattoIIIC = 1


class CoeffKind(IntEnum):
    Jacobi = 0
    GaussSeidelLower = 1
    UpperFactor = 2
    LowerFactor = 3
    Custom = 4


class CoeffStructure(IntEnum):
    Diagonal = 0
    LowerTriangular = 1
    UpperTriangular = 2


@dataclass
class ButcherTable:
    scheme: Scheme
    s: int
    A: np.ndarray
    b: np.ndarray
    c: np.ndarray
    q: int


def make_table(scheme: Scheme, s: int) -> ButcherTable:
    A = np.zeros(s * s)
    b = np.zeros(s)
    c = np.zeros(s)
    q = C.c_int()
    check(_abi.lib().irk_tableau(int(scheme), s, _abi.as_d(A), _abi.as_d(b), _abi.as_d(c), C.byref(q)))
    return ButcherTable(Scheme(scheme), s, A.reshape(s, s), b, c, q.value)


def make_radau_iia(s: int) -> ButcherTable:
    return make_table(Scheme.RadauIIA, s)


def make_lobatto_iiic(s: int) -> ButcherTable:
    return make_table(Scheme.LobattoIIIC, s)


def ldu_factorize(A: np.ndarray):
    A = np.ascontiguousarray(A, dtype=np.float64)
    s = A.shape[0]
    L, D, U = np.zeros(s * s), np.zeros(s), np.zeros(s * s)
    check(_abi.lib().irk_ldu(s, _abi.as_d(A.ravel()), _abi.as_d(L), _abi.as_d(D), _abi.as_d(U)))
    return L.reshape(s, s), D, U.reshape(s, s)


@dataclass
class PrecondCoeff:
    kind: CoeffKind
    Atilde: np.ndarray
    structure: CoeffStructure


def precond_coeff(table: ButcherTable, kind: CoeffKind) -> PrecondCoeff:
    s = table.s
    At = np.zeros(s * s)
    st = C.c_int()
    check(_abi.lib().irk_precond_coeff(int(table.scheme), s, int(kind), _abi.as_d(At), C.byref(st)))
    return PrecondCoeff(CoeffKind(kind), At.reshape(s, s), CoeffStructure(st.value))


def custom_coeff(Atilde: np.ndarray) -> PrecondCoeff:
    At = np.ascontiguousarray(Atilde, dtype=np.float64)
    if At.ndim != 2 or At.shape[0] != At.shape[1]:
        raise ValueError("custom_coeff: not square")
    st = C.c_int()
    check(_abi.lib().irk_custom_coeff(At.shape[0], _abi.as_d(At.ravel()), C.byref(st)))
    return PrecondCoeff(CoeffKind.Custom, At.copy(), CoeffStructure(st.value))


def read_coeff_file(path) -> np.ndarray:
    """read_coeff_file (butcher.cpp:300-313): the s x s matrix of a
    coefficient file ("s" then s*s row-major values).  IoError on a missing
    file, a bad stage count or truncated data."""
    L = _abi.lib()
    s = C.c_int()
    bp = str(path).encode()
    check(L.irk_read_coeff_file(bp, 0, C.byref(s), None))
    At = np.zeros(s.value * s.value)
    check(L.irk_read_coeff_file(bp, At.size, C.byref(s), _abi.as_d(At)))
    return At.reshape(s.value, s.value)


def make_coeff(table: ButcherTable, kind: CoeffKind, custom_coeff_path=None) -> PrecondCoeff:
    """make_coeff (study.cpp:269-282): precond_coeff for the built-in kinds; for
    Custom the matrix of `custom_coeff_path` (ValueError without a path or when
    its size is not table.s), validated by custom_coeff."""
    s = table.s
    At = np.zeros(s * s)
    st = C.c_int()
    path = None if custom_coeff_path is None else str(custom_coeff_path).encode()
    check(_abi.lib().irk_make_coeff(int(table.scheme), s, int(kind), path, _abi.as_d(At),
                                    C.byref(st)))
    return PrecondCoeff(CoeffKind(kind), At.reshape(s, s), CoeffStructure(st.value))


@dataclass
class AmgParams:
    """AmgParams (amg.hpp:14-29); library defaults = BASELINE's V(1,1) Jacobi."""
    theta: float = 0.25
    pre_sweeps: int = 1
    post_sweeps: int = 1
    smoother: int = 0
    jacobi_weight: float = 2.0 / 3.0
    prolongation_weight: float = 4.0 / 3.0
    prolongation_steps: int = 1
    max_coarse: int = 64
    max_levels: int = 10

    def c(self) -> _abi.irk_amg_params:
        return _abi.irk_amg_params(self.theta, self.pre_sweeps, self.post_sweeps, self.smoother,
                                   self.jacobi_weight, self.prolongation_weight,
                                   self.prolongation_steps, self.max_coarse, self.max_levels)


class AmgHierarchy:
    """Smoothed-aggregation hierarchy built by the host setup (amg.hpp:33-46)."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle

    def __del__(self):
        if getattr(self, "_h", None) and _abi is not None and _abi._lib is not None:
            _abi._lib.irk_hierarchy_free(self._h)
            self._h = None

    def n_levels(self) -> int:
        return _abi.lib().irk_hierarchy_levels(self._h)

    def level(self, l: int, which: str = "A") -> CsrMatrix:
        v = _abi.irk_csr()
        check(_abi.lib().irk_hierarchy_level(self._h, l, {"A": 0, "P": 1, "R": 2, "G": 3, "U": 4}[which], C.byref(v)))
        return CsrMatrix.from_view(v)

    def compose_lanes(self, l: int) -> tuple[int, int]:
        """Row-sum lanes (G, U) of level l's composed legs (csrc/host/compose.cpp)."""
        g, u = C.c_int(), C.c_int()
        check(_abi.lib().irk_hierarchy_compose_lanes(self._h, l, C.byref(g), C.byref(u)))
        return g.value, u.value

    def inv_diag(self, l: int) -> np.ndarray:
        n = self.level(l).n_rows
        return np.ctypeslib.as_array(_abi.lib().irk_hierarchy_inv_diag(self._h, l), (n,)).copy()

    def coarse_inverse(self) -> np.ndarray:
        n = C.c_int()
        p = _abi.lib().irk_hierarchy_coarse_inverse(self._h, C.byref(n))
        return np.ctypeslib.as_array(p, (n.value * n.value,)).copy().reshape(n.value, n.value)

    def sizes(self) -> list[int]:
        return [self.level(l).n_rows for l in range(self.n_levels())]

    def tail(self):
        """(level, B): the dense operator of the V-cycle below `level`
        (csrc/host/tail.cpp), B of shape (n, ld); (-1, None) if none."""
        f, n, ld = C.c_int(), C.c_int(), C.c_int()
        p = _abi.lib().irk_hierarchy_tail(self._h, C.byref(f), C.byref(n), C.byref(ld))
        if not p:
            return -1, None
        return f.value, np.ctypeslib.as_array(p, (n.value * ld.value,)).copy().reshape(n.value, ld.value)


def amg_setup(A: CsrMatrix, params: AmgParams | None = None) -> AmgHierarchy:
    h = C.c_void_p()
    v = A.view()
    check(_abi.lib().irk_amg_setup(C.byref(v), C.byref((params or AmgParams()).c()), C.byref(h)))
    return AmgHierarchy(h)


def amg_setup_device(A: CsrMatrix, params: AmgParams | None = None, device: int = 0) -> AmgHierarchy:
    """amg_setup (amg.cpp:172-227) with the sparse algebra on GPU `device`
    (SURVEY §8 f2); bit-identical to ``amg_setup``.  Raises without a GPU."""
    h = C.c_void_p()
    v = A.view()
    check(_abi.lib().irk_amg_setup_device(C.byref(v), C.byref((params or AmgParams()).c()), int(device),
                                          C.byref(h)))
    return AmgHierarchy(h)


# ---------------------------------------------------------- on-disk formats
def write_matrix_market(A: CsrMatrix, path) -> None:
    """write_matrix_market (csr.cpp:240-251): coordinate real general, %.17g."""
    check(_abi.lib().irk_mm_write(C.byref(A.view()), str(path).encode()))


def read_matrix_market(path) -> CsrMatrix:
    """read_matrix_market (csr.cpp:253-290): general or symmetric coordinate real."""
    L = _abi.lib()
    h = C.c_void_p()
    check(L.irk_mm_read(str(path).encode(), C.byref(h)))
    try:
        v = _abi.irk_csr()
        check(L.irk_matrix_view(h, C.byref(v)))
        rp, ci, vals, nc = _abi.csr_arrays(v)
        return CsrMatrix(rp.copy(), ci.copy(), vals.copy(), nc)
    finally:
        L.irk_matrix_free(h)


def csv_header() -> str:
    """study.cpp:334-337."""
    buf = C.create_string_buffer(256)
    check(_abi.lib().irk_csv_header(buf, len(buf)))
    return buf.value.decode()


def csv_row(table: ButcherTable, hx_inv: int, ht: float, n_free: int, coeff_kind: CoeffKind,
            cfg: GmresConfig, iterations: float, true_residual: float, rel_error: float,
            seconds: float, failed: bool = False) -> str:
    """study.cpp:339-360 (AMG subsolver: the only one on the device)."""
    buf = C.create_string_buffer(512)
    check(_abi.lib().irk_csv_row(int(table.scheme), table.s, hx_inv, ht, n_free, int(coeff_kind),
                                 0 if cfg.side == "left" else 1, 0, float(iterations),
                                 float(true_residual), float(rel_error), float(seconds),
                                 1 if failed else 0, buf, len(buf)))
    return buf.value.decode()


@dataclass
class LinearParabolicSystem:
    """M du/dt = -F u - f_lift + forcing(t) over the free dofs (irk.hpp:15-22).

    ``forcing`` (may be None) maps t to an n-vector, like the reference's
    ``std::function<Vec(double)>``; it is evaluated on the host at the stage
    times t_n + c_i h_t and uploaded."""
    M: CsrMatrix
    F: CsrMatrix
    f_lift: np.ndarray | None = None
    forcing: object = None

    def n(self) -> int:
        return self.M.n_rows


class ProblemSetup:
    """Host-assembled P1 problem (heat or double glazing) with its u0 recipe."""

    def __init__(self, handle: C.c_void_p, kind: str, cells: int):
        self._h = handle
        self.kind = kind
        self.cells = cells
        L = _abi.lib()
        mv, kv = _abi.irk_csr(), _abi.irk_csr()
        check(L.irk_problem_matrix(handle, 0, C.byref(mv)))
        check(L.irk_problem_matrix(handle, 1, C.byref(kv)))
        self.M = CsrMatrix.from_view(mv)
        self.F = CsrMatrix.from_view(kv)
        n = self.M.n_rows
        self.f_lift = np.ctypeslib.as_array(L.irk_problem_lift(handle), (n,)).copy()
        self.sys = LinearParabolicSystem(self.M, self.F, self.f_lift)

    def __del__(self):
        if getattr(self, "_h", None) and _abi is not None and _abi._lib is not None:
            _abi._lib.irk_problem_free(self._h)
            self._h = None

    def initial(self, noise: float = 0.0, seed: int = 1) -> np.ndarray:
        if self.kind == "double_glazing":
            return np.zeros(self.M.n_rows)
        u = np.zeros(self.M.n_rows)
        check(_abi.lib().irk_problem_initial(self._h, noise, seed, _abi.as_d(u)))
        return u


def make_heat_setup(cells: int) -> ProblemSetup:
    h = C.c_void_p()
    check(_abi.lib().irk_problem_heat(cells, C.byref(h)))
    return ProblemSetup(h, "heat", cells)


def make_double_glazing_setup(cells: int, eps: float = 0.005) -> ProblemSetup:
    h = C.c_void_p()
    check(_abi.lib().irk_problem_double_glazing(cells, eps, C.byref(h)))
    return ProblemSetup(h, "double_glazing", cells)


@dataclass
class GmresConfig:
    """GmresConfig (gmres.hpp:17-21) + GMRES(m) restart (0 = full GMRES)."""
    side: str = "right"
    rel_tol: float = 1e-8
    max_iter: int = 500
    restart: int = 0  # full GMRES, as the reference (gmres.hpp:20); BASELINE runs GMRES(50)

    def c(self) -> _abi.irk_gmres_cfg:
        if self.side not in ("right", "left"):
            raise ValueError("gmres: side must be 'right' or 'left'")
        return _abi.irk_gmres_cfg(1 if self.side == "right" else 0, self.rel_tol, self.max_iter,
                                  self.restart)


@dataclass
class SolveReport:
    iterations: int = 0
    history: list = field(default_factory=list)
    final_rel_residual: float = 0.0
    true_rel_residual: float = 0.0
    converged: bool = True
    solve_seconds: float = 0.0
    setup_seconds: float = 0.0
    cycles: int = 0
    n_reorth: int = 0
    rel_error: float = math.nan


@dataclass
class IrkStepResult:
    u_next: np.ndarray
    report: SolveReport
    K: np.ndarray | None = None


def _report(r: _abi.irk_report, hist: np.ndarray | None) -> SolveReport:
    return SolveReport(r.iterations, [] if hist is None else list(hist[: r.history_len]),
                       r.final_rel_residual, r.true_rel_residual, bool(r.converged),
                       r.solve_seconds, r.setup_seconds, r.cycles, r.n_reorth)


class _Device:
    """One irkdev handle: M, K, the Butcher matrix, Atilde and the hierarchies."""

    def __init__(self, M: CsrMatrix, F: CsrMatrix, A: np.ndarray, b: np.ndarray,
                 coeff: PrecondCoeff, ht: float, amg: AmgParams, hiers=None, device: int = 0):
        s = A.shape[0]
        self.s, self.n = s, M.n_rows
        self.A = np.ascontiguousarray(A, dtype=np.float64)
        self.b = np.ascontiguousarray(b, dtype=np.float64)
        self._keep = (M, F)
        mv, kv = M.view(), F.view()
        h = C.c_void_p()
        hp = None
        nh = 0
        if hiers:
            nh = len(hiers)
            hp = (C.c_void_p * nh)(*[x._h for x in hiers])
        check(_abi.lib().irkdev_create(
            C.byref(mv), C.byref(kv), s, _abi.as_d(self.A.ravel()),
            _abi.as_d(self.b),
            _abi.as_d(np.ascontiguousarray(coeff.Atilde, dtype=np.float64).ravel()),
            int(coeff.structure), ht, C.byref(amg.c()), nh, hp, device, C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) and _abi is not None and _abi._lib is not None:
            _abi._lib.irkdev_destroy(self._h)
            self._h = None

    def info(self):
        n, s, nh = C.c_int(), C.c_int(), C.c_int()
        sob = (C.c_int * self.s)()
        setup = C.c_double()
        check(_abi.lib().irkdev_info(self._h, C.byref(n), C.byref(s), C.byref(nh), sob, C.byref(setup)))
        return {"n": n.value, "s": s.value, "n_hier": nh.value, "solver_of_block": list(sob),
                "setup_seconds": setup.value}

    def _apply(self, fn, v: np.ndarray, *extra) -> np.ndarray:
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.empty_like(v)
        check(fn(self._h, *extra, _abi.as_d(v), _abi.as_d(out)))
        return out


class BlockPreconditioner:
    """I_s (x) M + ht Atilde (x) F with one AMG V-cycle per block (stage.hpp:54-95).

    Only the AMG subsolver runs on the device (BASELINE's path); ``ExactLU`` is
    analysis-only in the reference and out of scope here.
    """

    def __init__(self, M: CsrMatrix, F: CsrMatrix, coeff: PrecondCoeff, ht: float,
                 amg_params: AmgParams | None = None, table: ButcherTable | None = None,
                 hierarchies=None, device: int = 0):
        self.M, self.F, self.coeff, self.ht = M, F, coeff, ht
        self.amg_params = amg_params or AmgParams()
        self._hiers = hierarchies
        self._device = device
        s = coeff.Atilde.shape[0]
        A = table.A if table is not None else coeff.Atilde
        b = table.b if table is not None else np.zeros(s)
        self._dev = _Device(M, F, A, b, coeff, ht, self.amg_params, hierarchies, device)

    def stages(self) -> int:
        return self._dev.s

    def size(self) -> int:
        return self._dev.s * self._dev.n

    def distinct_subsolvers(self) -> int:
        return self._dev.info()["n_hier"]

    def hierarchy(self, k: int) -> AmgHierarchy:
        """The k-th distinct subsolver's hierarchy as built and uploaded."""
        h = C.c_void_p()
        check(_abi.lib().irkdev_hierarchy(self._dev._h, int(k), C.byref(h)))
        return AmgHierarchy(h)

    def setup_seconds(self) -> float:
        return self._dev.info()["setup_seconds"]

    def apply(self, v: np.ndarray) -> np.ndarray:
        return self._dev._apply(_abi.lib().irkdev_precond_apply, v)

    def vcycle(self, k: int, r: np.ndarray) -> np.ndarray:
        return self._dev._apply(_abi.lib().irkdev_vcycle, r, k)

    def bind_table(self, table: ButcherTable) -> None:
        """Rebuild the device handle with the stage operator of `table`."""
        if np.array_equal(self._dev.A, table.A) and np.array_equal(self._dev.b, table.b):
            return
        self._dev = None  # release the old handle before allocating the new one
        self._dev = _Device(self.M, self.F, table.A, table.b, self.coeff, self.ht,
                            self.amg_params, self._hiers, self._device)


class StageOperator:
    """I_s (x) M + ht A (x) F, applied on the device (stage.hpp:16-42)."""

    def __init__(self, P: BlockPreconditioner):
        self._dev = P._dev

    def apply(self, v: np.ndarray) -> np.ndarray:
        return self._dev._apply(_abi.lib().irkdev_stage_apply, v)


class _Forcing:
    """irk_forcing_fn around a Python callable; re-raises its exception."""

    def __init__(self, fn):
        self.fn, self.error = fn, None
        self.c = _abi.FORCING_FN(self._call) if fn is not None else _abi.FORCING_FN()

    def _call(self, t, out, n, user):
        try:
            f = np.ascontiguousarray(self.fn(t), dtype=np.float64)
            if f.shape != (n,):
                raise ValueError("stage_rhs: forcing size mismatch")
            C.memmove(out, f.ctypes.data, 8 * n)
            return 0
        except Exception as e:  # surfaced after the C call returns
            self.error = self.error or e
            return 1

    def reraise(self):
        if self.error is not None:
            raise self.error


def _check_precond(P, ht: float, table: ButcherTable, n: int) -> None:
    if P is None:
        raise Unsupported("the device path needs a BlockPreconditioner")
    if P.ht != ht:
        raise ValueError("irk_step: preconditioner built for a different ht")
    P.bind_table(table)
    if P._dev.n != n:
        raise ValueError("stage_rhs: dimension mismatch")


def irk_step(sys: LinearParabolicSystem, table: ButcherTable, ht: float, t_n: float,
             u_n: np.ndarray, P: BlockPreconditioner, cfg: GmresConfig | None = None,
             want_K: bool = False) -> IrkStepResult:
    """One IRK step (irk.cpp:35-68): stage rhs (with forcing at t_n + c_i h_t),
    GMRES(m) with P, u_{n+1}."""
    if ht <= 0.0:
        raise ValueError("irk_step: ht must be positive")
    u = np.ascontiguousarray(u_n, dtype=np.float64)
    _check_precond(P, ht, table, u.shape[0])
    cfg = cfg or GmresConfig()
    dev = P._dev
    un = np.empty_like(u)
    K = np.empty(dev.n * dev.s) if want_K else None
    hist = np.empty(cfg.max_iter + 1)
    rep = _abi.irk_report()
    lift = None if sys.f_lift is None else np.ascontiguousarray(sys.f_lift, dtype=np.float64)
    L = _abi.lib()
    if sys.forcing is None:
        check(L.irkdev_step(dev._h, _abi.as_d(u), None if lift is None else _abi.as_d(lift),
                            C.byref(cfg.c()), _abi.as_d(un), None if K is None else _abi.as_d(K),
                            C.byref(rep), _abi.as_d(hist)))
    else:
        fc = _Forcing(sys.forcing)
        c = np.ascontiguousarray(table.c, dtype=np.float64)
        rc = L.irkdev_step_forced(dev._h, _abi.as_d(u), None if lift is None else _abi.as_d(lift),
                                  float(t_n), _abi.as_d(c), fc.c, None, C.byref(cfg.c()),
                                  _abi.as_d(un), None if K is None else _abi.as_d(K),
                                  C.byref(rep), _abi.as_d(hist))
        fc.reraise()
        check(rc)
    return IrkStepResult(un, _report(rep, hist), K)


@dataclass
class TrajectorySummary:
    u_final: np.ndarray
    t_final: float = 0.0
    steps: int = 0
    reports: list = field(default_factory=list)
    all_converged: bool = True


def integrate(sys: LinearParabolicSystem, table: ButcherTable, u0: np.ndarray, t_final: float,
              ht: float, make_precond, cfg: GmresConfig | None = None) -> TrajectorySummary:
    """Time loop of irk.cpp:70-102 (truncated last step, factory consulted on a
    step-size change), device-resident: u stays in HBM between steps
    (irkdev_integrate); only the forcing is evaluated on the host."""
    if ht <= 0.0:
        raise ValueError("integrate: ht must be positive")
    if t_final < 0.0:
        raise ValueError("integrate: t_final must be nonnegative")
    cfg = cfg or GmresConfig()
    u = np.ascontiguousarray(u0, dtype=np.float64)
    L = _abi.lib()
    nsteps = C.c_int()
    check(L.irk_integrate_steps(float(t_final), float(ht), C.byref(nsteps)))
    if nsteps.value == 0:
        return TrajectorySummary(u.copy(), 0.0, 0, [], True)
    P = make_precond(ht)
    _check_precond(P, ht, table, u.shape[0])
    keep, errors = [P], []

    def factory(h, user):
        try:
            Q = make_precond(h)
            _check_precond(Q, h, table, u.shape[0])
            keep.append(Q)
            return Q._dev._h.value
        except Exception as e:
            errors.append(e)
            return None

    fac = _abi.FACTORY_FN(factory)
    fc = _Forcing(sys.forcing)
    c = np.ascontiguousarray(table.c, dtype=np.float64)
    lift = None if sys.f_lift is None else np.ascontiguousarray(sys.f_lift, dtype=np.float64)
    cap = nsteps.value
    reps = (_abi.irk_report * cap)()
    hl = cfg.max_iter + 1
    hist = np.empty(cap * hl)
    uf = np.empty_like(u)
    steps, t_out, conv = C.c_int(), C.c_double(), C.c_int()
    rc = L.irkdev_integrate(P._dev._h, fac, None, _abi.as_d(u),
                            None if lift is None else _abi.as_d(lift), _abi.as_d(c), fc.c, None,
                            float(t_final), float(ht), C.byref(cfg.c()), _abi.as_d(uf), reps, cap,
                            _abi.as_d(hist), C.byref(steps), C.byref(t_out), C.byref(conv))
    if errors:
        raise errors[0]
    fc.reraise()
    check(rc)
    return TrajectorySummary(uf, t_out.value, steps.value,
                             [_report(reps[k], hist[k * hl:(k + 1) * hl]) for k in range(steps.value)],
                             bool(conv.value))
