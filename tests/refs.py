"""Loaders for the two CPU checkers (test infrastructure only).

* ``Ref``    -- oracle/_ref/libirkref.so: the reference's own hot-path sources
               compiled in place (oracle/Makefile), driven through
               oracle/ref_harness.cpp.
* ``Oracle`` -- oracle/_build/liboracle.so: the C restatement (oracle/irk_oracle.c)
               whose operation order mirrors the device kernels.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
REF_SO = ROOT / "oracle" / "_ref" / "libirkref.so"
ORACLE_SO = ROOT / "oracle" / "_build" / "liboracle.so"

dptr = C.POINTER(C.c_double)
iptr = C.POINTER(C.c_int)


def _d(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64).ctypes.data_as(dptr)


def _i(a):
    return np.ascontiguousarray(a, dtype=np.int32).ctypes.data_as(iptr)


# ----------------------------------------------------------------- reference
class Ref:
    """The reference (irkprec) hot path, compiled from /root/reference sources."""

    _lib = None

    @classmethod
    def available(cls) -> bool:
        return REF_SO.exists()

    @classmethod
    def lib(cls):
        if cls._lib is None:
            L = C.CDLL(str(REF_SO))
            L.ref_last_error.restype = C.c_char_p
            L.ref_problem_flift.restype = dptr
            L.ref_amg_invdiag.restype = dptr
            L.ref_solver_setup_seconds.restype = C.c_double
            L.ref_dot.restype = C.c_double
            L.ref_problem_create.argtypes = [C.c_int, C.c_int, C.c_double, C.POINTER(C.c_void_p)]
            L.ref_solver_create.argtypes = [C.c_int, iptr, iptr, dptr, iptr, iptr, dptr, C.c_int,
                                            C.c_int, C.c_int, C.c_double, C.c_double, C.c_int,
                                            C.c_int, C.c_int, C.POINTER(C.c_void_p)]
            L.ref_solver_create_ex.argtypes = [C.c_int, iptr, iptr, dptr, iptr, iptr, dptr,
                                               C.c_int, C.c_int, C.c_int, dptr, C.c_double,
                                               dptr, iptr, C.POINTER(C.c_void_p)]
            L.ref_amg_setup_ex.argtypes = [C.c_int, iptr, iptr, dptr, dptr, iptr,
                                           C.POINTER(C.c_void_p)]
            L.ref_coeff_file.argtypes = [C.c_char_p, C.c_int, iptr, dptr, iptr]
            L.ref_amg_setup.argtypes = [C.c_int, iptr, iptr, dptr, C.c_double, C.c_int, C.c_int,
                                        C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
            L.ref_irk_step.argtypes = [C.c_void_p, dptr, dptr, C.c_double, C.c_int, C.c_int,
                                       dptr, dptr, iptr, iptr, dptr, iptr, dptr, dptr, C.c_int,
                                       iptr]
            L.ref_irk_step_forced.argtypes = [C.c_void_p, dptr, dptr, C.c_double, dptr, C.c_int,
                                              C.c_double, C.c_int, C.c_int, dptr, dptr, iptr,
                                              iptr, dptr, iptr, dptr, dptr, C.c_int, iptr]
            L.ref_integrate.argtypes = [C.c_void_p, C.c_void_p, dptr, dptr, dptr, C.c_double,
                                        C.c_double, C.c_int, dptr, iptr, dptr, iptr, C.c_int,
                                        iptr]
            for name in ("ref_problem_free", "ref_amg_free", "ref_solver_free"):
                getattr(L, name).argtypes = [C.c_void_p]
            L.ref_problem_csr.argtypes = [C.c_void_p, C.c_int, iptr, iptr, C.POINTER(iptr),
                                          C.POINTER(iptr), C.POINTER(dptr)]
            L.ref_problem_flift.argtypes = [C.c_void_p]
            L.ref_problem_initial.argtypes = [C.c_void_p, C.c_double, C.c_ulonglong, dptr]
            L.ref_amg_nlevels.argtypes = [C.c_void_p]
            L.ref_amg_level.argtypes = [C.c_void_p, C.c_int, C.c_int, iptr, iptr, iptr,
                                        C.POINTER(iptr), C.POINTER(iptr), C.POINTER(dptr)]
            L.ref_amg_invdiag.argtypes = [C.c_void_p, C.c_int]
            L.ref_amg_vcycle.argtypes = [C.c_void_p, dptr, dptr]
            L.ref_stage_apply.argtypes = [C.c_void_p, dptr, dptr]
            L.ref_precond_apply.argtypes = [C.c_void_p, dptr, dptr]
            L.ref_solver_setup_seconds.argtypes = [C.c_void_p]
            L.ref_solver_distinct.argtypes = [C.c_void_p]
            L.ref_butcher.argtypes = [C.c_int, C.c_int, dptr, dptr, dptr, iptr]
            L.ref_precond_coeff.argtypes = [C.c_int, C.c_int, C.c_int, dptr, iptr]
            L.ref_ldu.argtypes = [C.c_int, dptr, dptr, dptr, dptr]
            L.ref_spmv.argtypes = [C.c_int, C.c_int, iptr, iptr, dptr, dptr, dptr]
            L.ref_dot.argtypes = [C.c_int, dptr, dptr]
            L.ref_mm_write.argtypes = [C.c_int, C.c_int, iptr, iptr, dptr, C.c_char_p]
            L.ref_mm_read.argtypes = [C.c_char_p, iptr, iptr, iptr, iptr, iptr, dptr]
            cls._lib = L
        return cls._lib

    @classmethod
    def check(cls, status):
        if status != 0:
            raise RuntimeError(f"reference error {status}: {cls.lib().ref_last_error().decode()}")

    # -- problems
    @classmethod
    def problem(cls, kind: str, cells: int, eps: float = 0.005, initial=None):
        """M, K, f_lift of the reference assembly; with initial=(noise, seed) also
        the benchmark u0 computed from the reference mesh (ref_problem_initial)."""
        L = cls.lib()
        h = C.c_void_p()
        cls.check(L.ref_problem_create(0 if kind == "heat" else 1, cells, eps, C.byref(h)))
        out = {}
        for which, name in ((0, "M"), (1, "K")):
            n, nnz = C.c_int(), C.c_int()
            rp, ci, v = iptr(), iptr(), dptr()
            L.ref_problem_csr(h, which, C.byref(n), C.byref(nnz), C.byref(rp), C.byref(ci), C.byref(v))
            N, NZ = n.value, nnz.value
            out[name] = (np.ctypeslib.as_array(rp, (N + 1,)).copy(),
                         np.ctypeslib.as_array(ci, (NZ,)).copy(),
                         np.ctypeslib.as_array(v, (NZ,)).copy())
        out["f_lift"] = np.ctypeslib.as_array(L.ref_problem_flift(h), (len(out["M"][0]) - 1,)).copy()
        if initial is not None:
            u0 = np.empty(len(out["f_lift"]))
            cls.check(L.ref_problem_initial(h, float(initial[0]), int(initial[1]), _d(u0)))
            out["u0"] = u0
        L.ref_problem_free(h)
        return out

    @classmethod
    def tableau(cls, scheme: int, s: int):
        A, b, c = np.zeros(s * s), np.zeros(s), np.zeros(s)
        q = C.c_int()
        cls.check(cls.lib().ref_butcher(scheme, s, _d(A), _d(b), _d(c), C.byref(q)))
        # _d copies only when needed; A is already contiguous float64
        return A.reshape(s, s), b, c, q.value

    @classmethod
    def precond_coeff(cls, scheme: int, s: int, kind: int):
        At = np.zeros(s * s)
        st = C.c_int()
        cls.check(cls.lib().ref_precond_coeff(scheme, s, kind, _d(At), C.byref(st)))
        return At.reshape(s, s), st.value

    @classmethod
    def ldu(cls, A):
        s = A.shape[0]
        L, D, U = np.zeros(s * s), np.zeros(s), np.zeros(s * s)
        cls.check(cls.lib().ref_ldu(s, _d(np.ascontiguousarray(A).ravel()), _d(L), _d(D), _d(U)))
        return L.reshape(s, s), D, U.reshape(s, s)

    @classmethod
    def amg(cls, csr, theta=0.25, pre=1, post=1, max_coarse=64, max_levels=10, psteps=1):
        rp, ci, v = csr
        h = C.c_void_p()
        keep = [np.ascontiguousarray(rp, np.int32), np.ascontiguousarray(ci, np.int32),
                np.ascontiguousarray(v, np.float64)]
        cls.check(cls.lib().ref_amg_setup(len(rp) - 1, _i(keep[0]), _i(keep[1]), _d(keep[2]), theta,
                                          pre, post, max_coarse, max_levels, psteps, C.byref(h)))
        return RefHierarchy(h)

    @classmethod
    def amg_ex(cls, csr, amg):
        """amg_setup with every AmgParams field (amg: an AmgParams-like object)."""
        rp, ci, v = csr
        h = C.c_void_p()
        keep = [np.ascontiguousarray(rp, np.int32), np.ascontiguousarray(ci, np.int32),
                np.ascontiguousarray(v, np.float64)]
        d, i = _amg_arrays(amg)
        cls.check(cls.lib().ref_amg_setup_ex(len(rp) - 1, _i(keep[0]), _i(keep[1]), _d(keep[2]),
                                             _d(d), _i(i), C.byref(h)))
        return RefHierarchy(h)

    @classmethod
    def coeff_file(cls, path):
        """custom_coeff(read_coeff_file(path)) -> (At, structure); raises
        RuntimeError with the reference's status (6 = std::runtime_error)."""
        L = cls.lib()
        s = C.c_int()
        st = C.c_int()
        bp = str(path).encode()
        rc = L.ref_coeff_file(bp, 0, C.byref(s), None, C.byref(st))
        if rc != 0:
            raise RefError(rc, L.ref_last_error().decode())
        At = np.zeros(s.value * s.value)
        rc = L.ref_coeff_file(bp, At.size, C.byref(s), _d(At), C.byref(st))
        if rc != 0:
            raise RefError(rc, L.ref_last_error().decode())
        return At.reshape(s.value, s.value), st.value

    @classmethod
    def spmv(cls, csr, x, n_cols=None):
        rp, ci, v = csr
        n = len(rp) - 1
        y = np.zeros(n)
        x = np.ascontiguousarray(x, np.float64)
        cls.check(cls.lib().ref_spmv(n, n_cols or len(x), _i(rp), _i(ci), _d(v), _d(x), _d(y)))
        return y


class RefError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"reference error {status}: {msg}")
        self.status = status


def _amg_arrays(amg):
    d = np.array([amg.theta, amg.jacobi_weight, amg.prolongation_weight], np.float64)
    i = np.array([amg.pre_sweeps, amg.post_sweeps, amg.smoother, amg.prolongation_steps,
                  amg.max_coarse, amg.max_levels], np.int32)
    return d, i


class RefHierarchy:
    def __init__(self, h):
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            Ref.lib().ref_amg_free(self.h)
            self.h = None

    def n_levels(self):
        return Ref.lib().ref_amg_nlevels(self.h)

    def level(self, l, which="A"):
        nr, nc, nnz = C.c_int(), C.c_int(), C.c_int()
        rp, ci, v = iptr(), iptr(), dptr()
        Ref.check(Ref.lib().ref_amg_level(self.h, l, {"A": 0, "P": 1, "R": 2}[which], C.byref(nr),
                                          C.byref(nc), C.byref(nnz), C.byref(rp), C.byref(ci),
                                          C.byref(v)))
        N, NZ = nr.value, nnz.value
        if NZ == 0:
            return (np.ctypeslib.as_array(rp, (N + 1,)).copy() if N >= 0 and rp else np.zeros(1, np.int32),
                    np.zeros(0, np.int32), np.zeros(0)), nc.value
        return (np.ctypeslib.as_array(rp, (N + 1,)).copy(), np.ctypeslib.as_array(ci, (NZ,)).copy(),
                np.ctypeslib.as_array(v, (NZ,)).copy()), nc.value

    def inv_diag(self, l):
        n = len(self.level(l)[0][0]) - 1
        return np.ctypeslib.as_array(Ref.lib().ref_amg_invdiag(self.h, l), (n,)).copy()

    def vcycle(self, r):
        r = np.ascontiguousarray(r, np.float64)
        z = np.zeros_like(r)
        Ref.check(Ref.lib().ref_amg_vcycle(self.h, _d(r), _d(z)))
        return z


class RefSolver:
    """BlockPreconditioner(AMG) + StageOperator of the reference on given M, K."""

    def __init__(self, M, K, scheme, s, kind, ht, theta=0.25, pre=1, post=1, max_coarse=64,
                 amg=None, custom_At=None):
        """amg (an AmgParams-like object) overrides theta/pre/post/max_coarse
        and sets every AmgParams field; kind 4 with custom_At = custom_coeff."""
        self._keep = [np.ascontiguousarray(a) for a in (*M, *K)]
        m_rp, m_ci, m_v, k_rp, k_ci, k_v = self._keep
        self.n = len(m_rp) - 1
        self.s = s
        h = C.c_void_p()
        if amg is None and custom_At is None:
            Ref.check(Ref.lib().ref_solver_create(self.n, _i(m_rp), _i(m_ci), _d(m_v), _i(k_rp),
                                                  _i(k_ci), _d(k_v), scheme, s, kind, ht, theta,
                                                  pre, post, max_coarse, C.byref(h)))
        else:
            if amg is None:
                import paper_2010_11377_b200 as P
                amg = P.AmgParams(theta=theta, pre_sweeps=pre, post_sweeps=post,
                                  max_coarse=max_coarse)
            d, i = _amg_arrays(amg)
            At = None if custom_At is None else np.ascontiguousarray(custom_At, np.float64).ravel()
            self._keep.extend([d, i, At])
            Ref.check(Ref.lib().ref_solver_create_ex(self.n, _i(m_rp), _i(m_ci), _d(m_v), _i(k_rp),
                                                     _i(k_ci), _d(k_v), scheme, s, kind, _d(At), ht,
                                                     _d(d), _i(i), C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            Ref.lib().ref_solver_free(self.h)
            self.h = None

    def stage_apply(self, v):
        v = np.ascontiguousarray(v, np.float64)
        y = np.zeros_like(v)
        Ref.check(Ref.lib().ref_stage_apply(self.h, _d(v), _d(y)))
        return y

    def precond_apply(self, v):
        v = np.ascontiguousarray(v, np.float64)
        w = np.zeros_like(v)
        Ref.check(Ref.lib().ref_precond_apply(self.h, _d(v), _d(w)))
        return w

    def distinct(self):
        return Ref.lib().ref_solver_distinct(self.h)

    def integrate(self, u0, t_final, trunc=None, lift=None, fq=None, rtol=1e-8, max_iter=500,
                  cap=64):
        """The reference's integrate (irk.cpp:70-102), full GMRES; `trunc` is
        the RefSolver for the truncated last step size."""
        u0 = np.ascontiguousarray(u0, np.float64)
        uf = np.zeros_like(u0)
        its = (C.c_int * cap)()
        steps, cv = C.c_int(), C.c_int()
        t_out = C.c_double()
        fq = None if fq is None else np.ascontiguousarray(fq, np.float64)
        Ref.check(Ref.lib().ref_integrate(self.h, None if trunc is None else trunc.h, _d(u0),
                                          _d(lift), _d(fq), t_final, rtol, max_iter, _d(uf),
                                          C.byref(steps), C.byref(t_out), its, cap, C.byref(cv)))
        return {"u_final": uf, "steps": steps.value, "t_final": t_out.value,
                "iterations": list(its[: steps.value]), "all_converged": bool(cv.value)}

    def step(self, u, lift=None, rtol=1e-8, restart=50, max_iter=500, t_n=0.0, fq=None,
             side="right"):
        """fq: forcing(t) = cos(t) * fq (ref_harness.cpp cos_forcing), or None."""
        n, s = self.n, self.s
        u = np.ascontiguousarray(u, np.float64)
        un = np.zeros(n)
        K = np.zeros(n * s)
        hist = np.zeros(max_iter + 2)
        it, cyc, cv, hl = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        tr, sec = C.c_double(), C.c_double()
        fq = None if fq is None else np.ascontiguousarray(fq, np.float64)
        Ref.check(Ref.lib().ref_irk_step_forced(self.h, _d(u), _d(lift), t_n, _d(fq),
                                                0 if side == "left" else 1, rtol, restart,
                                                max_iter, _d(un), _d(K), C.byref(it), C.byref(cyc),
                                                C.byref(tr), C.byref(cv), C.byref(sec), _d(hist),
                                                len(hist), C.byref(hl)))
        return {"u_next": un, "K": K, "iterations": it.value, "cycles": cyc.value,
                "true_rel": tr.value, "converged": bool(cv.value), "seconds": sec.value,
                "history": hist[: min(hl.value, len(hist))].copy()}


# ----------------------------------------------------------------- oracle
class or_csr(C.Structure):
    _fields_ = [("rows", C.c_int), ("cols", C.c_int), ("ptr", iptr), ("idx", iptr), ("val", dptr)]


class or_hier(C.Structure):
    _fields_ = [("nlev", C.c_int), ("A", C.POINTER(or_csr)), ("P", C.POINTER(or_csr)),
                ("R", C.POINTER(or_csr)), ("inv_diag", C.POINTER(dptr)), ("cinv", dptr),
                ("nc", C.c_int), ("omega", C.c_double), ("pre", C.c_int), ("post", C.c_int),
                ("tail_from", C.c_int), ("tail_ld", C.c_int), ("tail", dptr),
                ("smoother", C.c_int), ("G", C.POINTER(or_csr)), ("U", C.POINTER(or_csr)),
                ("g_lanes", iptr), ("u_lanes", iptr)]


class or_sys(C.Structure):
    _fields_ = [("n", C.c_int), ("s", C.c_int), ("M", or_csr), ("K", or_csr), ("A", dptr),
                ("b", dptr), ("ht", C.c_double), ("At", dptr), ("structure", C.c_int),
                ("nh", C.c_int), ("h", C.POINTER(or_hier)), ("sob", iptr)]


class or_report(C.Structure):
    _fields_ = [("iterations", C.c_int), ("cycles", C.c_int), ("n_reorth", C.c_int),
                ("converged", C.c_int), ("true_rel", C.c_double), ("final_rel", C.c_double),
                ("seconds", C.c_double)]


class Oracle:
    """The C restatement (oracle/irk_oracle.c)."""

    _lib = None

    @classmethod
    def available(cls) -> bool:
        return ORACLE_SO.exists()

    @classmethod
    def lib(cls):
        if cls._lib is None:
            L = C.CDLL(str(ORACLE_SO))
            L.or_dot.restype = C.c_double
            L.or_dot.argtypes = [dptr, dptr, C.c_long]
            L.or_spmv.argtypes = [C.POINTER(or_csr), dptr, dptr]
            L.or_vcycle.argtypes = [C.POINTER(or_hier), dptr, dptr]
            L.or_stage_apply.argtypes = [C.POINTER(or_sys), dptr, dptr]
            L.or_precond_apply.argtypes = [C.POINTER(or_sys), dptr, dptr]
            L.or_irk_step.argtypes = [C.POINTER(or_sys), dptr, dptr, C.c_double, C.c_int, C.c_int,
                                      dptr, dptr, C.POINTER(or_report), dptr]
            L.or_irk_step_f.argtypes = [C.POINTER(or_sys), dptr, dptr, dptr, C.c_int, C.c_double,
                                        C.c_int, C.c_int, dptr, dptr, C.POINTER(or_report), dptr]
            L.or_set_ortho.argtypes = [C.c_int]
            cls._lib = L
        return cls._lib


class OracleSystem:
    """Packs M, K, Butcher data and hierarchies (arrays) into an or_sys.

    hiers: list of dicts {A:[(rp,ci,v,ncols)...], P:[...], R:[...], inv_diag:[...],
    cinv: 2-D array, omega, pre, post}.
    """

    def __init__(self, M, K, A, b, ht, At, structure, hiers, sob):
        self._keep = []
        self.n = len(M[0]) - 1
        self.s = A.shape[0]

        def csr(t, ncols=None):
            rp, ci, v = (np.ascontiguousarray(t[0], np.int32), np.ascontiguousarray(t[1], np.int32),
                         np.ascontiguousarray(t[2], np.float64))
            self._keep.extend([rp, ci, v])
            return or_csr(len(rp) - 1, ncols if ncols is not None else len(rp) - 1, _i(rp), _i(ci), _d(v))

        hs = []
        for h in hiers:
            L = len(h["A"])
            Aarr = (or_csr * L)(*[csr(h["A"][l][:3], h["A"][l][3]) for l in range(L)])
            Parr = (or_csr * max(L - 1, 1))(*[csr(h["P"][l][:3], h["P"][l][3]) for l in range(L - 1)])
            Rarr = (or_csr * max(L - 1, 1))(*[csr(h["R"][l][:3], h["R"][l][3]) for l in range(L - 1)])
            ids = [np.ascontiguousarray(d, np.float64) for d in h["inv_diag"]]
            cinv = np.ascontiguousarray(h["cinv"], np.float64).ravel()
            self._keep.extend([Aarr, Parr, Rarr, ids, cinv])
            idp = (dptr * L)(*[_d(d) for d in ids])
            self._keep.append(idp)
            tail_from, tail = h.get("tail", (-1, None))
            tl = None if tail is None else np.ascontiguousarray(tail, np.float64)
            self._keep.append(tl)
            Garr = Uarr = gl = ul = None
            if h.get("G") and any(len(g[0]) > 1 for g in h["G"]):
                gl = np.ascontiguousarray([x[0] for x in h["lanes"]], np.int32)
                ul = np.ascontiguousarray([x[1] for x in h["lanes"]], np.int32)
                self._keep.extend([gl, ul])
                # composed legs (csrc/host/compose.cpp); rows = 0 where absent
                Garr = (or_csr * max(L - 1, 1))(*[csr(g[:3], g[3]) for g in h["G"]])
                Uarr = (or_csr * max(L - 1, 1))(*[csr(u[:3], u[3]) for u in h["U"]])
                self._keep.extend([Garr, Uarr])
            hs.append(or_hier(L, Aarr, Parr, Rarr, idp, _d(cinv), int(round(np.sqrt(cinv.size))),
                              h["omega"], h["pre"], h["post"], tail_from,
                              0 if tl is None else tl.shape[1], None if tl is None else _d(tl),
                              int(h.get("smoother", 0)), Garr, Uarr,
                              None if gl is None else _i(gl), None if ul is None else _i(ul)))
        harr = (or_hier * len(hs))(*hs)
        arrs = [np.ascontiguousarray(x, np.float64).ravel() for x in (A, b, At)]
        sobv = np.ascontiguousarray(sob, np.int32)
        self._keep.extend([harr, arrs, sobv])
        self.sys = or_sys(self.n, self.s, csr(M), csr(K), _d(arrs[0]), _d(arrs[1]), ht, _d(arrs[2]),
                          int(structure), len(hs), harr, _i(sobv))

    def stage_apply(self, v):
        v = np.ascontiguousarray(v, np.float64)
        y = np.zeros_like(v)
        Oracle.lib().or_stage_apply(C.byref(self.sys), _d(v), _d(y))
        return y

    def precond_apply(self, v):
        v = np.ascontiguousarray(v, np.float64)
        w = np.zeros_like(v)
        Oracle.lib().or_precond_apply(C.byref(self.sys), _d(v), _d(w))
        return w

    def vcycle(self, k, r):
        r = np.ascontiguousarray(r, np.float64)
        z = np.zeros_like(r)
        Oracle.lib().or_vcycle(C.byref(self.sys.h[k]), _d(r), _d(z))
        return z

    def step(self, u, lift=None, rtol=1e-8, restart=50, max_iter=500, forcing=None,
             side="right"):
        """forcing: s*n stage-major forcing values at t_n + c_i ht, or None."""
        n, s = self.n, self.s
        u = np.ascontiguousarray(u, np.float64)
        un = np.zeros(n)
        K = np.zeros(n * s)
        hist = np.zeros(max_iter + 1)
        rep = or_report()
        lift_arr = None if lift is None else np.ascontiguousarray(lift, np.float64)
        f_arr = None if forcing is None else np.ascontiguousarray(forcing, np.float64)
        rc = Oracle.lib().or_irk_step_f(C.byref(self.sys), _d(u), _d(lift_arr), _d(f_arr),
                                        0 if side == "left" else 1, rtol, restart, max_iter,
                                        _d(un), _d(K), C.byref(rep), _d(hist))
        assert rc == 0, "oracle: left preconditioning needs the delayed CGS2 scheme"
        return {"u_next": un, "K": K, "iterations": rep.iterations, "cycles": rep.cycles,
                "n_reorth": rep.n_reorth, "converged": bool(rep.converged),
                "true_rel": rep.true_rel, "final_rel": rep.final_rel, "seconds": rep.seconds,
                "history": hist[: rep.iterations + 1].copy()}


def oracle_ortho(scheme: str) -> None:
    """Selects the oracle's orthogonalisation: 'dcgs2' (device default) or 'cgs2'."""
    Oracle.lib().or_set_ortho(1 if scheme == "dcgs2" else 0)


def oracle_dot(x, y):
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    return Oracle.lib().or_dot(_d(x), _d(y), len(x))


def hierarchy_dict(h, omega=2.0 / 3.0, pre=1, post=1, smoother=0):
    """Product AmgHierarchy -> oracle hierarchy dict."""
    L = h.n_levels()
    d = {"A": [], "P": [], "R": [], "G": [], "U": [], "inv_diag": [], "omega": omega, "pre": pre,
         "post": post, "smoother": smoother, "lanes": []}
    for l in range(L):
        a = h.level(l, "A")
        d["A"].append((a.row_ptr, a.col_idx, a.vals, a.n_cols))
        d["inv_diag"].append(h.inv_diag(l))
        if l + 1 < L:
            p, r = h.level(l, "P"), h.level(l, "R")
            d["P"].append((p.row_ptr, p.col_idx, p.vals, p.n_cols))
            d["R"].append((r.row_ptr, r.col_idx, r.vals, r.n_cols))
            g, u = h.level(l, "G"), h.level(l, "U")
            d["G"].append((g.row_ptr, g.col_idx, g.vals, g.n_cols))
            d["U"].append((u.row_ptr, u.col_idx, u.vals, u.n_cols))
            d["lanes"].append(h.compose_lanes(l))
    d["cinv"] = h.coarse_inverse()
    d["tail"] = h.tail()
    return d
