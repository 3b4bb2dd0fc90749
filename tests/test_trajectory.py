"""Time-dependent forcing and the device-resident time loop.

* stage_rhs with forcing (irk.cpp:9-33): block i gets forcing(t_n + c_i ht);
* integrate (irk.cpp:70-102): ht repeated, the last step truncated to land on
  t_final, the PrecondFactory consulted when the step size changes.

The forcing used everywhere is forcing(t) = cos(t) * q (q a seeded vector):
libm cos and one IEEE multiply, so the Python callback, the C oracle input and
the reference harness (ref_harness.cpp cos_forcing) produce the same bits.

CPU tests pin the oracle against the reference (forced step, the reference's
own integrate with a truncated step); GPU tests compare the device path with
the oracle bit for bit and with the reference at the BASELINE bar.
"""
import ctypes as C
import math

import numpy as np
import pytest

import paper_2010_11377_b200 as P
from conftest import has_gpu
from refs import Oracle, Ref, RefSolver
from systems import dg_case, heat_case, rel_l2

checkers = pytest.mark.skipif(not (Ref.available() and Oracle.available()),
                              reason="checkers not built")


def plan(t_final, ht):
    """The reference loop's step sizes (irk.cpp:85-99)."""
    out, t = [], 0.0
    while t < t_final - 1e-14 * t_final:
        step = ht
        if t + step > t_final:
            step = t_final - t
        out.append(step)
        t += step
    return out, t


def ref_solver(case, scheme, kind):
    M, K = case.M, case.K
    return RefSolver((M.row_ptr, M.col_idx, M.vals), (K.row_ptr, K.col_idx, K.vals), scheme,
                     case.s, kind, case.ht)


def stage_forcing(q, table, t_n, ht):
    """s*n stage-major forcing(t_n + c_i ht) = cos(t_n + c_i ht) * q."""
    return np.concatenate([math.cos(t_n + ci * ht) * q for ci in table.c])


def oracle_trajectory(cases, u0, t_final, ht, q=None, lift=None, restart=0):
    """integrate restated on top of the oracle step (one Case per step size)."""
    steps, _ = plan(t_final, ht)
    u, t, its = np.array(u0, np.float64), 0.0, []
    for step in steps:
        c = cases[step]
        f = None if q is None else stage_forcing(q, c.table, t, step)
        o = c.oracle.step(u, lift, restart=restart, forcing=f)
        u = o["u_next"]
        its.append(o["iterations"])
        t += step
    return u, t, its


# ------------------------------------------------------------------ host
def test_step_plan_matches_reference_loop():
    lib = P._abi.lib()
    for t_final, ht in [(0.035, 0.01), (0.03, 0.01), (1.0, 0.1), (0.0, 0.01), (1e-3, 1e-3),
                        (0.1, 0.3), (2.5e-3, 1e-3)]:
        n = C.c_int()
        P._abi.check(lib.irk_integrate_steps(t_final, ht, C.byref(n)))
        assert n.value == len(plan(t_final, ht)[0])
    with pytest.raises(ValueError):
        P._abi.check(lib.irk_integrate_steps(1.0, 0.0, C.byref(C.c_int())))
    with pytest.raises(ValueError):
        P._abi.check(lib.irk_integrate_steps(-1.0, 0.1, C.byref(C.c_int())))


@checkers
def test_oracle_forced_step_matches_reference():
    c = heat_case(32, s=3, ht=0.01)
    q = np.random.default_rng(11).uniform(-1.0, 1.0, c.n)
    u = c.problem.initial(0.01, 2)
    t_n = 0.37
    o = c.oracle.step(u, c.f_lift, restart=0, forcing=stage_forcing(q, c.table, t_n, c.ht))
    r = ref_solver(c, 0, 3).step(u, c.f_lift, restart=0, t_n=t_n, fq=q)
    assert abs(o["iterations"] - r["iterations"]) <= 1
    assert rel_l2(o["K"], r["K"]) <= 1e-9
    assert rel_l2(o["u_next"], r["u_next"]) <= 1e-9
    # the forcing moves the solution: not the unforced step
    z = c.oracle.step(u, c.f_lift, restart=0)
    assert rel_l2(z["K"], o["K"]) > 1e-3


@checkers
def test_reference_integrate_vs_oracle_loop_truncated():
    """The reference's own integrate (truncated last step through its factory)
    against the oracle loop: step count and final time exact, iterations +-1,
    u_final <= 1e-9."""
    ht, t_final = 0.01, 0.035
    steps, t_end = plan(t_final, ht)
    assert len(steps) == 4 and steps[-1] != ht
    cases = {h: heat_case(24, s=2, ht=h) for h in set(steps)}
    q = np.random.default_rng(5).uniform(-1.0, 1.0, cases[ht].n)
    u0 = cases[ht].problem.initial(0.01, 4)
    lift = cases[ht].f_lift
    r = ref_solver(cases[ht], 0, 3).integrate(u0, t_final, trunc=ref_solver(cases[steps[-1]], 0, 3),
                                              lift=lift, fq=q)
    uo, to, its = oracle_trajectory(cases, u0, t_final, ht, q=q, lift=lift)
    assert r["steps"] == len(steps) and r["t_final"] == t_end == to
    assert all(abs(a - b) <= 1 for a, b in zip(its, r["iterations"]))
    assert rel_l2(uo, r["u_final"]) <= 1e-9
    assert r["all_converged"]


# ------------------------------------------------------------------ device
@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
@pytest.mark.parametrize("restart", [50, 4])
def test_device_forced_step_bitwise(restart):
    c = heat_case(32, s=3, ht=0.01)
    q = np.random.default_rng(11).uniform(-1.0, 1.0, c.n)
    u = c.problem.initial(0.01, 2)
    t_n = 0.37
    sys = P.LinearParabolicSystem(c.M, c.K, c.f_lift, forcing=lambda t: math.cos(t) * q)
    g = P.irk_step(sys, c.table, c.ht, t_n, u, c.device(), P.GmresConfig(restart=restart),
                   want_K=True)
    o = c.oracle.step(u, c.f_lift, restart=restart, forcing=stage_forcing(q, c.table, t_n, c.ht))
    assert g.report.iterations == o["iterations"]
    assert np.array_equal(g.K, o["K"]) and np.array_equal(g.u_next, o["u_next"])
    if restart == 50:
        r = ref_solver(c, 0, 3).step(u, c.f_lift, restart=restart, t_n=t_n, fq=q)
        assert abs(g.report.iterations - r["iterations"]) <= 1
        assert rel_l2(g.u_next, r["u_next"]) <= 1e-9


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_device_integrate_bitwise_and_vs_reference():
    """Device-resident integrate with forcing and a truncated last step (a
    second solver from the factory) = the oracle loop bit for bit, and the
    reference's integrate at the BASELINE bar."""
    ht, t_final = 0.01, 0.035
    steps, t_end = plan(t_final, ht)
    cases = {h: heat_case(24, s=2, ht=h) for h in set(steps)}
    q = np.random.default_rng(5).uniform(-1.0, 1.0, cases[ht].n)
    u0 = cases[ht].problem.initial(0.01, 4)
    c0 = cases[ht]
    sys = P.LinearParabolicSystem(c0.M, c0.K, c0.f_lift, forcing=lambda t: math.cos(t) * q)
    made = []

    def make(h):
        made.append(h)
        return cases[h].device()

    tr = P.integrate(sys, c0.table, u0, t_final, ht, make, P.GmresConfig(restart=0))
    uo, to, its = oracle_trajectory(cases, u0, t_final, ht, q=q, lift=c0.f_lift)
    assert made == [ht, steps[-1]]
    assert tr.steps == len(steps) and tr.t_final == t_end == to
    assert [r.iterations for r in tr.reports] == its
    assert np.array_equal(tr.u_final, uo)
    assert tr.all_converged and all(len(r.history) == r.iterations + 1 for r in tr.reports)
    r = ref_solver(c0, 0, 3).integrate(u0, t_final, trunc=ref_solver(cases[steps[-1]], 0, 3),
                                       lift=c0.f_lift, fq=q)
    assert r["steps"] == tr.steps and r["t_final"] == tr.t_final
    assert all(abs(a - b) <= 1 for a, b in zip(its, r["iterations"]))
    assert rel_l2(tr.u_final, r["u_final"]) <= 1e-9


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_device_integrate_lift_matches_step_loop():
    """Double glazing (Dirichlet lift, no forcing), whole steps only: the
    device-resident loop equals repeated irk_step calls bit for bit."""
    c = dg_case(32, s=2, ht=0.01)
    sys = P.LinearParabolicSystem(c.M, c.K, c.f_lift)
    u0 = np.zeros(c.n)
    tr = P.integrate(sys, c.table, u0, 0.05, c.ht, lambda h: c.device(), P.GmresConfig())
    u, t = u0, 0.0
    for k in range(tr.steps):
        g = P.irk_step(sys, c.table, c.ht, t, u, c.device(), P.GmresConfig())
        assert g.report.iterations == tr.reports[k].iterations
        u, t = g.u_next, t + c.ht
    assert tr.steps == 5 and np.array_equal(tr.u_final, u)


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_device_integrate_errors():
    c = heat_case(16, s=2, ht=0.01)
    sys = P.LinearParabolicSystem(c.M, c.K, c.f_lift)
    u0 = c.problem.initial()

    def make(h):
        if h != c.ht:
            raise RuntimeError("no solver for the truncated step")
        return c.device()

    with pytest.raises(RuntimeError, match="truncated"):
        P.integrate(sys, c.table, u0, 0.025, c.ht, make)
    bad = P.LinearParabolicSystem(c.M, c.K, c.f_lift, forcing=lambda t: np.zeros(3))
    with pytest.raises(ValueError, match="forcing size"):
        P.integrate(bad, c.table, u0, 0.02, c.ht, make)
    with pytest.raises(ValueError):
        P.integrate(sys, c.table, u0, 0.02, -1.0, make)
    # C level: no factory although the step size changes
    lib = P._abi.lib()
    reps = (P._abi.irk_report * 8)()
    uf = np.empty_like(u0)
    cc = np.ascontiguousarray(c.table.c)
    cfg = P.GmresConfig().c()
    rc = lib.irkdev_integrate(c.device()._dev._h, P._abi.FACTORY_FN(), None, P._abi.as_d(u0), None,
                              P._abi.as_d(cc), P._abi.FORCING_FN(), None, 0.025, c.ht,
                              C.byref(cfg), P._abi.as_d(uf), reps, 8, None, None, None, None)
    assert rc == P._abi.IRK_EINVAL
