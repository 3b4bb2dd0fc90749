"""Pins the C oracle (oracle/irk_oracle.c) against the reference itself.

The reference (oracle/_ref) is the unmodified irkprec hot path compiled from
/root/reference, with a dense-LU stand-in for its Eigen coarse solve and a
GMRES(m) restart wrapper (oracle/ref_harness.cpp).  Expected agreement:
  * stage apply: bit-identical (same per-row and per-axpy operation order);
  * V-cycle / preconditioner: <= 1e-12 relative (only the coarsest direct
    solve differs: dense inverse vs LU substitution);
  * IRK step: iterations within +-1 and K, u_next within 1e-9 relative L2 --
    the BASELINE parity bar (MGS vs CGS, flexible vs plain right GMRES).
"""
import numpy as np
import pytest

import paper_2010_11377_b200 as P
from refs import Oracle, Ref, RefSolver
from systems import dg_case, heat_case, rel_l2

pytestmark = pytest.mark.skipif(not (Ref.available() and Oracle.available()),
                                reason="checkers not built")


def ref_solver(case, scheme, kind):
    M, K = case.M, case.K
    return RefSolver((M.row_ptr, M.col_idx, M.vals), (K.row_ptr, K.col_idx, K.vals), scheme,
                     case.s, kind, case.ht)


@pytest.mark.parametrize("s,kind", [(2, 3), (3, 3), (3, 0), (3, 1), (3, 2), (5, 3)])
def test_stage_apply_bitwise(s, kind):
    c = heat_case(32, s=s, kind=P.CoeffKind(kind))
    r = ref_solver(c, 0, kind)
    v = np.random.default_rng(7).uniform(-1, 1, c.n * s)
    assert np.array_equal(c.oracle.stage_apply(v), r.stage_apply(v))


@pytest.mark.parametrize("scheme,s,kind", [(0, 2, 3), (0, 3, 3), (0, 3, 0), (0, 3, 1), (0, 3, 2),
                                           (0, 5, 3), (1, 3, 3), (1, 5, 0)])
def test_precond_apply_matches_reference(scheme, s, kind):
    c = heat_case(64, scheme=P.Scheme(scheme), s=s, kind=P.CoeffKind(kind), ht=0.01)
    r = ref_solver(c, scheme, kind)
    assert r.distinct() == len(c.hiers)
    v = np.random.default_rng(11).uniform(-1, 1, c.n * s)
    assert rel_l2(c.oracle.precond_apply(v), r.precond_apply(v)) <= 1e-12


def test_vcycle_matches_reference_and_is_linear():
    c = heat_case(64, s=2, ht=0.01)
    B = c.hiers[0]
    ref = Ref.amg((c.M.row_ptr, c.M.col_idx, 1.0 * c.M.vals + (c.ht * c.coeff.Atilde[0, 0]) * c.K.vals))
    rng = np.random.default_rng(3)
    r1, r2 = rng.uniform(-1, 1, c.n), rng.uniform(-1, 1, c.n)
    z = c.oracle.vcycle(0, r1)
    assert rel_l2(z, ref.vcycle(r1)) <= 1e-12
    # linearity <= 1e-12 and bit-identical repeat (test_amg.cpp:90-107)
    al, be = 0.83, -2.31
    lhs = c.oracle.vcycle(0, al * r1 + be * r2)
    rhs = al * z + be * c.oracle.vcycle(0, r2)
    assert np.max(np.abs(lhs - rhs)) <= 1e-12 * max(np.linalg.norm(lhs), np.linalg.norm(rhs))
    assert np.array_equal(c.oracle.vcycle(0, r1), z)
    # zero residual -> zero correction (test_amg.cpp:52-57)
    assert not np.any(c.oracle.vcycle(0, np.zeros(c.n)))
    assert B.n_levels() == ref.n_levels()


def _step_pair(c, scheme, kind, u, restart=50, max_iter=500):
    r = ref_solver(c, scheme, kind).step(u, c.f_lift, restart=restart, max_iter=max_iter)
    o = c.oracle.step(u, c.f_lift, restart=restart, max_iter=max_iter)
    return r, o


def test_c1_step_parity():
    """BASELINE configs[0]: 64^2 heat, Radau IIA s=2, h=0.01, LD, GMRES(50)."""
    c = heat_case(64, s=2, ht=0.01)
    u = c.problem.initial()
    r, o = _step_pair(c, 0, 3, u)
    assert r["converged"] and o["converged"]
    assert r["iterations"] == 19  # survey probe / BASELINE.md §2
    assert abs(o["iterations"] - r["iterations"]) <= 1
    assert rel_l2(o["K"], r["K"]) <= 1e-9
    assert rel_l2(o["u_next"], r["u_next"]) <= 1e-9
    assert o["true_rel"] <= 1e-8


@pytest.mark.parametrize("scheme,s,kind", [(0, 3, 0), (0, 3, 1), (0, 3, 2), (1, 3, 3), (1, 4, 1)])
def test_step_parity_other_preconditioners(scheme, s, kind):
    c = heat_case(48, scheme=P.Scheme(scheme), s=s, kind=P.CoeffKind(kind), ht=0.005)
    u = c.problem.initial(0.01, 5)
    r, o = _step_pair(c, scheme, kind, u)
    assert abs(o["iterations"] - r["iterations"]) <= 1
    assert rel_l2(o["K"], r["K"]) <= 1e-9
    assert rel_l2(o["u_next"], r["u_next"]) <= 1e-9


def test_restart_cycles_parity():
    """GMRES(5) forces several restart cycles; both sides restart identically."""
    c = heat_case(48, s=3, ht=0.01)
    u = c.problem.initial(0.01, 9)
    r, o = _step_pair(c, 0, 3, u, restart=5)
    assert r["cycles"] >= 3 and o["cycles"] >= 3
    assert abs(o["iterations"] - r["iterations"]) <= 1
    assert rel_l2(o["K"], r["K"]) <= 1e-9


def test_double_glazing_step_parity():
    c = dg_case(48, s=2, ht=0.01)
    u = np.zeros(c.n)
    r, o = _step_pair(c, 0, 3, u)
    assert abs(o["iterations"] - r["iterations"]) <= 1
    assert rel_l2(o["K"], r["K"]) <= 1e-9
    assert rel_l2(o["u_next"], r["u_next"]) <= 1e-9


def test_zero_state_stays_zero():
    c = heat_case(16, s=2)
    o = c.oracle.step(np.zeros(c.n), None)
    assert o["iterations"] == 0 and o["converged"]
    assert not np.any(o["u_next"])


@pytest.mark.parametrize("s,upper", [(2, False), (3, True), (5, False), (7, False), (7, True)])
def test_custom_coeff_step_matches_reference(s, upper):
    """The Custom kind through a coefficient file (acceptance.cpp:171-241):
    the reference's BlockPreconditioner with custom_coeff(read_coeff_file)."""
    from systems import custom_case
    c = custom_case(32, s, upper)
    u = c.problem.initial()
    o = c.oracle.step(u, c.f_lift)
    M, K = c.M, c.K
    r = RefSolver((M.row_ptr, M.col_idx, M.vals), (K.row_ptr, K.col_idx, K.vals), 0, s, 4, c.ht,
                  custom_At=c.coeff.Atilde)
    v = np.random.default_rng(s).uniform(-1, 1, c.n * s)
    assert rel_l2(c.oracle.precond_apply(v), r.precond_apply(v)) <= 1e-12
    rr = r.step(u, c.f_lift)
    assert o["converged"] and rr["converged"]
    assert abs(o["iterations"] - rr["iterations"]) <= 1
    assert rel_l2(o["K"], rr["K"]) <= 1e-9
    assert rel_l2(o["u_next"], rr["u_next"]) <= 1e-9


@pytest.mark.parametrize("problem", ["heat", "dg"])
def test_gauss_seidel_study_cycle_matches_reference(problem):
    """The reference study driver's subsolve (study.hpp:44-47: Gauss-Seidel
    V(4,4), two prolongator smoothing steps) -- V-cycle, preconditioner and
    IRK step against the reference's own smooth_sweep (amg.cpp:125-140)."""
    from systems import study_amg
    amg = study_amg()
    c = (heat_case(64, s=2, ht=0.01, amg=amg) if problem == "heat" else dg_case(64, s=2, amg=amg))
    M, K = c.M, c.K
    B = (M.row_ptr, M.col_idx, 1.0 * M.vals + (c.ht * c.coeff.Atilde[0, 0]) * K.vals)
    ref = Ref.amg_ex(B, amg)
    r = np.random.default_rng(1).uniform(-1, 1, c.n)
    assert rel_l2(c.oracle.vcycle(0, r), ref.vcycle(r)) <= 1e-12
    rs = RefSolver((M.row_ptr, M.col_idx, M.vals), (K.row_ptr, K.col_idx, K.vals), 0, 2, 3, c.ht,
                   amg=amg)
    v = np.random.default_rng(2).uniform(-1, 1, 2 * c.n)
    assert rel_l2(c.oracle.precond_apply(v), rs.precond_apply(v)) <= 1e-12
    u = c.problem.initial() if problem == "heat" else np.zeros(c.n)
    o, rr = c.oracle.step(u, c.f_lift), rs.step(u, c.f_lift)
    assert abs(o["iterations"] - rr["iterations"]) <= 1
    assert rel_l2(o["K"], rr["K"]) <= 1e-9 and rel_l2(o["u_next"], rr["u_next"]) <= 1e-9


def test_gauss_seidel_without_tail_matches_reference(monkeypatch):
    """The whole cycle recursive (no dense tail): every level's sweeps."""
    from systems import study_amg
    monkeypatch.setenv("IRK_TAIL_MAX", "0")
    amg = P.AmgParams(pre_sweeps=2, post_sweeps=3, smoother=1)
    c = heat_case(128, s=2, ht=0.01, amg=amg)
    assert c.hiers[0].tail()[1] is None and c.hiers[0].n_levels() >= 3
    M, K = c.M, c.K
    B = (M.row_ptr, M.col_idx, 1.0 * M.vals + (c.ht * c.coeff.Atilde[0, 0]) * K.vals)
    r = np.random.default_rng(4).uniform(-1, 1, c.n)
    assert rel_l2(c.oracle.vcycle(0, r), Ref.amg_ex(B, amg).vcycle(r)) <= 1e-12
