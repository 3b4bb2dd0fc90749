"""Device parity through the C ABI (needs a B200).

The device kernels and the C oracle share the operation order (per-row
sequential sums, --fmad=false, fixed reduction tree), so kernel outputs and
whole IRK steps are compared BIT-FOR-BIT with the oracle; against the
reference itself (oracle/_ref) the BASELINE bar applies: iterations within +-1
and K, u_next within 1e-9 relative L2.
"""
import numpy as np
import pytest

import paper_2010_11377_b200 as P
from conftest import has_gpu
from refs import Oracle, Ref, RefSolver, oracle_dot
from systems import dg_case, heat_case, rel_l2

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


def ref_solver(case, scheme, kind):
    M, K = case.M, case.K
    return RefSolver((M.row_ptr, M.col_idx, M.vals), (K.row_ptr, K.col_idx, K.vals), scheme,
                     case.s, kind, case.ht)


@pytest.mark.parametrize("scheme,s,kind", [(0, 2, 3), (0, 3, 3), (0, 3, 0), (0, 3, 1), (0, 3, 2),
                                           (0, 5, 3), (0, 7, 2), (1, 3, 3), (1, 5, 0)])
def test_stage_and_precond_bitwise(scheme, s, kind):
    c = heat_case(64, scheme=P.Scheme(scheme), s=s, kind=P.CoeffKind(kind), ht=0.01)
    dev = c.device()
    v = np.random.default_rng(s * 10 + kind).uniform(-1, 1, c.n * s)
    assert np.array_equal(P.StageOperator(dev).apply(v), c.oracle.stage_apply(v))
    assert np.array_equal(dev.apply(v), c.oracle.precond_apply(v))


def test_vcycle_bitwise_every_hierarchy():
    c = heat_case(128, s=3, ht=1e-3)
    dev = c.device()
    rng = np.random.default_rng(5)
    for k in range(len(c.hiers)):
        r = rng.uniform(-1, 1, c.n)
        assert np.array_equal(dev.vcycle(k, r), c.oracle.vcycle(k, r))
    assert not np.any(dev.vcycle(0, np.zeros(c.n)))


def test_vcycle_general_sweeps_bitwise():
    c = heat_case(64, s=2, ht=0.01, amg=P.AmgParams(pre_sweeps=2, post_sweeps=3))
    r = np.random.default_rng(2).uniform(-1, 1, c.n)
    assert np.array_equal(c.device().vcycle(0, r), c.oracle.vcycle(0, r))


def test_dot_tree_bitwise():
    c = heat_case(16, s=2)
    lib = P._abi.lib()
    import ctypes as C
    for n in (1, 100, 4096, 4097, 3_000_001):
        x = np.random.default_rng(n).uniform(-1, 1, n)
        y = np.random.default_rng(n + 1).uniform(-1, 1, n)
        out = C.c_double()
        P._abi.check(lib.irkdev_dot(c.device()._dev._h, P._abi.as_d(x), P._abi.as_d(y), n, C.byref(out)))
        assert out.value == oracle_dot(x, y)


def _step(c, u, restart=50, max_iter=500):
    dev = c.device()
    sys = P.LinearParabolicSystem(c.M, c.K, c.f_lift)
    cfg = P.GmresConfig(restart=restart, max_iter=max_iter)
    return P.irk_step(sys, c.table, c.ht, 0.0, u, dev, cfg, want_K=True)


def test_c1_step_bitwise_and_vs_reference():
    """BASELINE configs[0] (64^2 heat, Radau IIA s=2, h=0.01, LD, GMRES(50))."""
    c = heat_case(64, s=2, ht=0.01)
    u = c.problem.initial()
    g = _step(c, u)
    o = c.oracle.step(u, c.f_lift)
    assert g.report.iterations == o["iterations"]
    assert g.report.n_reorth == o["n_reorth"]
    assert np.array_equal(g.K, o["K"])
    assert np.array_equal(g.u_next, o["u_next"])
    assert g.report.true_rel_residual == o["true_rel"]
    assert np.array_equal(np.array(g.report.history), o["history"])
    r = ref_solver(c, 0, 3).step(u, c.f_lift)
    assert abs(g.report.iterations - r["iterations"]) <= 1
    assert rel_l2(g.K, r["K"]) <= 1e-9
    assert rel_l2(g.u_next, r["u_next"]) <= 1e-9
    assert g.report.converged and g.report.true_rel_residual <= 1e-8


@pytest.mark.parametrize("scheme,s,kind,restart", [(0, 3, 0, 50), (0, 3, 1, 50), (0, 3, 2, 50),
                                                   (0, 3, 3, 5), (1, 5, 3, 50), (0, 7, 3, 8)])
def test_step_bitwise_variants(scheme, s, kind, restart):
    c = heat_case(48, scheme=P.Scheme(scheme), s=s, kind=P.CoeffKind(kind), ht=0.005)
    u = c.problem.initial(0.01, 3)
    g = _step(c, u, restart=restart)
    o = c.oracle.step(u, c.f_lift, restart=restart)
    assert g.report.iterations == o["iterations"]
    assert g.report.cycles == o["cycles"]
    assert np.array_equal(g.K, o["K"])
    assert np.array_equal(g.u_next, o["u_next"])


def test_double_glazing_step():
    c = dg_case(64, s=2, ht=0.01)
    u = np.zeros(c.n)
    g = _step(c, u)
    o = c.oracle.step(u, c.f_lift)
    assert np.array_equal(g.K, o["K"])
    r = ref_solver(c, 0, 3).step(u, c.f_lift)
    assert abs(g.report.iterations - r["iterations"]) <= 1
    assert rel_l2(g.u_next, r["u_next"]) <= 1e-9


def test_zero_state_and_nonconvergence():
    c = heat_case(16, s=2)
    g = _step(c, np.zeros(c.n))
    assert g.report.iterations == 0 and g.report.converged and not np.any(g.u_next)
    # max_iter = 3 with a tight tolerance: reported, not raised (gmres.hpp:45-48)
    sys = P.LinearParabolicSystem(c.M, c.K, c.f_lift)
    r = P.irk_step(sys, c.table, c.ht, 0.0, c.problem.initial(), c.device(),
                   P.GmresConfig(rel_tol=1e-14, max_iter=3, restart=50))
    assert not r.report.converged and r.report.iterations == 3
    assert len(r.report.history) == 4


def test_dahlquist_scalar():
    """N=1: u_next = R(-ht*lambda) u0 (test_blocksolve.cpp:324-338)."""
    lam, ht, u0 = 3.7, 0.29, 1.13
    one = P.CsrMatrix(np.array([0, 1], np.int32), np.array([0], np.int32), np.array([1.0]), 1)
    F = P.CsrMatrix(np.array([0, 1], np.int32), np.array([0], np.int32), np.array([lam]), 1)
    for s in (1, 2, 3, 5, 7):
        t = P.make_radau_iia(s)
        Pc = P.BlockPreconditioner(one, F, P.precond_coeff(t, P.CoeffKind.LowerFactor if s > 1
                                                           else P.CoeffKind.Jacobi), ht, table=t)
        r = P.irk_step(P.LinearParabolicSystem(one, F), t, ht, 0.0, np.array([u0]), Pc,
                       P.GmresConfig(rel_tol=1e-13))
        z = -ht * lam
        R = 1 + z * t.b @ np.linalg.solve(np.eye(s) - z * t.A, np.ones(s))
        assert r.u_next[0] == pytest.approx(R * u0, rel=1e-9)


@pytest.mark.slow
def test_c2_one_step_full_size():
    """BASELINE configs[1] size (1024^2, Radau IIA s=3, h=1e-3): bitwise vs the
    oracle and +-1 iteration / 1e-9 vs the reference, one step."""
    c = heat_case(1024, s=3, ht=1e-3)
    u = c.problem.initial(0.01, 1)
    g = _step(c, u)
    o = c.oracle.step(u, c.f_lift)
    assert g.report.iterations == o["iterations"]
    assert np.array_equal(g.K, o["K"])
    assert np.array_equal(g.u_next, o["u_next"])
    if Ref.available():
        r = ref_solver(c, 0, 3).step(u, c.f_lift)
        assert abs(g.report.iterations - r["iterations"]) <= 1
        assert rel_l2(g.K, r["K"]) <= 1e-9
        assert rel_l2(g.u_next, r["u_next"]) <= 1e-9


@pytest.mark.parametrize("cells", [256, 512])
def test_fused_coarse_levels_bitwise(cells):
    """Deep hierarchies (5-6 levels, every coarse-level kernel shape and the
    programmatic launches from level 2): V-cycles and a whole step stay
    bit-identical."""
    c = heat_case(cells, s=3, ht=1e-3)
    assert all(h.n_levels() >= 5 for h in c.hiers)
    rng = np.random.default_rng(cells)
    for k in range(len(c.hiers)):
        r = rng.standard_normal(c.n)
        assert np.array_equal(c.device().vcycle(k, r), c.oracle.vcycle(k, r))
    u = c.problem.initial(0.01, 2)
    g = _step(c, u)
    o = c.oracle.step(u, c.f_lift)
    assert g.report.iterations == o["iterations"]
    assert np.array_equal(g.K, o["K"])
