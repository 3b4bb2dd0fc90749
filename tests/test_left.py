"""Left preconditioning (gmres.cpp:41-46, 69-71).

GMRES on P^-1 A with the metric base P^-1 b: the stop test and the history use
the preconditioned residual, the report's true residual is ||b - A x|| / ||b||.
GMRES(m) restarts rescale the tolerance in the same metric,
rel_tol ||P^-1 b|| / ||P^-1 r_k||.  The device runs it
with the delayed CGS2 orthogonalisation; the oracle restates that order, so
device and oracle agree bit for bit, and both meet the BASELINE bar against
the reference's own left-preconditioned gmres.
"""
import numpy as np
import pytest

import paper_2010_11377_b200 as P
from conftest import has_gpu
from refs import Oracle, Ref, RefSolver
from systems import dg_case, heat_case, rel_l2

checkers = pytest.mark.skipif(not (Ref.available() and Oracle.available()),
                              reason="checkers not built")


def ref_solver(case, scheme, kind):
    M, K = case.M, case.K
    return RefSolver((M.row_ptr, M.col_idx, M.vals), (K.row_ptr, K.col_idx, K.vals), scheme,
                     case.s, kind, case.ht)


CASES = [("heat", 3, 3, 50), ("heat", 3, 3, 5), ("heat", 2, 0, 50), ("dg", 2, 3, 50)]


def build(kind_name, s, kind):
    if kind_name == "heat":
        c = heat_case(32, s=s, kind=P.CoeffKind(kind), ht=0.01)
        return c, c.problem.initial(0.01, 6)
    c = dg_case(32, s=s, kind=P.CoeffKind(kind), ht=0.01)
    return c, np.zeros(c.n)


@checkers
@pytest.mark.parametrize("prob,s,kind,restart", CASES)
def test_oracle_left_matches_reference(prob, s, kind, restart):
    c, u = build(prob, s, kind)
    o = c.oracle.step(u, c.f_lift, restart=restart, side="left")
    r = ref_solver(c, 0, kind).step(u, c.f_lift, restart=restart, side="left")
    assert o["converged"] and r["converged"]
    assert abs(o["iterations"] - r["iterations"]) <= 1
    assert o["cycles"] == r["cycles"]
    assert rel_l2(o["K"], r["K"]) <= 1e-9
    assert rel_l2(o["u_next"], r["u_next"]) <= 1e-9
    # the metric differs from the right-preconditioned solve
    rr = c.oracle.step(u, c.f_lift, restart=restart)
    assert not np.array_equal(rr["history"], o["history"])


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
@pytest.mark.parametrize("prob,s,kind,restart", CASES)
def test_device_left_bitwise(prob, s, kind, restart):
    c, u = build(prob, s, kind)
    sys = P.LinearParabolicSystem(c.M, c.K, c.f_lift)
    g = P.irk_step(sys, c.table, c.ht, 0.0, u, c.device(),
                   P.GmresConfig(side="left", restart=restart), want_K=True)
    o = c.oracle.step(u, c.f_lift, restart=restart, side="left")
    assert g.report.iterations == o["iterations"] and g.report.cycles == o["cycles"]
    assert np.array_equal(np.array(g.report.history), o["history"])
    assert np.array_equal(g.K, o["K"]) and np.array_equal(g.u_next, o["u_next"])
    assert g.report.true_rel_residual == o["true_rel"]
    # the whole solve stays one conditional graph (no host-driven fallback)
    import ctypes as C
    lp, mode = C.c_int(), C.c_int()
    P._abi.check(P._abi.lib().irkdev_graph_info(c.device()._dev._h, C.byref(lp), C.byref(mode)))
    assert mode.value == 1
    # switching sides on one handle rebuilds the graph and stays exact
    g2 = P.irk_step(sys, c.table, c.ht, 0.0, u, c.device(), P.GmresConfig(restart=restart),
                    want_K=True)
    o2 = c.oracle.step(u, c.f_lift, restart=restart)
    assert np.array_equal(g2.K, o2["K"])


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_left_with_cgs2_is_unsupported():
    import os
    import subprocess
    import sys as _sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    code = f"""
import sys; sys.path[:0] = [{str(root)!r}, {str(root / 'tests')!r}]
import paper_2010_11377_b200 as P
from systems import heat_case
c = heat_case(16, s=2)
sys_ = P.LinearParabolicSystem(c.M, c.K, c.f_lift)
try:
    P.irk_step(sys_, c.table, c.ht, 0.0, c.problem.initial(), c.device(), P.GmresConfig(side="left"))
except P.Unsupported:
    print("UNSUPPORTED")
"""
    r = subprocess.run([_sys.executable, "-c", code], env=dict(os.environ, IRK_ORTHO="cgs2"),
                       capture_output=True, text=True, timeout=300)
    assert "UNSUPPORTED" in r.stdout, r.stdout + r.stderr
