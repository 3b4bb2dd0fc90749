"""Long Arnoldi cycles (regression for the delayed-CGS2 column scaling).

DCGS2 applies the operator to the not yet normalised direction vt_j.  Unless
every Hessenberg column and the next direction are rescaled by 1/alpha_j, the
vector magnitudes shrink geometrically along a cycle and the breakdown test
(h_{j+1,j} <= 1e-14 beta, gmres.cpp:118) fires falsely after ~45 iterations --
which happened at BASELINE C3 (47 instead of the reference's 53 iterations).
These cases run ~50 iterations in one cycle: the oracle must match the
reference at the BASELINE bar and the device must match the oracle bit for bit.
"""
import numpy as np
import pytest

import paper_2010_11377_b200 as P
from conftest import has_gpu
from refs import Oracle, Ref, RefSolver
from systems import heat_case, rel_l2

CASES = [(64, 1, 5, 1e-13, 100), (64, 1, 5, 1e-13, 0), (96, 0, 5, 1e-13, 30)]


def build(cells, scheme, s):
    c = heat_case(cells, scheme=P.Scheme(scheme), s=s, ht=1e-3)
    return c, c.problem.initial(0.01, 1)


@pytest.mark.skipif(not (Ref.available() and Oracle.available()), reason="checkers not built")
@pytest.mark.parametrize("cells,scheme,s,rtol,restart", CASES)
def test_oracle_long_cycle_matches_reference(cells, scheme, s, rtol, restart):
    c, u = build(cells, scheme, s)
    o = c.oracle.step(u, c.f_lift, rtol=rtol, restart=restart)
    M, K = c.M, c.K
    r = RefSolver((M.row_ptr, M.col_idx, M.vals), (K.row_ptr, K.col_idx, K.vals), scheme, s, 3,
                  1e-3).step(u, c.f_lift, rtol=rtol, restart=restart)
    assert o["converged"] and o["true_rel"] <= rtol
    assert o["iterations"] >= 40
    assert abs(o["iterations"] - r["iterations"]) <= 1
    assert rel_l2(o["K"], r["K"]) <= 1e-9


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
@pytest.mark.parametrize("cells,scheme,s,rtol,restart", CASES)
def test_device_long_cycle_bitwise(cells, scheme, s, rtol, restart):
    c, u = build(cells, scheme, s)
    sys_ = P.LinearParabolicSystem(c.M, c.K, c.f_lift)
    g = P.irk_step(sys_, c.table, c.ht, 0.0, u, c.device(),
                   P.GmresConfig(rel_tol=rtol, restart=restart), want_K=True)
    o = c.oracle.step(u, c.f_lift, rtol=rtol, restart=restart)
    assert g.report.converged and g.report.iterations == o["iterations"]
    assert np.array_equal(g.K, o["K"])


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_device_cycle_longer_than_256_bitwise():
    """One Arnoldi cycle of 259 iterations (full GMRES, block Jacobi, s = 7):
    k_dgs_dot writes 2j + 2 partials per chunk, past the old (512 + 2)-slot
    partials buffer once j > 256."""
    c = heat_case(128, s=7, kind=P.CoeffKind.Jacobi, ht=1e-3)
    u = c.problem.initial(0.01, 1)
    sys_ = P.LinearParabolicSystem(c.M, c.K, c.f_lift)
    g = P.irk_step(sys_, c.table, c.ht, 0.0, u, c.device(),
                   P.GmresConfig(rel_tol=1e-20, restart=0, max_iter=300), want_K=True)
    o = c.oracle.step(u, c.f_lift, rtol=1e-20, restart=0, max_iter=300)
    assert o["iterations"] > 256 and o["cycles"] == 1
    assert g.report.iterations == o["iterations"] and g.report.cycles == 1
    assert g.report.converged == o["converged"]
    assert np.array_equal(g.K, o["K"])
