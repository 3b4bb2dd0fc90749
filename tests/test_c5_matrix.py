"""BASELINE C5's scheme x preconditioner matrix at a small grid.

Every tableau the reference builds (Radau IIA s = 1..7, Lobatto IIIC s = 2..5;
butcher.cpp:29-101) times every block preconditioner kind (P_J, P_GSL, P_DU,
P_LD; butcher.cpp:251-288), one IRK step on the 24^2 heat problem with
GMRES(50): the oracle matches the reference at the BASELINE bar (iterations
+-1, K within 1e-9) and the device matches the oracle bit for bit.
"""
import numpy as np
import pytest

import paper_2010_11377_b200 as P
from conftest import has_gpu
from refs import Oracle, Ref, RefSolver
from systems import heat_case, rel_l2

TABLES = [(0, s) for s in range(1, 8)] + [(1, s) for s in range(2, 6)]
KINDS = [0, 1, 2, 3]
CELLS = [(sch, s, k) for sch, s in TABLES for k in KINDS if not (s == 1 and k != 0)]


def build(scheme, s, kind):
    c = heat_case(24, scheme=P.Scheme(scheme), s=s, kind=P.CoeffKind(kind), ht=1e-2)
    return c, c.problem.initial(0.01, 3)


@pytest.mark.skipif(not (Ref.available() and Oracle.available()), reason="checkers not built")
@pytest.mark.parametrize("scheme,s,kind", CELLS)
def test_oracle_matches_reference(scheme, s, kind):
    c, u = build(scheme, s, kind)
    o = c.oracle.step(u, c.f_lift)
    M, K = c.M, c.K
    r = RefSolver((M.row_ptr, M.col_idx, M.vals), (K.row_ptr, K.col_idx, K.vals), scheme, s, kind,
                  c.ht).step(u, c.f_lift)
    assert o["converged"] and r["converged"]
    assert abs(o["iterations"] - r["iterations"]) <= 1
    assert rel_l2(o["K"], r["K"]) <= 1e-9
    assert rel_l2(o["u_next"], r["u_next"]) <= 1e-9


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
@pytest.mark.parametrize("scheme,s,kind", CELLS)
def test_device_bitwise(scheme, s, kind):
    c, u = build(scheme, s, kind)
    sys_ = P.LinearParabolicSystem(c.M, c.K, c.f_lift)
    g = P.irk_step(sys_, c.table, c.ht, 0.0, u, c.device(), P.GmresConfig(restart=50), want_K=True)
    o = c.oracle.step(u, c.f_lift)
    assert g.report.iterations == o["iterations"]
    assert np.array_equal(g.K, o["K"]) and np.array_equal(g.u_next, o["u_next"])
