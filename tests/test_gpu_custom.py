"""Custom preconditioner coefficients (the optimized block-GSL slot of
BASELINE C5) read from coefficient files on the device.

The reference exercises its Custom kind with seeded lower-triangular files
(acceptance.cpp:171-241); here lower AND upper triangular matrices at
s = 2..7 go through read_coeff_file -> custom_coeff -> the device
BlockPreconditioner: preconditioner applies and whole IRK steps are
bit-identical to the oracle, and the steps match the reference's own Custom
kind (iterations +-1, K and u_next <= 1e-9 relative L2).
"""
import numpy as np
import pytest

import paper_2010_11377_b200 as P
from conftest import has_gpu
from refs import RefSolver
from systems import custom_case, rel_l2

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


@pytest.mark.parametrize("s", [2, 3, 4, 5, 6, 7])
@pytest.mark.parametrize("upper", [False, True])
def test_custom_step_bitwise_and_vs_reference(s, upper):
    c = custom_case(32, s, upper)
    assert c.coeff.structure == (P.CoeffStructure.UpperTriangular if upper
                                 else P.CoeffStructure.LowerTriangular)
    dev = c.device()
    v = np.random.default_rng(s).uniform(-1, 1, c.n * s)
    assert np.array_equal(dev.apply(v), c.oracle.precond_apply(v))
    u = c.problem.initial()
    sys_ = P.LinearParabolicSystem(c.M, c.K, c.f_lift)
    g = P.irk_step(sys_, c.table, c.ht, 0.0, u, dev, P.GmresConfig(restart=50), want_K=True)
    o = c.oracle.step(u, c.f_lift)
    assert g.report.iterations == o["iterations"]
    assert np.array_equal(g.K, o["K"]) and np.array_equal(g.u_next, o["u_next"])
    M, K = c.M, c.K
    r = RefSolver((M.row_ptr, M.col_idx, M.vals), (K.row_ptr, K.col_idx, K.vals), 0, s, 4, c.ht,
                  custom_At=c.coeff.Atilde).step(u, c.f_lift)
    assert g.report.converged and r["converged"]
    assert abs(g.report.iterations - r["iterations"]) <= 1
    assert rel_l2(g.K, r["K"]) <= 1e-9 and rel_l2(g.u_next, r["u_next"]) <= 1e-9


def test_custom_at_size_lobatto():
    """A 256^2 Lobatto IIIC s=4 Custom step (the BASELINE-size code paths:
    DIA row classes, SELL transfer operators)."""
    c = custom_case(256, 4, False, scheme=P.Scheme.LobattoIIIC, ht=1e-3)
    u = c.problem.initial(noise=0.01, seed=3)
    sys_ = P.LinearParabolicSystem(c.M, c.K, c.f_lift)
    g = P.irk_step(sys_, c.table, c.ht, 0.0, u, c.device(), P.GmresConfig(restart=50), want_K=True)
    o = c.oracle.step(u, c.f_lift)
    assert g.report.iterations == o["iterations"] and g.report.converged
    assert np.array_equal(g.K, o["K"])
