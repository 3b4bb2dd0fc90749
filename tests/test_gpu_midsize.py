"""Mid-size device parity (bit for bit against the C oracle).

The small parity cases (tests/test_gpu_parity.py: 64^2, 128^2) have shallow
hierarchies; at 512^2 the device path takes the same routes as at BASELINE
size -- DIA row classes on the fine level, SELL-32 / CSR-vector operators with
the static preloads, the wave-capped CSR-vector lanes, the restriction's
wd.*r reuse, the single-CTA bottom kernel on the deepest levels, programmatic
launches -- for every preconditioner structure (diagonal, lower, upper) and
for the non-symmetric SUPG operators.  Each case runs one IRK step and
compares iterations, the residual history, K and u_next exactly.
"""
import numpy as np
import pytest

import paper_2010_11377_b200 as P
from conftest import has_gpu
from systems import dg_case, heat_case

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


def bitwise_step(c, u, lift=None):
    sys_ = P.LinearParabolicSystem(c.M, c.K, lift)
    g = P.irk_step(sys_, c.table, c.ht, 0.0, u, c.device(), P.GmresConfig(restart=50), want_K=True)
    o = c.oracle.step(u, lift, restart=50)
    assert g.report.converged
    assert g.report.iterations == o["iterations"], (g.report.iterations, o["iterations"])
    assert np.array_equal(np.array(g.report.history), o["history"])
    assert np.array_equal(g.K, o["K"])
    assert np.array_equal(g.u_next, o["u_next"])
    return g.report.iterations


@pytest.mark.parametrize("kind", [P.CoeffKind.Jacobi, P.CoeffKind.GaussSeidelLower,
                                  P.CoeffKind.UpperFactor, P.CoeffKind.LowerFactor])
def test_heat_512_every_preconditioner(kind):
    c = heat_case(512, s=3, kind=kind, ht=1e-3)
    u = c.problem.initial(0.01, 1)
    its = bitwise_step(c, u)
    assert 10 < its < 200


def test_double_glazing_256_lift():
    c = dg_case(256, s=4, ht=0.01)
    u = np.zeros(c.n)
    bitwise_step(c, u, np.ascontiguousarray(c.problem.f_lift))


def test_lobatto_512_s5():
    c = heat_case(512, scheme=P.Scheme.LobattoIIIC, s=5, ht=1e-3)
    bitwise_step(c, c.problem.initial(0.01, 1))


def test_left_preconditioning_512():
    c = heat_case(512, s=3, ht=1e-3)
    u = c.problem.initial(0.01, 1)
    sys_ = P.LinearParabolicSystem(c.M, c.K, None)
    g = P.irk_step(sys_, c.table, c.ht, 0.0, u, c.device(), P.GmresConfig(side="left", restart=50), want_K=True)
    o = c.oracle.step(u, None, restart=50, side="left")
    assert g.report.iterations == o["iterations"]
    assert np.array_equal(g.K, o["K"]) and np.array_equal(g.u_next, o["u_next"])


def test_restart_cycles_512():
    """Block Jacobi with Lobatto IIIC s=5 needs > 100 iterations: several
    GMRES(50) cycles, each ending with x += Z y and a true residual."""
    c = heat_case(512, scheme=P.Scheme.LobattoIIIC, s=5, kind=P.CoeffKind.Jacobi, ht=1e-3)
    u = c.problem.initial(0.01, 1)
    sys_ = P.LinearParabolicSystem(c.M, c.K, None)
    g = P.irk_step(sys_, c.table, c.ht, 0.0, u, c.device(), P.GmresConfig(restart=50), want_K=True)
    o = c.oracle.step(u, None, restart=50)
    assert g.report.cycles >= 3, g.report.cycles
    assert g.report.iterations == o["iterations"]
    assert np.array_equal(np.array(g.report.history), o["history"])
    assert np.array_equal(g.K, o["K"]) and np.array_equal(g.u_next, o["u_next"])
