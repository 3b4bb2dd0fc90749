"""Gauss-Seidel smoother on the device (amg.cpp:125-140).

The sweeps are level-scheduled (one CTA steps through the dependency depths
of the level's operator, csrc/device/kernels.cu k_gs_sweep) and compute every
row exactly as the reference's sequential loop does -- same column order,
same operands, the diagonal skipped -- so V-cycles, preconditioner applies and
whole IRK steps are bit-identical to the oracle; against the reference the
BASELINE bar applies.  The reference study driver's cycle (study.hpp:44-47:
GS V(4,4), two prolongator smoothing steps) is the main case.
"""
import numpy as np
import pytest

import paper_2010_11377_b200 as P
from conftest import has_gpu
from refs import Ref, RefSolver
from systems import dg_case, heat_case, rel_l2, study_amg

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]

CYCLES = {
    "study": study_amg(),
    "v11": P.AmgParams(smoother=1),
    "v23": P.AmgParams(smoother=1, pre_sweeps=2, post_sweeps=3),
}


@pytest.mark.parametrize("cyc", list(CYCLES))
@pytest.mark.parametrize("problem", ["heat", "dg"])
def test_vcycle_bitwise(problem, cyc):
    amg = CYCLES[cyc]
    c = heat_case(64, s=2, ht=0.01, amg=amg) if problem == "heat" else dg_case(64, s=2, amg=amg)
    dev = c.device()
    rng = np.random.default_rng(9)
    for k in range(len(c.hiers)):
        r = rng.uniform(-1, 1, c.n)
        assert np.array_equal(dev.vcycle(k, r), c.oracle.vcycle(k, r))
    assert not np.any(dev.vcycle(0, np.zeros(c.n)))


@pytest.mark.parametrize("cyc", ["study", "v23"])
def test_vcycle_every_level_bitwise(monkeypatch, cyc):
    """No dense tail: the sweeps run on every level above the coarsest
    (256^2: DIA row classes at level 0, SELL / CSR-vector below)."""
    monkeypatch.setenv("IRK_TAIL_MAX", "0")
    c = heat_case(256, s=2, ht=1e-3, amg=CYCLES[cyc])
    assert c.hiers[0].tail()[1] is None
    r = np.random.default_rng(1).uniform(-1, 1, c.n)
    assert np.array_equal(c.device().vcycle(0, r), c.oracle.vcycle(0, r))


@pytest.mark.parametrize("problem", ["heat", "dg"])
def test_step_bitwise_and_vs_reference(problem):
    amg = study_amg()
    c = heat_case(64, s=2, ht=0.01, amg=amg) if problem == "heat" else dg_case(64, s=2, amg=amg)
    u = c.problem.initial() if problem == "heat" else np.zeros(c.n)
    dev = c.device()
    v = np.random.default_rng(3).uniform(-1, 1, 2 * c.n)
    assert np.array_equal(dev.apply(v), c.oracle.precond_apply(v))
    sys_ = P.LinearParabolicSystem(c.M, c.K, c.f_lift)
    g = P.irk_step(sys_, c.table, c.ht, 0.0, u, dev, P.GmresConfig(restart=50), want_K=True)
    o = c.oracle.step(u, c.f_lift)
    assert g.report.iterations == o["iterations"]
    assert np.array_equal(g.K, o["K"]) and np.array_equal(g.u_next, o["u_next"])
    M, K = c.M, c.K
    r = RefSolver((M.row_ptr, M.col_idx, M.vals), (K.row_ptr, K.col_idx, K.vals), 0, 2, 3, c.ht,
                  amg=amg).step(u, c.f_lift)
    assert g.report.converged and r["converged"]
    assert abs(g.report.iterations - r["iterations"]) <= 1
    assert rel_l2(g.K, r["K"]) <= 1e-9 and rel_l2(g.u_next, r["u_next"]) <= 1e-9


def test_step_midsize_bitwise():
    """256^2 heat, Radau IIA s=3, LD, the study cycle: one IRK step."""
    c = heat_case(256, s=3, ht=1e-3, amg=study_amg())
    u = c.problem.initial(0.01, 1)
    sys_ = P.LinearParabolicSystem(c.M, c.K, c.f_lift)
    g = P.irk_step(sys_, c.table, c.ht, 0.0, u, c.device(), P.GmresConfig(restart=50), want_K=True)
    o = c.oracle.step(u, c.f_lift)
    assert g.report.converged and g.report.iterations == o["iterations"]
    assert np.array_equal(np.array(g.report.history), o["history"])
    assert np.array_equal(g.K, o["K"]) and np.array_equal(g.u_next, o["u_next"])


def test_device_setup_gs_hierarchy_matches_host():
    """amg_setup_device with the study parameters equals the host setup."""
    c = heat_case(128, s=2, ht=0.01, amg=study_amg())
    B = c.hiers[0]
    M, K = c.M, c.K
    A = P.CsrMatrix(M.row_ptr, M.col_idx, 1.0 * M.vals + (c.ht * c.coeff.Atilde[0, 0]) * K.vals,
                    M.n_cols)
    D = P.amg_setup_device(A, study_amg())
    assert D.sizes() == B.sizes()
    for l in range(B.n_levels()):
        for w in ("A", "P", "R") if l + 1 < B.n_levels() else ("A",):
            a, b = D.level(l, w), B.level(l, w)
            assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col_idx, b.col_idx)
            assert a.vals.tobytes() == b.vals.tobytes()
