"""Parity against committed golden fixtures from the reference build.

tests/golden/*.npz were produced by tests/golden/make_golden.py from the
reference's own code (oracle/_ref).  These tests need neither /root/reference
nor oracle/_ref, so they pin parity on any machine:
  * host setup: Butcher tables / coefficients equal; M, K, f_lift and every
    AMG level (A, P, R, inv_diag) bit-identical (SHA-256 of the raw arrays);
  * the C oracle's IRK step: iterations within +-1, K and u_next within 1e-9
    relative L2 of the reference's (BASELINE parity bar);
  * (gpu) the device step through the C ABI, same bar.
"""
import hashlib
from pathlib import Path

import numpy as np
import pytest

import paper_2010_11377_b200 as P
from conftest import has_gpu
from systems import Case, rel_l2

GOLD = Path(__file__).resolve().parent / "golden"
CASES = sorted(p.stem for p in GOLD.glob("*.npz") if p.stem != "butcher")


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def load(name):
    return dict(np.load(GOLD / f"{name}.npz"))


def build_case(g):
    cells, scheme, s, kind, ht = (int(g["cells"]), int(g["scheme"]), int(g["s"]), int(g["kind"]),
                                  float(g["ht"]))
    dg = "dg" in g.get("_name", "")
    prob = P.make_double_glazing_setup(cells, 0.005) if dg else P.make_heat_setup(cells)
    table = P.make_table(P.Scheme(scheme), s)
    c = Case(prob.M, prob.F, table, P.precond_coeff(table, P.CoeffKind(kind)), ht, None, prob.f_lift)
    c.problem = prob
    return c


def case(name):
    g = load(name)
    g["_name"] = name
    return g, build_case(g)


def test_butcher_tables_equal_reference():
    g = load("butcher")
    for scheme, ss in ((0, range(1, 8)), (1, range(2, 6))):
        for s in ss:
            t = P.make_table(P.Scheme(scheme), s)
            assert np.array_equal(t.A, g[f"tab_{scheme}_{s}_A"])
            assert np.array_equal(t.b, g[f"tab_{scheme}_{s}_b"])
            assert np.array_equal(t.c, g[f"tab_{scheme}_{s}_c"])
            for kind in range(4):
                pc = P.precond_coeff(t, P.CoeffKind(kind))
                assert np.array_equal(pc.Atilde, g[f"coeff_{scheme}_{s}_{kind}"])
                assert int(pc.structure) == int(g[f"struct_{scheme}_{s}_{kind}"])


@pytest.mark.parametrize("name", CASES)
def test_setup_bitwise_against_golden(name):
    g, c = case(name)
    M, K = c.problem.M, c.problem.F
    assert digest(M.row_ptr, M.col_idx, M.vals) == str(g["M_sha"])
    assert digest(K.row_ptr, K.col_idx, K.vals) == str(g["K_sha"])
    assert digest(c.problem.f_lift) == str(g["f_lift_sha"])
    for k, h in enumerate(c.hiers):
        assert h.sizes() == g[f"hier{k}_sizes"].tolist()
        for l in range(h.n_levels()):
            a = h.level(l, "A")
            parts = [a.row_ptr, a.col_idx, a.vals, h.inv_diag(l)]
            if l + 1 < h.n_levels():
                p, r = h.level(l, "P"), h.level(l, "R")
                parts += [p.row_ptr, p.col_idx, p.vals, r.row_ptr, r.col_idx, r.vals]
            assert digest(*parts) == str(g[f"hier{k}_sha"][l]), (k, l)


@pytest.mark.parametrize("name", CASES)
def test_oracle_step_against_golden(name):
    g, c = case(name)
    o = c.oracle.step(g["u0"], c.f_lift, restart=int(g["restart"]))
    assert abs(o["iterations"] - int(g["iterations"])) <= 1
    assert o["converged"]
    assert rel_l2(o["K"], g["K"]) <= 1e-9
    assert rel_l2(o["u_next"], g["u_next"]) <= 1e-9


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
@pytest.mark.parametrize("name", CASES)
def test_device_step_against_golden(name):
    g, c = case(name)
    sys_ = P.LinearParabolicSystem(c.M, c.K, c.f_lift)
    r = P.irk_step(sys_, c.table, c.ht, 0.0, g["u0"], c.device(),
                   P.GmresConfig(restart=int(g["restart"])), want_K=True)
    assert abs(r.report.iterations - int(g["iterations"])) <= 1
    assert r.report.converged
    assert rel_l2(r.K, g["K"]) <= 1e-9
    assert rel_l2(r.u_next, g["u_next"]) <= 1e-9
