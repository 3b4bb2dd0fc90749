"""Parity against committed golden fixtures from the reference build.

tests/golden/*.npz were produced by tests/golden/make_golden.py from the
reference's own code (oracle/_ref).  These tests need neither /root/reference
nor oracle/_ref, so they pin parity on any machine:
  * host setup: Butcher tables / coefficients equal; M, K, f_lift and every
    AMG level (A, P, R, inv_diag) bit-identical (SHA-256 of the raw arrays);
  * the C oracle's IRK step: iterations within +-1, K and u_next within 1e-9
    relative L2 of the reference's (BASELINE parity bar);
  * (gpu) the device step through the C ABI, same bar;
  * left preconditioning, a time-dependent forcing (cos(t) * fq) and a
    reference integrate() trajectory with a truncated last step, same bar.
"""
import hashlib
from pathlib import Path

import numpy as np
import pytest

import paper_2010_11377_b200 as P
from conftest import has_gpu
from systems import Case, rel_l2

GOLD = Path(__file__).resolve().parent / "golden"
CASES = sorted(p.stem for p in GOLD.glob("*.npz") if p.stem != "butcher" and not p.stem.startswith("traj_"))
TRAJ = sorted(p.stem for p in GOLD.glob("traj_*.npz"))


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


def side_of(g):
    return str(g["side"]) if "side" in g else "right"


def stage_forcing(g, table, ht):
    """s*n stage-major cos(t_n + c_i ht) * fq, or None."""
    if "fq" not in g:
        return None
    import math
    t_n = float(g["t_n"])
    return np.concatenate([math.cos(t_n + ci * ht) * g["fq"] for ci in table.c])


def forcing_fn(g):
    if "fq" not in g:
        return None
    import math
    fq = g["fq"]
    return lambda t: math.cos(t) * fq


@pytest.mark.parametrize("name", CASES)
def test_oracle_step_against_golden(name):
    g, c = case(name)
    o = c.oracle.step(g["u0"], c.f_lift, restart=int(g["restart"]), side=side_of(g),
                      forcing=stage_forcing(g, c.table, c.ht))
    assert abs(o["iterations"] - int(g["iterations"])) <= 1
    assert o["converged"]
    assert rel_l2(o["K"], g["K"]) <= 1e-9
    assert rel_l2(o["u_next"], g["u_next"]) <= 1e-9


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
@pytest.mark.parametrize("name", CASES)
def test_device_step_against_golden(name):
    g, c = case(name)
    sys_ = P.LinearParabolicSystem(c.M, c.K, c.f_lift, forcing=forcing_fn(g))
    t_n = float(g["t_n"]) if "t_n" in g else 0.0
    r = P.irk_step(sys_, c.table, c.ht, t_n, g["u0"], c.device(),
                   P.GmresConfig(side=side_of(g), restart=int(g["restart"])), want_K=True)
    assert abs(r.report.iterations - int(g["iterations"])) <= 1
    assert r.report.converged
    assert rel_l2(r.K, g["K"]) <= 1e-9
    assert rel_l2(r.u_next, g["u_next"]) <= 1e-9


def traj_cases(g):
    """One Case per step size of the reference loop (irk.cpp:85-99)."""
    cells, s, ht, t_final = int(g["cells"]), int(g["s"]), float(g["ht"]), float(g["t_final"])
    prob = P.make_heat_setup(cells)
    table = P.make_radau_iia(s)
    coeff = P.precond_coeff(table, P.CoeffKind.LowerFactor)
    t, steps = 0.0, []
    while t < t_final - 1e-14 * t_final:
        st = ht if t + ht <= t_final else t_final - t
        steps.append(st)
        t += st
    cases = {h: Case(prob.M, prob.F, table, coeff, h, None, prob.f_lift) for h in set(steps)}
    return prob, table, steps, cases


@pytest.mark.parametrize("name", TRAJ)
def test_oracle_trajectory_against_golden(name):
    import math
    g = load(name)
    prob, table, steps, cases = traj_cases(g)
    u, t, its = g["u0"].copy(), 0.0, []
    for st in steps:
        f = np.concatenate([math.cos(t + ci * st) * g["fq"] for ci in table.c])
        o = cases[st].oracle.step(u, prob.f_lift, restart=0, forcing=f)
        u, t = o["u_next"], t + st
        its.append(o["iterations"])
    assert len(steps) == int(g["steps"]) and t == float(g["t_end"])
    assert all(abs(a - b) <= 1 for a, b in zip(its, g["iterations"].tolist()))
    assert rel_l2(u, g["u_final"]) <= 1e-9


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
@pytest.mark.parametrize("name", TRAJ)
def test_device_trajectory_against_golden(name):
    import math
    g = load(name)
    prob, table, steps, cases = traj_cases(g)
    fq = g["fq"]
    sys_ = P.LinearParabolicSystem(prob.M, prob.F, prob.f_lift, forcing=lambda t: math.cos(t) * fq)
    tr = P.integrate(sys_, table, g["u0"], float(g["t_final"]), float(g["ht"]),
                     lambda h: cases[h].device(), P.GmresConfig(restart=0))
    assert tr.steps == int(g["steps"]) and tr.t_final == float(g["t_end"])
    assert all(abs(r.iterations - b) <= 1 for r, b in zip(tr.reports, g["iterations"].tolist()))
    assert rel_l2(tr.u_final, g["u_final"]) <= 1e-9
