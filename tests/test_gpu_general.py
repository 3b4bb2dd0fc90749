"""Operators the uniform-grid format heuristics were not tuned on, at sizes
that take the large-level code paths.

* diagonally scaled heat (D M D, D K D with a seeded random D): every stored
  value distinct -- no row classes, no value dictionaries: fp64 DIA for M, K
  and the fine level, fp64 SELL / CSR-vector below;
* symmetrically permuted heat (P M P^T, P K P^T, seeded permutation): no
  diagonal structure at all -- the fine level, M and K in SELL-32 / CSR-vector
  and the stage operator in its unfused form;
* the double-glazing operators permuted the same way (nonsymmetric SUPG).

Each runs one IRK step (Radau IIA s=3, P_LD, GMRES(50)) compared bit for bit
with the oracle on the same arrays, and reports the formats the device chose.
"""
import numpy as np
import pytest

import paper_2010_11377_b200 as P
from conftest import has_gpu
from systems import Case

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


def scaled(A: P.CsrMatrix, d: np.ndarray) -> P.CsrMatrix:
    rows = np.repeat(np.arange(A.n_rows), np.diff(A.row_ptr))
    return P.CsrMatrix(A.row_ptr.copy(), A.col_idx.copy(), d[rows] * A.vals * d[A.col_idx], A.n_cols)


def permuted(A: P.CsrMatrix, p: np.ndarray) -> P.CsrMatrix:
    """B[p[i], p[j]] = A[i, j] (columns sorted per row)."""
    n = A.n_rows
    rows = np.repeat(np.arange(n), np.diff(A.row_ptr))
    r, c = p[rows], p[A.col_idx]
    order = np.lexsort((c, r))
    r, c, v = r[order], c[order], A.vals[order]
    rp = np.zeros(n + 1, np.int32)
    np.add.at(rp, r + 1, 1)
    return P.CsrMatrix(np.cumsum(rp).astype(np.int32), c.astype(np.int32), v.copy(), n)


def formats(dev):
    import ctypes as C
    L = P._abi.lib()
    out = []
    for l in range(L.irkdev_num_levels(dev._h, 0)):
        vf = C.c_int()
        P._abi.check(L.irkdev_level_value_format(dev._h, 0, l, C.byref(vf)))
        out.append(vf.value)
    return out


def run(M, K, u, lift=None, ht=1e-3):
    t = P.make_radau_iia(3)
    c = Case(M, K, t, P.precond_coeff(t, P.CoeffKind.LowerFactor), ht, None, lift)
    sys_ = P.LinearParabolicSystem(c.M, c.K, lift)
    g = P.irk_step(sys_, t, ht, 0.0, u, c.device(), P.GmresConfig(restart=50), want_K=True)
    o = c.oracle.step(u, lift, restart=50)
    assert g.report.converged
    assert g.report.iterations == o["iterations"]
    assert np.array_equal(np.array(g.report.history), o["history"])
    assert np.array_equal(g.K, o["K"]) and np.array_equal(g.u_next, o["u_next"])
    return c, g


def test_scaled_heat_all_values_distinct():
    pr = P.make_heat_setup(384)
    d = np.random.default_rng(11).uniform(0.5, 2.0, pr.M.n_rows)
    M, K = scaled(pr.M, d), scaled(pr.F, d)
    c, g = run(M, K, pr.initial(0.01, 1) / d)
    assert formats(c.device()._dev)[0] == 0  # fine level in fp64 (no classes / codes)


@pytest.mark.parametrize("cells", [192, 320])
def test_permuted_heat_no_diagonal_structure(cells):
    pr = P.make_heat_setup(cells)
    p = np.random.default_rng(cells).permutation(pr.M.n_rows).astype(np.int32)
    M, K = permuted(pr.M, p), permuted(pr.F, p)
    u = np.empty(pr.M.n_rows)
    u[p] = pr.initial(0.01, 2)
    run(M, K, u)


def test_permuted_double_glazing():
    pr = P.make_double_glazing_setup(160, 0.005)
    p = np.random.default_rng(5).permutation(pr.M.n_rows).astype(np.int32)
    M, K = permuted(pr.M, p), permuted(pr.F, p)
    lift = np.empty(pr.M.n_rows)
    lift[p] = np.ascontiguousarray(pr.f_lift)
    run(M, K, np.zeros(pr.M.n_rows), lift=lift, ht=1e-2)
