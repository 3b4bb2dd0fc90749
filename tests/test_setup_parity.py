"""Host setup vs the reference (oracle/_ref), bit for bit.

The product's host setup (paper_2010_11377_b200/csrc/host) restates the
reference's FE assembly, Butcher construction, LDU and AMG coarsening.  The
BASELINE contract is "AMG hierarchy sparsity and integer index structures are
bit-exact"; we check that and, stronger, identical fp64 values.
"""
import numpy as np
import pytest

import paper_2010_11377_b200 as P
from refs import Ref

pytestmark = pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not built")


def same_csr(ours: P.CsrMatrix, ref, exact_values=True):
    rp, ci, v = ref
    assert np.array_equal(ours.row_ptr, rp)
    assert np.array_equal(ours.col_idx, ci)
    if exact_values:
        assert np.array_equal(ours.vals, v), np.max(np.abs(ours.vals - v))


@pytest.mark.parametrize("cells", [8, 64, 128])
def test_heat_assembly_bitwise(cells):
    ours = P.make_heat_setup(cells)
    ref = Ref.problem("heat", cells)
    same_csr(ours.M, ref["M"])
    same_csr(ours.F, ref["K"])
    assert np.array_equal(ours.f_lift, ref["f_lift"])


@pytest.mark.parametrize("cells", [16, 64])
def test_double_glazing_assembly_bitwise(cells):
    ours = P.make_double_glazing_setup(cells, 0.005)
    ref = Ref.problem("dg", cells, 0.005)
    same_csr(ours.M, ref["M"])
    same_csr(ours.F, ref["K"])
    assert np.array_equal(ours.f_lift, ref["f_lift"])


def test_shared_pattern_and_stencil():
    """M and K share one 7-point pattern (SURVEY §8 finding 4)."""
    pr = P.make_heat_setup(64)
    assert np.array_equal(pr.M.row_ptr, pr.F.row_ptr)
    assert np.array_equal(pr.M.col_idx, pr.F.col_idx)
    rows = np.repeat(np.arange(pr.M.n_rows), np.diff(pr.M.row_ptr))
    assert sorted(set((pr.M.col_idx - rows).tolist())) == [-64, -63, -1, 0, 1, 63, 64]


@pytest.mark.parametrize("scheme,smax", [(0, 7), (1, 5)])
def test_tableaux_bitwise(scheme, smax):
    for s in range(1 if scheme == 0 else 2, smax + 1):
        t = P.make_table(P.Scheme(scheme), s)
        A, b, c, q = Ref.tableau(scheme, s)
        assert np.array_equal(t.A, A), (s, np.max(np.abs(t.A - A)))
        assert np.array_equal(t.b, b)
        assert np.array_equal(t.c, c)
        assert t.q == q


def test_two_stage_constants():
    """Hand-checked s=2 values (test_butcher.cpp:47-65, 144-151)."""
    r = P.make_radau_iia(2)
    assert r.A[0, 0] == pytest.approx(5 / 12, rel=1e-14)
    assert r.A[0, 1] == pytest.approx(-1 / 12, rel=1e-13)
    assert r.A[1, 0] == pytest.approx(3 / 4, rel=1e-14)
    assert r.A[1, 1] == pytest.approx(1 / 4, rel=1e-14)
    L, D, U = P.ldu_factorize(r.A)
    assert D[0] == pytest.approx(5 / 12, rel=1e-13)
    assert D[1] == pytest.approx(2 / 5, rel=1e-13)
    assert L[1, 0] == pytest.approx(9 / 5, rel=1e-13)
    assert U[0, 1] == pytest.approx(-1 / 5, rel=1e-13)
    l2 = P.make_lobatto_iiic(2)
    assert np.allclose(l2.A, [[0.5, -0.5], [0.5, 0.5]], rtol=1e-14)


@pytest.mark.parametrize("kind", [0, 1, 2, 3])
def test_precond_coeff_bitwise(kind):
    for scheme, ss in ((0, range(1, 8)), (1, range(2, 6))):
        for s in ss:
            t = P.make_table(P.Scheme(scheme), s)
            pc = P.precond_coeff(t, P.CoeffKind(kind))
            At, st = Ref.precond_coeff(scheme, s, kind)
            assert np.array_equal(pc.Atilde, At)
            assert int(pc.structure) == st


def test_ldu_errors_and_custom():
    with pytest.raises(P.SingularError):
        P.ldu_factorize(np.array([[0.0, 1.0], [1.0, 0.0]]))
    with pytest.raises(ValueError):
        P.custom_coeff(np.array([[1.0, 2.0], [3.0, 4.0]]))
    with pytest.raises(ValueError):
        P.custom_coeff(np.array([[0.0, 0.0], [1.0, 1.0]]))
    assert P.custom_coeff(np.array([[1.0, 0.0], [2.0, 3.0]])).structure == P.CoeffStructure.LowerTriangular


def _compare_hierarchies(ours, ref):
    assert ours.n_levels() == ref.n_levels()
    for l in range(ours.n_levels()):
        for which in ("A", "P", "R") if l + 1 < ours.n_levels() else ("A",):
            a = ours.level(l, which)
            (rp, ci, v), nc = ref.level(l, which)
            assert a.n_cols == nc
            same_csr(a, (rp, ci, v))
        assert np.array_equal(ours.inv_diag(l), ref.inv_diag(l))


@pytest.mark.parametrize("cells,ht,d", [(64, 0.01, 5 / 12), (64, 0.01, 0.4), (128, 1e-3, 0.2)])
def test_amg_hierarchy_bitwise_heat(cells, ht, d):
    pr = P.make_heat_setup(cells)
    B = P.CsrMatrix(pr.M.row_ptr, pr.M.col_idx, 1.0 * pr.M.vals + (ht * d) * pr.F.vals, pr.M.n_cols)
    ours = P.amg_setup(B)
    ref = Ref.amg((B.row_ptr, B.col_idx, B.vals))
    _compare_hierarchies(ours, ref)


def test_amg_hierarchy_bitwise_dg():
    pr = P.make_double_glazing_setup(64, 0.005)
    B = P.CsrMatrix(pr.M.row_ptr, pr.M.col_idx, 1.0 * pr.M.vals + 0.0025 * pr.F.vals, pr.M.n_cols)
    _compare_hierarchies(P.amg_setup(B), Ref.amg((B.row_ptr, B.col_idx, B.vals)))


def test_amg_hierarchy_bitwise_poisson_and_psteps():
    pr = P.make_heat_setup(32)
    _compare_hierarchies(P.amg_setup(pr.F), Ref.amg((pr.F.row_ptr, pr.F.col_idx, pr.F.vals)))
    prm = P.AmgParams(prolongation_steps=2, theta=0.1)
    _compare_hierarchies(P.amg_setup(pr.F, prm),
                         Ref.amg((pr.F.row_ptr, pr.F.col_idx, pr.F.vals), theta=0.1, psteps=2))


def test_amg_setup_errors():
    empty = P.CsrMatrix(np.zeros(1, np.int32), np.zeros(0, np.int32), np.zeros(0), 0)
    with pytest.raises(ValueError):
        P.amg_setup(empty)
    pr = P.make_heat_setup(8)
    with pytest.raises(ValueError):
        P.amg_setup(pr.F, P.AmgParams(theta=1.5))
    z = P.CsrMatrix(pr.F.row_ptr, pr.F.col_idx, np.where(pr.F.col_idx == np.repeat(
        np.arange(pr.F.n_rows), np.diff(pr.F.row_ptr)), 0.0, pr.F.vals), pr.F.n_cols)
    with pytest.raises(P.SingularError):
        P.amg_setup(z)


def test_small_matrix_single_level():
    """n <= max_coarse gives one exact level (test_amg.cpp:40-50)."""
    n = 40
    rp = np.arange(0, 3 * n - 1, dtype=np.int32)
    rows, cols, vals = [], [], []
    for i in range(n):
        for j, v in ((i - 1, -1.0), (i, 2.0), (i + 1, -1.0)):
            if 0 <= j < n:
                rows.append(i)
                cols.append(j)
                vals.append(v)
    rp = np.searchsorted(np.array(rows), np.arange(n + 1)).astype(np.int32)
    A = P.CsrMatrix(rp, np.array(cols, np.int32), np.array(vals), n)
    h = P.amg_setup(A)
    assert h.n_levels() == 1
    Ainv = h.coarse_inverse()
    dense = np.zeros((n, n))
    dense[np.array(rows), np.array(cols)] = vals
    assert np.allclose(Ainv @ dense, np.eye(n), atol=1e-10)
