"""On-disk formats around the solve path.

* MatrixMarket (csr.cpp:240-290): our writer produces the reference writer's
  bytes; each side reads the other's files to the identical CSR (values
  round-trip exactly through %.17g); symmetric files are mirrored; malformed
  files raise the reference's error classes.
* Study CSV rows (study.cpp:334-360): header and row layout, including the
  "failed" row.
* A device step on reference-written M / K files equals the step on the
  in-memory matrices bit for bit (GPU).
"""
import ctypes as C

import numpy as np
import pytest

import paper_2010_11377_b200 as P
from conftest import has_gpu
from refs import Ref
from systems import Case, heat_case

ref_only = pytest.mark.skipif(not Ref.available(), reason="reference not built")


def _i(a):
    return np.ascontiguousarray(a, np.int32).ctypes.data_as(C.POINTER(C.c_int))


def _d(a):
    return np.ascontiguousarray(a, np.float64).ctypes.data_as(C.POINTER(C.c_double))


def ref_write(A: P.CsrMatrix, path):
    Ref.check(Ref.lib().ref_mm_write(A.n_rows, A.n_cols, _i(A.row_ptr), _i(A.col_idx), _d(A.vals),
                                     str(path).encode()))


def ref_read(path) -> P.CsrMatrix:
    nr, nc, nz = C.c_int(), C.c_int(), C.c_int()
    L = Ref.lib()
    Ref.check(L.ref_mm_read(str(path).encode(), C.byref(nr), C.byref(nc), C.byref(nz), None, None,
                            None))
    rp = np.zeros(nr.value + 1, np.int32)
    ci = np.zeros(max(nz.value, 1), np.int32)
    v = np.zeros(max(nz.value, 1))
    Ref.check(L.ref_mm_read(str(path).encode(), C.byref(nr), C.byref(nc), C.byref(nz), _i(rp),
                            _i(ci), _d(v)))
    return P.CsrMatrix(rp, ci[: nz.value], v[: nz.value], nc.value)


def same(a: P.CsrMatrix, b: P.CsrMatrix) -> bool:
    return (a.n_rows == b.n_rows and a.n_cols == b.n_cols and np.array_equal(a.row_ptr, b.row_ptr)
            and np.array_equal(a.col_idx, b.col_idx)
            and np.array_equal(a.vals.view(np.int64), b.vals.view(np.int64)))


def test_roundtrip_exact(tmp_path):
    prob = P.make_double_glazing_setup(16)
    for A in (prob.M, prob.F):
        f = tmp_path / "a.mtx"
        P.write_matrix_market(A, f)
        assert same(P.read_matrix_market(f), A)
    # awkward values: subnormal, negative zero, huge
    A = P.CsrMatrix(np.array([0, 2, 3], np.int32), np.array([0, 1, 1], np.int32),
                    np.array([5e-324, -0.0, 1.7976931348623157e308]), 2)
    P.write_matrix_market(A, tmp_path / "b.mtx")
    assert same(P.read_matrix_market(tmp_path / "b.mtx"), A)


@ref_only
def test_writer_bytes_and_cross_reading_match_reference(tmp_path):
    K = P.make_heat_setup(12).F
    ours, theirs = tmp_path / "ours.mtx", tmp_path / "ref.mtx"
    P.write_matrix_market(K, ours)
    ref_write(K, theirs)
    assert ours.read_bytes() == theirs.read_bytes()
    assert same(P.read_matrix_market(theirs), K)
    assert same(ref_read(ours), K)


@ref_only
def test_symmetric_duplicates_and_comments(tmp_path):
    text = ("%%MatrixMarket matrix coordinate real symmetric\n"
            "% a comment line\n\n"
            "3 3 5\n"
            "1 1 4.0\n2 1 -1.5\n3 2 0.25\n3 3 2.0\n2 1 0.5\n")
    f = tmp_path / "sym.mtx"
    f.write_text(text)
    a, b = P.read_matrix_market(f), ref_read(f)
    assert same(a, b)
    dense = np.zeros((3, 3))
    for i in range(3):
        for k in range(a.row_ptr[i], a.row_ptr[i + 1]):
            dense[i, a.col_idx[k]] = a.vals[k]
    assert np.array_equal(dense, dense.T) and dense[1, 0] == -1.0


@pytest.mark.parametrize("text,exc", [
    ("%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n", ValueError),
    ("%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n", RuntimeError),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n", ValueError),
])
def test_malformed_files_raise(tmp_path, text, exc):
    f = tmp_path / "bad.mtx"
    f.write_text(text)
    with pytest.raises(exc):
        P.read_matrix_market(f)


def test_missing_file_raises(tmp_path):
    with pytest.raises(RuntimeError, match="cannot open"):
        P.read_matrix_market(tmp_path / "missing.mtx")


def test_csv_header_and_rows():
    assert P.csv_header() == ("scheme,s,hx_inv,ht,dof,precond,side,subsolver,iterations,"
                              "true_residual,rel_error,seconds\n")
    t = P.make_radau_iia(3)
    row = P.csv_row(t, 1024, 1e-3, 1046529, P.CoeffKind.LowerFactor, P.GmresConfig(), 30.1,
                    6.76e-9, 0.0, 0.0199)
    assert row == "radau_iia,3,1024,0.001,3139587,ld,right,amg,30.1,6.760000e-09,0.000000e+00,0.0199\n"
    row = P.csv_row(P.make_lobatto_iiic(5), 2048, 1e-3, 4190209, P.CoeffKind.Jacobi,
                    P.GmresConfig(side="left"), 0, 0, 0, 0, failed=True)
    assert row == "lobatto_iiic,5,2048,0.001,20951045,jacobi,left,amg,failed,,,\n"


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_device_step_on_matrix_market_inputs(tmp_path):
    c = heat_case(32, s=2, ht=0.01)
    P.write_matrix_market(c.M, tmp_path / "M.mtx")
    P.write_matrix_market(c.K, tmp_path / "K.mtx")
    M, K = P.read_matrix_market(tmp_path / "M.mtx"), P.read_matrix_market(tmp_path / "K.mtx")
    c2 = Case(M, K, c.table, c.coeff, c.ht, f_lift=c.f_lift)
    u = c.problem.initial(0.01, 3)
    sys = P.LinearParabolicSystem(c.M, c.K, c.f_lift)
    sys2 = P.LinearParabolicSystem(M, K, c.f_lift)
    a = P.irk_step(sys, c.table, c.ht, 0.0, u, c.device(), want_K=True)
    b = P.irk_step(sys2, c2.table, c2.ht, 0.0, u, c2.device(), want_K=True)
    assert np.array_equal(a.K, b.K) and a.report.iterations == b.report.iterations
