"""Coefficient files: read_coeff_file (butcher.cpp:300-313) and make_coeff
(study.cpp:269-282) against the reference build, including the error classes.

The files are written the way the reference's acceptance criterion 3 writes
its custom kind (acceptance.cpp:195-215): the stage count, then s rows of
"%.17g " values from a seeded generator.
"""
import numpy as np
import pytest

import paper_2010_11377_b200 as P
from refs import Ref, RefError
from systems import seeded_triangular, write_coeff

needs_ref = pytest.mark.skipif(not Ref.available(), reason="reference build missing")


@needs_ref
@pytest.mark.parametrize("s", [1, 2, 3, 5, 7])
@pytest.mark.parametrize("shape", ["lower", "upper", "diagonal"])
def test_read_matches_reference(tmp_path, s, shape):
    At = seeded_triangular(s, 777 + s, upper=shape == "upper")
    if shape == "diagonal":
        At = np.diag(np.diag(At))
    path = tmp_path / "coeff.txt"
    write_coeff(path, At)
    got = P.read_coeff_file(path)
    want, want_structure = Ref.coeff_file(path)
    assert got.tobytes() == want.tobytes() == At.tobytes()
    c = P.custom_coeff(got)
    assert int(c.structure) == want_structure
    assert c.kind == P.CoeffKind.Custom


@needs_ref
@pytest.mark.parametrize("text", [
    "2\n1 0\n0.5 2\n",
    "2 1e0 0 -5e-1 2.0",                       # one line, exponents
    "  3\n\n1\t0 0\n 0.25 1 0\n0.125 0.5 1\n trailing words ignored",
    "2\n+1.5 0\n1e-310 3\n",                     # subnormal
    "2\n0.1000000000000000055511151231257827 0\n-0.2 1\n",  # more digits than a double holds
])
def test_parse_variants_bitwise(tmp_path, text):
    path = tmp_path / "c.txt"
    path.write_text(text)
    got = P.read_coeff_file(path)
    want, _ = Ref.coeff_file(path)
    assert got.tobytes() == want.tobytes()


@needs_ref
@pytest.mark.parametrize("text,exc", [
    (None, P.IoError),            # missing file
    ("", P.IoError),              # no stage count
    ("0\n", P.IoError),           # bad stage count
    ("-2\n1 2 3 4", P.IoError),
    ("abc", P.IoError),
    ("2\n1 0 0\n", P.IoError),    # truncated
    ("2\n1 0 x 1\n", P.IoError),  # parse failure mid-matrix
])
def test_read_errors_match_reference(tmp_path, text, exc):
    path = tmp_path / "bad.txt"
    if text is not None:
        path.write_text(text)
    with pytest.raises(exc):
        P.read_coeff_file(path)
    with pytest.raises(RefError) as e:
        Ref.coeff_file(path)
    assert e.value.status == 6  # std::runtime_error


@needs_ref
@pytest.mark.parametrize("text", ["2\n1 1\n1 1\n", "2\n0 0\n1 1\n"])
def test_custom_validation_matches_reference(tmp_path, text):
    """Full matrix -> 'neither diagonal nor triangular'; zero diagonal entry;
    both std::invalid_argument (butcher.cpp:225-247)."""
    path = tmp_path / "c.txt"
    path.write_text(text)
    with pytest.raises(ValueError):
        P.custom_coeff(P.read_coeff_file(path))
    with pytest.raises(RefError) as e:
        Ref.coeff_file(path)
    assert e.value.status == 1


def test_make_coeff(tmp_path):
    t = P.make_radau_iia(3)
    for kind in (P.CoeffKind.Jacobi, P.CoeffKind.GaussSeidelLower, P.CoeffKind.UpperFactor,
                 P.CoeffKind.LowerFactor):
        a, b = P.make_coeff(t, kind), P.precond_coeff(t, kind)
        assert a.Atilde.tobytes() == b.Atilde.tobytes() and a.structure == b.structure
    with pytest.raises(ValueError, match="without --custom-coeff"):
        P.make_coeff(t, P.CoeffKind.Custom)
    path = tmp_path / "c.txt"
    write_coeff(path, seeded_triangular(2, 1))
    with pytest.raises(ValueError, match="expected s = 3"):
        P.make_coeff(t, P.CoeffKind.Custom, path)
    At = seeded_triangular(3, 4, upper=True)
    write_coeff(path, At)
    c = P.make_coeff(t, P.CoeffKind.Custom, path)
    assert c.kind == P.CoeffKind.Custom and c.structure == P.CoeffStructure.UpperTriangular
    assert c.Atilde.tobytes() == At.tobytes()
    with pytest.raises(P.IoError):
        P.make_coeff(t, P.CoeffKind.Custom, tmp_path / "missing.txt")
