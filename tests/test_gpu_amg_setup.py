"""AMG setup on the device vs the host setup and the
reference's own amg_setup (oracle/_ref), bit for bit: every level's A, P, R
(row pointers, column indices, fp64 values), inverse diagonals and the
coarsest dense inverse.  The host setup is itself pinned to the reference
(tests/test_setup_parity.py), and where the reference build is present the
device hierarchy is also compared with it directly.
"""
import numpy as np
import pytest

import paper_2010_11377_b200 as P
from conftest import has_gpu
from refs import Ref

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


def same_hierarchy(a: P.AmgHierarchy, b: P.AmgHierarchy):
    assert a.n_levels() == b.n_levels()
    for l in range(a.n_levels()):
        for which in ("A", "P", "R") if l + 1 < a.n_levels() else ("A",):
            x, y = a.level(l, which), b.level(l, which)
            assert x.n_rows == y.n_rows and x.n_cols == y.n_cols, (l, which)
            assert np.array_equal(x.row_ptr, y.row_ptr), (l, which)
            assert np.array_equal(x.col_idx, y.col_idx), (l, which)
            assert np.array_equal(x.vals, y.vals), (l, which, np.max(np.abs(x.vals - y.vals)))
        assert np.array_equal(a.inv_diag(l), b.inv_diag(l)), l
    assert np.array_equal(a.coarse_inverse(), b.coarse_inverse())


def same_as_reference(dev: P.AmgHierarchy, B: P.CsrMatrix, **kw):
    if not Ref.available():
        return
    ref = Ref.amg((B.row_ptr, B.col_idx, B.vals), **kw)
    assert dev.n_levels() == ref.n_levels()
    for l in range(dev.n_levels()):
        for which in ("A", "P", "R") if l + 1 < dev.n_levels() else ("A",):
            a = dev.level(l, which)
            (rp, ci, v), nc = ref.level(l, which)
            assert a.n_cols == nc
            assert np.array_equal(a.row_ptr, rp) and np.array_equal(a.col_idx, ci)
            assert np.array_equal(a.vals, v), (l, which)
        assert np.array_equal(dev.inv_diag(l), ref.inv_diag(l))


def block(pr, ht, d):
    return P.CsrMatrix(pr.M.row_ptr, pr.M.col_idx, 1.0 * pr.M.vals + (ht * d) * pr.F.vals, pr.M.n_cols)


@pytest.mark.parametrize("cells,ht,d", [(64, 0.01, 5 / 12), (64, 0.01, 0.4), (128, 1e-3, 0.2),
                                        (256, 1e-3, 0.15505102572168222)])
def test_device_setup_heat(cells, ht, d):
    B = block(P.make_heat_setup(cells), ht, d)
    dev = P.amg_setup_device(B)
    same_hierarchy(dev, P.amg_setup(B))
    same_as_reference(dev, B)


def test_device_setup_double_glazing():
    """Non-symmetric operator (SUPG convection): the transposes matter."""
    pr = P.make_double_glazing_setup(64, 0.005)
    B = block(pr, 0.01, 0.25)
    dev = P.amg_setup_device(B)
    same_hierarchy(dev, P.amg_setup(B))
    same_as_reference(dev, B)


def test_device_setup_params():
    """Threshold, two prolongator smoothing steps, level and size caps."""
    pr = P.make_heat_setup(48)
    for prm, kw in ((P.AmgParams(theta=0.1, prolongation_steps=2), dict(theta=0.1, psteps=2)),
                    (P.AmgParams(theta=0.5), dict(theta=0.5)),
                    (P.AmgParams(max_coarse=10, max_levels=3), dict(max_coarse=10, max_levels=3))):
        dev = P.amg_setup_device(pr.F, prm)
        same_hierarchy(dev, P.amg_setup(pr.F, prm))
        if kw is not None:
            same_as_reference(dev, pr.F, **kw)


def test_device_setup_c2_size():
    """The C2 block M + h*0.2*K at 1024^2 (1,046,529 rows, six levels)."""
    B = block(P.make_heat_setup(1024), 1e-3, 0.2)
    dev = P.amg_setup_device(B)
    host = P.amg_setup(B)
    assert dev.sizes() == host.sizes()
    same_hierarchy(dev, host)


def test_device_setup_errors():
    pr = P.make_heat_setup(8)
    with pytest.raises(ValueError):
        P.amg_setup_device(pr.F, P.AmgParams(theta=1.5))
    rows = np.repeat(np.arange(pr.F.n_rows), np.diff(pr.F.row_ptr))
    z = P.CsrMatrix(pr.F.row_ptr, pr.F.col_idx, np.where(pr.F.col_idx == rows, 0.0, pr.F.vals), pr.F.n_cols)
    with pytest.raises(P.SingularError):
        P.amg_setup_device(z)
    # a single level when n <= max_coarse (test_amg.cpp:40-50)
    h = P.amg_setup_device(pr.F, P.AmgParams(max_coarse=100))
    assert h.n_levels() == 1
    same_hierarchy(h, P.amg_setup(pr.F, P.AmgParams(max_coarse=100)))


def test_solver_builds_device_hierarchies():
    """irkdev_create without caller hierarchies builds them on the device;
    the IRK step equals the one built from host hierarchies bit for bit."""
    pr = P.make_heat_setup(64)
    t = P.make_radau_iia(3)
    pc = P.precond_coeff(t, P.CoeffKind.LowerFactor)
    u = pr.initial(noise=0.01, seed=3)
    sys_ = P.LinearParabolicSystem(pr.M, pr.F, pr.f_lift)
    a = P.irk_step(sys_, t, 1e-3, 0.0, u, P.BlockPreconditioner(pr.M, pr.F, pc, 1e-3, table=t),
                   P.GmresConfig(restart=50), want_K=True)
    blocks = []
    for j in range(3):
        d = pc.Atilde[j, j]
        if d not in blocks:
            blocks.append(d)
    hiers = [P.amg_setup(block(pr, 1e-3, d)) for d in blocks]
    b = P.irk_step(sys_, t, 1e-3, 0.0, u, P.BlockPreconditioner(pr.M, pr.F, pc, 1e-3, table=t,
                                                                  hierarchies=hiers),
                   P.GmresConfig(restart=50), want_K=True)
    assert a.report.iterations == b.report.iterations
    assert np.array_equal(a.K, b.K) and np.array_equal(a.u_next, b.u_next)


def test_device_setup_c3_size():
    """The C3 block (2048^2: 4,190,209 rows, seven levels; Lobatto IIIC s=5
    diagonal coefficient scale), device vs host bit for bit."""
    B = block(P.make_heat_setup(2048), 1e-3, 0.25)
    dev = P.amg_setup_device(B)
    host = P.amg_setup(B)
    assert dev.n_levels() >= 6
    same_hierarchy(dev, host)


def test_device_setup_double_glazing_256():
    pr = P.make_double_glazing_setup(256, 0.005)
    B = block(pr, 0.01, 0.2)
    same_hierarchy(P.amg_setup_device(B), P.amg_setup(B))
