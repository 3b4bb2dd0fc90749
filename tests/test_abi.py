"""C ABI surface (CPU): the library loads, exports every symbol irkdev.h
declares, and the device entry points fail loudly without a GPU."""
import ctypes as C

import numpy as np
import pytest

import paper_2010_11377_b200 as P
from paper_2010_11377_b200 import _abi
from conftest import has_gpu


def test_library_loads_and_exports_header_symbols():
    L = _abi.lib()
    names = _abi.exported_symbols()
    assert len(names) >= 30
    for name in names:
        assert hasattr(L, name), name


def test_every_export_has_a_python_signature():
    for name in _abi.exported_symbols():
        assert name in _abi._SIGS, name


def test_defaults_match_reference():
    p = _abi.irk_amg_params()
    _abi.lib().irk_amg_params_default(C.byref(p))
    # AmgParams defaults (amg.hpp:14-29)
    assert (p.theta, p.pre_sweeps, p.post_sweeps, p.smoother) == (0.25, 1, 1, 0)
    assert p.jacobi_weight == 2.0 / 3.0 and p.prolongation_weight == 4.0 / 3.0
    assert (p.prolongation_steps, p.max_coarse, p.max_levels) == (1, 64, 10)
    g = _abi.irk_gmres_cfg()
    _abi.lib().irk_gmres_cfg_default(C.byref(g))
    assert (g.side, g.rel_tol, g.max_iter, g.restart) == (1, 1e-8, 500, 0)  # full GMRES, gmres.hpp:20


def test_errors_map_to_reference_exceptions():
    with pytest.raises(ValueError):
        P.make_radau_iia(8)  # require(s in 1..7)
    with pytest.raises(ValueError):
        P.make_lobatto_iiic(6)
    with pytest.raises(P.SingularError):
        P.ldu_factorize(np.array([[0.0, 1.0], [1.0, 0.0]]))
    bad = P.CsrMatrix(np.array([0, 2], np.int32), np.array([1, 0], np.int32), np.ones(2), 2)
    with pytest.raises(ValueError):
        P.amg_setup(bad)  # columns not strictly increasing -> validate()


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure path")
def test_device_fails_loudly_without_gpu():
    pr = P.make_heat_setup(8)
    t = P.make_radau_iia(2)
    with pytest.raises(P.CudaError):
        P.BlockPreconditioner(pr.M, pr.F, P.precond_coeff(t, P.CoeffKind.LowerFactor), 0.01,
                              table=t)


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure path")
def test_device_amg_setup_fails_loudly_without_gpu():
    """amg_setup_device has no CPU fallback."""
    pr = P.make_heat_setup(8)
    with pytest.raises(P.CudaError):
        P.amg_setup_device(pr.F)
    with pytest.raises(ValueError):  # argument checks come first, as in amg_setup
        P.amg_setup_device(pr.F, P.AmgParams(theta=1.5))


def test_tuning_switches_are_settable_without_gpu():
    """irk_set_option only records the override (read when graphs are recorded)."""
    from paper_2010_11377_b200 import _abi
    _abi.check(_abi.lib().irk_set_option(b"IRK_ZR", 1))
    with pytest.raises(ValueError):
        _abi.check(_abi.lib().irk_set_option(None, 1))


def test_gauss_seidel_setup_and_no_cpu_fallback():
    """The Gauss-Seidel smoother (amg.cpp:125-140) runs on the device only:
    host setup accepts it, an unknown smoother is an invalid argument, and
    without a GPU the device solver fails loudly (no CPU emulation)."""
    from conftest import has_gpu
    pr = P.make_heat_setup(8)
    t = P.make_radau_iia(2)
    B = P.CsrMatrix(pr.M.row_ptr, pr.M.col_idx, pr.M.vals + 0.01 * pr.F.vals, pr.M.n_cols)
    h = P.amg_setup(B, P.AmgParams(smoother=1, pre_sweeps=4, post_sweeps=4, prolongation_steps=2))
    assert h.n_levels() >= 1
    with pytest.raises(ValueError):
        P.amg_setup(B, P.AmgParams(smoother=2))
    if not has_gpu():
        with pytest.raises(P.CudaError):
            P.BlockPreconditioner(pr.M, pr.F, P.precond_coeff(t, P.CoeffKind.LowerFactor), 0.01,
                                  P.AmgParams(smoother=1), table=t)
