"""Every runtime tuning switch of the device path changes how the work is
scheduled, never the arithmetic: an IRK step (iterations, residual history,
K, u_next) and a V-cycle are bit-identical with each switch on and off.

Switches (irk_set_option, same names as the IRK_* environment variables):
  IRK_BOTTOM       single-CTA bottom V-cycle kernel vs per-level kernels
  IRK_ZR           restriction writes wd.*r for the next level vs on-the-fly
  IRK_PDL_DGS      programmatic launches of the DCGS2 block-dot / update
  IRK_PDL_COARSE   first AMG level launched programmatically
  IRK_PDL_FINE     level-0/1 SpMVs launched programmatically, late trigger
  IRK_DOM_CLASS    row-class SpMV with the dominant class in the kernel
                   parameters vs class-table loads for every row
"""
import numpy as np
import pytest

import paper_2010_11377_b200 as P
from paper_2010_11377_b200 import _abi
from conftest import has_gpu

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]

DEFAULTS = {"IRK_BOTTOM": 1, "IRK_ZR": 1, "IRK_PDL_DGS": 1, "IRK_PDL_COARSE": 2, "IRK_DOM_CLASS": 1,
            "IRK_PDL_FINE": 1}


def set_opt(name, value):
    _abi.check(_abi.lib().irk_set_option(name.encode(), int(value)))


@pytest.fixture(autouse=True)
def restore_defaults():
    yield
    for k, v in DEFAULTS.items():
        set_opt(k, v)


@pytest.fixture(scope="module")
def case():
    pr = P.make_heat_setup(256)
    t = P.make_radau_iia(3)
    pc = P.precond_coeff(t, P.CoeffKind.LowerFactor)
    dev = P.BlockPreconditioner(pr.M, pr.F, pc, 1e-3, table=t)
    u = pr.initial(noise=0.01, seed=7)
    return pr, t, dev, u


def step(case):
    pr, t, dev, u = case
    sys_ = P.LinearParabolicSystem(pr.M, pr.F, pr.f_lift)
    return P.irk_step(sys_, t, 1e-3, 0.0, u, dev, P.GmresConfig(restart=50), want_K=True)


@pytest.mark.parametrize("name,off", [("IRK_BOTTOM", 0), ("IRK_ZR", 0), ("IRK_PDL_DGS", 0),
                                      ("IRK_PDL_COARSE", 0), ("IRK_PDL_COARSE", 99),
                                      ("IRK_DOM_CLASS", 0), ("IRK_PDL_FINE", 0)])
def test_switch_is_bit_identical(case, name, off):
    a = step(case)
    set_opt(name, off)
    b = step(case)
    assert a.report.iterations == b.report.iterations
    assert np.array_equal(a.report.history, b.report.history)
    assert np.array_equal(a.K, b.K) and np.array_equal(a.u_next, b.u_next)


def test_vcycle_bottom_kernel_bit_identical(case):
    _, _, dev, _ = case
    r = np.random.default_rng(3).uniform(-1, 1, dev.size() // dev.stages())
    z1 = dev.vcycle(0, r)
    set_opt("IRK_BOTTOM", 0)
    z0 = dev.vcycle(0, r)
    assert np.array_equal(z1, z0)
