"""Composed V-cycle operators (csrc/host/compose.cpp).

One damped-Jacobi V(1,1) level of amg.cpp:144-168 as two sparse products,
r_{l+1} = G_l r_l and z_l = [S_l Q_l] [r_l; z_{l+1}] with G = R (I - A W),
S = W (I - A W) + W, Q = P - W A P, W = omega D^-1.  CPU: the operators against
an independent dense computation, the lane rule, the composed oracle cycle
against the recursive cycle and the reference's amg_vcycle.  GPU: device ==
oracle bit for bit in both forms and across the storage switches.
"""
import numpy as np
import pytest

import paper_2010_11377_b200 as P
from conftest import has_gpu
from refs import Ref
from systems import dg_case, heat_case, rel_l2

def dense(m: P.CsrMatrix) -> np.ndarray:
    d = np.zeros((m.n_rows, m.n_cols))
    rows = np.repeat(np.arange(m.n_rows), np.diff(m.row_ptr))
    d[rows, m.col_idx] = m.vals
    return d


@pytest.mark.parametrize("make", [lambda: heat_case(24, s=2, ht=0.01), lambda: dg_case(28, s=2)])
def test_composed_operators_against_dense_algebra(make, monkeypatch):
    monkeypatch.setenv("IRK_TAIL_MAX", "0")  # compose every level above the coarsest
    c = make()
    h = c.hiers[0]
    L = h.n_levels()
    assert L >= 2
    for l in range(L - 1):
        A, Pm, R = dense(h.level(l, "A")), dense(h.level(l, "P")), dense(h.level(l, "R"))
        G, U = h.level(l, "G"), h.level(l, "U")
        n, nc = A.shape[0], Pm.shape[1]
        assert (G.n_rows, G.n_cols) == (nc, n) and (U.n_rows, U.n_cols) == (n, n + nc)
        W = np.diag(c.amg.jacobi_weight * h.inv_diag(l))
        E = np.eye(n) - A @ W
        assert np.allclose(dense(G), R @ E, rtol=1e-13, atol=1e-15)
        Ud = dense(U)
        assert np.allclose(Ud[:, :n], W @ E + W, rtol=1e-13, atol=1e-15)
        assert np.allclose(Ud[:, n:], Pm - W @ A @ Pm, rtol=1e-13, atol=1e-15)
        # CSR invariants: strictly increasing columns per row
        for m in (G, U):
            for i in range(m.n_rows):
                cols = m.col_idx[m.row_ptr[i]:m.row_ptr[i + 1]]
                assert np.all(np.diff(cols) > 0)
    last = h.level(L - 1, "G")
    assert last.n_rows == 0 and h.level(L - 1, "U").n_rows == 0


def test_lane_rule_and_scope(monkeypatch):
    c = heat_case(64, s=2, ht=0.01)
    h = c.hiers[0]
    tail_from, _ = h.tail()
    assert tail_from == 1  # 687 rows: the dense tail starts right below the fine level
    g, u = h.compose_lanes(0)
    assert u == 1  # 7-point fine level: sequential row sums (row classes + SELL on the device)
    assert g in (2, 4, 8, 16, 32)
    G = h.level(0, "G")
    assert 6.0 * g >= G.nnz / G.n_rows > 6.0 * g / 2
    # levels at or below the tail are not composed
    assert all(h.level(l, "G").n_rows == 0 for l in range(1, h.n_levels()))
    # Gauss-Seidel and V(2,3) hierarchies keep the recursive form
    for amg in (P.AmgParams(smoother=1), P.AmgParams(pre_sweeps=2, post_sweeps=3)):
        hh = heat_case(32, s=2, ht=0.01, amg=amg).hiers[0]
        assert hh.level(0, "G").n_rows == 0
    monkeypatch.setenv("IRK_COMPOSE", "0")
    assert heat_case(32, s=2, ht=0.01).hiers[0].level(0, "G").n_rows == 0


@pytest.mark.parametrize("make", [lambda: heat_case(64, s=2, ht=0.01), lambda: dg_case(48, s=2)])
@pytest.mark.parametrize("tail", [True, False])
def test_composed_cycle_matches_recursive_and_reference(make, tail, monkeypatch):
    if not tail:
        monkeypatch.setenv("IRK_TAIL_MAX", "0")
    comp = make()
    assert comp.hiers[0].level(0, "G").n_rows > 0
    monkeypatch.setenv("IRK_COMPOSE", "0")
    rec = make()
    assert rec.hiers[0].level(0, "G").n_rows == 0
    B = comp.M.vals * 1.0 + (comp.ht * comp.coeff.Atilde[0, 0]) * comp.K.vals
    ref = Ref.amg((comp.M.row_ptr, comp.M.col_idx, B))
    rng = np.random.default_rng(9)
    for _ in range(2):
        r = rng.uniform(-1, 1, comp.n)
        zc, zr = comp.oracle.vcycle(0, r), rec.oracle.vcycle(0, r)
        assert not np.array_equal(zc, zr)  # a different rounding, the same operator
        assert rel_l2(zc, zr) <= 1e-13
        assert rel_l2(zc, ref.vcycle(r)) <= 1e-12
    assert not np.any(comp.oracle.vcycle(0, np.zeros(comp.n)))


# ------------------------------------------------------------------ device
@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
@pytest.mark.parametrize("make", [lambda: heat_case(128, s=3, ht=1e-3), lambda: dg_case(96, s=2)])
@pytest.mark.parametrize("compose", [True, False])
@pytest.mark.parametrize("tail", [True, False])
def test_device_cycle_bitwise_both_forms(make, compose, tail, monkeypatch):
    if not compose:
        monkeypatch.setenv("IRK_COMPOSE", "0")
    if not tail:
        monkeypatch.setenv("IRK_TAIL_MAX", "0")
    c = make()
    assert (c.hiers[0].level(0, "G").n_rows > 0) == compose
    dev = c.device()
    rng = np.random.default_rng(4)
    for k in range(len(c.hiers)):
        r = rng.uniform(-1, 1, c.n)
        assert np.array_equal(dev.vcycle(k, r), c.oracle.vcycle(k, r))
    v = rng.uniform(-1, 1, c.n * c.s)
    assert np.array_equal(dev.apply(v), c.oracle.precond_apply(v))


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
@pytest.mark.parametrize("env", [{"IRK_UP_CLS": "0"}, {"IRK_LT_MM": "4"}, {"IRK_LT_MM": "6"},
                                 {"IRK_ROW_CLASSES": "0"}, {"IRK_ROW_SIG": "1"}, {"IRK_ROW_SIG": "7"}, {"IRK_PACK8": "0"}])
def test_storage_switches_are_bit_identical(env, monkeypatch):
    """The up leg as row classes + SELL or as one split SELL operator, the
    lane-tree operators as CSR or row signatures (opt-in), and the pipelined
    kernels' staging depth, are storage choices: same row sums."""
    c = heat_case(256, s=3, ht=1e-3)
    assert c.hiers[0].compose_lanes(0)[1] == 1  # k_up_cls path (exact grid spacing: few row classes)
    r = np.random.default_rng(12).uniform(-1, 1, c.n)
    base = c.device().vcycle(0, r)
    assert np.array_equal(base, c.oracle.vcycle(0, r))
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    other = P.BlockPreconditioner(c.M, c.K, c.coeff, c.ht, c.amg, table=c.table, hierarchies=c.hiers)
    assert np.array_equal(other.vcycle(0, r), base)


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_recursive_step_still_bitwise(monkeypatch):
    """IRK_COMPOSE=0 keeps the four-kernel levels: a whole step equals the oracle."""
    monkeypatch.setenv("IRK_COMPOSE", "0")
    c = heat_case(96, s=3, ht=1e-3)
    u = c.problem.initial(noise=0.01, seed=3)
    sys_ = P.LinearParabolicSystem(c.M, c.K, c.f_lift)
    d = P.irk_step(sys_, c.table, c.ht, 0.0, u, c.device(), P.GmresConfig(restart=50), want_K=True)
    o = c.oracle.step(u, c.f_lift, restart=50, max_iter=500)
    assert d.report.iterations == o["iterations"]
    assert np.array_equal(d.K, o["K"]) and np.array_equal(d.u_next, o["u_next"])


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_level0_leg_timing_hooks(monkeypatch):
    """irkdev_time_kernel(7 | 8) time the composed level-0 legs alone and report
    their algorithmic bytes (bench.py's vcycle_level0_roofline); a recursive
    hierarchy rejects them."""
    import ctypes as C
    from paper_2010_11377_b200 import _abi
    L = _abi.lib()
    c = heat_case(256, s=2, ht=0.01)
    h = c.device()._dev._h
    n, nc = c.n, c.hiers[0].level(1, "A").n_rows
    for which in (7, 8):
        ms, b = C.c_double(), C.c_double()
        _abi.check(L.irkdev_time_kernel(h, which, 5, C.byref(ms)))
        _abi.check(L.irkdev_last_timed_bytes(h, C.byref(b)))
        assert ms.value > 0.0
        # at least the operand and result vectors once
        assert b.value >= 8.0 * (n + nc)
    monkeypatch.setenv("IRK_COMPOSE", "0")
    r = heat_case(64, s=2, ht=0.01)
    ms = C.c_double()
    assert L.irkdev_time_kernel(r.device()._dev._h, 7, 1, C.byref(ms)) != 0
