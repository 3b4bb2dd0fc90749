"""Builds matching product / oracle / reference systems for parity tests."""
from __future__ import annotations

import numpy as np

import paper_2010_11377_b200 as P
from refs import OracleSystem, hierarchy_dict


def stage_blocks(M: P.CsrMatrix, K: P.CsrMatrix, ht: float, At: np.ndarray):
    """Distinct diagonal blocks M + ht*d*K (stage.cpp:85-106, csr_add fast path)."""
    s = At.shape[0]
    distinct, sob = [], []
    for j in range(s):
        d = At[j, j]
        if d not in distinct:
            distinct.append(d)
        sob.append(distinct.index(d))
    assert np.array_equal(M.row_ptr, K.row_ptr) and np.array_equal(M.col_idx, K.col_idx)
    blocks = [P.CsrMatrix(M.row_ptr.copy(), M.col_idx.copy(), 1.0 * M.vals + (ht * d) * K.vals,
                          M.n_cols) for d in distinct]
    return blocks, sob


class Case:
    """One IRK configuration: problem matrices, table, coefficients, hierarchies."""

    def __init__(self, M: P.CsrMatrix, K: P.CsrMatrix, table: P.ButcherTable,
                 coeff: P.PrecondCoeff, ht: float, amg: P.AmgParams | None = None,
                 f_lift=None):
        self.M, self.K, self.table, self.coeff, self.ht = M, K, table, coeff, ht
        self.amg = amg or P.AmgParams()
        self.f_lift = f_lift
        blocks, self.sob = stage_blocks(M, K, ht, coeff.Atilde)
        self.hiers = [P.amg_setup(B, self.amg) for B in blocks]
        self.oracle = OracleSystem(
            (M.row_ptr, M.col_idx, M.vals), (K.row_ptr, K.col_idx, K.vals), table.A, table.b, ht,
            coeff.Atilde, int(coeff.structure),
            [hierarchy_dict(h, self.amg.jacobi_weight, self.amg.pre_sweeps, self.amg.post_sweeps,
                            self.amg.smoother)
             for h in self.hiers], self.sob)
        self._P = None

    @property
    def n(self):
        return self.M.n_rows

    @property
    def s(self):
        return self.table.s

    def device(self) -> P.BlockPreconditioner:
        if self._P is None:
            self._P = P.BlockPreconditioner(self.M, self.K, self.coeff, self.ht, self.amg,
                                            table=self.table, hierarchies=self.hiers)
        return self._P


def heat_case(cells=64, scheme=P.Scheme.RadauIIA, s=2, kind=P.CoeffKind.LowerFactor, ht=0.01,
              amg=None):
    prob = P.make_heat_setup(cells)
    table = P.make_table(scheme, s)
    c = Case(prob.M, prob.F, table, P.precond_coeff(table, kind), ht, amg, prob.f_lift)
    c.problem = prob
    return c


def dg_case(cells=64, eps=0.005, s=2, kind=P.CoeffKind.LowerFactor, ht=0.01, amg=None):
    prob = P.make_double_glazing_setup(cells, eps)
    table = P.make_radau_iia(s)
    c = Case(prob.M, prob.F, table, P.precond_coeff(table, kind), ht, amg, prob.f_lift)
    c.problem = prob
    return c


def rel_l2(a, b):
    a, b = np.asarray(a), np.asarray(b)
    den = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (den if den > 0 else 1.0)


def custom_case(cells, s, upper=False, seed=None, scheme=P.Scheme.RadauIIA, ht=0.01, path=None):
    """Heat with a Custom preconditioner read from a coefficient file written
    like the reference's acceptance criterion 3 (acceptance.cpp:195-215)."""
    import os
    import tempfile
    At = seeded_triangular(s, 777 + s if seed is None else seed, upper=upper)
    prob = P.make_heat_setup(cells)
    table = P.make_table(scheme, s)
    with tempfile.TemporaryDirectory() as d:
        f = path or os.path.join(d, "coeff.txt")
        write_coeff(f, At)
        coeff = P.make_coeff(table, P.CoeffKind.Custom, f)
    c = Case(prob.M, prob.F, table, coeff, ht, None, prob.f_lift)
    c.problem = prob
    return c


def write_coeff(path, At, fmt="%.17g "):
    """A coefficient file as acceptance.cpp:195-215 writes it."""
    s = At.shape[0]
    with open(path, "w") as f:
        f.write(f"{s}\n")
        for i in range(s):
            f.write("".join(fmt % At[i, j] for j in range(s)) + "\n")


def seeded_triangular(s, seed, upper=False):
    """acceptance.cpp:201-211: diagonal U(0.3, 1.2), off-diagonal 0.4 U(0.3, 1.2)."""
    rng = np.random.default_rng(seed)
    At = np.zeros((s, s))
    for i in range(s):
        for j in range(s):
            if (j > i and not upper) or (j < i and upper):
                continue
            u = rng.uniform(0.3, 1.2)
            At[i, j] = u if i == j else 0.4 * u
    return At


def study_amg():
    """The reference study driver's subsolve cycle (study.hpp:44-47):
    Gauss-Seidel V(4,4) with two prolongator smoothing steps."""
    return P.AmgParams(pre_sweeps=4, post_sweeps=4, smoother=1, prolongation_steps=2)
