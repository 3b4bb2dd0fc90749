"""Bit-exact pins of the integer structures at the BASELINE sizes.

north_star: "AMG hierarchy sparsity and integer index structures are
bit-exact".  tests/golden/fullsize_digests.json holds SHA-256 digests of the
REFERENCE's own assembly (fem.cpp) and amg_setup (amg.cpp:172-227) output at
C2 (heat 1024^2, 3 hierarchies), C4 (double glazing 1024^2, 4) and C3 (heat
2048^2, 5), made by tests/golden/make_fullsize_digests.py -- integer
structure (row_ptr, col_idx) and values digested separately.  Checked here:

* (CPU) the product's host assembly and host amg_setup on the same blocks;
* (GPU) the hierarchies the device solver builds itself (irkdev_create's
  default device setup, amg_device.cu), fetched back with irkdev_hierarchy.

Neither needs /root/reference at run time.
"""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2010_11377_b200 as P
from conftest import has_gpu

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "fullsize_digests.json").read_text())
NAMES = ["C2", "C4", "C3"]


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def check_csr(A: P.CsrMatrix, g: dict, what: str):
    assert (A.n_rows, A.nnz) == (g["n"], g["nnz"]), what
    assert sha(A.row_ptr.astype(np.int32), A.col_idx.astype(np.int32)) == g["int"], f"{what}: index structure"
    assert sha(A.vals.astype(np.float64)) == g["val"], f"{what}: values"


def check_hierarchy(h: P.AmgHierarchy, g: dict, what: str):
    lv = g["levels"]
    assert h.sizes() == [x["A"]["n"] for x in lv], what
    for l, x in enumerate(lv):
        check_csr(h.level(l, "A"), x["A"], f"{what} level {l} A")
        assert sha(h.inv_diag(l)) == x["inv_diag"], f"{what} level {l} inv_diag"
        if "P" in x:
            Pl = h.level(l, "P")
            assert Pl.n_cols == x["P"]["n_cols"], f"{what} level {l}: aggregate count"
            check_csr(Pl, x["P"], f"{what} level {l} P (aggregates)")
            check_csr(h.level(l, "R"), x["R"], f"{what} level {l} R")


def problem(g):
    if g["problem"] == "heat":
        return P.make_heat_setup(g["cells"])
    return P.make_double_glazing_setup(g["cells"], 0.005)


def blocks(pr, g):
    table = P.make_table(P.Scheme(g["scheme"]), g["s"])
    coeff = P.precond_coeff(table, P.CoeffKind(g["kind"]))
    d = []
    for j in range(g["s"]):
        if coeff.Atilde[j, j] not in d:
            d.append(coeff.Atilde[j, j])
    assert d == [h["d"] for h in g["hierarchies"]]
    return table, coeff, d


@pytest.mark.parametrize("name", NAMES)
def test_host_setup_matches_reference_digests(name):
    g = GOLD[name]
    pr = problem(g)
    check_csr(pr.M, g["M"], f"{name} M")
    check_csr(pr.F, g["K"], f"{name} K")
    assert sha(pr.f_lift) == g["f_lift"]
    _, _, ds = blocks(pr, g)
    for k, d in enumerate(ds):
        B = P.CsrMatrix(pr.M.row_ptr, pr.M.col_idx, 1.0 * pr.M.vals + (g["ht"] * d) * pr.F.vals, pr.M.n_cols)
        check_hierarchy(P.amg_setup(B), g["hierarchies"][k], f"{name} host hierarchy {k}")


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
@pytest.mark.parametrize("name", NAMES)
def test_device_solver_hierarchies_match_reference_digests(name):
    g = GOLD[name]
    pr = problem(g)
    table, coeff, ds = blocks(pr, g)
    dev = P.BlockPreconditioner(pr.M, pr.F, coeff, g["ht"], table=table)
    assert dev.distinct_subsolvers() == len(ds)
    for k in range(len(ds)):
        check_hierarchy(dev.hierarchy(k), g["hierarchies"][k], f"{name} device hierarchy {k}")
