"""SHA-256 pins of the reference's integer structures (and values) at the
BASELINE sizes, generated from the reference itself.

Run in the build container (needs /root/reference and oracle/_ref):
    python tests/golden/make_fullsize_digests.py [C2 C4 C3]

For each BASELINE workload -- C2 heat 1024^2 Radau IIA s=3 h=1e-3, C4 double
glazing 1024^2 Radau IIA s=4 h=1e-2, C3 heat 2048^2 Lobatto IIIC s=5 h=1e-3,
all P_LD -- the reference's own assembly (fem.cpp:174-304 via
ref_problem_create) gives M, K, f_lift, and the reference's amg_setup
(amg.cpp:172-227) one hierarchy per distinct diagonal block M + h*Atilde_jj*K
(stage.cpp:85-106; csr_add's shared-pattern path, csr.cpp:147-186).  Stored
per array: the digest of the integer structure (row_ptr, col_idx) apart from
the digest of the values, so a failure says which one broke.  The aggregates
are pinned through P's pattern (P = (I - w D^-1 A) T, T's columns are the
aggregate ids).  Output: tests/golden/fullsize_digests.json (~60 KB of digests).
"""
import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))

from refs import Ref  # noqa: E402

# name: (problem, cells, scheme, s, coeff kind (3 = LD), ht)
WORKLOADS = {
    "C2": ("heat", 1024, 0, 3, 3, 1e-3),
    "C4": ("dg", 1024, 0, 4, 3, 1e-2),
    "C3": ("heat", 2048, 1, 5, 3, 1e-3),
}


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def csr_digests(csr) -> dict:
    rp, ci, v = csr
    return {"n": int(len(rp) - 1), "nnz": int(len(ci)), "int": sha(np.asarray(rp, np.int32),
                                                                np.asarray(ci, np.int32)),
            "val": sha(np.asarray(v, np.float64))}


def distinct_diagonals(At):
    d = []
    for j in range(At.shape[0]):
        if At[j, j] not in d:
            d.append(At[j, j])
    return d


def workload(name):
    kind, cells, scheme, s, ck, ht = WORKLOADS[name]
    t0 = time.time()
    prob = Ref.problem(kind, cells, 0.005)
    out = {"problem": kind, "cells": cells, "scheme": scheme, "s": s, "kind": ck, "ht": ht,
           "M": csr_digests(prob["M"]), "K": csr_digests(prob["K"]),
           "f_lift": sha(prob["f_lift"]), "hierarchies": []}
    At, _ = Ref.precond_coeff(scheme, s, ck)
    for d in distinct_diagonals(At):
        rp, ci, mv = prob["M"]
        B = (rp, ci, 1.0 * mv + (ht * d) * prob["K"][2])
        h = Ref.amg(B)
        levels = []
        for l in range(h.n_levels()):
            (a, _) = h.level(l, "A")
            lv = {"A": csr_digests(a), "inv_diag": sha(h.inv_diag(l))}
            if l + 1 < h.n_levels():
                (p, pc) = h.level(l, "P")
                (r, _) = h.level(l, "R")
                lv["P"] = csr_digests(p)
                lv["P"]["n_cols"] = int(pc)
                lv["R"] = csr_digests(r)
            levels.append(lv)
        out["hierarchies"].append({"d": float(d), "levels": levels})
        del h
    print(name, "levels", [[lv["A"]["n"] for lv in hh["levels"]] for hh in out["hierarchies"]],
          f"{time.time() - t0:.1f} s", flush=True)
    return out


def main(names):
    path = HERE / "fullsize_digests.json"
    data = json.loads(path.read_text()) if path.exists() else {}
    for n in names:
        data[n] = workload(n)
    path.write_text(json.dumps(data, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main(sys.argv[1:] or list(WORKLOADS))
