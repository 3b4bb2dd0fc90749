"""Full-size parity record for the BASELINE workloads (C2/C3/C4): one IRK step
of the device path against the C oracle (bit for bit) and against the
reference built from its own sources (iterations +-1, K and u_next <= 1e-9
relative L2).  Prints one JSON line per workload; the output is kept under
profiles/.  Test infrastructure: imports the checkers from tests/.

  python tools/fullsize_parity.py C4 C3
"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]

import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2010_11377_b200 as P  # noqa: E402
from refs import Ref, RefSolver  # noqa: E402
from systems import Case, rel_l2  # noqa: E402


def run(name, with_oracle=True):
    bench.set_workload(name)
    prob, table, u0, lift = bench.make_problem(P)
    coeff = P.precond_coeff(table, P.CoeffKind.LowerFactor)
    t0 = time.time()
    c = Case(prob.M, prob.F, table, coeff, bench.HT, f_lift=lift)
    setup = time.time() - t0
    sys_ = P.LinearParabolicSystem(prob.M, prob.F, lift)
    g = P.irk_step(sys_, table, bench.HT, 0.0, u0, c.device(), P.GmresConfig(restart=50),
                   want_K=True)
    out = {"workload": bench.WORKLOAD, "unknowns": int(g.K.size),
           "device": {"iterations": g.report.iterations, "cycles": g.report.cycles,
                      "true_rel": g.report.true_rel_residual,
                      "solve_seconds": g.report.solve_seconds},
           "host_setup_seconds": setup}
    if with_oracle:
        t0 = time.time()
        o = c.oracle.step(u0, lift, restart=50)
        out["oracle"] = {"iterations": o["iterations"], "seconds": time.time() - t0,
                         "K_bitwise": bool(np.array_equal(g.K, o["K"])),
                         "u_next_bitwise": bool(np.array_equal(g.u_next, o["u_next"])),
                         "history_bitwise": bool(np.array_equal(np.array(g.report.history),
                                                                o["history"]))}
    if Ref.available():
        M, K = prob.M, prob.F
        t0 = time.time()
        rs = RefSolver((M.row_ptr, M.col_idx, M.vals), (K.row_ptr, K.col_idx, K.vals),
                       bench.WL["scheme"], bench.S, 3, bench.HT)
        rsetup = time.time() - t0
        r = rs.step(u0, lift, restart=50)
        out["reference"] = {"iterations": r["iterations"], "solve_seconds": r["seconds"],
                            "setup_seconds": rsetup,
                            "iterations_within_1": abs(r["iterations"] - g.report.iterations) <= 1,
                            "rel_l2_K": rel_l2(g.K, r["K"]),
                            "rel_l2_u_next": rel_l2(g.u_next, r["u_next"])}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    for w in sys.argv[1:] or ["C4"]:
        run(w, with_oracle=True)
