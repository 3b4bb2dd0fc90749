"""Full-size C5 cells against the reference build on identical inputs:
1024^2 heat, h_t = 1e-3, one step, GMRES(50), the reference's own irk_step
through oracle/_ref (RefSolver), the device through the product API.  Prints
one JSON line per cell (iterations, K / u_next relative L2).  Test
infrastructure (imports the checkers from tests/).

  python tools/c5_ref_check.py radau:7:0 radau:7:3 lobatto:5:0 ...
  (scheme:s:kind, kind 0 J, 1 GSL, 2 DU, 3 LD)
"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]

import paper_2010_11377_b200 as P  # noqa: E402
from refs import RefSolver  # noqa: E402
from systems import rel_l2  # noqa: E402

cells, ht = 1024, 1e-3
prob = P.make_heat_setup(cells)
u0 = prob.initial(0.01, 1)
sys_ = P.LinearParabolicSystem(prob.M, prob.F, None)
M, K = prob.M, prob.F
for spec in sys.argv[1:]:
    sc, s, kind = spec.split(":")
    scheme = P.Scheme.RadauIIA if sc == "radau" else P.Scheme.LobattoIIIC
    s, kind = int(s), int(kind)
    table = P.make_table(scheme, s)
    pc = P.BlockPreconditioner(M, K, P.precond_coeff(table, P.CoeffKind(kind)), ht, table=table)
    g = P.irk_step(sys_, table, ht, 0.0, u0, pc, P.GmresConfig(restart=50), want_K=True)
    t0 = time.time()
    rs = RefSolver((M.row_ptr, M.col_idx, M.vals), (K.row_ptr, K.col_idx, K.vals), int(scheme), s, kind, ht)
    r = rs.step(u0, None, restart=50)
    print(json.dumps({"cell": spec, "device_iterations": g.report.iterations,
                      "reference_iterations": r["iterations"],
                      "rel_l2_K": rel_l2(g.K, r["K"]), "rel_l2_u_next": rel_l2(g.u_next, r["u_next"]),
                      "device_ms": 1e3 * g.report.solve_seconds, "reference_s": time.time() - t0}), flush=True)
    del pc
