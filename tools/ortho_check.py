"""One step of a BASELINE workload on the device: iterations, restart cycles
and the true relative residual for the orthogonalisation scheme selected by
IRK_ORTHO (dcgs2 default / cgs2).  python tools/ortho_check.py C3"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT)]
import bench  # noqa: E402
import paper_2010_11377_b200 as P  # noqa: E402

for name in sys.argv[1:] or ["C3"]:
    bench.set_workload(name)
    prob, table, u0, lift = bench.make_problem(P)
    Pc = P.BlockPreconditioner(prob.M, prob.F, P.precond_coeff(table, P.CoeffKind.LowerFactor),
                               bench.HT, table=table)
    sys_ = P.LinearParabolicSystem(prob.M, prob.F, lift)
    u = u0
    for step in range(2):
        r = P.irk_step(sys_, table, bench.HT, 0.0, u, Pc, P.GmresConfig(restart=50))
        rep = r.report
        print(f"{name} ortho={os.environ.get('IRK_ORTHO', 'dcgs2')} step {step}: iterations "
              f"{rep.iterations} cycles {rep.cycles} est {rep.final_rel_residual:.3e} "
              f"true {rep.true_rel_residual:.3e} ms {1e3 * rep.solve_seconds:.1f}", flush=True)
        u = r.u_next
