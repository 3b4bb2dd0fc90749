"""BASELINE C5 on the device: 1024^2 heat, h_t = 1e-3, one step per cell,
{Radau IIA s = 2..7, Lobatto IIIC s = 2..5} x {J, GSL, DU, LD}, GMRES(50),
written in the reference study's CSV schema (study.cpp:334-360) to stdout.
(P~_GSL needs an external coefficient file the repository does not have.)

  python tools/c5_sweep.py [cells] > profiles/r1/c5_sweep.csv
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2010_11377_b200 as P  # noqa: E402

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
ht = 1e-3
prob = P.make_heat_setup(cells)
u0 = prob.initial(0.01, 1)
sys_ = P.LinearParabolicSystem(prob.M, prob.F, None)
cfg = P.GmresConfig(restart=50)
sys.stdout.write(P.csv_header())
for scheme, ss in ((P.Scheme.RadauIIA, range(2, 8)), (P.Scheme.LobattoIIIC, range(2, 6))):
    for s in ss:
        table = P.make_table(scheme, s)
        for kind in (P.CoeffKind.Jacobi, P.CoeffKind.GaussSeidelLower, P.CoeffKind.UpperFactor,
                     P.CoeffKind.LowerFactor):
            try:
                pc = P.BlockPreconditioner(prob.M, prob.F, P.precond_coeff(table, kind), ht,
                                           table=table)
                P.irk_step(sys_, table, ht, 0.0, u0, pc, cfg)  # warm (graph capture)
                r = P.irk_step(sys_, table, ht, 0.0, u0, pc, cfg)
                rep = r.report
                row = P.csv_row(table, cells, ht, prob.M.n_rows, kind, cfg, rep.iterations,
                                rep.true_rel_residual, float("nan"), rep.solve_seconds,
                                failed=not rep.converged)
                del pc
            except Exception as e:  # recorded as a failed cell, like the study driver
                print(f"# {scheme.name} s={s} {kind.name}: {e}", file=sys.stderr)
                row = P.csv_row(table, cells, ht, prob.M.n_rows, kind, cfg, 0, 0, 0, 0, failed=True)
            sys.stdout.write(row)
            sys.stdout.flush()
