"""BASELINE C5 on the device: 1024^2 heat, h_t = 1e-3, one step per cell,
{Radau IIA s = 2..7, Lobatto IIIC s = 2..5} x {J, GSL, DU, LD} (+ Custom,
the P~_GSL slot, when --custom-coeff DIR holds coeff_<scheme>_<s>.txt files in
the read_coeff_file format), GMRES(50), written in the reference study's CSV
schema (study.cpp:334-360) to stdout.

With --json FILE each cell also gets a JSON line: iterations, solve seconds,
solves/s and HBM GB/s -- the algorithmic bytes of the solve in the stored
formats (irkdev_model_bytes over the cell's actual GMRES cycles, bench.py
format_model_bytes) and SURVEY §8(d)'s CSR formula (survey_model_bytes), each
divided by the device-timed solve.

  python tools/c5_sweep.py [--cells N] [--json F] [--custom-coeff DIR] > c5.csv
"""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402  (byte models)
import paper_2010_11377_b200 as P  # noqa: E402
from paper_2010_11377_b200 import _abi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cells", type=int, default=1024)
ap.add_argument("--json", default=None)
ap.add_argument("--custom-coeff", default=None)
args = ap.parse_args()

cells, ht = args.cells, 1e-3
prob = P.make_heat_setup(cells)
u0 = prob.initial(0.01, 1)
sys_ = P.LinearParabolicSystem(prob.M, prob.F, None)
cfg = P.GmresConfig(restart=50)
L = _abi.lib()
jout = open(args.json, "w") if args.json else None
peak = bench.peaks().get("hbm_gbs", 6550.0)


def levels_of(dev, info):
    out = []
    for k in range(info["n_hier"]):
        lv = []
        for l in range(L.irkdev_num_levels(dev._h, k)):
            a, b_, c_, d_, f_ = (C.c_int() for _ in range(5))
            _abi.check(L.irkdev_level_info(dev._h, k, l, C.byref(a), C.byref(b_), C.byref(c_),
                                           C.byref(d_), C.byref(f_)))
            lv.append((a.value, b_.value, c_.value, d_.value))
        out.append(lv)
    return out


sys.stdout.write(P.csv_header())
kinds = [P.CoeffKind.Jacobi, P.CoeffKind.GaussSeidelLower, P.CoeffKind.UpperFactor,
         P.CoeffKind.LowerFactor]
if args.custom_coeff:
    kinds.append(P.CoeffKind.Custom)
for scheme, ss in ((P.Scheme.RadauIIA, range(2, 8)), (P.Scheme.LobattoIIIC, range(2, 6))):
    for s in ss:
        table = P.make_table(scheme, s)
        for kind in kinds:
            rec = {"scheme": scheme.name, "s": s, "kind": kind.name}
            try:
                path = None
                if kind == P.CoeffKind.Custom:
                    path = Path(args.custom_coeff) / f"coeff_{scheme.name}_{s}.txt"
                pc = P.BlockPreconditioner(prob.M, prob.F, P.make_coeff(table, kind, path), ht,
                                           table=table)
                P.irk_step(sys_, table, ht, 0.0, u0, pc, cfg)  # warm (graph capture)
                r = P.irk_step(sys_, table, ht, 0.0, u0, pc, cfg)
                rep = r.report
                row = P.csv_row(table, cells, ht, prob.M.n_rows, kind, cfg, rep.iterations,
                                rep.true_rel_residual, float("nan"), rep.solve_seconds,
                                failed=not rep.converged)
                dev = pc._dev
                info = dev.info()
                mb = (C.c_double * 8)()
                _abi.check(L.irkdev_model_bytes(dev._h, mb))
                fmt = bench.format_model_bytes(list(mb), rep.iterations)
                sv = bench.survey_model_bytes(info, levels_of(dev, info), rep.iterations,
                                              prob.M.n_rows, s, prob.M.nnz)
                sec = rep.solve_seconds
                rec.update(iterations=rep.iterations, converged=bool(rep.converged),
                           seconds=sec, solves_per_s=1.0 / sec,
                           hbm_gbs_stored_formats=fmt / sec / 1e9,
                           hbm_frac_stored_formats=fmt / sec / 1e9 / peak,
                           hbm_gbs_survey_model=sv / sec / 1e9,
                           bytes_stored_formats=fmt, bytes_survey_model=sv, peak_gbs=peak)
                del pc
            except Exception as e:  # recorded as a failed cell, like the study driver
                print(f"# {scheme.name} s={s} {kind.name}: {e}", file=sys.stderr)
                row = P.csv_row(table, cells, ht, prob.M.n_rows, kind, cfg, 0, 0, 0, 0, failed=True)
                rec["failed"] = str(e)
            sys.stdout.write(row)
            sys.stdout.flush()
            if jout:
                jout.write(json.dumps(rec) + "\n")
                jout.flush()
