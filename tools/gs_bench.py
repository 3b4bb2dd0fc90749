"""The reference study driver's subsolve cycle at BASELINE size: heat 1024^2,
Radau IIA s=3, h_t=1e-3, P_LD, AMG Gauss-Seidel V(4,4) with two prolongator
smoothing steps (study.hpp:44-47), GMRES(50).  Device steps (one warm-up,
then --steps timed, device events) and, with --ref, one step of the
reference build (oracle/_ref) on the same inputs with its iteration count and
relative differences.  Prints one JSON line.

  python tools/gs_bench.py [--cells N] [--steps K] [--ref]
"""
import argparse
import ctypes as C
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import paper_2010_11377_b200 as P  # noqa: E402
from paper_2010_11377_b200 import _abi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cells", type=int, default=1024)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--ref", action="store_true")
ap.add_argument("--pre", type=int, default=4)
ap.add_argument("--post", type=int, default=4)
ap.add_argument("--psteps", type=int, default=2)
args = ap.parse_args()

amg = P.AmgParams(pre_sweeps=args.pre, post_sweeps=args.post, smoother=1,
                  prolongation_steps=args.psteps)
prob = P.make_heat_setup(args.cells)
t = P.make_radau_iia(3)
coeff = P.precond_coeff(t, P.CoeffKind.LowerFactor)
t0 = time.time()
pc = P.BlockPreconditioner(prob.M, prob.F, coeff, 1e-3, amg, table=t)
setup = time.time() - t0
u = prob.initial(0.01, 1)
sys_ = P.LinearParabolicSystem(prob.M, prob.F, None)
cfg = P.GmresConfig(restart=50)
P.irk_step(sys_, t, 1e-3, 0.0, u, pc, cfg)  # warm-up (graph capture)
its, secs = [], []
uu = u
for _ in range(args.steps):
    r = P.irk_step(sys_, t, 1e-3, 0.0, uu, pc, cfg, want_K=True)
    its.append(r.report.iterations)
    secs.append(r.report.solve_seconds)
    first = first if _ else r
    uu = r.u_next
L = _abi.lib()
vc = C.c_double()
_abi.check(L.irkdev_time_kernel(pc._dev._h, 3, 5, C.byref(vc)))
sweeps = {}
for l in range(3):
    for back in (0, 1):
        ms = C.c_double()
        if L.irkdev_time_kernel(pc._dev._h, 60 + 2 * l + back, 5, C.byref(ms)) == 0:
            sweeps[f"L{l}_{'bwd' if back else 'fwd'}_ms"] = ms.value
h0 = pc.hierarchy(0)
out = {"workload": f"heat {args.cells}^2, Radau IIA s=3, h_t=1e-3, P_LD, AMG GS V({args.pre},{args.post}) "
                   f"x{args.psteps} prolongator steps, GMRES(50) rtol 1e-8",
       "levels": h0.sizes(), "tail_from": h0.tail()[0], "iterations": its,
       "ms_per_step": [1e3 * s for s in secs], "solves_per_s": len(secs) / sum(secs),
       "ms_per_vcycle": vc.value, "sweep_ms": sweeps, "setup_s": setup}
if args.ref:
    from refs import RefSolver
    from systems import rel_l2
    M, K = prob.M, prob.F
    rs = RefSolver((M.row_ptr, M.col_idx, M.vals), (K.row_ptr, K.col_idx, K.vals), 0, 3, 3, 1e-3,
                   amg=amg)
    rr = rs.step(u, None)
    out["reference"] = {"iterations": rr["iterations"], "seconds": rr["seconds"],
                        "rel_K": rel_l2(first.K, rr["K"]),
                        "rel_u_next": rel_l2(first.u_next, rr["u_next"])}
print(json.dumps(out))
