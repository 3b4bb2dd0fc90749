"""Same-process A/B of tuning switches (irk_set_option): one C2 solver, the
variants alternate ROUNDS times on identical memory placement; each variant
records its graph (one untimed step) and then times REPS steps.

  python tools/ab_inproc.py IRK_PDL_DGS=1,0 [NAME=a,b ...] [--rounds 6] [--reps 3]

Variants are the cartesian product of the listed values.  Prints, per
variant, the min and median step time over all timed steps."""
import argparse
import ctypes as C
import itertools
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2010_11377_b200 as P  # noqa: E402
from paper_2010_11377_b200 import _abi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("switches", nargs="*")
ap.add_argument("--construct", default=None,
                help="NAME=a,b: one solver per value (set before construction), alternated")
ap.add_argument("--rounds", type=int, default=6)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--cells", type=int, default=1024)
ap.add_argument("--s", type=int, default=3)
ap.add_argument("--dg", action="store_true", help="C4-style double glazing (u0 = 0, lift, h_t = 1e-2)")
args = ap.parse_args()
names, values = [], []
for sw in args.switches:
    k, v = sw.split("=")
    names.append(k)
    values.append([int(x) for x in v.split(",")])
L = _abi.lib()
prob = P.make_double_glazing_setup(args.cells, 0.005) if args.dg else P.make_heat_setup(args.cells)
table = P.make_radau_iia(args.s)
HT = 1e-2 if args.dg else 1e-3
solvers = {}
cname, cvals = None, [None]
if args.construct:
    cname, cv = args.construct.split("=")
    cvals = [int(x) for x in cv.split(",")]
for cvv in cvals:
    if cname:
        _abi.check(L.irk_set_option(cname.encode(), cvv))
    solvers[cvv] = P.BlockPreconditioner(prob.M, prob.F, P.precond_coeff(table, P.CoeffKind.LowerFactor),
                                         HT, table=table)
    solvers[cvv]._dev  # construct now
if cname:
    names.insert(0, cname)
    values.insert(0, cvals)
else:
    names.insert(0, "_")
    values.insert(0, [None])
variants = list(itertools.product(*values))
import numpy as np  # noqa: E402
u0 = np.zeros(prob.M.n_rows) if args.dg else prob.initial(0.01, 1)
d_u = torch.from_numpy(u0).cuda()
d_lift = torch.from_numpy(np.ascontiguousarray(prob.f_lift)).cuda() if args.dg else None
d_un = torch.empty_like(d_u)
cfg = P.GmresConfig(restart=50).c()
rep = _abi.irk_report()


def step(Pc):
    lift = C.c_void_p(d_lift.data_ptr()) if d_lift is not None else None
    _abi.check(L.irkdev_step_device(Pc._dev._h, C.c_void_p(d_u.data_ptr()), lift, C.byref(cfg),
                                    C.c_void_p(d_un.data_ptr()), None, C.byref(rep)))
    return rep.solve_seconds * 1e3, rep.iterations


times = {v: [] for v in variants}
its = {}
for r in range(args.rounds):
    for v in variants:
        for k, x in zip(names[1:], v[1:]):
            _abi.check(L.irk_set_option(k.encode(), x))
        Pc = solvers[v[0]]
        step(Pc)
        for _ in range(args.reps):
            t, it = step(Pc)
            times[v].append(t)
            its[v] = it
for v in variants:
    label = " ".join(f"{k}={x}" for k, x in zip(names, v) if k != "_")
    ts = times[v]
    print(f"{label:40s} iterations {its[v]}  min {min(ts):.3f}  med {statistics.median(ts):.3f} ms")
