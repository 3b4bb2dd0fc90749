"""One IRK step for profiling: setup and one warm step run outside the
profiled range; the second step is bracketed by cudaProfilerStart/Stop so
`ncu --profile-from-start off` sees exactly one step's launches.

  python tools/profile_step.py [cells s kind]     heat, Radau IIA (default C2)
  python tools/profile_step.py C1|C2|C3|C4        a BASELINE workload (bench.py)
"""
import ctypes as C
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np
import torch

import paper_2010_11377_b200 as P
from paper_2010_11377_b200 import _abi

kind = P.CoeffKind.LowerFactor
lift = None
if len(sys.argv) > 1 and sys.argv[1].startswith("C"):
    import bench
    bench.set_workload(sys.argv[1])
    prob, table, u0, lift = bench.make_problem(P)
    ht = bench.HT
else:
    cells = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    s = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    kind = P.CoeffKind(int(sys.argv[3])) if len(sys.argv) > 3 else kind
    prob = P.make_heat_setup(cells)
    table = P.make_radau_iia(s)
    u0 = prob.initial(0.01, 1)
    ht = 1e-3
Pc = P.BlockPreconditioner(prob.M, prob.F, P.precond_coeff(table, kind), ht, table=table)
cfg = P.GmresConfig(restart=50).c()
L = _abi.lib()
d_u = torch.from_numpy(u0).cuda()
d_un = torch.empty_like(d_u)
d_lift = torch.from_numpy(lift).cuda() if lift is not None else None
rep = _abi.irk_report()


def step():
    _abi.check(L.irkdev_step_device(Pc._dev._h, C.c_void_p(d_u.data_ptr()),
                                    C.c_void_p(d_lift.data_ptr()) if d_lift is not None else None,
                                    C.byref(cfg), C.c_void_p(d_un.data_ptr()), None, C.byref(rep)))


step()
torch.cuda.synchronize()
torch.cuda.profiler.start()
step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
first = rep.solve_seconds * 1e3
# IRK_AB_REPS=k: k more timed steps (same input) -> min / median for A/B runs
reps = int(__import__("os").environ.get("IRK_AB_REPS", "0"))
ts = [first]
for _ in range(reps):
    step()
    ts.append(rep.solve_seconds * 1e3)
ts.sort()
extra = f" min {ts[0]:.3f} med {ts[len(ts) // 2]:.3f}" if reps else ""
print("iterations", rep.iterations, "reorth", rep.n_reorth, "ms", first, extra)
