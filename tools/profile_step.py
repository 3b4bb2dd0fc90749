"""One C2 IRK step for profiling: setup and one warm step run outside the
profiled range; the second step is bracketed by cudaProfilerStart/Stop so
`ncu --profile-from-start off` sees exactly one step's launches."""
import ctypes as C
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np
import torch

import paper_2010_11377_b200 as P
from paper_2010_11377_b200 import _abi

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
s = int(sys.argv[2]) if len(sys.argv) > 2 else 3
kind = P.CoeffKind(int(sys.argv[3])) if len(sys.argv) > 3 else P.CoeffKind.LowerFactor
prob = P.make_heat_setup(cells)
table = P.make_radau_iia(s)
Pc = P.BlockPreconditioner(prob.M, prob.F, P.precond_coeff(table, kind), 1e-3,
                           table=table)
u0 = prob.initial(0.01, 1)
cfg = P.GmresConfig(restart=50).c()
L = _abi.lib()
d_u = torch.from_numpy(u0).cuda()
d_un = torch.empty_like(d_u)
rep = _abi.irk_report()


def step():
    _abi.check(L.irkdev_step_device(Pc._dev._h, C.c_void_p(d_u.data_ptr()), None, C.byref(cfg),
                                    C.c_void_p(d_un.data_ptr()), None, C.byref(rep)))


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
