"""Isolated launch times of the fine-level kernels (time_kernel hooks 0-3) for
the environment's variant."""
import ctypes as C
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2010_11377_b200 as P
from paper_2010_11377_b200 import _abi

prob = P.make_heat_setup(1024)
t = P.make_radau_iia(3)
Pc = P.BlockPreconditioner(prob.M, prob.F, P.precond_coeff(t, P.CoeffKind.LowerFactor), 1e-3, table=t)
L = _abi.lib()
tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("IRK_")) or "default"
out = []
for which, name in ((0, "stage op"), (1, "fine smoother"), (2, "precond"), (3, "V-cycle"),
                    (4, "V-cycle below L0"), (5, "below L1")):
    ms = C.c_double()
    _abi.check(L.irkdev_time_kernel(Pc._dev._h, which, 100, C.byref(ms)))
    out.append(f"{name} {1e3 * ms.value:.1f}us")
print(tag + ": " + ", ".join(out))
