"""Isolated timing of the DCGS2 block-dot at j=15 (17 vectors of sN) and of
the CGS block-dot for comparison; prints achieved GB/s."""
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
n = prob.M.n_rows
for which, name in ((115, "CGS block-dot j=15"), (615, "DCGS2 block-dot j=15")):
    ms = C.c_double()
    _abi.check(L.irkdev_time_kernel(Pc._dev._h, which, 50, C.byref(ms)))
    b = 17 * 8 * 3 * n
    print(f"{name}: {1e3 * ms.value:.1f} us, {b / ms.value / 1e6:.0f} GB/s")
