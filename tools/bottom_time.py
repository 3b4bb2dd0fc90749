"""Bottom-kernel timing: back to back (50) and alternating with a level-1
smoother launch (51), plus the smoother alone (time_kernel 1 is the fine one;
here the difference 51 - 50 estimates the smoother + carveout switch)."""
import ctypes as C
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2010_11377_b200 as P
from paper_2010_11377_b200 import _abi
prob = P.make_heat_setup(1024)
t = P.make_radau_iia(3)
Pc = P.BlockPreconditioner(prob.M, prob.F, P.precond_coeff(t, P.CoeffKind.LowerFactor), 1e-3, table=t)
L = _abi.lib()
for which, name in ((50, "bottom back to back"), (51, "bottom + level-1 smoother")):
    ms = C.c_double()
    _abi.check(L.irkdev_time_kernel(Pc._dev._h, which, 200, C.byref(ms)))
    print(f"{name}: {1e3 * ms.value:.2f} us per pair/launch")
