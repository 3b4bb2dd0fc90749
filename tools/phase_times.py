"""Warm per-phase device times at C2 (CUDA events on the solver stream, each
phase launched back to back `reps` times): stage operator, fine smoother,
preconditioner apply, full V-cycle, V-cycle below level 1 / 2 / 3."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2010_11377_b200 as P
from paper_2010_11377_b200 import _abi

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
prob = P.make_heat_setup(cells)
t = P.make_radau_iia(3)
Pc = P.BlockPreconditioner(prob.M, prob.F, P.precond_coeff(t, P.CoeffKind.LowerFactor), 1e-3, table=t)
L = _abi.lib()
names = {0: "stage operator", 1: "fine smoother SpMV", 2: "precond apply (3 V-cycles + 2 sweeps)",
         3: "V-cycle (hierarchy 0)", 4: "V-cycle below level 1", 5: "V-cycle below level 2",
         6: "V-cycle below level 3", 115: "GMRES block-dot j=15 (17 vectors)",
         20: "empty kernel, graph launch (per kernel)", 21: "empty kernel, stream launch (per kernel)",
         30: "graph: V-cycle (hot, repeated)", 31: "graph: V-cycle below level 1",
         32: "graph: V-cycle below level 2", 33: "graph: V-cycle below level 3",
         34: "graph: V-cycle below level 4", 35: "graph: coarse solve only",
         40: "graph: dense tail matvec (cycling hierarchies)"}
for w, name in names.items():
    ms = C.c_double()
    _abi.check(L.irkdev_time_kernel(Pc._dev._h, w, 50, C.byref(ms)))
    print(f"{name:40s} {1e3 * ms.value:9.1f} us")
