import ctypes as C, os, sys
sys.path.insert(0, '/root/repo' if os.path.exists('/root/repo') else '.')
import paper_2010_11377_b200 as P
from paper_2010_11377_b200 import _abi
prob = P.make_heat_setup(1024); t = P.make_radau_iia(3)
Pc = P.BlockPreconditioner(prob.M, prob.F, P.precond_coeff(t, P.CoeffKind.LowerFactor), 1e-3, table=t)
L = _abi.lib()
for w in (32, 33, 34, 35):
    ms = C.c_double(); _abi.check(L.irkdev_time_kernel(Pc._dev._h, w, 50, C.byref(ms)))
    print(os.environ.get('IRK_TAIL_ROWS','-'), w, round(1e3*ms.value,1), 'us')
