"""Repeatability stress of the device V-cycle (race hunt): REPS V-cycles of
one residual with the bottom kernel on and off and the step graph in between,
each compared with the C oracle bit for bit.  Prints the mismatch counts.

  python tools/vcycle_stress.py [cells] [reps]
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_2010_11377_b200 as P  # noqa: E402
from paper_2010_11377_b200 import _abi  # noqa: E402
from systems import heat_case  # noqa: E402

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
c = heat_case(cells, s=3, ht=1e-3)
dev = c.device()
r = np.random.default_rng(3).uniform(-1, 1, c.n)
want = c.oracle.vcycle(0, r)
u = c.problem.initial(0.01, 7)
sys_ = P.LinearParabolicSystem(c.M, c.K, c.f_lift)
for bottom in (1, 0, 1):
    _abi.check(_abi.lib().irk_set_option(b"IRK_BOTTOM", bottom))
    bad = 0
    for i in range(reps):
        z = dev.vcycle(0, r)
        if not np.array_equal(z, want):
            bad += 1
            if bad <= 3:
                d = np.abs(z - want)
                print(f"bottom={bottom} rep {i}: {np.count_nonzero(d)} entries differ, max {d.max():.3e}",
                      flush=True)
        if i % 10 == 9:
            P.irk_step(sys_, c.table, c.ht, 0.0, u, dev, P.GmresConfig(restart=50))
    print(f"bottom={bottom}: {bad}/{reps} V-cycles differ from the oracle", flush=True)
