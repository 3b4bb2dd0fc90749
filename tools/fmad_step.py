"""One process of the --fmad A/B (tools/fmad_ab.sh): `steps` C2 steps with the
library IRK_LIB points at; saves iterations, K and u_next of every step to
an .npz and prints the device ms per step."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2010_11377_b200 as P  # noqa: E402

out, steps = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 4
prob = P.make_heat_setup(1024)
t = P.make_radau_iia(3)
pc = P.BlockPreconditioner(prob.M, prob.F, P.precond_coeff(t, P.CoeffKind.LowerFactor), 1e-3, table=t)
sys_ = P.LinearParabolicSystem(prob.M, prob.F, None)
u = prob.initial(0.01, 1)
cfg = P.GmresConfig(restart=50)
P.irk_step(sys_, t, 1e-3, 0.0, u, pc, cfg)  # warm-up
rec = {}
for k in range(steps):
    r = P.irk_step(sys_, t, 1e-3, 0.0, u, pc, cfg, want_K=True)
    rec[f"it{k}"] = r.report.iterations
    rec[f"ms{k}"] = 1e3 * r.report.solve_seconds
    rec[f"K{k}"] = r.K
    rec[f"u{k}"] = r.u_next
    u = r.u_next
np.savez(out, **rec)
print(out, [rec[f"it{k}"] for k in range(steps)], [round(rec[f"ms{k}"], 3) for k in range(steps)])
