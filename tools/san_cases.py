"""Small device workloads for compute-sanitizer (tools/sanitize.sh): the C1
step (BASELINE configs[0]) in both graph modes with the programmatic launches
on, a V-cycle with the single-CTA bottom kernel, a DCGS2 cycle longer than
the restart default, and a Gauss-Seidel study-cycle step.  Each result is
checked against the oracle, so a run under a sanitizer also proves it did
not change the arithmetic."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import paper_2010_11377_b200 as P  # noqa: E402
from paper_2010_11377_b200 import _abi  # noqa: E402
from systems import heat_case, study_amg  # noqa: E402


def step(c, u, cfg=None):
    sys_ = P.LinearParabolicSystem(c.M, c.K, c.f_lift)
    return P.irk_step(sys_, c.table, c.ht, 0.0, u, c.device(), cfg or P.GmresConfig(), want_K=True)


c = heat_case(64, s=2, ht=0.01)
u = c.problem.initial()
o = c.oracle.step(u, c.f_lift)
for mode in (0, 1):
    _abi.check(_abi.lib().irk_set_option(b"IRK_NO_COND_GRAPH", mode))
    r = step(c, u)
    assert r.report.iterations == o["iterations"] and np.array_equal(r.K, o["K"]), mode
    print(f"C1 step (host-driven={mode}): {r.report.iterations} iterations, bit-identical")
_abi.check(_abi.lib().irk_set_option(b"IRK_NO_COND_GRAPH", 0))
c3 = heat_case(128, s=3, ht=1e-3)
rv = np.random.default_rng(1).uniform(-1, 1, c3.n)
assert np.array_equal(c3.device().vcycle(0, rv), c3.oracle.vcycle(0, rv))
print("V-cycle 128^2 (bottom kernel): bit-identical")
r = step(c3, c3.problem.initial(0.01, 2), P.GmresConfig(restart=0, rel_tol=1e-13, max_iter=80))
o3 = c3.oracle.step(c3.problem.initial(0.01, 2), c3.f_lift, rtol=1e-13, restart=0, max_iter=80)
assert r.report.iterations == o3["iterations"] and np.array_equal(r.K, o3["K"])
print(f"long DCGS2 cycle: {r.report.iterations} iterations, bit-identical")
g = heat_case(64, s=2, ht=0.01, amg=study_amg())
og = g.oracle.step(u, g.f_lift)
rg = step(g, u)
assert rg.report.iterations == og["iterations"] and np.array_equal(rg.K, og["K"])
print(f"Gauss-Seidel V(4,4) step: {rg.report.iterations} iterations, bit-identical")
