"""Alternate device execution modes stay bit-identical to the oracle.

The switches are read once per process, so each mode runs in a subprocess:
  * IRK_NO_COND_GRAPH=1 -- host-driven GMRES loop (the mode ncu profiles);
  * IRK_ORTHO=cgs2      -- CGS with the reference's conditional second pass
                           (oracle scheme 0) instead of delayed CGS2;
  * IRK_NO_VALUE_CODES=1, IRK_SPARSE_FMT=0/2 -- fp64 values, all-SELL /
                           all-CSR-vector sparse formats;
  * IRK_PDL=1           -- programmatic dependent launch for every kernel;
  * IRK_PDL_COARSE=-1/0 -- programmatic launches on no / every AMG level
                           (default: levels >= 2);
  * IRK_SERIAL_JACOBI=1 -- block-Jacobi V-cycles in stage order on one stream
                           instead of one graph branch per hierarchy;
  * IRK_CODES_MIN_ROWS=0 -- value dictionaries on every operator (the
                           full-size defaults use them at level 0 only), read
                           through L1 (default) or staged in shared memory
                           (IRK_U8_TAB_SMEM=1).
"""
import os
import subprocess
import sys
from pathlib import Path

import pytest

from conftest import has_gpu

ROOT = Path(__file__).resolve().parent.parent
pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import paper_2010_11377_b200 as P
from systems import heat_case
from refs import oracle_ortho
oracle_ortho({ortho!r})
for s, restart, kind in ((2, 50, 3), (3, 5, 3), (3, 50, 0), (5, 8, 0)):
    c = heat_case(48, s=s, ht=0.01, kind=P.CoeffKind(kind))
    u = c.problem.initial(0.01, 7)
    r = P.irk_step(P.LinearParabolicSystem(c.M, c.K, c.f_lift), c.table, c.ht, 0.0, u, c.device(),
                   P.GmresConfig(restart=restart), want_K=True)
    o = c.oracle.step(u, c.f_lift, restart=restart)
    assert r.report.iterations == o["iterations"], (r.report.iterations, o["iterations"])
    assert np.array_equal(r.K, o["K"]) and np.array_equal(r.u_next, o["u_next"])
print("MODE-OK")
"""


@pytest.mark.parametrize("env,ortho", [
    ({"IRK_NO_COND_GRAPH": "1"}, "dcgs2"),
    ({"IRK_ORTHO": "cgs2"}, "cgs2"),
    ({"IRK_ORTHO": "cgs2", "IRK_NO_COND_GRAPH": "1"}, "cgs2"),
    ({"IRK_NO_VALUE_CODES": "1"}, "dcgs2"),
    ({"IRK_SPARSE_FMT": "0"}, "dcgs2"),
    ({"IRK_SPARSE_FMT": "2"}, "dcgs2"),
    ({"IRK_PDL": "1"}, "dcgs2"),
    ({"IRK_PDL_COARSE": "-1"}, "dcgs2"),
    ({"IRK_PDL_COARSE": "0"}, "dcgs2"),
    ({"IRK_SERIAL_JACOBI": "1"}, "dcgs2"),
    ({"IRK_CODES_MIN_ROWS": "0"}, "dcgs2"),
    ({"IRK_CODES_MIN_ROWS": "0", "IRK_U8_TAB_SMEM": "1"}, "dcgs2"),
])
def test_mode_bitwise(env, ortho):
    code = SCRIPT.format(root=str(ROOT), tests=str(ROOT / "tests"), ortho=ortho)
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "MODE-OK" in r.stdout, r.stdout + r.stderr
