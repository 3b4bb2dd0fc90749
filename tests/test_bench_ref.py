"""The bench's reference arm runs the reference alone.

* ref_problem_initial (oracle/ref_harness.cpp, the project's u0 recipe on the
  reference mesh) equals the product's irk_problem_initial bit for bit, so both
  arms start from the same u0;
* `bench.py --impl reference` never imports the product package nor maps
  libirkdev.so: the timed region and its setup are the reference's own code.
"""
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2010_11377_b200 as P
from refs import Ref

ROOT = Path(__file__).resolve().parent.parent
needs_ref = pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("cells,noise,seed", [(16, 0.0, 0), (64, 0.01, 1), (257, 0.01, 7)])
def test_ref_initial_matches_product(cells, noise, seed):
    ours = P.make_heat_setup(cells).initial(noise, seed)
    ref = Ref.problem("heat", cells, initial=(noise, seed))["u0"]
    assert ours.shape == ref.shape
    assert np.array_equal(ours, ref)


@needs_ref
def test_reference_arm_is_reference_only():
    code = (
        "import sys, json; sys.argv=['bench.py']; import bench\n"
        "bench.set_workload('C1')\n"
        "t, its, st, w = bench.run_reference_steps(2, 1)\n"
        "maps = open('/proc/self/maps').read()\n"
        "print(json.dumps({'its': its, 'steps': st, 'pkg': 'paper_2010_11377_b200' in sys.modules,\n"
        "  'irkdev': 'libirkdev' in maps, 'irkref': 'libirkref' in maps}))\n")
    env = dict(os.environ, OMP_NUM_THREADS="2")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, check=True,
                         capture_output=True, text=True, timeout=300).stdout
    r = json.loads(out.strip().splitlines()[-1])
    assert r["steps"] == 2 and r["its"][0] == 19, r
    assert not r["pkg"] and not r["irkdev"] and r["irkref"], r
