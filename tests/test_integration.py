"""The reference-side adapter of INTEGRATION.md (integration/irk_step_b200.cpp)
is real code: it compiles against the reference's own headers, links with the
reference build and the B200 library, and -- through irkprec's API, beside the
reference's own irk_step on the same inputs -- reproduces its iteration count
and u_{n+1} (integration/demo.cpp).  Without a GPU it fails loudly."""
import subprocess
from pathlib import Path

import pytest

from conftest import has_gpu

ROOT = Path(__file__).resolve().parent.parent
DEMO = ROOT / "integration" / "_build" / "irk_b200_demo"


@pytest.mark.skipif(not Path("/root/reference/proj/include").exists(), reason="needs the reference headers")
def test_adapter_compiles_against_reference_headers():
    subprocess.run(["make", "-s", "-C", str(ROOT / "integration")], check=True)
    assert DEMO.exists()


@pytest.mark.skipif(has_gpu() or not DEMO.exists(), reason="checks the no-GPU failure path")
def test_adapter_fails_loudly_without_gpu():
    r = subprocess.run([str(DEMO), "32", "2"], capture_output=True, text=True, timeout=120)
    assert r.returncode != 0
    assert "no CUDA device" in r.stderr


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
@pytest.mark.skipif(not DEMO.exists(), reason="integration demo not built (needs /root/reference at build time)")
@pytest.mark.parametrize("cells,s,problem", [(128, 2, "heat"), (256, 3, "heat"), (64, 2, "dg"), (128, 4, "dg")])
def test_adapter_matches_reference_irk_step(cells, s, problem):
    r = subprocess.run([str(DEMO), str(cells), str(s), problem], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "device" in r.stdout and "reference" in r.stdout
