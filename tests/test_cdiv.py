"""Host check of the lean kernel's division by a per-simulation constant (sim_kernel.cuh `cdiv`): RN(a y) with
y = RN(1/b) and two FMA-residual corrections must equal IEEE a / b bit for bit (the batch-latency terms of Eq. (3),
PAPER.md:1727, divide by flops, bw, tp and link_bw).  tools/check_cdiv.c is the same five-operation
sequence in C (libm fma, no contraction) over the cost models' divisors and random ones."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("gcc") is None, reason="needs gcc")
def test_cdiv_matches_ieee_division(tmp_path):
    exe = tmp_path / "check_cdiv"
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-o", str(exe), os.path.join(ROOT, "tools", "check_cdiv.c"), "-lm"],
                   check=True)
    r = subprocess.run([str(exe), "300000"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().startswith("0 of 19200000"), r.stdout
