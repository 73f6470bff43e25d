"""The reference's own test-suite on the CUDA line kernels.

oracle/build.py installs the reference package into oracle/_ref/site and
stages its tests in oracle/_ref/reftests; tests/ref_suite_plugin.py
registers the sm_100a kernels as the reference backend "cuda" and
activates it.  Every sweep of these tests then runs through
paper_1803_02143_b200.kernels (H2D -> kernel -> D2H), including
test_kernels_backends.py's bitwise strategy / worker-count contracts
parametrised over the new backend."""

from __future__ import annotations

import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

from oracle import build

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
# (suite, whether it sweeps: the poisson / grid suites never reach a line kernel)
SUITES = [("test_dg.py", True), ("test_spline.py", True), ("test_kernels_backends.py", True),
          ("test_driver.py", True), ("test_poisson.py", False), ("test_grid.py", False)]


@pytest.mark.parametrize("suite,sweeps", SUITES)
def test_reference_suite_on_cuda_backend(suite, sweeps):
    site, tests = build.ref_site_dir(), build.ref_tests_dir()
    assert (site / "slvp").exists() and (tests / suite).exists(), "python -m oracle.build"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(site), str(ROOT), str(ROOT / "tests"),
                                         env.get("PYTHONPATH", "")])
    env.pop("SLVP_BACKEND", None)
    proc = subprocess.run(
        [sys.executable, "-m", "pytest", "-q", "-p", "ref_suite_plugin", "-p", "no:cacheprovider",
         "--rootdir", str(tests), "-c", str(tests / "pytest.ini"), str(tests / suite)],
        cwd=str(tests), env=env, capture_output=True, text=True, timeout=1800)
    out = proc.stdout + proc.stderr
    print(out[-3000:])
    assert proc.returncode == 0, out[-3000:]
    calls = int(re.search(r"cuda backend calls: (\d+)", out).group(1))
    if sweeps:
        assert calls > 0, "no sweep reached the CUDA backend"
