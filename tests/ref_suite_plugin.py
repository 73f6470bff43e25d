"""pytest plugin: register this package's CUDA line kernels as a
third backend ``"cuda"`` of the reference's plugin registry
(/root/reference/pkg/src/slvp/kernels.py:17-47) and make it the active one,
so the reference's OWN tests (test_dg.py, test_spline.py,
test_kernels_backends.py, ...) run their sweeps on the B200.

Used by tests/test_gpu_reference_suite.py:

    python -m pytest -p ref_suite_plugin oracle/_ref/reftests/test_dg.py ...

with oracle/_ref/site (the installed reference) and tests/ on PYTHONPATH.
The terminal summary reports how many line-kernel calls went to CUDA."""

from __future__ import annotations

import functools

CALLS = {"n": 0}


def _counted(fn):
    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        CALLS["n"] += 1
        return fn(*args, **kwargs)

    return staticmethod(wrapper)


def pytest_configure(config):
    import slvp.kernels as kr

    from paper_1803_02143_b200.kernels import _CudaBackend

    class Cuda:  # the reference's backend module interface (four entry points)
        spline_sweep_contig = _counted(_CudaBackend.spline_sweep_contig)
        spline_sweep_strided = _counted(_CudaBackend.spline_sweep_strided)
        dg_sweep_contig = _counted(_CudaBackend.dg_sweep_contig)
        dg_sweep_strided = _counted(_CudaBackend.dg_sweep_strided)

    kr._BACKENDS["cuda"] = Cuda
    kr.set_backend("cuda")


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    terminalreporter.write_line(f"cuda backend calls: {CALLS['n']}")
