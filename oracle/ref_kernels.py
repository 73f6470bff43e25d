"""ORACLE -- TEST INFRASTRUCTURE ONLY.

Loader for the reference's own compiled line kernels built into
``oracle/_ref`` by ``oracle/build.py`` (entry points of
/root/reference/pkg/src/slvp/_kernels.pyx:126-279).  Used to pin the
oracle restatement bitwise and as the ``--impl reference`` CPU arm.
"""

from __future__ import annotations

import sys

from . import build

_mod = None


def load():
    """The reference kernel module, or None when it was not built."""
    global _mod
    if _mod is None:
        d = str(build.ref_module_dir())
        if d not in sys.path:
            sys.path.insert(0, d)
        try:
            import refkern._kernels as k  # type: ignore
        except ImportError:
            return None
        _mod = k
    return _mod


class RefKernels:
    """Adapter with the oracle's sweep-kernel interface (oracle.core.sweep)."""

    def __init__(self, block: int = 8):
        self.mod = load()
        if self.mod is None:
            raise RuntimeError("reference kernels not built (oracle/build.py)")
        self.block = block

    def dg(self, lines, idx, a, b, q, alpha, ncells, p, threads):
        from .core import host_threads

        return self.mod.dg_sweep_contig(lines, idx, a, b, q, alpha, ncells, p,
                                        threads or host_threads())

    def spline(self, lines, idx, table, h, threads):
        from .core import host_threads

        return self.mod.spline_sweep_contig(lines, idx, table, float(h), threads or host_threads())
