"""ORACLE -- TEST INFRASTRUCTURE ONLY.  Build recipe for the checkers.

* ``_build/liboracle.so``: the C restatement ``lines.c`` (gcc, OpenMP,
  -ffp-contract=off, like the reference's ``-O3 -fopenmp`` build without
  fast-math, /root/reference/pkg/setup.py:5-15).
* ``_ref/refkern/``: the reference's OWN compiled line kernels, cythonized
  from /root/reference/pkg/src/slvp/_kernels.pyx where it lies and compiled
  with the reference's flags.  The .pyx imports ``_factors`` from its sibling
  ``_kernels_py``; the generated shim supplies the oracle's restatement of
  it (pinned bitwise against the reference's factors by the golden tests).
  Nothing from /root/reference is copied: only build outputs land in _ref/.
"""

from __future__ import annotations

import subprocess
import sys
import sysconfig
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF_PYX = Path("/root/reference/pkg/src/slvp/_kernels.pyx")
GCC = "/usr/bin/gcc"


def build_oracle(force: bool = False) -> Path:
    out = HERE / "_build" / "liboracle.so"
    src = HERE / "lines.c"
    if not force and out.exists() and out.stat().st_mtime >= src.stat().st_mtime:
        return out
    out.parent.mkdir(exist_ok=True)
    subprocess.run([GCC, "-O3", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared", "-o",
                    str(out), str(src), "-lm"], check=True)
    return out


def ref_module_dir() -> Path:
    return HERE / "_ref"


def build_ref(force: bool = False) -> Path | None:
    """Compile the reference's Cython kernels into _ref/ (needs /root/reference)."""
    pkg = HERE / "_ref" / "refkern"
    suffix = sysconfig.get_config_var("EXT_SUFFIX")
    so = pkg / f"_kernels{suffix}"
    if not REF_PYX.exists():
        return so if so.exists() else None
    if not force and so.exists() and so.stat().st_mtime >= REF_PYX.stat().st_mtime:
        return so
    import numpy as np

    pkg.mkdir(parents=True, exist_ok=True)
    (pkg / "__init__.py").write_text("# build output of oracle/build.py (reference kernels)\n")
    (pkg / "_kernels_py.py").write_text(
        "# generated shim: the reference kernel module imports _factors from here\n"
        "from oracle.core import spline_factors as _factors  # noqa: F401\n"
    )
    csrc = pkg / "_kernels.c"
    subprocess.run([sys.executable, "-m", "cython", "-3", "--module-name", "refkern._kernels",
                    str(REF_PYX), "-o", str(csrc)], check=True)
    inc = sysconfig.get_paths()["include"]
    subprocess.run([GCC, "-O3", "-fopenmp", "-fPIC", "-shared",
                    "-DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION",
                    f"-I{inc}", f"-I{np.get_include()}", str(csrc), "-o", str(so)], check=True)
    return so


def build(force: bool = False) -> None:
    build_oracle(force)
    build_ref(force)


if __name__ == "__main__":
    build(force="--force" in sys.argv)
    print("ok")
