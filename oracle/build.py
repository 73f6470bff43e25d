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
* ``_ref/site/slvp``: the WHOLE reference package, installed with the
  base contract's own command (``pip install --no-index --no-build-isolation
  --no-deps --target``) from a scratch copy under /tmp (its build writes
  into the source tree, /root/reference is read-only).  This is the
  unmodified reference (``slvp.strang_step``, its compiled ``_kernels``);
  the reference CPU arm of bench.py and the full-size GPU parity tests run
  it on the GPU box's host cores.
* ``_ref/reftests``: the reference's own test-suite, staged next to the
  install so ``tests/test_gpu_reference_suite.py`` can run it with the CUDA
  line kernels registered as the reference backend ``"cuda"``.
  Both are git-ignored build outputs that travel to the GPU box.
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


REF_PKG = Path("/root/reference/pkg")


def ref_site_dir() -> Path:
    return HERE / "_ref" / "site"


def ref_tests_dir() -> Path:
    return HERE / "_ref" / "reftests"


def build_ref_pkg(force: bool = False) -> Path | None:
    """pip-install the reference package into _ref/site (needs /root/reference)."""
    import shutil
    import tempfile

    site = ref_site_dir()
    so = list((site / "slvp").glob("_kernels*.so")) if (site / "slvp").exists() else []
    if not REF_PKG.exists():
        return site if so else None
    if so and not force:
        return site
    scratch = Path(tempfile.mkdtemp(prefix="slvp_pkg_"))
    try:
        for name in ("src", "setup.py", "pyproject.toml", "README.md"):
            src = REF_PKG / name
            (shutil.copytree if src.is_dir() else shutil.copy)(src, scratch / name)
        if site.exists():
            shutil.rmtree(site)
        env = dict(__import__("os").environ, CC=GCC, LDSHARED=f"{GCC} -shared")
        subprocess.run([sys.executable, "-m", "pip", "install", "--no-index",
                        "--no-build-isolation", "--no-deps", "--find-links", "/opt/wheelhouse",
                        "--target", str(site), str(scratch)], check=True, env=env,
                       stdout=subprocess.DEVNULL)
    finally:
        shutil.rmtree(scratch, ignore_errors=True)
    tests = ref_tests_dir()
    if tests.exists():
        shutil.rmtree(tests)
    shutil.copytree(REF_PKG / "tests", tests)
    # the reference's pytest settings (pkg/pyproject.toml [tool.pytest.ini_options])
    (tests / "pytest.ini").write_text(
        "[pytest]\nmarkers =\n    slow: long-running end-to-end runs\n")
    return site


def load_ref_pkg():
    """Import the installed reference package ``slvp`` (None when not built)."""
    site = ref_site_dir()
    if not list((site / "slvp").glob("_kernels*.so")):
        return None
    if str(site) not in sys.path:
        sys.path.insert(0, str(site))
    import slvp  # type: ignore

    return slvp


def build(force: bool = False) -> None:
    build_oracle(force)
    build_ref(force)
    build_ref_pkg(force)


if __name__ == "__main__":
    build(force="--force" in sys.argv)
    print("ok")
