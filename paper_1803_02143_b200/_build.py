"""In-tree build of the CUDA C-ABI library ``libvpb200.so`` (sm_100a).

The library is compiled with nvcc directly (no torch extension machinery):
the product boundary is a plain C ABI loaded with ctypes, so the shared
object must not depend on torch.  Host code is compiled with
``-ffp-contract=off`` so the host-side constant tables (spline factors,
Gauss rules) round exactly like the reference's NumPy code.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libvpb200.so"
SOURCES = ["common.cu", "dg.cu", "fused.cu", "fused2.cu", "xcomp.cu", "spline.cu", "field.cu", "halo.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# fused2.cu instantiates 18 large kernels (the "exact" merged x pass): let
# nvcc compile them in parallel (258 s -> ~95 s; only register numbering in
# the SASS changes)
EXTRA = {"fused2.cu": ["-split-compile=0"]}


def nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "vpb200.h"]
    if not force and not _stale(LIB, deps):
        return LIB
    objdir = ROOT / "build" / "obj"
    objdir.mkdir(parents=True, exist_ok=True)
    objs = []
    procs = []
    headers = list(CSRC.glob("*.cuh")) + [ROOT / "include" / "vpb200.h", Path(__file__)]
    for s in SOURCES:
        obj = objdir / (Path(s).stem + ".o")
        objs.append(obj)
        if not force and not _stale(obj, [CSRC / s, *headers]):
            continue  # object newer than its source and every header
        cmd = [
            nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17",
            "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
            "-I", str(ROOT / "include"),
            *EXTRA.get(s, []), "-c", str(CSRC / s), "-o", str(obj),
        ]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    failed = []
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            failed.append((cmd, out.decode(errors="replace")))
        elif verbose and out:
            sys.stdout.write(out.decode(errors="replace"))
    if failed:
        msg = "\n".join(" ".join(c) + "\n" + o for c, o in failed)
        raise RuntimeError(f"nvcc failed:\n{msg}")
    tmp = LIB.with_suffix(".so.tmp")
    link = [nvcc(), *ARCH, "-shared", "-cudart=static", "-o", str(tmp), *map(str, objs)]
    subprocess.run(link, check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
