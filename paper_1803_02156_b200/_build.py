"""In-tree build of libchebfd_b200.so (sm_100a) and of the CPU checker libraries.

The product library is compiled with nvcc for ``-gencode arch=compute_100a,code=sm_100a``
only (no other architectures, no JIT fallback) and lands next to this file so it
travels with the repository snapshot to the GPU box.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libchebfd_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _sources():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp")) + sorted(CSRC.glob("*.hpp")) + [
        ROOT / "include" / "chebfd_b200.h"
    ]


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _run(cmd, cwd=None):
    r = subprocess.run(cmd, cwd=cwd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {' '.join(map(str, cmd))}")
    return r


def build_library(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale(LIB, _sources()):
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    bdir = PKG / "build"
    bdir.mkdir(exist_ok=True)
    headers = sorted(CSRC.glob("*.hpp")) + [ROOT / "include" / "chebfd_b200.h"]
    jobs = []
    for cu in sorted(CSRC.glob("*.cu")):
        jobs.append((cu, bdir / (cu.stem + ".o"), [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler",
                                                   "-fPIC", "-Xptxas", "-v", "-c", str(cu)]))
    for cpp in sorted(CSRC.glob("*.cpp")):
        jobs.append((cpp, bdir / (cpp.stem + ".o"), ["g++", "-O3", "-std=c++17", "-fPIC", "-pthread", "-Wall", "-c",
                                                     str(cpp)]))
    # an object is rebuilt when its source or any shared header is newer
    todo = [(cmd + ["-o", str(o)]) for src, o, cmd in jobs if force or _stale(o, [src, *headers])]
    with ThreadPoolExecutor(max(1, min(len(todo), os.cpu_count() or 1))) as ex:
        list(ex.map(_run, todo))
    objs = [o for _, o, _ in jobs]
    tmp = LIB.with_suffix(".so.tmp")
    _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs), "-lpthread"])
    os.replace(tmp, LIB)
    if verbose:
        print(f"built {LIB}")
    return LIB


def build_oracle(with_ref: bool = True) -> None:
    """CPU checker (test infrastructure only): oracle/liboracle.so and, where the
    reference tree is present, oracle/_ref/libchebref.so."""
    odir = ROOT / "oracle"
    _run(["make", "-s", "-C", str(odir), "liboracle.so"])
    if with_ref and Path("/root/reference/proj/include/chebfilter").is_dir():
        _run(["make", "-s", "-C", str(odir), "ref"])


if __name__ == "__main__":
    build_library(force="--force" in sys.argv, verbose=True)
    build_oracle()
