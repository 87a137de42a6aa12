"""Build the in-tree CUDA library ``libsptrsv_b200.so`` for sm_100a.

Plain nvcc, one object per translation unit (compiled in parallel), linked
into a shared library next to this file so it travels with the repo snapshot
to the GPU box. No JIT cache, no torch extension machinery: the library is a
C ABI (include/sptrsv_b200.h) loaded with ctypes.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
BUILD = PKG.parent / "build" / "csrc"
LIB = PKG / "libsptrsv_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr"]


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False, defines: tuple[str, ...] = (), lib: Path | None = None,
          build_dir: Path | None = None) -> Path:
    """Compile and link; ``defines``/``lib``/``build_dir`` build a variant (tools/variants.sh)."""
    BUILD = build_dir or globals()["BUILD"]
    LIB = lib or globals()["LIB"]
    BUILD.mkdir(parents=True, exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.hpp")) + [PKG.parent / "include" / "sptrsv_b200.h"]
    objs = []
    jobs = []
    for src in sources():
        obj = BUILD / (src.stem + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + headers):
            cmd = [NVCC, *ARCH, *FLAGS, *defines, "-c", str(src), "-o", str(obj)]
            jobs.append(cmd)

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        return r

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        list(ex.map(run, jobs))
    if force or jobs or _stale(LIB, objs):
        run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(LIB), *map(str, objs)])
    return LIB


if __name__ == "__main__":
    # python -m paper_2012_06959_b200.build [--force] [--variant NAME -DX=Y ...]
    args = sys.argv[1:]
    if "--variant" in args:
        name = args[args.index("--variant") + 1]
        defs = tuple(a for a in args if a.startswith("-D"))
        print(build(verbose=True, force=True, defines=defs, lib=PKG / f"libsptrsv_b200_{name}.so",
                    build_dir=PKG.parent / "build" / f"csrc_{name}"))
    else:
        build(verbose=True, force="--force" in args)
        print(LIB)
