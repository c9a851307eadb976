"""Build libbamg_sm100.so in-tree with nvcc for sm_100a.

`python -m paper_1402_4005_b200.build` (or `__graft_entry__.build()`) compiles
every `csrc/*.cu` to an object with
`-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo` and links them into
`paper_1402_4005_b200/libbamg_sm100.so` (static CUDA runtime, so the library
does not depend on the runtime version torch ships).  Rebuilds only what
changed.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
BUILD = PKG / "_build"
LIB = PKG / "libbamg_sm100.so"
INCLUDE = PKG.parent / "include"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
              "--expt-relaxed-constexpr", "-Xptxas", "-O3"] + ARCH


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build libbamg_sm100.so")


def _headers_mtime() -> float:
    hs = list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))
    return max((h.stat().st_mtime for h in hs), default=0.0)


def _compile(src: Path, verbose: bool, bdir: Path = BUILD, extra=()) -> Path:
    obj = bdir / (src.stem + ".o")
    if obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, _headers_mtime()):
        return obj
    cmd = [nvcc(), "-c", str(src), "-o", str(obj), "-I", str(INCLUDE)] + NVCC_FLAGS + list(extra)
    if verbose:
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src.name}:\n{res.stdout}\n{res.stderr}")
    return obj


def build(verbose: bool = False, force: bool = False, variant: str = "", defines=()) -> Path:
    """Build the library; `variant`/`defines` build a tuning variant
    (`_build_<variant>/`, `libbamg_sm100_<variant>.so`, extra -D flags) that
    BAMG_LIB_PATH can select."""
    bdir = BUILD if not variant else PKG / f"_build_{variant}"
    lib = LIB if not variant else PKG / f"libbamg_sm100_{variant}.so"
    extra = [f"-D{d}" for d in defines]
    bdir.mkdir(exist_ok=True)
    if force:
        for o in bdir.glob("*.o"):
            o.unlink()
    sources = sorted(CSRC.glob("*.cu"))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, bdir, extra), sources))
    newest = max(o.stat().st_mtime for o in objs)
    if lib.exists() and lib.stat().st_mtime >= newest and not force:
        return lib
    tmp = lib.with_suffix(".so.tmp")
    cmd = [nvcc(), "-shared", "-o", str(tmp)] + [str(o) for o in objs] + ARCH + [
        "-lcudart_static", "-Xlinker", "-rpath=/usr/local/cuda/lib64"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, lib)
    if verbose:
        print(f"built {lib}", flush=True)
    return lib


if __name__ == "__main__":
    args = sys.argv[1:]
    var = next((a.split("=", 1)[1] for a in args if a.startswith("--variant=")), "")
    defs = [a.split("=", 1)[1] for a in args if a.startswith("-D=")]
    build(verbose=True, force="--force" in args, variant=var, defines=defs)
