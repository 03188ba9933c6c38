"""In-tree build of libtidepool_gpu.so (sm_100a) and the C oracle.

`python -m paper_1810_08723_b200.build` (or __graft_entry__.build()) compiles
every .cu under csrc/ with nvcc for sm_100a only and links them into
paper_1810_08723_b200/libtidepool_gpu.so.  Objects are rebuilt only when a
source or header is newer than the object.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = PKG / "_build"
LIB = PKG / "libtidepool_gpu.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
          "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", f"-I{ROOT / 'include'}"]
# files whose double arithmetic must not be contracted into FMAs (the
# reference computes every + - * as a separately rounded CPython float op)
NO_FMA_PREFIX = ("tpg_ewise", "tpg_reduce", "tpg_chain")


def _headers():
    return list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [ROOT / "include" / "tidepool_gpu.h"]


def _stale(obj: Path, src: Path, deps) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return src.stat().st_mtime > t or any(d.stat().st_mtime > t for d in deps)


def _compile(src: Path, verbose: bool) -> Path:
    obj = BUILD / (src.stem + ".o")
    cmd = [NVCC, *ARCH, *COMMON, "-c", str(src), "-o", str(obj)]
    if src.name.startswith(NO_FMA_PREFIX):
        cmd.insert(1, "-fmad=false")
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return obj


def build_library(verbose: bool = False, jobs: int | None = None) -> Path:
    BUILD.mkdir(exist_ok=True)
    srcs = sorted(CSRC.glob("*.cu"))
    deps = _headers()
    todo = [s for s in srcs if _stale(BUILD / (s.stem + ".o"), s, deps)]
    if todo:
        with cf.ThreadPoolExecutor(max_workers=jobs or min(len(todo), os.cpu_count() or 4)) as ex:
            list(ex.map(lambda s: _compile(s, verbose), todo))
    objs = [BUILD / (s.stem + ".o") for s in srcs]
    if todo or not LIB.exists() or any(o.stat().st_mtime > LIB.stat().st_mtime for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs),
               "-lcudart", "-ldl", "-lcuda"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    build_pyext(verbose)
    return LIB


def build_pyext(verbose: bool = False) -> Path:
    """The drop-in plugin's CPython host fast path (hostsrc/tpg_pyfast.c):
    plain C against the interpreter's headers, no CUDA, no link-time
    dependency on libtidepool_gpu.so (it receives C-ABI function addresses)."""
    import sysconfig
    src = PKG / "hostsrc" / "tpg_pyfast.c"
    out = PKG / ("_tpg_pyfast" + sysconfig.get_config_var("EXT_SUFFIX"))
    if out.exists() and out.stat().st_mtime >= src.stat().st_mtime:
        return out
    cc = os.environ.get("CC", "gcc")
    cmd = [cc, "-O2", "-shared", "-fPIC", "-Wall", "-Wno-missing-field-initializers",
           f"-I{sysconfig.get_paths()['include']}", str(src), "-o", str(out)]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return out


def build_oracle(verbose: bool = False) -> Path:
    sys.path.insert(0, str(ROOT))
    from oracle import build as ob  # the checker, not the product
    return ob.build(verbose=verbose)


if __name__ == "__main__":
    v = "-v" in sys.argv
    print(build_library(verbose=v))
    print(build_oracle(verbose=v))
