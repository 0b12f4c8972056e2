"""Build the in-tree CUDA library libqqq_b200.so for sm_100a with nvcc.

The product never JIT-compiles: `__graft_entry__.build()` (and `make`) call
`build_library()`, the resulting .so lives in `paper_2406_09904_b200/lib/` and
travels with the repo snapshot to the GPU box.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libqqq_b200.so")
# developer variant with the in-kernel %globaltimer timeline (scripts/timeline.py)
LIB_TL = os.path.join(LIBDIR, "libqqq_b200_tl.so")
INCLUDE = os.path.join(ROOT, "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", INCLUDE, "-I", CSRC,
                     "--expt-relaxed-constexpr"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the B200 library cannot be built")


def _sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _deps():
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(INCLUDE, "qqq_b200.h")]
    return files + [os.path.abspath(__file__)]


def up_to_date(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return False
    t = os.path.getmtime(lib)
    return all(os.path.getmtime(f) <= t for f in _deps())


def build_library(force: bool = False, verbose: bool = False, timeline: bool = False, defines=(), name=None) -> str:
    """Build the product library (or, for developer A/B runs, a variant with
    extra -D defines written to lib/<name>.so)."""
    lib = LIB_TL if timeline else LIB
    if name:
        lib = os.path.join(LIBDIR, name + ".so")
    if not force and up_to_date(lib):
        return lib
    nvcc = _nvcc()
    objdir = os.path.join(PKG, "build", name or ("tl" if timeline else "prod"))
    extra = (["-DQQQ_TIMELINE"] if timeline else []) + ["-D" + d for d in defines]
    os.makedirs(objdir, exist_ok=True)
    os.makedirs(LIBDIR, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [nvcc, *NVCC_FLAGS, *extra, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        if verbose and r.stderr:
            sys.stderr.write(r.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
        objs = list(ex.map(compile_one, _sources()))
    tmp = lib + ".tmp"
    # libcuda is resolved at run time (cudaGetDriverEntryPoint), so the library
    # loads on a GPU-less build host too; cudart is linked statically.
    cmd = [nvcc, *ARCH, "-shared", "-o", tmp, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    names = [a[7:] for a in sys.argv[1:] if a.startswith("--name=")]
    print(build_library(force="--force" in sys.argv, verbose=True, timeline="--timeline" in sys.argv, defines=defs,
                        name=names[0] if names else None))
