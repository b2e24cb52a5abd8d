"""Build libspamm_b200.so in-tree with nvcc for sm_100a (no JIT, no torch extension)."""
from __future__ import annotations

import glob
import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libspamm_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3",
]
LINK_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "--cudart", "static", "-shared"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [
        os.path.join(HERE, "..", "include", "spamm.h")]


def up_to_date(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return False
    t = os.path.getmtime(lib)
    return all(os.path.getmtime(f) <= t for f in sources() + headers())


LIB_DEBUG = os.path.join(HERE, "libspamm_b200_debug.so")


def build_debug(force: bool = False, verbose: bool = False) -> str:
    """The SPAMM_DEBUG variant (device-side bounds asserts, common.cuh SPAMM_ASSERT);
    select it with SPAMM_LIB=<path> for a checked test run."""
    return build(force, verbose, lib=LIB_DEBUG, extra=["-DSPAMM_DEBUG"])


LIB_CLOCKS = os.path.join(HERE, "libspamm_b200_clocks.so")


def build_clocks(force: bool = False, verbose: bool = False) -> str:
    """Diagnostic variant: the leaf GEMM's consumer warps count the cycles they wait for
    stages and queue entries (tools/gemm_clocks.py; select it with SPAMM_LIB=<path>)."""
    return build(force, verbose, lib=LIB_CLOCKS, extra=["-DSPAMM_GEMM_CLOCKS"])


def build_variant(name: str, defines, force: bool = False) -> str:
    """An experimental variant (extra -D flags) built to libspamm_b200_<name>.so for A/B
    timing with SPAMM_LIB."""
    return build(force, lib=os.path.join(HERE, f"libspamm_b200_{name}.so"), extra=[f"-D{d}" for d in defines])


def build(force: bool = False, verbose: bool = False, lib: str = LIB, extra=()) -> str:
    if not force and up_to_date(lib):
        return lib
    # one nvcc per translation unit, in parallel, then one link
    tmp = lib + f".tmp{os.getpid()}"
    objdir = os.path.join(HERE, "build", f"obj{os.getpid()}")
    os.makedirs(objdir, exist_ok=True)
    objs = [os.path.join(objdir, os.path.basename(s)[:-3] + ".o") for s in sources()]
    cmds = [[NVCC, *NVCC_FLAGS, *extra, "-c", "-o", o, s] for s, o in zip(sources(), objs)]
    if verbose:
        for c in cmds:
            print(" ".join(c))
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 4)) as ex:
        rcs = list(ex.map(lambda c: subprocess.call(c), cmds))
    if any(rcs):
        raise subprocess.CalledProcessError(max(rcs), "nvcc (see the errors above)")
    subprocess.check_call([NVCC, *LINK_FLAGS, "-o", tmp, *objs])
    os.replace(tmp, lib)
    shutil.rmtree(objdir, ignore_errors=True)
    return lib


if __name__ == "__main__":
    import sys
    if "--debug" in sys.argv:
        print(build_debug(force="-f" in sys.argv, verbose=True))
    else:
        print(build(force="-f" in sys.argv, verbose=True))
