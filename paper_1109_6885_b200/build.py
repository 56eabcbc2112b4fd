"""Build libdictmerge.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
LIB = os.path.join(HERE, "libdictmerge.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-warn-spills"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _inputs():
    return sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(INCLUDE, "*.h"))


def up_to_date() -> bool:
    return os.path.exists(LIB) and os.path.getmtime(LIB) >= max(os.path.getmtime(p) for p in _inputs())


def build_trace() -> str:
    """Diagnostic variant with %globaltimer phase stamps (-DDM_TRACE); not used by the product path."""
    out = os.path.join(HERE, "libdictmerge_trace.so")
    subprocess.check_call([NVCC, *FLAGS, "-DDM_TRACE", *sources(), "-o", out])
    return out


def build_check() -> str:
    """Diagnostic variant with device-side bounds assertions (-DDM_CHECK); load it
    with DM_LIB_PATH.  Not used by the product path."""
    out = os.path.join(HERE, "libdictmerge_check.so")
    subprocess.check_call([NVCC, *FLAGS, "-DDM_CHECK", *sources(), "-o", out])
    return out


def build_variant(name: str, *defines: str) -> str:
    """Experiment variant libdictmerge_<name>.so built with extra -D flags (load via DM_LIB_PATH)."""
    out = os.path.join(HERE, f"libdictmerge_{name}.so")
    subprocess.check_call([NVCC, *FLAGS, *[f"-D{d}" for d in defines], *sources(), "-o", out])
    return out


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *FLAGS, *sources(), "-o", tmp]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
