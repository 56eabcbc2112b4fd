"""Build libdictmerge.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

Each csrc/*.cu compiles to its own object under build/ (in parallel, rebuilt only
when the source or a header changed), then one link makes the shared library."""
from __future__ import annotations

import glob
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
OBJ = os.path.join(os.path.dirname(HERE), "build", "obj")
LIB = os.path.join(HERE, "libdictmerge.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-warn-spills"]
LDFLAGS = [*ARCH, "-shared", "-Xcompiler", "-fPIC"]
FLAGS = [*CFLAGS, "-shared"]  # single-command form (kept for callers that compile in one step)


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _headers():
    return glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(INCLUDE, "*.h"))


def _inputs():
    return sources() + _headers()


def up_to_date() -> bool:
    return os.path.exists(LIB) and os.path.getmtime(LIB) >= max(os.path.getmtime(p) for p in _inputs())


def _compile(src: str, tag: str, defines: tuple, verbose: bool) -> str:
    os.makedirs(OBJ, exist_ok=True)
    obj = os.path.join(OBJ, os.path.basename(src)[:-3] + (f".{tag}" if tag else "") + ".o")
    newest = max([os.path.getmtime(src)] + [os.path.getmtime(h) for h in _headers()])
    if os.path.exists(obj) and os.path.getmtime(obj) >= newest:
        return obj
    tmp = obj + f".tmp{os.getpid()}"
    cmd = [NVCC, *CFLAGS, *[f"-D{d}" for d in defines], "-c", src, "-o", tmp]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(tmp, obj)
    return obj


def _build(out: str, tag: str = "", defines: tuple = (), verbose: bool = False, only: tuple = ()) -> str:
    """Compile (in parallel) and link.  `only`: sources that get `defines`/`tag`
    (the others reuse the default objects)."""
    srcs = sources()
    with ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        objs = list(ex.map(lambda s: _compile(s, tag if (not only or os.path.basename(s) in only) else "",
                                              defines if (not only or os.path.basename(s) in only) else (),
                                              verbose), srcs))
    tmp = out + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *LDFLAGS, *objs, "-o", tmp])
    os.replace(tmp, out)
    return out


def build_trace() -> str:
    """Diagnostic variant with %globaltimer phase stamps (-DDM_TRACE); not used by the product path."""
    return _build(os.path.join(HERE, "libdictmerge_trace.so"), "trace", ("DM_TRACE",))


def build_check() -> str:
    """Diagnostic variant with device-side bounds assertions (-DDM_CHECK); load it
    with DM_LIB_PATH.  Not used by the product path."""
    return _build(os.path.join(HERE, "libdictmerge_check.so"), "check", ("DM_CHECK",))


def build_variant(name: str, *defines: str, only: tuple = ()) -> str:
    """Experiment variant libdictmerge_<name>.so built with extra -D flags (load via DM_LIB_PATH)."""
    return _build(os.path.join(HERE, f"libdictmerge_{name}.so"), name, tuple(defines), only=only)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    return _build(LIB, verbose=verbose)


if __name__ == "__main__":
    import sys
    if len(sys.argv) > 2 and sys.argv[1] == "variant":  # python -m ... variant <name> DEF=1 ... [--only f.cu]
        args = sys.argv[2:]
        only = tuple(a for a in args if a.endswith(".cu"))
        print(build_variant(args[0], *[a for a in args[1:] if not a.endswith(".cu")], only=only))
    else:
        print(build(force=True, verbose=True))
