"""In-tree build of libpcg.so for sm_100a (nvcc cross-compiles; no GPU needed).

    python -m paper_1210_1878_b200.build [--force]

Device code: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo.  Host setup code
(AINV, packing) is compiled with -ffp-contract=off so its fp64 arithmetic is exactly the
sequence written.  NCCL comes from the venv's nvidia-nccl wheel (the same
libnccl.so.2 torch loads); cudart is linked statically.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libpcg.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_paths():
    import nvidia.nccl as n
    root = os.path.dirname(n.__file__) if getattr(n, "__file__", None) else list(n.__path__)[0]
    return os.path.join(root, "include"), os.path.join(root, "lib")


def _sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    return hs + [os.path.join(INCLUDE, "libpcg.h")]


def _compile(src, nccl_inc, bdir=BUILD, defines=()):
    path = os.path.join(CSRC, src)
    obj = os.path.join(bdir, src + ".o")
    common = ["-I" + CSRC, "-I" + INCLUDE, "-I" + nccl_inc, "-std=c++17"] + ["-D" + d for d in defines]
    if src.endswith(".cu"):
        cmd = [NVCC] + ARCH + ["-O3", "-lineinfo", "-Xptxas", "-v", "-Xcompiler", "-fPIC,-O2,-ffp-contract=off",
                               "-c", path, "-o", obj] + common
    else:
        # host-only translation units: plain g++, no contraction of a*b+c
        cmd = ["g++", "-O2", "-fPIC", "-ffp-contract=off", "-fno-fast-math", "-Wall", "-c", path, "-o", obj,
               "-I/usr/local/cuda/include"] + common
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False, variant: str = "", defines=()) -> str:
    """Build libpcg.so (or, with `variant`, a tuning variant _build/<variant>/libpcg.so
    compiled with extra -D defines; load it with PCG_LIB=<path>)."""
    bdir = os.path.join(BUILD, variant) if variant else BUILD
    lib = os.path.join(bdir, "libpcg.so") if variant else LIB
    os.makedirs(bdir, exist_ok=True)
    srcs = _sources()
    deps = [os.path.join(CSRC, s) for s in srcs] + _headers() + [os.path.abspath(__file__)]
    if not force and os.path.exists(lib):
        t = os.path.getmtime(lib)
        if all(os.path.getmtime(d) <= t for d in deps):
            return lib
    nccl_inc, nccl_lib = nccl_paths()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        outs = list(ex.map(lambda s: _compile(s, nccl_inc, bdir, defines), srcs))
    if verbose:
        for _, log in outs:
            if log:
                print(log, file=sys.stderr)
    tmp = lib + ".tmp"
    cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + [o for o, _ in outs] + [
        "-L" + nccl_lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + nccl_lib, "-cudart", "static", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    if "--variant" in sys.argv:
        k = sys.argv.index("--variant")
        name, defs = sys.argv[k + 1], sys.argv[k + 2:]
        print(build(force=True, verbose="-v" in sys.argv, variant=name, defines=[d for d in defs if d != "-v"]))
    else:
        print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
