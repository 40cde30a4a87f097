"""Build libfp8lm.so in-tree with nvcc for sm_100a (no JIT, no torch extension cache).

    python paper_2310_18313_b200/build.py [--force]     # or __graft_entry__.build()

Flags: -gencode arch=compute_100a,code=sm_100a (arch-specific: the packed FP8 cvt and
256-bit ld/st are sm_100a instructions); -fmad=false + IEEE div/sqrt so that every
binary32 rounding matches the oracle's (R16); -lineinfo for ncu source
correlation.  NCCL: the torch-bundled libnccl.so.2 (the same library torch loads).
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libfp8lm.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    try:
        import nvidia.nccl as nn
        base = list(nn.__path__)[0]
    except Exception:
        return None, None
    inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
    if os.path.exists(os.path.join(inc, "nccl.h")) and glob.glob(os.path.join(lib, "libnccl.so*")):
        return inc, lib
    return None, None


def nvcc():
    for c in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def needs_rebuild() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))
    deps.append(os.path.join(ROOT, "include", "fp8lm.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """Each source compiles to an object in parallel (kernels.cu dominates), then one link.
    out / defines: an experiment build (A/B runs load it through FP8LM_LIB)."""
    lib_out = out or LIB
    if out: os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
    if not force and out is None and not defines and not needs_rebuild():
        return LIB
    inc, lib = nccl_dirs()
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
             "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
             "-Xcompiler", "-fPIC,-O2,-ffp-contract=off", "-I", os.path.join(ROOT, "include")]
    if inc:
        flags += ["-DFP8LM_WITH_NCCL", "-I", inc]
    flags += [f"-D{d}" for d in defines]
    objdir = os.path.join(HERE, "build" if not defines else "build_" + "_".join(defines).replace("=", ""))
    os.makedirs(objdir, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [nvcc(), *flags, "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd))
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src} ({r.returncode}):\n{r.stdout}\n{r.stderr}")
        return obj

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=len(sources())) as ex:
        objs = list(ex.map(compile_one, sources()))
    cmd = [nvcc(), *ARCH, "-shared", *objs]
    if lib:
        cmd += ["-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{lib}"]
    cmd += ["-o", lib_out + ".tmp"]
    if verbose:
        print(" ".join(cmd))
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed ({r.returncode}):\n{r.stdout}\n{r.stderr}")
    os.replace(lib_out + ".tmp", lib_out)
    return lib_out


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--out", default=None, help="experiment build: output path")
    ap.add_argument("-D", dest="defines", action="append", default=[], help="extra -D for an experiment build")
    a = ap.parse_args()
    print(build(force=a.force or bool(a.out), verbose=True, out=a.out, defines=a.defines))
