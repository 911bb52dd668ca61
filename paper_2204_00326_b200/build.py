"""Build the product's shared library paper_2204_00326_b200/_lib/libdafmm.so.

nvcc compiles the CUDA kernels for sm_100a only (-gencode arch=compute_100a,code=sm_100a,
-lineinfo) and the host setup / C-ABI C++ with OpenMP; cudart is linked statically so the
library does not depend on the runtime torch happens to load.  Cross-compiles without a GPU.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT_DIR, "libdafmm.so")
# experiments: DAFMM_NVCC_FLAGS adds nvcc flags, DAFMM_LIB_NAME builds a differently named library
# (the binding loads DAFMM_LIB_NAME too when it is set)
EXTRA = os.environ.get("DAFMM_NVCC_FLAGS", "").split()
if os.environ.get("DAFMM_LIB_NAME"):
    LIB = os.path.join(OUT_DIR, os.environ["DAFMM_LIB_NAME"])
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SOURCES = ["kernels.cu", "setup_device.cu", "hodlr.cu"]
CPP_SOURCES = ["setup.cpp", "capi.cpp"]


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)


def build(verbose=False, force=False, ptxas_verbose=False):
    os.makedirs(OUT_DIR, exist_ok=True)
    srcs = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "dafmm.h")]
    if not force and os.path.exists(LIB) and all(os.path.getmtime(LIB) >= os.path.getmtime(s) for s in srcs):
        return LIB
    inc = ["-I" + CSRC, "-I" + os.path.join(ROOT, "include")]
    objs = []
    for f in CU_SOURCES:
        o = os.path.join(OUT_DIR, f + ".o")
        o = os.path.join(OUT_DIR, os.path.basename(LIB) + "." + f + ".o")
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", *EXTRA, *inc, "-c",
               os.path.join(CSRC, f), "-o", o]
        if ptxas_verbose:
            cmd += ["-Xptxas", "-v"]
        _run(cmd, verbose)
        objs.append(o)
    for f in CPP_SOURCES:
        o = os.path.join(OUT_DIR, f + ".o")
        _run(["g++", "-O3", "-std=c++17", "-fPIC", "-fopenmp", "-mfma", "-mavx2", "-g", *inc,
              "-I/usr/local/cuda/include", "-c", os.path.join(CSRC, f), "-o", o], verbose)
        objs.append(o)
    _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs, "-Xcompiler", "-fopenmp", "-lgomp"],
         verbose)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv, ptxas_verbose="-v" in sys.argv))
