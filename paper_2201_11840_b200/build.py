"""Builds libgc3.so (in-tree) for sm_100a, and the oracle library used by the tests.

    python -m paper_2201_11840_b200.build          # incremental
    python -m paper_2201_11840_b200.build --force

The product library: C++ host runtime (g++) + the CUDA interpreter (nvcc, sm_100a only, -lineinfo),
linked with -Bsymbolic so its nccl* entry points never bind to another libnccl in the process.
"""
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build" + os.environ.get("GC3_BUILD_TAG", ""))
LIB = os.environ.get("GC3_LIB_OUT", os.path.join(PKG, "libgc3.so"))
# extra nvcc defines for tuning builds, e.g. GC3_NVCC_DEFS="-DGC3_THREADS=256 -DGC3_UNROLL=8"
NVCC_DEFS = os.environ.get("GC3_NVCC_DEFS", "").split()
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

CXX_SRCS = ["json.cpp", "ir.cpp", "msccl_xml.cpp", "timed.cpp", "runtime.cpp"]
CU_SRCS = ["interp_launch.cu", "interp_k_copy.cu", "interp_k_sum.cu", "interp_k_prod.cu", "interp_k_max.cu", "interp_k_min.cu",
           "interp_k_sum_df.cu", "interp_k_prod_df.cu", "interp_k_max_df.cu", "interp_k_min_df.cu"]
HEADERS = ["json.hpp", "ir.hpp", "msccl_xml.hpp", "timed.hpp", "devplan.hpp", "interp.cuh"]
CU_HEADERS = ["devplan.hpp", "interp.cuh"]

ORACLE_DIR = os.path.join(REPO, "oracle")
ORACLE_LIB = os.path.join(ORACLE_DIR, "liboracle.so")


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        sys.stderr.write(p.stdout + p.stderr)
        raise RuntimeError("build step failed: " + " ".join(cmd[:3]))
    return p.stdout + p.stderr


def build_oracle(force=False, verbose=False):
    src = os.path.join(ORACLE_DIR, "gc3_oracle.c")
    hdr = os.path.join(ORACLE_DIR, "gc3_oracle.h")
    if force or _newer(ORACLE_LIB, [src, hdr]):
        _run(["gcc", "-O2", "-std=c11", "-Wall", "-Wextra", "-fPIC", "-shared", "-pthread", "-o", ORACLE_LIB, src], verbose)
    return ORACLE_LIB


def build_ref_harness(verbose=False):
    """oracle/_ref from the reference headers, only when /root/reference exists (never on the GPU box)."""
    if not os.path.isdir("/root/reference/proj/include"):
        return None
    out = os.path.join(ORACLE_DIR, "_ref", "libref.so")
    src = os.path.join(ORACLE_DIR, "ref_harness", "ref_tool.cpp")
    if _newer(out, [src]):
        _run(["make", "-s", "-C", os.path.join(ORACLE_DIR, "ref_harness")], verbose)
    return out


def build(force=False, verbose=False):
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(REPO, "include", "gc3.h")]
    objs, jobs = [], []
    for s in CXX_SRCS:
        src, obj = os.path.join(CSRC, s), os.path.join(BUILD, s + ".o")
        objs.append(obj)
        if force or _newer(obj, [src] + hdrs):
            jobs.append(["g++", "-std=c++17", "-O2", "-g", "-fPIC", "-fvisibility=hidden", "-Wall", "-Wextra",
                         "-Wno-unused-parameter", "-I" + os.path.join(CUDA, "include"), *NVCC_DEFS, "-c", src, "-o", obj])
    cu_hdrs = [os.path.join(CSRC, h) for h in CU_HEADERS]  # what the kernels include
    for s in CU_SRCS:
        src, obj = os.path.join(CSRC, s), os.path.join(BUILD, s + ".o")
        objs.append(obj)
        if force or _newer(obj, [src] + cu_hdrs):
            jobs.append([NVCC, *ARCH, "-std=c++17", "-O3", "-lineinfo", "-Xptxas", "-v", "-Xcompiler", "-fPIC",
                         "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr", *NVCC_DEFS, "-c", src, "-o", obj])
    logs = []
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
            logs = list(ex.map(lambda c: _run(c, verbose), jobs))
    if force or jobs or not os.path.exists(LIB):
        _run([NVCC, *ARCH, "-shared", "-o", LIB + ".tmp", *objs, "-lcudart", "-Xlinker", "-Bsymbolic",
              "-Xlinker", "--no-undefined"], verbose)
        os.replace(LIB + ".tmp", LIB)
        with open(os.path.join(BUILD, "ptxas.log"), "w") as f:
            f.write("\n".join(logs))
    return LIB


def main():
    force = "--force" in sys.argv
    verbose = "-v" in sys.argv
    build_oracle(force, verbose)
    build_ref_harness(verbose)
    print(build(force, verbose))


if __name__ == "__main__":
    main()
