"""In-tree build of the native library (no pip install, no JIT cache).

  csrc/*.cu                 -> nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo
  csrc/layer.cpp capi.cpp   -> host C++20
  => paper_2505_11580_b200/libfipa_b200.so   (C ABI: include/fipa_b200.h)
  csrc/bindings.cpp         -> paper_2505_11580_b200/_fipa_b200.<abi>.so (pybind11, links the C ABI)

Objects go to build/; both .so files are written next to this file so they travel with the
repo snapshot to the GPU box.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import sysconfig
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "native")
INCLUDE = os.path.join(ROOT, "include")

CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SOURCES = ["gemm_tc.cu", "pack.cu", "attn_fwd_tc.cu", "attn_fwd_2sm.cu", "attn_fwd_pass.cu", "dense.cu", "simt_f32.cu", "attn_bwd.cu",
              "bwd.cu", "pair_features.cu", "proj_pack.cu", "attn_fwd_f32tc.cu"]
CXX_SOURCES = ["layer.cpp", "host_path.cpp", "capi.cpp", "comm.cpp", "trunk.cpp", "producer.cpp"]
HEADERS = ["ptx.cuh", "kernels.hpp", "layer.hpp", "tma_host.hpp", "trunk.hpp", "producer.hpp"]

LIB_NAME = "libfipa_b200.so"
EXT_NAME = "_fipa_b200" + (sysconfig.get_config_var("EXT_SUFFIX") or ".so")
LIB_PATH = os.path.join(PKG, LIB_NAME)
EXT_PATH = os.path.join(PKG, EXT_NAME)


def _cxx():
    # Prefer the system g++: it links libstdc++ dynamically.  A g++ that links it statically puts
    # a second, exported libstdc++ inside the pybind module, and libraries loaded after it
    # (torch's cuSPARSELt) then crash in their static constructors.
    # (The image's CXX wrapper links parts of libstdc++ statically, so CXX is not honoured here;
    # FIPA_CXX overrides.)
    if os.environ.get("FIPA_CXX"):
        return os.environ["FIPA_CXX"]
    if os.access("/usr/bin/g++", os.X_OK):
        return "/usr/bin/g++"
    return shutil.which("g++") or "g++"


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _run(cmd):
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        raise RuntimeError("build step failed:\n" + " ".join(cmd) + "\n" + r.stdout)
    return r.stdout


def _compile(src):
    path = os.path.join(CSRC, src)
    obj = os.path.join(BUILD, src + ".o")
    deps = [path] + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "fipa_b200.h")]
    if not _stale(obj, deps):
        return obj
    if src.endswith(".cu"):
        cmd = [NVCC, *GENCODE, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "-Xptxas", "-v", "--expt-relaxed-constexpr", "-I", CSRC, "-I", INCLUDE,
               "-c", path, "-o", obj]
    else:
        cmd = [_cxx(), "-O3", "-std=c++20", "-fPIC", "-Wall", "-I", CSRC, "-I", INCLUDE,
               "-I", os.path.join(CUDA_HOME, "include"), "-c", path, "-o", obj]
    log = _run(cmd)
    with open(obj + ".log", "w") as f:
        f.write(log)
    return obj


def build_native(verbose=False):
    os.makedirs(BUILD, exist_ok=True)
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
        objs = list(ex.map(_compile, CU_SOURCES + CXX_SOURCES))
    if _stale(LIB_PATH, objs):
        tmp = LIB_PATH + ".tmp"
        # CUDA runtime linked SHARED (rpath to the toolkit): a static cudart claims glibc's static-TLS
        # surplus, which made torch's CUDA libraries fail to load after this library
        _run([NVCC, *GENCODE, "-shared", "-cudart", "shared", "-o", tmp, *objs, "-Xlinker", "-soname=" + LIB_NAME,
              "-Xlinker", "-rpath=" + os.path.join(CUDA_HOME, "lib64"), "-ldl"])
        os.replace(tmp, LIB_PATH)
    import pybind11

    bsrc = os.path.join(CSRC, "bindings.cpp")
    if _stale(EXT_PATH, [bsrc, LIB_PATH, os.path.join(INCLUDE, "fipa_b200.h")]):
        tmp = EXT_PATH + ".tmp"
        _run([_cxx(), "-O2", "-std=c++17", "-shared", "-fPIC", "-fvisibility=hidden",
              "-I", pybind11.get_include(), "-I", sysconfig.get_paths()["include"], "-I", INCLUDE,
              bsrc, "-o", tmp, "-L", PKG, "-l:" + LIB_NAME, "-Wl,-rpath,$ORIGIN"])
        os.replace(tmp, EXT_PATH)
    if verbose:
        print(f"built {LIB_PATH}\nbuilt {EXT_PATH}")
    return LIB_PATH, EXT_PATH


def build_oracle():
    """Compile the reference oracle (test infrastructure) when the reference is mounted."""
    oracle = os.path.join(ROOT, "oracle")
    if os.path.isdir("/root/reference/proj/src") and shutil.which("make"):
        _run(["make", "-C", oracle, "-j8"])
        return True
    return False


if __name__ == "__main__":
    build_native(verbose=True)
    print("oracle built" if build_oracle() else "oracle skipped (no /root/reference)")
    sys.exit(0)
