"""Build libptg.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

``python -m paper_1810_05628_b200._build`` compiles every ``csrc/*.cu`` to an
object with ``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` and
links ``paper_1810_05628_b200/lib/libptg.so``.  The .so is git-ignored but
travels to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
OBJDIR = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(LIBDIR, "libptg.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
           "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")]
# PTG_NVCC_DEFS="-DFOO=1 ...": extra defines for kernel-variant experiments
NVFLAGS += os.environ.get("PTG_NVCC_DEFS", "").split()


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise FileNotFoundError("nvcc not found")


def host_cxx() -> list:
    # the image's $CXX may point at a toolchain without libgomp; use the system g++
    gxx = shutil.which("g++", path="/usr/bin") or shutil.which("g++")
    return ["-ccbin", gxx] if gxx else []


def _stale(obj: str, deps: list) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, jobs: int = 8) -> str:
    os.makedirs(LIBDIR, exist_ok=True)
    os.makedirs(OBJDIR, exist_ok=True)
    srcs = sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(ROOT, "include", "ptg.h"))
    cmds = []
    objs = []
    for s in srcs:
        src = os.path.join(CSRC, s)
        obj = os.path.join(OBJDIR, s.replace(".cu", ".o"))
        objs.append(obj)
        if _stale(obj, [src] + headers):
            cmds.append([nvcc(), *host_cxx(), *ARCH, *NVFLAGS, "-c", src, "-o", obj])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        return cmd, r

    with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
        for cmd, r in ex.map(run, cmds):
            log = r.stdout + r.stderr
            if r.returncode != 0:
                sys.stderr.write(log)
                raise RuntimeError("nvcc failed: " + " ".join(cmd))
            if verbose:
                sys.stderr.write(log)
            with open(os.path.join(OBJDIR, os.path.basename(cmd[-1]) + ".ptxas.txt"), "w") as f:
                f.write(log)
    if cmds or not os.path.exists(LIB):
        link = [nvcc(), *host_cxx(), *ARCH, "-shared", "-o", LIB, *objs, "-lcudart", "-ldl"]
        r = subprocess.run(link, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
    build_cpp_tests()
    return LIB


CPP = os.path.join(PKG, "cpp")
CPP_INC = os.path.join(CPP, "include")
SHIM = os.path.join(CPP, "doctest_shim")
EXT_TEST = os.path.join(LIBDIR, "test_dropin_ext")
REF_TEST = os.path.join(LIBDIR, "ref_tests_dropin")
REF_TESTS_DIR = "/root/reference/proj/tests"
REF_TEST_FILES = ("test_objectives.cpp", "test_solvers.cpp", "test_multigrid.cpp")


def _cxx():
    return shutil.which("g++", path="/usr/bin") or "g++"


def _cpp_headers():
    out = [os.path.join(ROOT, "include", "ptg.h"), os.path.join(SHIM, "doctest.h"), LIB]
    for d, _, fs in os.walk(CPP_INC):
        out += [os.path.join(d, f) for f in fs if f.endswith(".hpp")]
    return out


def build_cpp_tests() -> str:
    """C++ tests of the drop-in headers (cpp/include/ptycho), linked to libptg.so:
    test_dropin_ext (the additive API) and, where the reference sources exist,
    ref_tests_dropin = the reference's UNMODIFIED unit tests
    (proj/tests/test_objectives.cpp, test_solvers.cpp, test_multigrid.cpp,
    compiled in place with the doctest shim; never copied) -- the binary
    travels to the GPU box with the rest of lib/."""
    flags = ["-std=c++20", "-O2", "-Wall", "-I" + CPP_INC, "-I" + CPP, "-I" + SHIM, "-I" + os.path.join(ROOT, "include")]
    link = ["-L" + LIBDIR, "-lptg", "-Wl,-rpath,$ORIGIN"]
    deps = _cpp_headers()
    src = os.path.join(CPP, "test_dropin_ext.cpp")
    if _stale(EXT_TEST, deps + [src]):
        r = subprocess.run([_cxx(), *flags, src, "-o", EXT_TEST, *link], capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("C++ drop-in extension test build failed")
    if os.path.isdir(REF_TESTS_DIR):
        srcs = [os.path.join(REF_TESTS_DIR, f) for f in REF_TEST_FILES] + [os.path.join(CPP, "ref_tests_main.cpp")]
        if _stale(REF_TEST, deps + srcs):
            cmd = [_cxx(), *flags, "-I" + REF_TESTS_DIR, *srcs, "-o", REF_TEST, *link]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError("reference unit tests against the drop-in failed to build")
    return EXT_TEST


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
