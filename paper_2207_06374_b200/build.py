"""Builds the in-tree CUDA library paper_2207_06374_b200/_lib/libtrstmi_b200.so.

nvcc -gencode arch=compute_100a,code=sm_100a for every translation unit;
-fmad=false so only the explicit fma() sites of the Canonical Arithmetic Spec
fuse; host code with -ffp-contract=off for the same reason.
Also builds the C++ host-API test binary when its sources exist.
"""
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIBDIR = os.path.join(HERE, "_lib")
LIB = os.path.join(LIBDIR, "libtrstmi_b200.so")
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "--expt-relaxed-constexpr",
                 "-Xcompiler", "-fPIC,-ffp-contract=off,-O2", "-I", os.path.join(HERE, "..", "include")]

# (complex, S, stored-Gram layout): the set kernel_table.hpp declares
INSTANCES = [(c, s, g) for c in (1, 0) for (s, g) in ((64, 1), (128, 1), (128, 0), (256, 1), (256, 0), (512, 1))]


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed: %s\n%s\n%s" % (" ".join(cmd), r.stdout, r.stderr))
    return r.stdout + r.stderr


def _newer(target, deps):
    if not os.path.exists(target):
        return False
    t = os.path.getmtime(target)
    return all(os.path.getmtime(d) <= t for d in deps)


def sources():
    out = []
    for root, _, files in os.walk(CSRC):
        for f in files:
            if f.endswith((".cu", ".cuh", ".hpp", ".h", ".cpp")):
                out.append(os.path.join(root, f))
    out.append(os.path.join(HERE, "..", "include", "trstmi_b200.h"))
    return out


def _includes(path, seen=None):
    """Transitive local #include "..." closure of a source file."""
    import re
    seen = set() if seen is None else seen
    if path in seen or not os.path.exists(path):
        return seen
    seen.add(path)
    for m in re.finditer(r'^\s*#\s*include\s+"([^"]+)"', open(path).read(), re.M):
        _includes(os.path.normpath(os.path.join(os.path.dirname(path), m.group(1))), seen)
    return seen


def build(verbose=False, force=False, jobs=None):
    os.makedirs(BUILD, exist_ok=True)
    os.makedirs(LIBDIR, exist_ok=True)
    deps = sources()
    if not force and _newer(LIB, deps):
        return LIB
    jobs = jobs or max(2, min(8, os.cpu_count() or 2))
    tasks = []
    objs = []
    me = [os.path.abspath(__file__)]

    def add(src, o, extra):
        objs.append(o)
        if force or not _newer(o, sorted(_includes(src)) + me):  # per-object: only stale objects rebuild
            tasks.append(COMMON + extra + ["-c", src, "-o", o])

    for cplx, s, g in INSTANCES:
        o = os.path.join(BUILD, "inst_%s_%d_%s.o" % ("c" if cplx else "r", s, "g" if g else "r"))
        add(os.path.join(CSRC, "instantiate.cu"), o, ["-DINST_CPLX=%d" % cplx, "-DINST_S=%d" % s, "-DINST_GS=%d" % g])
    for src in ("trstmi_capi.cu", "large_engine.cu", "analysis.cu", "sharding.cu", "bde_engine.cu", "altproj.cu"):
        add(os.path.join(CSRC, src), os.path.join(BUILD, src.replace(".cu", ".o")), [])
    with cf.ThreadPoolExecutor(jobs) as ex:
        for log in ex.map(lambda c: _run([NVCC] + c), tasks):
            if verbose and log.strip():
                print(log)
    tmp = LIB + ".tmp"
    _run([NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-cudart", "static", "-lnccl"])
    os.replace(tmp, LIB)
    build_host_tests()
    return LIB


HOST_TEST_SRC = os.path.join(HERE, "..", "tests", "cpp", "test_host_api.cpp")
HOST_TEST_BIN = os.path.join(LIBDIR, "test_host_api")


def build_host_tests():
    """C++ host-mirror tests (tests/cpp), linked against the in-tree library."""
    if not os.path.exists(HOST_TEST_SRC):
        return None
    gxx = shutil.which("g++") or "g++"
    _run([gxx, "-std=c++17", "-O2", "-ffp-contract=off", "-o", HOST_TEST_BIN, HOST_TEST_SRC, "-L" + LIBDIR,
          "-ltrstmi_b200", "-Wl,-rpath,$ORIGIN"])
    return HOST_TEST_BIN


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
