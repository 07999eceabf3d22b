"""In-tree build of libauxmc_b200.so (sm_100a) — nvcc, no JIT cache.

`python -m paper_2303_00301_b200.build` or `build()` from __graft_entry__.
Object files go to paper_2303_00301_b200/build/ and the shared library to
paper_2303_00301_b200/libauxmc_b200.so; both travel to the GPU box with the
repo snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import pathlib
import subprocess
import sys

PKG = pathlib.Path(__file__).resolve().parent
CSRC = PKG / "csrc"
HOST = PKG / "host"
OUT = PKG / "build"
LIB = PKG / "libauxmc_b200.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                  "-Xcompiler", "-Wall", "--expt-relaxed-constexpr",
                  "-Wno-deprecated-gpu-targets", "-I", str(PKG.parent / "include")]
CXXFLAGS = ["-O2", "-fPIC", "-std=c++17", "-Wall", "-I", str(PKG.parent / "include"),
            "-I", "/usr/local/cuda/include"]


def _sources():
    cu = sorted(CSRC.glob("*.cu"))
    cpp = sorted(HOST.glob("*.cpp")) if HOST.exists() else []
    return cu, cpp


def _deps():
    return sorted(CSRC.glob("*.cuh")) + sorted(HOST.glob("*.hpp")) + [
        PKG.parent / "include" / "auxmc_gpu.h"]


def _stale(obj: pathlib.Path, src: pathlib.Path, deps) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return src.stat().st_mtime > t or any(d.stat().st_mtime > t for d in deps)


def _compile(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r.stderr


def build(verbose: bool = False) -> pathlib.Path:
    OUT.mkdir(exist_ok=True)
    cu, cpp = _sources()
    deps = _deps()
    jobs, objs = [], []
    for src in cu:
        obj = OUT / (src.stem + ".o")
        objs.append(obj)
        if _stale(obj, src, deps):
            jobs.append([NVCC, *NVFLAGS, "-c", str(src), "-o", str(obj)])
    for src in cpp:
        obj = OUT / (src.stem + ".host.o")
        objs.append(obj)
        if _stale(obj, src, deps):
            jobs.append(["g++", *CXXFLAGS, "-c", str(src), "-o", str(obj)])
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        for msg in ex.map(_compile, jobs):
            if verbose and msg.strip():
                print(msg, file=sys.stderr)
    if jobs or not LIB.exists():
        _compile([NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs),
                  "-lcudart", "-Xlinker", "-rpath,/usr/local/cuda/lib64"])
    return LIB


TEST_SRC = PKG.parent / "tests" / "cpp" / "test_facade.cpp"
TEST_BIN = PKG.parent / "tests" / "cpp" / "build" / "test_facade"


def build_tests() -> pathlib.Path:
    """C++ facade parity test (tests/cpp/test_facade.cpp), linked against the
    product library and the CPU oracle (test infrastructure; build it first with
    oracle/pyoracle.build()).  rpaths are relative so the binary runs from any
    checkout, including the GPU box's copy of the repo."""
    oracle_lib = PKG.parent / "oracle" / "build" / "liboracle.so"
    TEST_BIN.parent.mkdir(parents=True, exist_ok=True)
    deps = [TEST_SRC, LIB, oracle_lib, PKG.parent / "include" / "auxmc_b200.hpp"]
    if TEST_BIN.exists() and all(d.stat().st_mtime <= TEST_BIN.stat().st_mtime for d in deps):
        return TEST_BIN
    _compile(["g++", "-O2", "-std=c++17", "-Wall", "-I", str(PKG.parent / "include"),
              "-I", str(PKG.parent / "oracle"), str(TEST_SRC), "-o", str(TEST_BIN),
              "-L", str(PKG), "-lauxmc_b200", "-L", str(oracle_lib.parent), "-loracle",
              "-Wl,-rpath,$ORIGIN/../../../paper_2303_00301_b200",
              "-Wl,-rpath,$ORIGIN/../../../oracle/build"])
    return TEST_BIN


if __name__ == "__main__":
    print(build(verbose=True))
