"""In-tree build of libdistattn_b200.so (sm_100a) with plain nvcc.

The shared library is the product: CUDA kernels + the C ABI declared in
include/distattn_b200.h. Objects are compiled in parallel and relinked only
when a source or header is newer than the library.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = Path(os.environ.get("DA_BUILD_DIR", PKG / "_build"))
LIB = Path(os.environ.get("DA_LIB_OUT", PKG / "libdistattn_b200.so"))
EXTRA = os.environ.get("DA_BUILD_DEFINES", "").split()

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-fvisibility=hidden", "-DNDEBUG", "-I", str(ROOT / "include"),
              "-I", str(CSRC)]


# kernels that redistribute registers with setmaxnreg need a known launch budget
PER_FILE = {"attn_bwd_ws_sm100.cu": ["-maxrregcount=128"],
            "attn_bwd_pair_sm100.cu": ["-maxrregcount=128"]}


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _sources() -> list[Path]:
    return sorted(list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cpp")))


def _headers() -> list[Path]:
    return sorted(list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) +
                  list((ROOT / "include").rglob("*.h")))


def _newest(paths) -> float:
    return max((p.stat().st_mtime for p in paths), default=0.0)


def _compile(src: Path, verbose: bool, ptxas_v: bool) -> Path:
    obj = BUILD / (src.name + ".o")
    cmd = [nvcc(), *ARCH, *NVCC_FLAGS, *PER_FILE.get(src.name, []), *EXTRA, "-c", str(src), "-o",
           str(obj)]
    if ptxas_v and src.suffix == ".cu":
        cmd += ["-Xptxas", "-v"]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stdout}\n{r.stderr}")
    if ptxas_v and r.stderr:
        print(r.stderr, file=sys.stderr)
    return obj


def build(force: bool = False, verbose: bool = False, ptxas_v: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    srcs = _sources()
    hdr_time = _newest(_headers())
    if LIB.exists() and not force and not ptxas_v:
        if LIB.stat().st_mtime >= max(_newest(srcs), hdr_time):
            return LIB
    todo = []
    for s in srcs:
        obj = BUILD / (s.name + ".o")
        if force or ptxas_v or not obj.exists() or obj.stat().st_mtime < max(s.stat().st_mtime, hdr_time):
            todo.append(s)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        list(ex.map(lambda s: _compile(s, verbose, ptxas_v), todo))
    objs = [BUILD / (s.name + ".o") for s in srcs]
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcuda", "-lpthread"]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


def build_cpp_tests() -> Path:
    """tests/cpp/_build/test_b200_api: the C++ drop-in API (include/distattn/b200.hpp)
    against the C oracle; tests/cpp/_build/test_rank_cpp: the multi-process
    RankRuntime driven from C++ only. Needs libdistattn_b200.so and
    oracle/liboracle.so."""
    exe = _build_cpp_test("test_b200_api")
    _build_cpp_test("test_rank_cpp")
    return exe


def _build_cpp_test(name: str) -> Path:
    out_dir = ROOT / "tests" / "cpp" / "_build"
    out_dir.mkdir(parents=True, exist_ok=True)
    exe = out_dir / name
    src = ROOT / "tests" / "cpp" / f"{name}.cpp"
    deps = [src, ROOT / "include" / "distattn" / "b200.hpp", ROOT / "include" / "distattn_b200.h", LIB]
    if exe.exists() and exe.stat().st_mtime >= _newest(deps):
        return exe
    cuda = Path(nvcc()).resolve().parents[1]
    cxx = shutil.which("g++") or "g++"
    cmd = [cxx, "-std=c++17", "-O2", "-Wall", "-I", str(ROOT / "include"), "-I", str(ROOT / "oracle"),
           "-I", str(cuda / "include"), str(src), "-o", str(exe),
           "-L", str(PKG), "-ldistattn_b200", "-L", str(ROOT / "oracle"), "-loracle",
           "-L", str(cuda / "lib64"), "-lcudart_static", "-ldl", "-lrt", "-lpthread",
           "-Wl,-rpath,$ORIGIN/../../../paper_2310_03294_b200", "-Wl,-rpath,$ORIGIN/../../../oracle"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"C++ API test build failed:\n{r.stdout}\n{r.stderr}")
    return exe


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv, ptxas_v="--ptxas" in sys.argv)
    print(LIB)
