"""In-tree build of the native libraries (nvcc / g++, no torch JIT cache).

    libdsdv.so      sm_100a kernels + the C-ABI of include/dsdv/dsdv.h
    libdsd_b200.so  the C++ drop-in `dsd::` verifier API (include/dsd/) over the C-ABI

Outputs land next to this file so they travel with a gpurun snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
HOSTSRC = PKG / "host"
INCLUDE = ROOT / "include"
BUILD = ROOT / "build"

LIB_DSDV = PKG / "libdsdv.so"
LIB_DSD = PKG / "libdsd_b200.so"

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
CUDA_HOME = Path(NVCC).resolve().parent.parent
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-std=c++17", "-O3", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC",
              f"-I{INCLUDE}", "--expt-relaxed-constexpr"]

CU_SOURCES = ["verify.cu", "rows.cu", "shard.cu", "topm.cu", "calib.cu", "abi.cu"]
HOST_SOURCES = ["dsd_api.cpp", "calib_api.cpp"]


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("build step failed: " + " ".join(cmd))


def _stale(out: Path, deps: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _headers() -> list[Path]:
    return sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.rglob("*.h")) + sorted(INCLUDE.rglob("*.hpp"))


def build_dsdv(force: bool = False, trace: bool = False) -> Path:
    """libdsdv.so; trace=True builds the cycle-accounting variant
    libdsdv_trace.so (-DDSDV_TRACE, development aid, load with DSDV_LIB)."""
    hdrs = _headers()
    lib = PKG / "libdsdv_trace.so" if trace else LIB_DSDV
    bdir = BUILD / ("trace" if trace else "release")
    flags = [*NVCC_FLAGS, *(["-DDSDV_TRACE"] if trace else [])]
    if not force and not _stale(lib, [*(CSRC / s for s in CU_SOURCES), *hdrs]):
        return lib  # up to date (also on GPU boxes, where build/ is not shipped)
    bdir.mkdir(parents=True, exist_ok=True)
    objs = []
    jobs = []
    for src in CU_SOURCES:
        s = CSRC / src
        o = bdir / (s.stem + ".o")
        objs.append(o)
        if force or _stale(o, [s, *hdrs]):
            jobs.append([NVCC, *flags, "-c", str(s), "-o", str(o)])
    with ThreadPoolExecutor(max_workers=min(4, max(1, len(jobs)))) as ex:
        list(ex.map(_run, jobs))
    if force or jobs or _stale(lib, objs):
        _run([NVCC, *ARCH, "-shared", "-o", str(lib), *map(str, objs)])
    return lib


def build_variant(name: str, defines: list[str], force: bool = False) -> Path:
    """libdsdv_<name>.so with extra -D flags (development aid: kernel variants
    timed side by side on one box through DSDV_LIB)."""
    hdrs = _headers()
    lib = PKG / f"libdsdv_{name}.so"
    bdir = BUILD / f"var_{name}"
    if not force and not _stale(lib, [*(CSRC / s for s in CU_SOURCES), *hdrs]):
        return lib
    bdir.mkdir(parents=True, exist_ok=True)
    flags = [*NVCC_FLAGS, *(f"-D{d}" for d in defines)]
    objs, jobs = [], []
    for src in CU_SOURCES:
        s = CSRC / src
        o = bdir / (s.stem + ".o")
        objs.append(o)
        jobs.append([NVCC, *flags, "-c", str(s), "-o", str(o)])
    with ThreadPoolExecutor(max_workers=4) as ex:
        list(ex.map(_run, jobs))
    _run([NVCC, *ARCH, "-shared", "-o", str(lib), *map(str, objs)])
    return lib


def build_dsd_api(force: bool = False) -> Path | None:
    srcs = [HOSTSRC / s for s in HOST_SOURCES if (HOSTSRC / s).exists()]
    if not srcs:
        return None
    deps = [*srcs, *_headers(), LIB_DSDV]
    if force or _stale(LIB_DSD, deps):
        _run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-Wall", "-Wextra",
              f"-I{INCLUDE}", f"-I{CUDA_HOME}/include", *map(str, srcs), "-o", str(LIB_DSD),
              f"-L{PKG}", "-ldsdv", f"-L{CUDA_HOME}/lib64", "-lcudart", "-Wl,-rpath,$ORIGIN"])
    return LIB_DSD


CPP_TESTS = ROOT / "tests" / "cpp"


def build_cpp_tests(force: bool = False) -> list[Path]:
    """C++ test programs of the drop-in API (tests/cpp/*.cpp -> build/cpp/)."""
    outs = []
    for src in sorted(CPP_TESTS.glob("*.cpp")):
        exe = PKG / "bin" / src.stem
        if force or _stale(exe, [src, *_headers(), LIB_DSD]):
            exe.parent.mkdir(parents=True, exist_ok=True)
            _run(["g++", "-std=c++20", "-O2", "-Wall", f"-I{INCLUDE}", str(src), "-o", str(exe),
                  f"-L{PKG}", "-ldsd_b200", "-ldsdv", f"-Wl,-rpath,{PKG}", "-Wl,-rpath,$ORIGIN/.."])
        outs.append(exe)
    return outs


def build_all(force: bool = False) -> None:
    build_dsdv(force)
    build_dsd_api(force)
    build_cpp_tests(force)


if __name__ == "__main__":
    if "--variant" in sys.argv:
        i = sys.argv.index("--variant")
        print(build_variant(sys.argv[i + 1], sys.argv[i + 2:], force=True))
    elif "--trace" in sys.argv:
        print(build_dsdv(force="--force" in sys.argv, trace=True))
    else:
        build_all(force="--force" in sys.argv)
        print(LIB_DSDV)
