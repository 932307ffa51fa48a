"""In-tree build of libh2mmp_b200.so (sm_100a) and of the oracle checker.

The library is plain nvcc/g++ objects linked into one shared object with a
C-ABI (include/h2c.h); Python reaches it through ctypes.  Objects are rebuilt
only when a source or header is newer than the library.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "lib"
LIB = LIBDIR / "libh2mmp_b200.so"
OBJDIR = PKG / "build"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUDA_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                     "-Xptxas", "-v"]
CXX_FLAGS = ["-O3", "-std=c++17", "-fPIC", "-Wall", "-Wextra", "-pthread", "-I/usr/local/cuda/include"]

CU_SOURCES = ["engine.cu", "construct_dev.cu"]
CPP_SOURCES = ["plan.cpp", "counters.cpp", "structure.cpp", "construct.cpp", "capi_inputs.cpp", "capi.cpp"]
# CPU-only input generator (structure + synthetic BASELINE operands) for bench.py's reference arm
INPUT_SOURCES = ["structure.cpp", "construct.cpp", "capi_inputs.cpp", "construct_dev_stub.cpp"]
INPUTS_LIB = ROOT / "oracle" / "_build" / "libh2inputs.so"


def _host_blas() -> list[str]:
    """Link flags for the scipy wheel's OpenBLAS (host BLAS/LAPACK of the input constructor only)."""
    import scipy
    libs = Path(scipy.__path__[0]).parent / "scipy.libs"
    so = sorted(libs.glob("libscipy_openblas*.so"))
    if not so:
        raise RuntimeError(f"no libscipy_openblas in {libs}")
    return [f"-L{libs}", f"-l:{so[0].name}", "-Xlinker", f"-rpath={libs}"]


def _headers() -> list[Path]:
    return list(CSRC.glob("*.hpp")) + list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h"))


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _run(cmd: list[str], log: Path | None = None) -> None:
    res = subprocess.run(cmd, capture_output=True, text=True)
    if log is not None:
        log.write_text(res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd)}")


def build_library(force: bool = False, verbose: bool = False) -> Path:
    OBJDIR.mkdir(exist_ok=True)
    LIBDIR.mkdir(exist_ok=True)
    headers = _headers()
    objs = []
    for src in CU_SOURCES:
        s = CSRC / src
        o = OBJDIR / (src + ".o")
        if force or _stale(o, [s] + headers):
            if verbose:
                print(f"[nvcc] {src}", flush=True)
            _run([NVCC, *CUDA_FLAGS, "-c", str(s), "-o", str(o)], OBJDIR / (src + ".ptxas.log"))
        objs.append(o)
    for src in CPP_SOURCES:
        s = CSRC / src
        o = OBJDIR / (src + ".o")
        if force or _stale(o, [s] + headers):
            if verbose:
                print(f"[g++ ] {src}", flush=True)
            _run(["g++", *CXX_FLAGS, "-c", str(s), "-o", str(o)])
        objs.append(o)
    if force or _stale(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart", *_host_blas(),
              "-Xcompiler", "-pthread"])
    return LIB


def build_inputs_library(force: bool = False) -> Path:
    """oracle/_build/libh2inputs.so: the host-only entry points of include/h2c.h that build the
    structure and the synthetic inputs (no CUDA), so bench.py's reference arm never maps
    libh2mmp_b200.so."""
    INPUTS_LIB.parent.mkdir(parents=True, exist_ok=True)
    srcs = [CSRC / s for s in INPUT_SOURCES]
    if force or _stale(INPUTS_LIB, srcs + _headers()):
        _run(["g++", *CXX_FLAGS, "-DH2C_INPUTS_ONLY", "-shared", "-o", str(INPUTS_LIB), *map(str, srcs),
              *[("-Wl," + a) if a.startswith("-rpath") else a for a in _host_blas() if a != "-Xlinker"]])
    return INPUTS_LIB


def build_oracle(force: bool = False) -> Path | None:
    """The CPU oracle (test infrastructure) — built here so it travels with the snapshot."""
    odir = ROOT / "oracle"
    if not (odir / "Makefile").exists():
        return None
    cmd = ["make", "-s", "-C", str(odir), f"PY={sys.executable}"]
    if force:
        subprocess.run(["make", "-s", "-C", str(odir), "clean"], check=False)
    _run(cmd)
    # the reference's own MMP path (unmodified sources + oracle/eigen_shim) and its unit tests, only
    # where /root/reference exists (this container; the GPU box never needs them)
    if Path("/root/reference/proj/core/src/mmp.cpp").exists():
        _run(["make", "-s", "-C", str(odir), f"PY={sys.executable}", "ref", "ref-tests"])
    return odir / "_build" / "liboracle.so"


if __name__ == "__main__":
    force = "--force" in sys.argv
    print(build_library(force=force, verbose=True))
    print(build_oracle(force=force))
    print(build_inputs_library(force=force))
