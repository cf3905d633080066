"""Native build of libhiccl.so (host C++20 + sm_100a CUDA, one C-ABI library).

Host sources compile with g++, the executor with nvcc for sm_100a only
(``-gencode arch=compute_100a,code=sm_100a``), cudart is linked statically
so the library loads on CPU-only hosts (the CPU test suite binds it too).
Incremental: objects are rebuilt when a source or any header is newer.

    python -m paper_2408_05962_b200.build          # build
    python -m paper_2408_05962_b200.build --clean  # rebuild from scratch
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
INCLUDE = ROOT / "include"
# HICCL_BUILD_VARIANT=name + HICCL_BUILD_DEFINES="-DX ...": an A/B build of
# the same sources into _build/<name> and lib/<name>/libhiccl.so (load it
# with HICCL_LIB_PATH); the default build is untouched.
VARIANT = os.environ.get("HICCL_BUILD_VARIANT", "")
BUILD = PKG / "_build" / VARIANT if VARIANT else PKG / "_build"
LIB = PKG / "lib" / VARIANT / "libhiccl.so" if VARIANT else PKG / "lib" / "libhiccl.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

HOST_FLAGS = ["-std=c++20", "-O2", "-fPIC", "-Wall", "-Wextra", "-g",
              f"-I{INCLUDE}", f"-I{CSRC / 'host'}", "-I/usr/local/cuda/include"]
CUDA_FLAGS = ["-std=c++20", "-O3", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC",
              "--fmad=false", "-Xptxas", "-v", f"-I{INCLUDE}", f"-I{CSRC}",
              *os.environ.get("HICCL_BUILD_DEFINES", "").split()]


def _headers() -> list[Path]:
    hs = list(INCLUDE.rglob("*.h")) + list(INCLUDE.rglob("*.hpp"))
    hs += list(CSRC.rglob("*.hpp")) + list(CSRC.rglob("*.cuh"))
    return hs


def _stale(obj: Path, src: Path, newest_header: float) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return src.stat().st_mtime > t or newest_header > t


def _run(cmd: list[str], log: Path | None = None) -> None:
    res = subprocess.run(cmd, capture_output=True, text=True)
    if log is not None:
        log.write_text(res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd[:4])} ...")


def build(clean: bool = False, verbose: bool = False) -> Path:
    if clean and BUILD.exists():
        shutil.rmtree(BUILD)
    BUILD.mkdir(parents=True, exist_ok=True)
    LIB.parent.mkdir(parents=True, exist_ok=True)
    newest = max((h.stat().st_mtime for h in _headers()), default=0.0)
    jobs = []
    objs = []
    for src in sorted((CSRC / "host").glob("*.cpp")):
        obj = BUILD / (src.stem + ".o")
        objs.append(obj)
        if _stale(obj, src, newest):
            jobs.append((["g++", *HOST_FLAGS, "-c", str(src), "-o", str(obj)], None))
    for src in sorted((CSRC / "cuda").glob("*.cu")):
        obj = BUILD / (src.stem + ".cu.o")
        objs.append(obj)
        if _stale(obj, src, newest):
            jobs.append(([NVCC, *CUDA_FLAGS, "-c", str(src), "-o", str(obj)],
                         BUILD / (src.stem + ".ptxas.log")))
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        for fut in [ex.submit(_run, cmd, log) for cmd, log in jobs]:
            fut.result()
    if jobs or not LIB.exists() or any(o.stat().st_mtime > LIB.stat().st_mtime for o in objs):
        tmp = LIB.with_suffix(".so.tmp")
        _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs),
              "-lpthread", "-ldl", "-lrt"])
        os.replace(tmp, LIB)
    if verbose:
        print(f"built {LIB}")
    return LIB


def build_oracle() -> None:
    """The parity checkers (test infrastructure, see oracle/Makefile)."""
    _run(["make", "-s", "-C", str(ROOT / "oracle"), "port"])
    if Path("/root/reference/proj/src").is_dir():
        _run(["make", "-s", "-j8", "-C", str(ROOT / "oracle"), "ref"])


if __name__ == "__main__":
    build(clean="--clean" in sys.argv, verbose=True)
    if "--no-oracle" not in sys.argv:
        build_oracle()
