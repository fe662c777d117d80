"""Build liblagtrans_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2211_12616_b200._build        (or __graft_entry__.build())

The library is compiled with -fmad=false: the reference evaluates every
product and sum separately (numpy), and keeping nvcc from contracting them
into FMAs is what makes the float64 arithmetic bit-identical.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "_lib"
LIB = LIBDIR / "liblagtrans_b200.so"
SOURCES = ["lt_capi.cu", "lt_kernels.cu", "lt_step.cu", "lt_output.cu", "lt_host.cpp",
           "lt_comm.cu"]
HEADERS = ["lt_device.cuh", "lt_step.cuh", "lt_kernels.cuh", "lt_comm.cuh", "lt_logtab.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "--expt-relaxed-constexpr",
         "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-v"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; set NVCC or install the CUDA toolkit")


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [PKG.parent / "include" / "lagtrans_b200.h",
                                                   Path(__file__)]
    return any(d.stat().st_mtime > t for d in deps)


LAST_MODE = None   # "compiled" | "up-to-date" (the shipped .so is newer than every source)


def build(force: bool = False, verbose: bool = False, outdir: Path | None = None,
          defines: tuple[str, ...] = ()) -> Path:
    """Compile and link; `outdir`/`defines` build an experimental variant."""
    libdir = Path(outdir) if outdir else LIBDIR
    lib = libdir / LIB.name
    global LAST_MODE
    if not force and outdir is None and not defines and not _stale():
        LAST_MODE = "up-to-date"
        return LIB
    LAST_MODE = "compiled"
    libdir.mkdir(parents=True, exist_ok=True)

    def compile_one(src):
        obj = libdir / (Path(src).stem + ".o")
        cmd = [nvcc(), *ARCH, *FLAGS, *[f"-D{d}" for d in defines],
               "-I", str(PKG.parent / "include"), "-c",
               str(CSRC / src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
        return str(obj), r.stdout + r.stderr

    # the translation units compile independently: build them in parallel
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(len(SOURCES)) as pool:
        results = list(pool.map(compile_one, SOURCES))
    objs = [o for o, _ in results]
    log = [text for _, text in results]
    tmp = lib.with_suffix(".so.tmp")
    cmd = [nvcc(), *ARCH, "-shared", "--cudart", "static", "-o", str(tmp), *objs, "-lpthread", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, lib)
    (libdir / "ptxas.log").write_text("\n".join(log))
    if verbose:
        print("\n".join(log))
    return lib


if __name__ == "__main__":
    args = sys.argv[1:]
    defs = tuple(a[2:] for a in args if a.startswith("-D"))
    out = next((a.split("=", 1)[1] for a in args if a.startswith("--out=")), None)
    print(build(force="--force" in args, verbose="-v" in args, outdir=out, defines=defs))
