"""Build the in-tree native library ``lib/libgdvfs.so`` for sm_100a.

    python -m paper_2004_08177_b200._build

Every translation unit (the .cu kernels and the C++ host runtime behind the
C ABI) goes through nvcc with ``-gencode arch=compute_100a,code=sm_100a``;
nvcc cross-compiles here without a GPU.  ``--fmad=false`` keeps every double
expression free of contraction (bit parity with the reference's no-FMA
Release build; the kernels also spell their sums with __dadd_rn/__dmul_rn).
"""
from __future__ import annotations

import concurrent.futures
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "lib" / "libgdvfs.so"
SOURCES = ["gd_grid.cu", "gd_kernels.cu", "gd_capi.cpp", "gd_pack.cpp", "gd_model_io.cpp", "gd_edf.cpp", "gd_multi.cpp", "gd_train.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def ccbin() -> list:
    """Host compiler: the system g++ links libstdc++ dynamically (the /opt/gcc
    wrapper would embed a second, static libstdc++ into the library)."""
    return ["-ccbin", "/usr/bin/g++"] if Path("/usr/bin/g++").exists() else []


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.hpp"))
    deps.append(ROOT / "include" / "gdvfs.h")
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = True, out: Path = None, defines=()) -> Path:
    """Build lib/libgdvfs.so (or `out` with extra -D `defines`, for experiments)."""
    lib = Path(out) if out else LIB
    if not force and out is None and not _stale():
        return LIB
    objdir = lib.parent / ("obj" if out is None else f"obj_{lib.stem}")
    objdir.mkdir(parents=True, exist_ok=True)
    common = ["-O3", "-std=c++17", "-lineinfo", "--fmad=false", "-Xcompiler", "-fPIC,-O3,-Wall",
              f"-I{ROOT / 'include'}", f"-I{CSRC}"] + [f"-D{d}" for d in defines] + ccbin() + ARCH
    cmds, objs = [], []
    for s in SOURCES:
        src = CSRC / s
        obj = objdir / (src.stem + ".o")
        cmd = [nvcc(), *common, "-c", str(src), "-o", str(obj)]
        if s.endswith(".cu") and os.environ.get("GD_PTXAS_VERBOSE"):
            cmd += ["-Xptxas", "-v"]
        cmds.append(cmd)
        objs.append(str(obj))
    with concurrent.futures.ThreadPoolExecutor(max_workers=len(cmds)) as pool:
        for cmd in cmds:
            if verbose:
                print(" ".join(cmd), flush=True)
        list(pool.map(lambda c: subprocess.run(c, check=True), cmds))
    tmp = lib.with_suffix(".so.tmp")
    cmd = [nvcc(), *ccbin(), *ARCH, "-shared", "-o", str(tmp), *objs, "-lcudart_static", "-lrt", "-lpthread",
           "-ldl"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    # python -m paper_2004_08177_b200._build [--force] [--out PATH -DNAME=V ...]
    args = sys.argv[1:]
    out = args[args.index("--out") + 1] if "--out" in args else None
    defs = [a[2:] for a in args if a.startswith("-D")]
    build(force="--force" in args, out=out, defines=defs)
