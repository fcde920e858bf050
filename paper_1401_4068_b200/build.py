"""Build libente_b200.so in-tree with nvcc for sm_100a (B200).

    python -m paper_1401_4068_b200.build [--verbose]

Each .cu under csrc/ is compiled to an object in build/ (in parallel) and
linked into paper_1401_4068_b200/libente_b200.so.  No GPU is needed: nvcc
cross-compiles.  -lineinfo keeps the SASS <-> source map for ncu.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "ente_b200")
LIB = os.path.join(PKG, "libente_b200.so")
PYHOST_SRC = os.path.join(CSRC, "pyhost.cpp")
PYHOST = os.path.join(PKG, "_pyhost" + sysconfig.get_config_var("EXT_SUFFIX"))

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--fmad=false",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
    "-I", os.path.join(ROOT, "include"),
]


def nvcc() -> str:
    path = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(path):
        raise RuntimeError("nvcc not found; CUDA 12.9 toolkit required")
    return path


def _sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = _sources() + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    deps.append(os.path.join(ROOT, "include", "ente_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build_pyhost(force: bool = False) -> str:
    """The CPython host helper (_pyhost: chunk pointers via the buffer protocol)."""
    if not force and os.path.exists(PYHOST) and os.path.getmtime(PYHOST) > os.path.getmtime(PYHOST_SRC):
        return PYHOST
    cxx = shutil.which("g++") or "c++"
    tmp = PYHOST + ".tmp"
    cmd = [cxx, "-O2", "-shared", "-fPIC", "-std=c++17", "-I", sysconfig.get_paths()["include"],
           PYHOST_SRC, "-o", tmp]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"g++ failed for {PYHOST_SRC}:\n{r.stderr}")
    os.replace(tmp, PYHOST)
    return PYHOST


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Compile and link; `defines` (-D flags) + `out` make development variants."""
    lib_path = out or LIB
    if out is None and not defines:
        build_pyhost(force)
    if not force and not defines and out is None and not _needs_build():
        return LIB
    bdir = BUILD if not defines else BUILD + "_" + "_".join(d.replace("=", "") for d in defines)
    os.makedirs(bdir, exist_ok=True)
    cc = nvcc()
    extra = ["-Xptxas", "-v"] if verbose else []

    def compile_one(src):
        obj = os.path.join(bdir, os.path.basename(src)[:-3] + ".o")
        cmd = [cc, *NVCC_FLAGS, *[f"-D{d}" for d in defines], *extra, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        if verbose and r.stderr:
            sys.stderr.write(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, _sources()))
    tmp = lib_path + ".tmp"
    cmd = [cc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", tmp,
           "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, lib_path)
    return lib_path


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv, defines=defs,
                out=outs[0] if outs else None))
